# bench sweep over streams per GPU / groups / host threads (one GPU call)
mkdir -p gpurun_out/sweep
for cfg in "8 4 0" "8 4 1" "8 8 1" "16 8 1" "16 4 1" "24 8 1" "32 8 1" "32 16 1"; do
  set -- $cfg
  timeout 300 python bench.py --no-cpu-baseline --streams $1 --groups $2 --host-threads $3 \
      > gpurun_out/sweep/s$1_g$2_t$3.json 2> gpurun_out/sweep/s$1_g$2_t$3.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep/s$1_g$2_t$3.json')); print('$cfg', round(d['value']), round(d['e2e']['value']), d['clocks'])" || tail -3 gpurun_out/sweep/s$1_g$2_t$3.err
done
