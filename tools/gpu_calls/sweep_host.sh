# host enqueue time per step vs device time per step
mkdir -p gpurun_out/sweep6
for cfg in "16 4 1" "16 4 0" "32 8 1" "16 1 1"; do
  set -- $cfg
  n=s$1_g$2_t$3
  timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 --streams $1 --groups $2 --host-threads $3 > gpurun_out/sweep6/$n.json 2> gpurun_out/sweep6/$n.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep6/$n.json')); print('$cfg', round(d['value']), round(d['ms_per_step'],3), d['host_ms_per_step'])" || tail -3 gpurun_out/sweep6/$n.err
done
