# streams / groups at the final build
mkdir -p gpurun_out/sweep11
for cfg in "16 4" "20 5" "24 6" "24 4" "32 8" "16 4"; do
  set -- $cfg
  n=s$1_g$2
  timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 --streams $1 --groups $2 > gpurun_out/sweep11/$n.json 2> gpurun_out/sweep11/$n.err
  python -c "import json; d=json.load(open('gpurun_out/sweep11/$n.json')); print('$cfg', round(d['value']), round(d['ms_per_step'],3), d['host_ms_per_step'])" || tail -3 gpurun_out/sweep11/$n.err
done
