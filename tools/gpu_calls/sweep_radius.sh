# candidate-list radius at the throughput config (16 streams / 4 groups)
mkdir -p gpurun_out/sweep7
for r in 1e30 256 128 64; do
  LIVECAP_LIST_RADIUS=$r timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/sweep7/r$r.json 2> gpurun_out/sweep7/r$r.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep7/r$r.json')); print('$r', round(d['value']), round(d['ms_per_step'],3), d['roofline']['kernel_ms_per_launch'])" || tail -3 gpurun_out/sweep7/r$r.err
done
