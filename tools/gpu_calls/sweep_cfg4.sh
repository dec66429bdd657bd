# cfg4 (x20k, 4 GN x 8 PCG): surface team size 4 / 8 / 16
mkdir -p gpurun_out/sweep10
for cs in 8 16 4; do
  LIVECAP_SURFACE_CLUSTER=$cs timeout 400 python bench.py --preset x20k --gn 4 --pcg 8 --no-cpu-baseline --no-e2e-u8 > gpurun_out/sweep10/cs$cs.json 2> gpurun_out/sweep10/cs$cs.err
  python -c "import json; d=json.load(open('gpurun_out/sweep10/cs$cs.json')); print('cfg4 surface cs $cs', round(d['value']), round(d['ms_per_step'],3), d['pcg_iter_us'])" || tail -3 gpurun_out/sweep10/cs$cs.err
done
