# 2-CTA teams (two runs each) vs the 4/4 default
mkdir -p gpurun_out/sweep9
for cfg in "2 4" "4 2" "2 2" "4 4"; do
  set -- $cfg
  for i in 1 2; do
    n=p$1_s$2_$i
    LIVECAP_POSE_CLUSTER=$1 LIVECAP_SURFACE_CLUSTER=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/sweep9/$n.json 2> gpurun_out/sweep9/$n.err
    python -c "import json; d=json.load(open('gpurun_out/sweep9/$n.json')); print('$cfg', round(d['value']), round(d['ms_per_step'],3), d['pcg_iter_us'])" || tail -3 gpurun_out/sweep9/$n.err
  done
done
