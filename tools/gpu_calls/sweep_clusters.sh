# bench sweep over per-solver cluster sizes at larger stream counts (one GPU call)
mkdir -p gpurun_out/sweep2
for cfg in "16 4 8 16" "16 4 4 16" "16 4 8 8" "16 4 4 8" "32 8 4 8" "32 8 4 16" "32 8 8 8"; do
  set -- $cfg
  n=s$1_g$2_p$3_s$4
  LIVECAP_POSE_CLUSTER=$3 LIVECAP_SURFACE_CLUSTER=$4 timeout 300 python bench.py --no-cpu-baseline --streams $1 --groups $2 \
      > gpurun_out/sweep2/$n.json 2> gpurun_out/sweep2/$n.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep2/$n.json')); r=d['roofline']; print('$cfg', round(d['value']), round(d['e2e']['value']), round(r['kernel_ms_per_launch'],3), d['pcg_iter_us'], d['clocks']['samples'])" || tail -3 gpurun_out/sweep2/$n.err
done
