# third cluster-size sweep (one GPU call); the last line also runs the u8 e2e leg
mkdir -p gpurun_out/sweep4
free -g | head -2
for cfg in "16 4 4 1" "16 8 4 1" "16 8 4 4" "24 6 4 4" "32 8 4 1" "16 4 4 4"; do
  set -- $cfg
  n=s$1_g$2_p$3_s$4
  extra="--no-e2e-u8"; [ "$cfg" = "16 4 4 4" ] && extra=""
  LIVECAP_POSE_CLUSTER=$3 LIVECAP_SURFACE_CLUSTER=$4 timeout 300 python bench.py --no-cpu-baseline --streams $1 --groups $2 $extra \
      > gpurun_out/sweep4/$n.json 2> gpurun_out/sweep4/$n.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep4/$n.json')); r=d['roofline']; print('$cfg', round(d['value']), round(d['e2e']['value']), d.get('e2e_u8') and round(d['e2e_u8']['value']), round(r['kernel_ms_per_launch'],3), d['pcg_iter_us'], d['clocks']['samples'])" || tail -3 gpurun_out/sweep4/$n.err
done
