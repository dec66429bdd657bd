# surface-kernel block size / residency variants (rebuilds the library on the box)
mkdir -p gpurun_out/sweep5
for v in "256 2 4" "256 2 8" "512 1 4"; do
  set -- $v
  LIVECAP_NVCC_EXTRA="-DLC_SURF_NT=$1 -DLC_SURF_MINB=$2" python -c "from paper_1810_02648_b200 import _build; _build.build(force=True)" > gpurun_out/sweep5/build_$1.log 2>&1 || { tail -5 gpurun_out/sweep5/build_$1.log; continue; }
  n=nt$1_mb$2_s$3
  LIVECAP_SURFACE_CLUSTER=$3 timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/sweep5/$n.json 2> gpurun_out/sweep5/$n.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep5/$n.json')); r=d['roofline']; print('$v', round(d['value']), round(d['e2e']['value']), round(r['kernel_ms_per_launch'],3), d['pcg_iter_us'], d['clocks']['samples'])" || tail -3 gpurun_out/sweep5/$n.err
done
