# surface block size 256 (2 CTAs/SM) vs 512, two runs each, then cfg4 at the default build
mkdir -p gpurun_out/sweep8
for v in "256 2" "512 1"; do
  set -- $v
  LIVECAP_NVCC_EXTRA="-DLC_SURF_NT=$1 -DLC_SURF_MINB=$2" python -c "from paper_1810_02648_b200 import _build; _build.build(force=True)" > gpurun_out/sweep8/build_$1.log 2>&1 || { tail -5 gpurun_out/sweep8/build_$1.log; continue; }
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/sweep8/nt$1_$i.json 2> gpurun_out/sweep8/nt$1_$i.err
    python -c "import json; d=json.load(open('gpurun_out/sweep8/nt$1_$i.json')); print('$v', round(d['value']), round(d['ms_per_step'],3), d['pcg_iter_us'])" || tail -3 gpurun_out/sweep8/nt$1_$i.err
  done
done
timeout 600 python bench.py --preset x20k --gn 4 --pcg 8 --no-cpu-baseline > gpurun_out/sweep8/cfg4.json 2> gpurun_out/sweep8/cfg4.err
python -c "import json; d=json.load(open('gpurun_out/sweep8/cfg4.json')); print('cfg4', round(d['value']), d['e2e']['value'], d['pcg_iter_us'])" || tail -3 gpurun_out/sweep8/cfg4.err
