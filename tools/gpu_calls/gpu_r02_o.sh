# r02: PCG sub-phase timing under the shared-memory modes and team sizes
O=gpurun_out/r02o; mkdir -p $O
for m in 0 1 2; do
  echo "== pcg mode $m"; LIVECAP_PCG_MODE=$m timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8
done > $O/pcg_modes.txt 2>&1
for cs in 2 8 16; do
  echo "== surface cluster $cs"; LIVECAP_SURFACE_CLUSTER=$cs timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8
done > $O/surf_cs.txt 2>&1
for m in 0 2; do for s in 16 24; do
  echo "== bench mode $m streams $s"; LIVECAP_PCG_MODE=$m timeout 300 python bench.py --streams $s --groups $((s/4)) --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']), d['pcg_iter_us'], d['roofline']['kernel_ms_per_launch'])"
done; done > $O/bench_modes.txt 2>&1
cat $O/*.txt
