# r02: PCG mode 3 (z + ELL ids in shared memory) + light mbarrier reductions: parity, phases, bench
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_frame.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8 > $O/phases4.txt; cat $O/phases4.txt
for m in 0 3; do
  echo "== bench mode $m"; LIVECAP_PCG_MODE=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']), d['pcg_iter_us'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], d['roofline']['frac_concurrent'])"
done > $O/bench_modes.txt 2>&1; cat $O/bench_modes.txt
