# r02: line-search batching per solver (pose: full step first; surface: all trials at once)
O=gpurun_out/r02aq; mkdir -p $O
cat gpurun_out/r02ap/pytest.log 2>/dev/null | tail -2
timeout 1200 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_frame.py tests/test_gpu_rng.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8 > $O/phases4.txt; cat $O/phases4.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
echo "== new defaults (pose 1, surf 4)"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== old (pose 4, surf 1)"; LIVECAP_POSE_FIRST_TRIALS=4 LIVECAP_SURF_FIRST_TRIALS=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pose 1, surf 1"; LIVECAP_SURF_FIRST_TRIALS=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== new defaults again"; timeout 300 $B 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
