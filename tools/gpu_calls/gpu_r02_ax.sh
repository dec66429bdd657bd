# r02: pyramid grid-stride loop (parity) + grid cap sweep
O=gpurun_out/r02ax; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_frame.py -q -rf -x -k "pyramid" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
LIVECAP_PYR_GRID=64 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_frame.py -q -rf -x -k "pyramid" > $O/pytest_cap.log 2>&1; echo "pytest cap rc=$?"; tail -2 $O/pytest_cap.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
for g in 0 148 296 592 0; do echo "== pyr grid $g"; LIVECAP_PYR_GRID=$g timeout 300 $B 2>/dev/null | python -c "$P"; done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
