# r02: line search without the step rescale pass (power-of-two trial scales)
O=gpurun_out/r02av; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_sets.py tests/test_gpu_frame.py tests/test_gpu_bench_parity.py tests/test_gpu_kernels.py tests/test_gpu_golden.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python tools/trace_step.py --streams 4 --steps 1 > $O/trace4.txt 2>&1; tail -18 $O/trace4.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
for i in 1 2; do timeout 300 $B 2>/dev/null | python -c "$P"; done
