# r02: register-column QR for the 36x36 pose system (two warps, named barrier per step)
O=gpurun_out/r02ab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stages.py tests/test_gpu_bench_parity.py tests/test_gpu_golden.py tests/test_gpu_frame.py -q -rf > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8 > $O/phases4.txt; cat $O/phases4.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
timeout 300 $B 2>/dev/null | python -c "$P"
