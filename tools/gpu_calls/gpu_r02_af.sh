# r02: branch-free packed DSMEM gathers in the PCG matvec
O=gpurun_out/r02af; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_frame.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8 > $O/phases4.txt; cat $O/phases4.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality --no-graph"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
timeout 300 $B 2>/dev/null | python -c "$P"
