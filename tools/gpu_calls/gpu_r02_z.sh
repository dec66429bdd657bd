# r02: device random stream (generator on the GPU), PCG id prologue, racecheck of the full-sync variant, bench
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_frame.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
timeout 300 $B 2>/dev/null | python -c "$P"
bash tools/sanitize_racecheck.sh $O
