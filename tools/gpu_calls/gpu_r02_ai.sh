# r02: pyramid store loop flattened; bench variance check
O=gpurun_out/r02ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_frame.py -q -rf -x -k "pyramid or raster" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none -k regex:k_pyramid_fused -s 8 -c 1 -o $O/k_pyramid_fused $NB > $O/ncu_pyr.log 2>&1; echo "ncu pyr rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
for i in 1 2 3; do timeout 300 $B 2>/dev/null | python -c "$P"; done
