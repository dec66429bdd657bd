# r02: pyramid 16-byte loads / coalesced stores; rng scratch reuse; ncu crash diagnosis
O=gpurun_out/r02ah; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rng.py tests/test_gpu_frame.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
timeout 300 $NB > $O/plain.json 2> $O/plain.err; echo "plain rc=$?"; tail -2 $O/plain.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nograph.csv $NB --no-graph > $O/ncu_nograph.log 2>&1; echo "ncu nograph rc=$?"; tail -3 $O/ncu_nograph.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_graph.csv $NB > $O/ncu_graph.log 2>&1; echo "ncu graph rc=$?"; tail -3 $O/ncu_graph.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality --no-graph"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
timeout 300 $B 2>/dev/null | python -c "$P"
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none -k regex:k_pyramid_fused -s 8 -c 1 -o $O/k_pyramid_fused $NB --no-graph > $O/ncu_pyr.log 2>&1; echo "ncu pyr rc=$?"
