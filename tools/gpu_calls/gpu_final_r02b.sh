# final-build profile pass (session 4): full gpu suite, smoke, bench lines (ours + reference arm),
# launch list, ncu --set full of the solver kernels at the bench's launch shape, memcheck on the smoke scene
O=gpurun_out/r02fin; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -6 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench.err; echo "bench rc=$?"; head -c 400 $O/bench_n1.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err; echo "ref rc=$?"; head -c 300 $O/bench_reference.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu list rc=$?"
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
for k in k_surface_solve k_pose_solve; do
  BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -o $O/$k $NB > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
for k in k_pyramid_fused k_cand_build k_rt_tiles; do
  BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o $O/$k $NB > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > $O/memcheck_small.txt 2>&1; echo "memcheck rc=$?"; tail -3 $O/memcheck_small.txt
ls -la $O
