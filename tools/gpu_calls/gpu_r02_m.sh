# r02 (session 3): full gpu suite, smoke, bench line, launch list, ncu full of the two solver kernels at the bench launch shape
set -x
O=gpurun_out/r02m; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" $O/pytest_gpu.log | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json; tail -5 $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; cat $O/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu rc=$?"
for k in k_surface_solve k_pose_solve; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/$k \
      python tools/profile_step.py --streams 4 --frames 5 > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
ls -la $O
