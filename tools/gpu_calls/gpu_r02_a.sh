# r02 first GPU call: full gpu test suite, smoke, bench line (in-track workload), launch list
set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; echo "bench rc=$?"
cat gpurun_out/r02a/bench.json; tail -5 gpurun_out/r02a/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu rc=$?"
