# r02: full gpu suite + smoke + bench after the LU preconditioner fix
set -x
mkdir -p gpurun_out/r02f
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=12 > gpurun_out/r02f/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02f/pytest_gpu.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r02f/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err; echo "bench rc=$?"
cat gpurun_out/r02f/bench.json; tail -3 gpurun_out/r02f/bench.err
