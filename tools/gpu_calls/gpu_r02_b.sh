# r02 second GPU call: new PCG (smem z/p/Ap, 2 barriers/iteration) -- tests, smoke, bench, phases
set -x
mkdir -p gpurun_out/r02b
timeout 1200 python -m pytest tests -m gpu -q -rf -x --durations=10 > gpurun_out/r02b/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r02b/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r02b/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e-u8 > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err; echo "bench rc=$?"
cat gpurun_out/r02b/bench.json; tail -5 gpurun_out/r02b/bench.err
timeout 300 python tools/profile_step.py --streams 4 --frames 5 --phases > gpurun_out/r02b/phases.txt 2>&1; echo "phases rc=$?"
tail -12 gpurun_out/r02b/phases.txt
