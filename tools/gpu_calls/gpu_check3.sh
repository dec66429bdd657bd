# parity + two bench runs + solver phase stamps
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/b$i.json 2> gpurun_out/b$i.err
  python -c "import json; d=json.load(open('gpurun_out/b$i.json')); print('bench', round(d['value']), round(d['ms_per_step'],3), d['roofline']['kernel_ms_per_launch'])" || tail -3 gpurun_out/b$i.err
done
python tools/profile_step.py --streams 4 --frames 5 --phases 2>&1 | tail -8
