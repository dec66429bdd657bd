# parity + two bench runs (noise) + the pyramid kernel's launch times
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/b$i.json 2> gpurun_out/b$i.err
  python -c "import json; d=json.load(open('gpurun_out/b$i.json')); print('bench', round(d['value']), round(d['ms_per_step'],3))" || tail -3 gpurun_out/b$i.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_pyramid_fused|k_cand_build" -s 6 -c 4 python tools/profile_step.py --streams 8 --frames 4 2>&1 | grep -E "k_pyramid|k_cand|duration|dram__bytes" | head -20
