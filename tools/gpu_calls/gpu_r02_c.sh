# r02: parity diagnostics at the bench workload, PCG variants, phases, bench, ncu captures
set -x
mkdir -p gpurun_out/r02c
timeout 600 python tools/dbg_bench_frames.py --frames 8 > gpurun_out/r02c/dbg_frames.txt 2>&1; echo "dbg rc=$?"
head -60 gpurun_out/r02c/dbg_frames.txt
timeout 600 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_kernels.py -q -rf > gpurun_out/r02c/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02c/pytest.log
timeout 300 python tools/profile_step.py --streams 4 --frames 5 --phases > gpurun_out/r02c/phases.txt 2>&1
grep -A9 "^frame 3" gpurun_out/r02c/phases.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e-u8 --no-cpu-baseline --no-quality > gpurun_out/r02c/bench.json 2> gpurun_out/r02c/bench.err; echo "bench rc=$?"
cat gpurun_out/r02c/bench.json
for k in k_surface_solve k_pose_solve; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/r02c/$k \
      python tools/profile_step.py --streams 8 --frames 5 > gpurun_out/r02c/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
ls -la gpurun_out/r02c
