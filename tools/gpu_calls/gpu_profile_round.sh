# One GPU call: bench line, cfg4 bench line, launch list, ncu full captures of the top kernels.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
python bench.py --preset x20k --gn 4 --pcg 8 --no-cpu-baseline --no-e2e-u8 > gpurun_out/prof/bench_cfg4.json 2> gpurun_out/prof/bench_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 > /dev/null 2>&1
for k in k_surface_solve k_pose_solve k_rt_tiles k_cand_build k_pyramid_fused k_rim; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof/$k \
      python tools/profile_step.py --streams 8 --frames 5 > gpurun_out/prof/ncu_$k.log 2>&1
done
python tools/profile_step.py --streams 4 --frames 5 --phases > gpurun_out/prof/phases.txt 2>&1
ls -la gpurun_out/prof
