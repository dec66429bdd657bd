# One GPU call: bench line, launch list, ncu full captures of the top kernels.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for k in k_surface_solve k_pose_solve k_rt_tiles k_cand_build k_pyramid_fused k_rim; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof/$k \
      python tools/profile_step.py --streams 8 --frames 5 > gpurun_out/prof/ncu_$k.log 2>&1
done
ls -la gpurun_out/prof
