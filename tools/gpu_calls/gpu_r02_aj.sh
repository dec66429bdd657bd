# r02: final ncu evidence at the bench's launch shape (current build): launch list + full captures
O=gpurun_out/r02aj; mkdir -p $O
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu list rc=$?"
for k in k_surface_solve k_pose_solve; do
  BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -o $O/$k $NB > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
for k in k_pyramid_fused k_cand_build k_rt_tiles; do
  BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none -k regex:$k -s 8 -c 1 -o $O/$k $NB > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
ls -la $O
