# ncu --set full (with source) of k_rt_tiles, k_rim (both stages), k_cand_build, k_own_cells at the bench's launch shape
O=gpurun_out/r02p3; mkdir -p $O
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rt_tiles|k_rim|k_cand_build|k_own_cells|k_pyramid_fused" -s 40 -c 8 -o $O/mix $NB > $O/ncu_mix.log 2>&1; echo "ncu rc=$?"
ls -la $O
