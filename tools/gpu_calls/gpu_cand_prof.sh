# ncu --set full (with source) of k_cand_build at the bench's launch shape; launch list of the new build
O=gpurun_out/r02cprof; mkdir -p $O
NB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cand_build -s 8 -c 1 -o $O/k_cand_build $NB > $O/ncu_cand.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu list rc=$?"
ls -la $O
