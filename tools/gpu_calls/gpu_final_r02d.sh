# final build (after the rim launch bounds and the raster merge exit): full gpu suite, smoke, bench lines, launch list
O=gpurun_out/r02fd; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -6 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench.err; echo "bench rc=$?"; head -c 300 $O/bench_n1.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err; echo "ref rc=$?"; head -c 200 $O/bench_reference.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > /dev/null 2>&1; echo "ncu list rc=$?"
ls -la $O
