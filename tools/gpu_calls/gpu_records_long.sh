# final build: cfg4 (x20k, 4 GN x 8 PCG) and cfg5 (8 streams) records with CPU baselines; the long
# teacher-forced sequences (cfg3 300 frames, cfg2 100 frames pose-only)
O=gpurun_out/r02rec; mkdir -p $O
timeout 900 python bench.py --preset x20k --gn 4 --pcg 8 --steps 10 --warmup 3 --no-e2e-u8 > $O/bench_cfg4_x20k.json 2> $O/cfg4.err; echo "cfg4 rc=$?"; head -c 250 $O/bench_cfg4_x20k.json; echo
timeout 900 python bench.py --streams 8 --groups 2 --steps 20 --warmup 3 --no-e2e-u8 > $O/bench_cfg5_8streams.json 2> $O/cfg5.err; echo "cfg5 rc=$?"; head -c 250 $O/bench_cfg5_8streams.json; echo
LIVECAP_LONG_TESTS=1 timeout 1500 python -m pytest tests/test_gpu_bench_parity.py -q -rf -s -k "cfg3_300 or cfg2_pose" --durations=3 > $O/long.log 2>&1; echo "long rc=$?"; grep -E "worst|frames|passed|failed" $O/long.log | tail -8
