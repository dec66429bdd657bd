# r02: SURVEY 8c long sequences (cfg3 300 frames, cfg2 100 frames), teacher-forced
O=gpurun_out/r02long; mkdir -p $O
LIVECAP_LONG_TESTS=1 timeout 3300 python -m pytest tests/test_gpu_bench_parity.py -q -rf -s -k "cfg3_300 or cfg2_pose" --durations=5 > $O/long.log 2>&1; echo "long rc=$?"; tail -15 $O/long.log
