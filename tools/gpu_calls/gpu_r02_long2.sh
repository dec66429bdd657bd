O=gpurun_out/r02long2; mkdir -p $O
LIVECAP_LONG_TESTS=1 timeout 1800 python -m pytest tests/test_gpu_bench_parity.py -q -rf -s -k "cfg2_pose" > $O/long.log 2>&1; echo "long rc=$?"; tail -5 $O/long.log
