O=gpurun_out/r02ao; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -rf -s -k directional > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
