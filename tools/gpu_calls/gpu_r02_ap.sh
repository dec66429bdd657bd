O=gpurun_out/r02ap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_frame.py tests/test_gpu_rng.py -q -rf > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
