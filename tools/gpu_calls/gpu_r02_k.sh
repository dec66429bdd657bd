set -x
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_sets.py tests/test_gpu_frame.py tests/test_gpu_golden.py -q -rf > gpurun_out/r02k/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02k/pytest.log | tail -12
timeout 600 python bench.py --no-cpu-baseline --no-e2e-u8 --steps 20 --warmup 5 > gpurun_out/r02k/bench.json 2>gpurun_out/r02k/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02k/bench.json')); print(round(d['value']), d['pcg_iter_us'], d['roofline']['kernel_ms_per_launch'], d['tracking']['iou_mean'], d['tracking']['streams_iou_ge_0_9'])"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py > gpurun_out/r02k/racecheck_small.txt 2>&1; echo "racecheck rc=$?"
tail -5 gpurun_out/r02k/racecheck_small.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > gpurun_out/r02k/memcheck_small.txt 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/r02k/memcheck_small.txt
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize.py --x5k > gpurun_out/r02k/memcheck_x5k.txt 2>&1; echo "memcheck x5k rc=$?"
tail -4 gpurun_out/r02k/memcheck_x5k.txt
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize.py > gpurun_out/r02k/synccheck_small.txt 2>&1; echo "synccheck rc=$?"
tail -4 gpurun_out/r02k/synccheck_small.txt
