# r02: CUDA-graph mode of the tracker step: parity + bench graph leg
O=gpurun_out/r02ae; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_frame.py -q -rf -k "graph or pyramid or pipeline" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -25 $O/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -5 $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(round(d['value']), d['graph'])"
