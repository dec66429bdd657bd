# r02 final build: full gpu suite, smoke, bench line (ours + reference), graph leg
set -x
O=gpurun_out/r02final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" $O/pytest_gpu.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --graph --steps 20 --warmup 5 --no-cpu-baseline --no-e2e-u8 --no-quality > $O/bench_graph.json 2> $O/bench_graph.err; echo "graph rc=$?"
python -c "
import json
d=json.load(open('$O/bench_n1.json')); print(round(d['value']), d['e2e']['value'], d['e2e_u8']['value'], d['pcg_iter_us'], d['roofline']['frac'], d['roofline']['frac_concurrent'], d['tracking']['iou_mean'], d['cpu_baseline'])
g=json.load(open('$O/bench_graph.json')); print('graph', round(g['value']), g['graph'])
"
