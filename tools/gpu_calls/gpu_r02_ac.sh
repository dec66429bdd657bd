# r02: cfg4 / cfg5 records with CPU baselines; surface team 16 at x5k; pose team 8
O=gpurun_out/r02ac; mkdir -p $O
timeout 900 python bench.py --preset x20k --gn 4 --pcg 8 --steps 10 --warmup 3 --no-e2e-u8 > $O/bench_cfg4_x20k.json 2> $O/cfg4.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --streams 8 --groups 2 --steps 20 --warmup 3 --no-e2e-u8 > $O/bench_cfg5_8streams.json 2> $O/cfg5.err; echo "cfg5 rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== surf cs 16"; LIVECAP_SURFACE_CLUSTER=16 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pose cs 8"; LIVECAP_POSE_CLUSTER=8 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 20 streams 5 groups"; timeout 300 $B --streams 20 --groups 5 2>/dev/null | python -c "$P"
echo "== 12 streams 4 groups"; timeout 300 $B --streams 12 --groups 4 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
python -c "
import json
for f in ['bench_cfg4_x20k','bench_cfg5_8streams']:
    d=json.load(open('$O/'+f+'.json')); print(f, round(d['value']), d['e2e']['value'], d['pcg_iter_us'], d['roofline']['frac'], d['cpu_baseline'])
"
