# knob sweep on the final build: candidate-list radius, pyramid margin, pose team 8
O=gpurun_out/r02kn; mkdir -p $O
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== radius 256"; LIVECAP_LIST_RADIUS=256 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== radius 384"; LIVECAP_LIST_RADIUS=384 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== radius 128"; LIVECAP_LIST_RADIUS=128 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pyr margin 32"; LIVECAP_PYR_MARGIN=32 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pyr margin 96"; LIVECAP_PYR_MARGIN=96 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pose cs 8"; LIVECAP_POSE_CLUSTER=8 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
