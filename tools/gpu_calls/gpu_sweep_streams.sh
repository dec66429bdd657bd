# stream / group / team-size sweep on the current build
O=gpurun_out/r02sw; mkdir -p $O
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
echo "== 16 streams 4 groups"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 24 streams 6 groups"; timeout 300 $B --streams 24 --groups 6 2>/dev/null | python -c "$P"
echo "== 32 streams 8 groups"; timeout 300 $B --streams 32 --groups 8 2>/dev/null | python -c "$P"
echo "== 24 streams 4 groups"; timeout 300 $B --streams 24 --groups 4 2>/dev/null | python -c "$P"
echo "== 32 streams 4 groups"; timeout 300 $B --streams 32 --groups 4 2>/dev/null | python -c "$P"
echo "== 16 streams 8 groups"; timeout 300 $B --streams 16 --groups 8 2>/dev/null | python -c "$P"
echo "== 16/4 pose cs 2"; LIVECAP_POSE_CLUSTER=2 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 16/4 surf cs 4"; LIVECAP_SURFACE_CLUSTER=4 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 24/6 surf cs 4"; LIVECAP_SURFACE_CLUSTER=4 timeout 300 $B --streams 24 --groups 6 2>/dev/null | python -c "$P"
echo "== 32/8 pose cs 2 surf cs 4"; LIVECAP_POSE_CLUSTER=2 LIVECAP_SURFACE_CLUSTER=4 timeout 300 $B --streams 32 --groups 8 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
