# r02: what saturates frames/s: per-kernel concurrency probe, skip-preprocessing probe, team-size / stream sweeps
O=gpurun_out/r02q; mkdir -p $O
timeout 600 python tools/busy_probe.py --streams 16 --groups 4 --steps 10 > $O/busy16.txt 2>&1; cat $O/busy16.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3))'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== skip prep probe"; LIVECAP_PROBE_SKIP_PREP=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pose cs 2"; LIVECAP_POSE_CLUSTER=2 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pose cs 2, 24 streams"; LIVECAP_POSE_CLUSTER=2 timeout 300 $B --streams 24 --groups 6 2>/dev/null | python -c "$P"
echo "== surf cs 8"; LIVECAP_SURFACE_CLUSTER=8 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pcg mode 1"; LIVECAP_PCG_MODE=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 8 streams 2 groups"; timeout 300 $B --streams 8 --groups 2 2>/dev/null | python -c "$P"
echo "== 8 streams 1 group"; timeout 300 $B --streams 8 --groups 1 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
