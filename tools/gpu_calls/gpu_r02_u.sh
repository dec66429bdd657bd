# r02: preprocessing cost split (grid vs pyramid) and candidate-list radius on the in-track workload
O=gpurun_out/r02u; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== skip grid"; LIVECAP_PROBE_SKIP_GRID=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== skip pyr"; LIVECAP_PROBE_SKIP_PYR=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== skip both"; LIVECAP_PROBE_SKIP_PREP=1 timeout 300 $B 2>/dev/null | python -c "$P"
for r in 32 64 128; do echo "== radius $r"; LIVECAP_LIST_RADIUS=$r timeout 300 $B 2>/dev/null | python -c "$P"; done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 600 python tools/busy_probe.py --streams 16 --groups 4 --steps 10 > $O/busy16.txt 2>&1; cat $O/busy16.txt
