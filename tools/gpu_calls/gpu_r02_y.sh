# r02: candidate-list radius after the disabled-row query skip; concurrency probe
O=gpurun_out/r02y; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
for r in 48 64 96 128 192; do echo "== radius $r"; LIVECAP_LIST_RADIUS=$r timeout 300 $B 2>/dev/null | python -c "$P"; done
echo "== skip pyr"; LIVECAP_PROBE_SKIP_PYR=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== 24 streams 6 groups"; timeout 300 $B --streams 24 --groups 6 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 600 python tools/busy_probe.py --streams 16 --groups 4 --steps 10 > $O/busy16.txt 2>&1; cat $O/busy16.txt
