# r02: bounding the auxiliary stream's candidate-list grid
O=gpurun_out/r02aw; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
for g in 0 32 64 128 256 0; do echo "== cand grid $g"; LIVECAP_CAND_GRID=$g timeout 300 $B 2>/dev/null | python -c "$P"; done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
