# aux-kernel grid caps on the final build (pyramid / candidate lists)
O=gpurun_out/r02gr; mkdir -p $O
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pyr grid 148"; LIVECAP_PYR_GRID=148 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== pyr grid 0 (one CTA per tile)"; LIVECAP_PYR_GRID=0 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== cand grid 128"; LIVECAP_CAND_GRID=128 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== cand grid 512"; LIVECAP_CAND_GRID=512 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
