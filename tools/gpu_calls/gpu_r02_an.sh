# r02: stream / group sweep on the final build
O=gpurun_out/r02an; mkdir -p $O
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
for sg in "16 2" "16 4" "16 8" "24 6" "32 8" "16 4"; do set -- $sg; echo "== $1 streams $2 groups"; timeout 400 $B --streams $1 --groups $2 2>/dev/null | python -c "$P"; done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
