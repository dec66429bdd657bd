# r02: surface kernel register budget / CTAs per SM (LC_SURF_MINB 3: 85 registers, 3 CTAs per SM) and 128-thread CTAs
O=gpurun_out/r02al; mkdir -p $O
python -c "from paper_1810_02648_b200 import _build as b; b.build_variant('/tmp/lc_minb3/liblivecap.so', ['LC_SURF_MINB=3'])" && echo built3
python -c "from paper_1810_02648_b200 import _build as b; b.build_variant('/tmp/lc_nt128/liblivecap.so', ['LC_SURF_NT=128', 'LC_SURF_MINB=4'])" && echo built128
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), d["input_generation_s"])'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== minb3"; LIVECAP_LIB=/tmp/lc_minb3/liblivecap.so timeout 300 $B 2>/dev/null | python -c "$P"
echo "== minb3 cs16"; LIVECAP_SURFACE_CLUSTER=16 LIVECAP_LIB=/tmp/lc_minb3/liblivecap.so timeout 300 $B 2>/dev/null | python -c "$P"
echo "== nt128 minb4 cs16"; LIVECAP_SURFACE_CLUSTER=16 LIVECAP_LIB=/tmp/lc_nt128/liblivecap.so timeout 300 $B 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
LIVECAP_LIB=/tmp/lc_minb3/liblivecap.so timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8
