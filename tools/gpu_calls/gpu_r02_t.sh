# r02: hybrid assembly (edge pass + owner-computes rows/blocks); 8-CTA default surface team at x5k
O=gpurun_out/r02t; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_stages.py tests/test_gpu_frame.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for cs in 4 8; do echo "== cs $cs"; LIVECAP_SURFACE_CLUSTER=$cs timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases 2>&1 | grep -E "^frame 3" -A8; done > $O/phases4.txt; cat $O/phases4.txt
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== mode 0"; LIVECAP_PCG_MODE=0 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== mode 1"; LIVECAP_PCG_MODE=1 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== cfg4"; timeout 300 $B --preset x20k --gn 4 --pcg 8 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
