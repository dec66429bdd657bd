# r02: pyramid region of interest (+ exact on-demand blur outside): parity, bench
O=gpurun_out/r02v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_frame.py tests/test_gpu_bench_parity.py tests/test_gpu_stages.py -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4))'
{
echo "== default (margin 64)"; timeout 300 $B 2>/dev/null | python -c "$P"
echo "== margin 32"; LIVECAP_PYR_MARGIN=32 timeout 300 $B 2>/dev/null | python -c "$P"
echo "== margin -1 (full)"; LIVECAP_PYR_MARGIN=-1 timeout 300 $B 2>/dev/null | python -c "$P"
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 600 python tools/busy_probe.py --streams 16 --groups 4 --steps 10 > $O/busy16.txt 2>&1; cat $O/busy16.txt
