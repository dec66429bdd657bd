# final check after the k_rim launch-bounds edit: full gpu suite, smoke, one bench line
O=gpurun_out/r02chk; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["frac"],4))'
