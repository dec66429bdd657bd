# PCG vertex-batch (LC_PCG_VA / LC_PCG_VB) parity + sweep; variant libraries in build_var/
O=gpurun_out/r02pcg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_bench_parity.py tests/test_gpu_frame.py tests/test_gpu_kernels.py -m gpu -q -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
for v in default v11 v22 v21 v33 v42 default v11; do
  if [ $v = default ]; then L=""; else L="LIVECAP_LIB=build_var/$v/liblivecap.so"; fi
  echo "== $v"; env $L timeout 300 $B 2>/dev/null | python -c "$P"
done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 300 python tools/profile_step.py --streams 4 --frames 4 --phases > $O/phases.txt 2>&1; tail -8 $O/phases.txt
