# PDL early trigger (build_var/pdl, -DLC_PDL_EARLY_TRIGGER) vs the default build on the final code
O=gpurun_out/r02pdl; mkdir -p $O
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
for v in default pdl default pdl default pdl; do
  if [ $v = default ]; then L=""; else L="LIVECAP_LIB=build_var/$v/liblivecap.so"; fi
  echo "== $v"; env $L timeout 300 $B 2>/dev/null | python -c "$P"
done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
LIVECAP_LIB=build_var/pdl/liblivecap.so timeout 600 python -m pytest tests -m gpu -q -x -k "tracker or frame or golden" > $O/pytest_pdl.log 2>&1; echo "pytest pdl rc=$?"; tail -1 $O/pytest_pdl.log
