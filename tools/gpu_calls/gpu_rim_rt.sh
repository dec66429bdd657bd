# rim: warp-cooperative scans + per-vertex near list; raster: work items from a per-stream counter. A/B against build_var/prev
O=gpurun_out/r02rr; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "render or raster or contour or sets or tracker or frame or golden or bench or edge or stages or dropin" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{
for v in default prev default prev; do
  if [ $v = default ]; then L=""; else L="LIVECAP_LIB=build_var/$v/liblivecap.so"; fi
  echo "== $v"; env $L timeout 300 $B 2>/dev/null | python -c "$P"
done
} > $O/sweep.txt 2>&1; cat $O/sweep.txt
for v in default prev; do
  if [ $v = default ]; then L=""; else L="LIVECAP_LIB=build_var/$v/liblivecap.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rim|k_rt_tiles|k_rt_scan|k_own_cells" --csv python tools/profile_step.py --streams 4 --frames 4 > $O/ncu_list_$v.csv 2>&1
done
python tools/launch_summary.py $O/ncu_list_default.csv | head -8
python tools/launch_summary.py $O/ncu_list_prev.csv | head -8
