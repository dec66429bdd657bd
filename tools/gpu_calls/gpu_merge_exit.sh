# raster merge returns at once when no tile was split; raster/frame parity + bench + launch times
O=gpurun_out/r02mg; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "render or raster or tracker or frame or golden or bench or sets or edge" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e-u8 --no-quality"
P='import json,sys; d=json.load(sys.stdin); print(round(d["value"]), round(d["ms_per_step"],3), d["pcg_iter_us"], round(d["roofline"]["kernel_ms_per_launch"],3), round(d["roofline"]["frac"],4), round(d["roofline"]["frac_concurrent"],4))'
{ for i in 1 2; do echo "== default"; timeout 300 $B 2>/dev/null | python -c "$P"; done; } > $O/sweep.txt 2>&1; cat $O/sweep.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rt_merge|k_rt_tiles" --csv python tools/profile_step.py --streams 4 --frames 4 > $O/ncu_list.csv 2>&1
python tools/launch_summary.py $O/ncu_list.csv | head -4
