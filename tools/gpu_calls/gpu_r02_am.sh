O=gpurun_out/r02am; mkdir -p $O
timeout 300 python tools/trace_step.py --streams 4 --steps 2 > $O/trace4.txt 2>&1; echo "trace rc=$?"; tail -40 $O/trace4.txt
