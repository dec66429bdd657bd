# r02: dropin fix check, solver phase breakdown, device timeline, surface ncu full capture
set -x
O=gpurun_out/r02n; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dropin.py -q -rf > $O/pytest_dropin.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_dropin.log
timeout 300 python tools/profile_step.py --streams 4 --frames 5 --phases > $O/phases4.txt 2>&1; echo "phases rc=$?"
timeout 300 python tools/profile_step.py --streams 1 --frames 5 --phases > $O/phases1.txt 2>&1; echo "phases rc=$?"
timeout 300 python tools/trace_step.py --streams 4 --steps 2 > $O/trace4.txt 2>&1; echo "trace rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_surface_solve -s 3 -c 1 -o $O/k_surface_solve \
      python tools/profile_step.py --streams 4 --frames 5 > $O/ncu_k_surface_solve.log 2>&1; echo "ncu rc=$?"
