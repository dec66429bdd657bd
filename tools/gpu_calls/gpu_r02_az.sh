# r02: nearest-contour query statistics (LC_NN_STATS variant build)
O=gpurun_out/r02az; mkdir -p $O
python -c "from paper_1810_02648_b200 import _build as b; b.build_variant('/tmp/lc_nnstats/liblivecap.so', ['LC_NN_STATS'])" && echo built
LIVECAP_LIB=/tmp/lc_nnstats/liblivecap.so timeout 300 python tools/profile_step.py --streams 4 --frames 5 > $O/nnstats.txt 2>&1; echo "rc=$?"; tail -12 $O/nnstats.txt
