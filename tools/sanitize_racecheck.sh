# racecheck of the solver kernels: the in-tree build (its only reports are the
# light team reductions' remote-mbarrier handshake, which racecheck does not
# model) and the LC_TEAM_FULL_SYNC variant (cluster barriers everywhere)
set -x
O=${1:-gpurun_out/racecheck}; mkdir -p $O
python -c "from paper_1810_02648_b200 import _build as b; print(b.build_variant('/tmp/lc_fullsync/liblivecap.so', ['LC_TEAM_FULL_SYNC']))"
LIVECAP_LIB=/tmp/lc_fullsync/liblivecap.so timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py > $O/racecheck_fullsync_small.txt 2>&1; echo "racecheck fullsync rc=$?"; tail -3 $O/racecheck_fullsync_small.txt
LIVECAP_LIB=/tmp/lc_fullsync/liblivecap.so timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize.py --x5k > $O/racecheck_fullsync_x5k.txt 2>&1; echo "racecheck fullsync x5k rc=$?"; tail -3 $O/racecheck_fullsync_x5k.txt
