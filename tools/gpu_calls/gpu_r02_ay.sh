# r02: does FMA in the pose J^T J change Stage I parity? cfg2 100 frames, pose-parameter deviation per build
O=gpurun_out/r02ay; mkdir -p $O
python -c "from paper_1810_02648_b200 import _build as b; b.build_variant('/tmp/lc_nofma/liblivecap.so', ['LC_POSE_JTJ_NOFMA'])" && echo built
cat > /tmp/posedev.py <<'PY'
import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from helpers import scene_bench, oracle_state_to_mirror
from oracle import frame as OF
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
actor, cam, frames = scene_bench("x5k", 1024, 40, seed=0)
cfg = SequenceConfig(mode="pose_only")
A = Tracker(actor, cam, cfg, 1)
st = OF.State(); devs = []
for fr in frames:
    prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
    xo, vo, _, st_new, plogs, _ = OF.solve_frame(prep, actor, cam, cfg, st)
    A.set_state(0, oracle_state_to_mirror(st)); A.set_frame(0, fr.image, fr.mask, fr.detections); A.step()
    x, v, _, _ = A.result(0)
    devs.append(float(np.abs(x - xo).max())); st = st_new
print("max pose dev", max(devs), "frame", int(np.argmax(devs)), "median", float(np.median(devs)))
PY
timeout 900 python /tmp/posedev.py > $O/fma.txt 2>&1; echo "fma rc=$?"; tail -1 $O/fma.txt
LIVECAP_LIB=/tmp/lc_nofma/liblivecap.so timeout 900 python /tmp/posedev.py > $O/nofma.txt 2>&1; echo "nofma rc=$?"; tail -1 $O/nofma.txt
