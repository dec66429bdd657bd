import sys, numpy as np
_R = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, _R + '/tests')
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
ctx = _lib.default_context()
preset, res, nf = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
actor = S.build_actor(preset, with_skirt=True); cam = suggest_camera(res, res)
frames = bench.make_stream_frames(actor, cam, nf, 0, bench.device_renderer(ctx), bench.device_posing(ctx))
tr = Tracker(actor, cam, SequenceConfig(), 1, ctx=ctx)
for f in range(nf):
    fr = frames[f]
    tr.set_frame(0, fr.image, fr.mask, fr.detections); tr.step()
    x, v, vs, rep = tr.result(0)
    p = rep.pose; n = rep.nonrigid
    gt = fr.gt_vertices
    print(f, 'x finite', np.isfinite(x).all(), 'v finite', np.isfinite(v).all(), 'verr', np.abs(v-gt).max(),
          'pose e', [round(p.energy_after[k],1) for k in range(p.n_iterations)][-3:], 'halv', [p.halvings[k] for k in range(p.n_iterations)][-6:],
          'nr', [(round(n.energy_before[k],1), n.halvings[k]) for k in range(n.n_iterations)], 'P', n.n_visible, 'B', n.n_boundary, 'contour', p.n_contour)
