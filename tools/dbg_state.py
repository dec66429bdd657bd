import sys, numpy as np
_R = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, _R + '/tests')
from helpers import scene
from oracle import frame as OF
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
actor, cam, frames = scene('small', 128, 3)
cfg = SequenceConfig(directional=False)
tr = Tracker(actor, cam, cfg, 1)
st = OF.State()
for k, fr in enumerate(frames):
    tr.set_frame(0, fr.image, fr.mask, fr.detections); tr.step()
    x, v, vs, rep = tr.result(0)
    prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
    xo, vo, vso, st, pl, sl = OF.solve_frame(prep, actor, cam, cfg, st)
    g = tr.get_state(0)
    def d(a, b):
        if a is None or b is None: return (a is None, b is None)
        a = a.to_vector() if hasattr(a, 'to_vector') else a
        return float(np.abs(np.asarray(a) - np.asarray(b)).max())
    print(k, 'x', d(x, xo), 'v', d(v, vo), 'vs', d(vs, vso),
          'state: xp', d(g.pose_prev, st.x_prev), 'xp2', d(g.pose_prev2, st.x_prev2), 'jp', d(g.joints_prev, st.joints_prev),
          'disp', d(g.disp_rest, st.disp_rest), 'vp', d(g.v_prev, st.v_prev), 'vp2', d(g.v_prev2, st.v_prev2))
    print('   pose halv gpu', [rep.pose.halvings[i] for i in range(rep.pose.n_iterations)], 'oracle', [o['halvings'] for o in pl])
    print('   nr halv gpu', [rep.nonrigid.halvings[i] for i in range(rep.nonrigid.n_iterations)], 'oracle', [o['halvings'] for o in sl], 'B', rep.nonrigid.n_boundary, 'P', rep.nonrigid.n_visible, 'snap', rep.nonrigid.snap_walked, rep.nonrigid.snap_reached, rep.nonrigid.snap_stuck)
