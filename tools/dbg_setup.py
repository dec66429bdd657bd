import sys, numpy as np
_R = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, _R + '/tests')
from helpers import scene
from oracle import frame as OF
from paper_1810_02648_b200.config import SequenceConfig, TrackState
from paper_1810_02648_b200.device import Tracker
actor, cam, frames = scene('small', 128, 3)
cfg = SequenceConfig(directional=False)
tr = Tracker(actor, cam, cfg, 1)
st = OF.State()
for k, fr in enumerate(frames):
    tr.set_state(0, TrackState(st.x_prev, st.x_prev2, st.joints_prev, st.disp_rest, st.v_prev, st.v_prev2))
    tr.set_frame(0, fr.image, fr.mask, fr.detections); tr.step()
    ins = tr.inspect(0)
    prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
    trace = []
    xo, vo, vso, st2, pl, sl = OF.solve_frame(prep, actor, cam, cfg, st, trace)
    pb = [t for t in trace if t[0] == 'surface_problem'][0][1]['problem']
    vi = [t for t in trace if t[0] == 'surface_problem'][0][1]['v_init']
    print(k, 'v_init', np.abs(ins['v_init'] - vi).max(), 'vs', np.abs(ins['skinned'] - pb.skinned).max())
    print('   boundary equal', np.array_equal(ins['boundary'], pb.boundary_idx), len(ins['boundary']), len(pb.boundary_idx),
          'visible equal', np.array_equal(ins['visible'], pb.visible))
    if np.array_equal(ins['boundary'], pb.boundary_idx):
        diff = np.flatnonzero(ins['enabled'] != pb.enabled)
        print('   enabled diffs', diff, ins['enabled'][diff], pb.enabled[diff], 'n2d', np.abs(ins['normals2d'] - pb.normals2d).max())
    st = st2
