import sys, numpy as np
_R = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, _R + '/tests')
from test_gpu_stages import _surface, _mirror
from helpers import scene, bbox_diag
from oracle import surface as OS
from paper_1810_02648_b200.nonrigid_stage import solve_nonrigid, snap_vertices
actor, cam, frames = scene('small', 128, 3)
for frame in (0, 1, 2):
    pb, v_init = _surface(actor, cam, frames, directional=False, frame=frame)
    vo, logs, tot = OS.solve_surface(pb, v_init)
    vg, rep = solve_nonrigid(_mirror(pb, actor), v_init)
    print(frame, 'solve dv', np.abs(vg - vo).max(), [(round(o['energy_before'], 6), o['halvings']) for o in logs])
    print('   gpu', [(round(it.energy_before, 6), it.halvings) for it in rep.iterations])
    so, info = OS.snap(vo, pb)
    sg, ginfo = snap_vertices(vo, _mirror(pb, actor))
    print('   snap dv', np.abs(sg - so).max(), info['walked'], info['reached'], info['stuck'], '| gpu', ginfo.walked, ginfo.reached, ginfo.stuck)
    bad = np.argsort(-np.abs(sg - so).max(1))[:3]
    print('   worst', bad, np.abs(sg - so).max(1)[bad])
