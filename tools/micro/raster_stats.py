"""Triangle bbox statistics of the Stage II raster input (vinit) on the bench workload."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import ctypes as C
import numpy as np
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
ctx = _lib.default_context()
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
F = 6
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx)) for s in range(8)]
tr = Tracker(actor, cam, SequenceConfig(), 8, ctx=ctx)
tris = actor.mesh.triangles
N = actor.mesh.n_vertices
for f in range(F):
    for s in range(8):
        tr.set_frame(s, frames[s][f].image, frames[s][f].mask, frames[s][f].detections)
    tr.step()
    ctx.synchronize()
    line = []
    for s in range(8):
        v = np.empty((N, 3)); n = C.c_int64()
        _lib.check(ctx.lib.lc_tracker_inspect(tr.handle, s, 4, _lib.ptr(v), 3 * N, C.byref(n)))
        px = cam.fx * v[:, 0] / v[:, 2] + cam.cx
        py = cam.fy * v[:, 1] / v[:, 2] + cam.cy
        P = np.stack([px[tris], py[tris]], -1)
        x0 = np.clip(np.floor(P[..., 0].min(1)), 0, 1023); x1 = np.clip(np.ceil(P[..., 0].max(1)), 0, 1023)
        y0 = np.clip(np.floor(P[..., 1].min(1)), 0, 1023); y1 = np.clip(np.ceil(P[..., 1].max(1)), 0, 1023)
        bb = np.maximum(x1 - x0 + 1, 0) * np.maximum(y1 - y0 + 1, 0)
        big = bb > 256
        area = 0.5 * np.abs((P[:, 1, 0] - P[:, 0, 0]) * (P[:, 2, 1] - P[:, 0, 1]) - (P[:, 2, 0] - P[:, 0, 0]) * (P[:, 1, 1] - P[:, 0, 1]))
        line.append(f"s{s}: big {big.sum()} bbpx {int(bb[big].sum())} area {int(area[big].sum())} small_bbpx {int(bb[~big].sum())}")
    print(f"frame {f}: " + " | ".join(line[:4]))
