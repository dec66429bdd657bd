"""CPU model of the tile binning on late bench frames (Stage II raster input)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import ctypes as C
import numpy as np
import torch
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
ctx = _lib.default_context()
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
F = 30
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx)) for s in range(2)]
tr = Tracker(actor, cam, SequenceConfig(), 2, ctx=ctx)
tris = actor.mesh.triangles
N = actor.mesh.n_vertices
for f in range(F):
    for s in range(2):
        tr.set_frame(s, frames[s][f].image, frames[s][f].mask, frames[s][f].detections)
    tr.step()
    if f < 24:
        continue
    ctx.synchronize()
    v = np.empty((N, 3)); n = C.c_int64()
    _lib.check(ctx.lib.lc_tracker_inspect(tr.handle, 0, 4, _lib.ptr(v), 3 * N, C.byref(n)))
    z = v[:, 2]
    px = cam.fx * v[:, 0] / z + cam.cx
    py = cam.fy * v[:, 1] / z + cam.cy
    P = np.stack([px[tris], py[tris]], -1)
    D = z[tris]
    ok = (D > 0).all(1)
    area = (P[:, 1, 0] - P[:, 0, 0]) * (P[:, 2, 1] - P[:, 0, 1]) - (P[:, 2, 0] - P[:, 0, 0]) * (P[:, 1, 1] - P[:, 0, 1])
    ok &= np.abs(area) >= 1e-12
    x0 = np.clip(np.floor(P[..., 0].min(1)), 0, 1023); x1 = np.clip(np.ceil(P[..., 0].max(1)), 0, 1023)
    y0 = np.clip(np.floor(P[..., 1].min(1)), 0, 1023); y1 = np.clip(np.ceil(P[..., 1].max(1)), 0, 1023)
    ok &= (x0 <= x1) & (y0 <= y1)
    ntiles = ((x1 // 16 - x0 // 16 + 1) * (y1 // 16 - y0 // 16 + 1)) * ok
    big = np.abs(P).max((1, 2))
    print(f"frame {f}: ok {ok.sum()} bbox-tile entries {int(ntiles.sum())}, tris >64 tiles {(ntiles > 64).sum()}, "
          f"max tiles {int(ntiles.max())}, max|P| {big[ok].max():.3g}, min|area| of big {np.abs(area[ntiles > 64]).min() if (ntiles > 64).any() else 0:.3g}, "
          f"zmin {z.min():.3g}")
