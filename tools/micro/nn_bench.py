"""Time DistanceField queries on an x5k 1024^2 silhouette (near-contour and far
queries) and check them against the oracle on a subsample.
  python tools/micro/nn_bench.py [libpath]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1810_02648_b200 import _lib
if len(sys.argv) > 1:
    _lib.load_library(sys.argv[1])
import bench
from paper_1810_02648_b200 import synthetic as S, imageproc as G
from paper_1810_02648_b200.camera import suggest_camera
from oracle import imaging as OI
ctx = _lib.default_context()
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
fr = bench.make_stream_frames(actor, cam, 1, 0, bench.device_renderer(ctx), bench.device_posing(ctx))[0]
g = G.DistanceField(fr.mask)
o = OI.DistanceField(fr.mask)
rng = np.random.default_rng(0)
pts = o.points
for name, q in (("near", pts[rng.integers(0, len(pts), 200000)] + rng.uniform(-6, 6, (200000, 2))),
                ("far", rng.uniform(0, 1023, (200000, 2)))):
    g.sample_value(q[:1000])
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        gd, _ = g.sample_value(q)
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / 5
    od, _ = o.sample_value(q[:20000])
    print(f"{name}: {len(q) / dt / 1e6:.1f} Mq/s (incl. transfer) exact={np.array_equal(gd[:20000], od)}")
