"""Distribution of line-search halvings on the bench workload (pose and surface)."""
import os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker
ctx = _lib.default_context()
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
F = 30
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx)) for s in range(8)]
tr = Tracker(actor, cam, SequenceConfig(), 8, ctx=ctx)
hp, hs = collections.Counter(), collections.Counter()
for f in range(F):
    for s in range(8):
        tr.set_frame(s, frames[s][f].image, frames[s][f].mask, frames[s][f].detections)
    tr.step()
    if f < 3:
        continue
    for s in range(8):
        _, _, _, rep = tr.result(s)
        for k in range(rep.pose.n_iterations):
            hp[rep.pose.halvings[k]] += 1
        for k in range(rep.nonrigid.n_iterations):
            hs[rep.nonrigid.halvings[k]] += 1
print("pose halvings", sorted(hp.items()))
print("surface halvings", sorted(hs.items()))
