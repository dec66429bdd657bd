"""Does a pinned H2D copy overlap a running solve?"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker

stream = torch.cuda.Stream(priority=-1)
ctx = _lib.Context(0, stream.cuda_stream)
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
F = 4
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx)) for s in range(8)]
img_d = torch.empty((8, F, 1024, 1024, 3), dtype=torch.float64, device="cuda")
msk_d = torch.empty((8, F, 1024, 1024), dtype=torch.uint8, device="cuda")
for s in range(8):
    for f in range(F):
        img_d[s, f].copy_(torch.from_numpy(frames[s][f].image))
        msk_d[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
tr = Tracker(actor, cam, SequenceConfig(), 8, ctx=ctx)
host = torch.empty((8, 1024, 1024, 3), dtype=torch.float64, pin_memory=True)
dev = torch.empty_like(host, device="cuda")
cs = torch.cuda.Stream()
def q(f):
    for s in range(8):
        tr.set_frame(s, img_d[s, f % F].data_ptr(), msk_d[s, f % F].data_ptr(), frames[s][f % F].detections, on_device=True)
for mode in ("solve", "copy", "both", "solve", "both"):
    torch.cuda.synchronize(); ctx.synchronize()
    t0 = time.perf_counter()
    for f in range(4):
        if mode in ("copy", "both"):
            with torch.cuda.stream(cs):
                dev.copy_(host, non_blocking=True)
        if mode in ("solve", "both"):
            q(f); tr.step()
    torch.cuda.synchronize(); ctx.synchronize()
    print(f"{mode}: {1e3 * (time.perf_counter() - t0) / 4:.2f} ms/iter")
