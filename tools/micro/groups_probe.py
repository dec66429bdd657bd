"""Throughput of S streams split into G concurrently stepped groups (one
context / CUDA stream / Tracker per group) -- value-style loop, inputs in HBM."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker

NS, K, W = 8, 20, 3
F = K + W + 2
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
ctx0 = _lib.Context(0)
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx0), bench.device_posing(ctx0)) for s in range(NS)]
img = torch.empty((NS, F, 1024, 1024, 3), dtype=torch.float64, device="cuda")
msk = torch.empty((NS, F, 1024, 1024), dtype=torch.uint8, device="cuda")
for s in range(NS):
    for f in range(F):
        img[s, f].copy_(torch.from_numpy(frames[s][f].image))
        msk[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
torch.cuda.synchronize()
for G in [int(x) for x in sys.argv[1:]] or [1, 2, 4]:
    per = NS // G
    strs = [torch.cuda.Stream(priority=-1) for _ in range(G)]
    ctxs = [_lib.Context(0, st.cuda_stream) for st in strs]
    trs = [Tracker(actor, cam, SequenceConfig(), per, ctx=c) for c in ctxs]
    def q(f):
        for g in range(G):
            for s in range(per):
                gs = g * per + s
                trs[g].set_frame(s, img[gs, f].data_ptr(), msk[gs, f].data_ptr(), frames[gs][f].detections, on_device=True)
    q(0); q(1)
    for f in range(W):
        q(f + 2)
        for t in trs: t.step()
    for c in ctxs: c.synchronize()
    t0 = time.perf_counter()
    for f in range(W, W + K):
        q(f + 2)
        for t in trs: t.step()
    for c in ctxs: c.synchronize()
    dt = time.perf_counter() - t0
    print(f"G={G}: {NS * K / dt:.0f} frames/s ({1e3 * dt / K:.3f} ms/step)", flush=True)
    for t in trs: t.close()
