"""Probe the e2e path: pinned H2D bandwidth, host enqueue time per step."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_1810_02648_b200 import _lib, synthetic as S
from paper_1810_02648_b200.camera import suggest_camera
from paper_1810_02648_b200.config import SequenceConfig
from paper_1810_02648_b200.device import Tracker

x = torch.empty((8, 1024, 1024, 3), dtype=torch.float64, pin_memory=True)
d = torch.empty_like(x, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize()
print(f"torch pinned H2D: {x.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
stream = torch.cuda.Stream(priority=-1)
ctx = _lib.Context(0, stream.cuda_stream)
actor = S.build_actor("x5k", with_skirt=True)
cam = suggest_camera(1024, 1024)
F = 8
frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx)) for s in range(8)]
img_h = torch.empty((8, F, 1024, 1024, 3), dtype=torch.float64, pin_memory=True)
msk_h = torch.empty((8, F, 1024, 1024), dtype=torch.uint8, pin_memory=True)
for s in range(8):
    for f in range(F):
        img_h[s, f].copy_(torch.from_numpy(frames[s][f].image))
        msk_h[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
tr = Tracker(actor, cam, SequenceConfig(), 8, ctx=ctx)
# upload-only timing through set_frame (copy stream)
for f in range(2):
    ctx.synchronize(); t0 = time.perf_counter()
    for s in range(8):
        tr.set_frame(s, img_h[s, f].numpy(), msk_h[s, f].numpy(), frames[s][f].detections)
    t1 = time.perf_counter(); ctx.synchronize(); t2 = time.perf_counter()
    print(f"set_frame x8: host {1e3*(t1-t0):.2f} ms, upload done after {1e3*(t2-t0):.2f} ms "
          f"({8 * (1024*1024*25) / (t2 - t0) / 1e9:.1f} GB/s)")
    tr.step(); ctx.synchronize()
# host enqueue time of a step
for f in range(2, 6):
    for s in range(8):
        tr.set_frame(s, img_h[s, f].numpy(), msk_h[s, f].numpy(), frames[s][f].detections)
    ctx.synchronize()
    t0 = time.perf_counter(); tr.step(); t1 = time.perf_counter(); ctx.synchronize(); t2 = time.perf_counter()
    print(f"step: host enqueue {1e3*(t1-t0):.2f} ms, device done after {1e3*(t2-t0):.2f} ms")

# e2e loop variants
tr.close()
def loop(readback, ahead, nsteps=5):
    t = Tracker(actor, cam, SequenceConfig(), 8, ctx=ctx)
    N = actor.mesh.n_vertices
    xh = torch.empty((2, 8, 36), dtype=torch.float64, pin_memory=True)
    vh = torch.empty((2, 8, N, 3), dtype=torch.float64, pin_memory=True)
    ev = [torch.cuda.Event(), torch.cuda.Event()]
    def q(f):
        for s in range(8):
            t.set_frame(s, img_h[s, f % F].numpy(), msk_h[s, f % F].numpy(), frames[s][f % F].detections)
    for f in range(ahead):
        q(f)
    ctx.synchronize()
    t0 = time.perf_counter()
    for f in range(nsteps):
        q(f + ahead)
        t.step()
        if readback:
            for s in range(8):
                t.result_async(s, xh[f & 1, s], vh[f & 1, s])
            ev[f & 1].record(stream)
            if f:
                ev[(f - 1) & 1].synchronize()
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / nsteps
    t.close()
    print(f"loop readback={readback} ahead={ahead}: {1e3 * dt:.2f} ms/step")
for rb in (False, True):
    for ah in (1, 2):
        loop(rb, ah)
