"""Device timeline of the bench workload's steady steps (LIVECAP_TRACE=1):
solve-stream (lane 0) and preprocessing-stream (lane 1) marks, in ms.
  python tools/trace_step.py [--streams 8 --steps 3]"""
import argparse
import ctypes as C
import os
import sys

os.environ["LIVECAP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--skip", type=int, default=4, help="untraced steps first")
    a = ap.parse_args()
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    stream = torch.cuda.Stream(priority=-1)
    ctx = _lib.Context(0, stream.cuda_stream)
    actor = S.build_actor("x5k", with_skirt=True)
    cam = suggest_camera(1024, 1024)
    F = a.skip + a.steps + 2
    frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx))
              for s in range(a.streams)]
    img = torch.empty((a.streams, F, 1024, 1024, 3), dtype=torch.float64, device="cuda")
    msk = torch.empty((a.streams, F, 1024, 1024), dtype=torch.uint8, device="cuda")
    for s in range(a.streams):
        for f in range(F):
            img[s, f].copy_(torch.from_numpy(frames[s][f].image))
            msk[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
    torch.cuda.synchronize()
    tr = Tracker(actor, cam, SequenceConfig(directional=False), a.streams, ctx=ctx)   # the bench workload

    def q(f):
        for s in range(a.streams):
            tr.set_frame(s, img[s, f].data_ptr(), msk[s, f].data_ptr(), frames[s][f].detections, on_device=True)
    buf = C.create_string_buffer(1 << 20)
    q(0)
    q(1)
    for f in range(a.skip):
        q(f + 2)
        tr.step()
    ctx.synchronize()
    ctx.lib.lc_trace_dump(ctx.handle, buf, len(buf))   # discard warm-up marks
    for f in range(a.skip, a.skip + a.steps):
        q(f + 2)
        tr.step()
    ctx.synchronize()
    ctx.lib.lc_trace_dump(ctx.handle, buf, len(buf))
    prev = {0: 0.0, 1: 0.0}
    for line in buf.value.decode().splitlines():
        lane, name, t = line.split()
        lane, t = int(lane), float(t)
        print(f"{'  ' * 0 if lane == 0 else ' ' * 40}{name:<20} {t:8.3f}  (+{t - prev.get(lane, 0):.3f})")
        prev[lane] = t


if __name__ == "__main__":
    main()
