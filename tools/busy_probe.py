"""Per-kernel concurrency on the bench workload: for each kernel, the sum of
its launch durations and the union of its launch intervals (CUDA events on
each group's solve stream) per step, next to the step time.  union << sum:
the groups' launches of that kernel overlap; union ~ sum: they serialise.

  python tools/busy_probe.py [--streams 16 --groups 4 --steps 10]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

KERNELS = ["k_pose_solve", "k_surface_solve", "k_cand_build", "k_pyramid_fused", "k_rt_tiles", "k_rim", "k_fk",
           "k_own_cells", "k_contour_compact", "k_cell_jfa"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--groups", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import BatchTracker
    ctx = _lib.default_context()
    actor = S.build_actor("x5k", with_skirt=True)
    cam = suggest_camera(1024, 1024)
    n_runs = len(KERNELS) + 1
    F = 3 + n_runs * a.steps + 2
    frames = [bench.make_stream_frames(actor, cam, F, s, bench.device_renderer(ctx), bench.device_posing(ctx))
              for s in range(a.streams)]
    img = torch.empty((a.streams, F, 1024, 1024, 3), dtype=torch.float64, device="cuda")
    msk = torch.empty((a.streams, F, 1024, 1024), dtype=torch.uint8, device="cuda")
    for s in range(a.streams):
        for f in range(F):
            img[s, f].copy_(torch.from_numpy(frames[s][f].image))
            msk[s, f].copy_(torch.from_numpy(frames[s][f].mask.astype(np.uint8)))
    torch.cuda.synchronize()
    tr = BatchTracker(actor, cam, SequenceConfig(directional=False), a.streams, groups=a.groups)

    def q(f):
        for s in range(a.streams):
            tr.set_frame(s, img[s, f].data_ptr(), msk[s, f].data_ptr(), frames[s][f].detections, on_device=True)
    q(0)
    q(1)
    f = 0
    for _ in range(3):
        q(f + 2)
        tr.step()
        f += 1
    tr.synchronize()
    for name in [None] + KERNELS:
        tr.profile_kernel(name)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            q(f + 2)
            tr.step()
            f += 1
        tr.synchronize()
        step_ms = 1e3 * (time.perf_counter() - t0) / a.steps
        if name is None:
            print(f"step {step_ms:.3f} ms ({a.streams} streams, {a.groups} groups, no profiling)")
            continue
        ms, n = tr.profile_read()
        busy = tr.profile_busy_ms()
        print(f"{name:<20} launches/step {n / a.steps:5.1f}  sum {ms / a.steps:7.3f} ms/step  "
              f"union {busy / a.steps:7.3f} ms/step  (step {step_ms:.3f} ms)")
        tr.profile_kernel(None)


if __name__ == "__main__":
    main()
