"""Run the bench workload's tracker for a few frames (for ncu captures).

  python tools/profile_step.py --streams 8 --frames 4
Input generation (device renders) happens first: ncu filters should skip the
8*frames mode-1 renders when targeting raster kernels.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--preset", default="x5k")
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--phases", action="store_true")
    a = ap.parse_args()
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    ctx = _lib.default_context()
    actor = S.build_actor(a.preset, with_skirt=True)
    cam = suggest_camera(a.res, a.res)
    frames = [bench.make_stream_frames(actor, cam, a.frames, s, bench.device_renderer(ctx),
                                       bench.device_posing(ctx)) for s in range(a.streams)]
    tr = Tracker(actor, cam, SequenceConfig(directional=False), a.streams, ctx=ctx)   # the bench workload
    stats = hasattr(ctx.lib, "lc_debug_nn_stats_pose") if False else None
    try:
        import ctypes
        raw = ctypes.CDLL(_lib.LIB_PATH)
        stats = [getattr(raw, "lc_debug_nn_stats_" + k) for k in ("pose", "surface")]
    except (AttributeError, OSError):
        stats = None
    for f in range(a.frames):
        t0 = time.perf_counter()
        for s in range(a.streams):
            fr = frames[s][f]
            tr.set_frame(s, fr.image, fr.mask, fr.detections)
        tr.step()
        ctx.synchronize()
        print(f"frame {f}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
        if stats:
            import numpy as np
            for k, fn in zip(("pose", "surface"), stats):
                o = np.zeros(16, dtype=np.uint64)
                fn(o.ctypes.data, 1)
                q = max(int(o[0]), 1)
                print(f"   nn {k}: list queries {int(o[0])} entries/query {int(o[1]) / q:.1f} "
                      f"quadtree {int(o[2])} hinted {int(o[3])}"
                      + (f" | snap: slowest walk {int(o[4])} cyc / {int(o[5])} steps, max steps {int(o[6])}, "
                         f"total steps {int(o[7])}" if k == "surface" else "")
                      + f" | max scanned {int(o[8])} max list {int(o[9])} hist/64 {[int(x) for x in o[10:16]]}")
        if a.phases:
            import numpy as np
            worst = {}
            for st in range(a.streams):
                pp, ss = np.zeros(64, dtype=np.int64), np.zeros(64, dtype=np.int64)
                _lib.check(ctx.lib.lc_tracker_phase_times(tr.handle, st, _lib.ptr(pp), _lib.ptr(ss)))
                for name, arr, n in (("pose", pp, 19), ("surface", ss, 11)):
                    d = np.diff(arr[:n]) / 1e3
                    if d.min() < 0:
                        continue
                    if name not in worst or d.sum() > worst[name][1].sum():
                        worst[name] = (st, d)
            for name, (st, d) in worst.items():
                print(f"   slowest {name} stream {st} (us): " + " ".join(f"{x:.0f}" for x in d) + f"  total {d.sum():.0f}")
            # fine sub-phase stamps (GN iteration 1): pose eval+J [32..37], pose trial [40..45],
            # surface assembly [16..21], snap [24..29]
            pp, ss = np.zeros(64, dtype=np.int64), np.zeros(64, dtype=np.int64)
            _lib.check(ctx.lib.lc_tracker_phase_times(tr.handle, 0, _lib.ptr(pp), _lib.ptr(ss)))
            for name, arr, a0, n in (("pose evalJ", pp, 32, 6), ("pose rows|jtj", pp[[34, 38, 35]], 0, 3), ("pose trial", pp, 40, 6),
                                     ("surf asm", ss, 16, 5), ("surf snap", ss, 24, 5),
                                     ("surf pcg init|mv|red1|upd|red2|p", ss, 40, 7)):
                d = np.diff(arr[a0:a0 + n]) / 1e3
                print(f"   stream0 {name} (us): " + " ".join(f"{x:.1f}" for x in d))


if __name__ == "__main__":
    main()
