"""Free-running tracking quality of the CPU oracle (bit-identical to the
reference) on the bench's synthetic streams: per frame, the silhouette IoU of
the solved surface against the observed mask and the centred mean vertex error
against the ground truth (metrics.py:26-46).  Used to choose a workload whose
timed frames are in track.

  python tools/track_quality.py --preset x5k --res 1024 --frames 40 --seeds 0-15 [--directional]
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    preset, res, n, seed, directional = a
    os.environ["OMP_NUM_THREADS"] = "1"
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import frame as OF, geometry as OG, imaging as OI, post as OP
    from paper_1810_02648_b200 import synthetic as S
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.config import SequenceConfig

    def posing(actor, pose, rest):
        fk = OG.Fk(actor.skeleton, pose.to_vector())
        return OG.skin(rest, actor.skinning, fk.dqs)[0], fk.pos, fk.markers

    actor = S.build_actor(preset, with_skirt=True)
    cam = suggest_camera(res, res)
    frames = S.generate_sequence(actor, cam, S.default_script(n, noise=S.NoiseParams(sigma2d=1.0, sigma3d=0.008,
                                                                                      seed=seed)),
                                 OI.render_attributes, posing)
    cfg = SequenceConfig(directional=directional)
    st = OF.State()
    ious, errs = [], []
    with threadpool_limits(1):
        for fr in frames:
            prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
            _, v, _, st, _, _ = OF.solve_frame(prep, actor, cam, cfg, st)
            m = np.isfinite(OI.render_depth(cam, v, actor.mesh.triangles))
            ious.append(OP.iou(m, fr.mask))
            errs.append(float(np.mean(np.linalg.norm((v - v.mean(0)) - (fr.gt_vertices - fr.gt_vertices.mean(0)),
                                                     axis=1))))
    return seed, ious, errs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="x5k")
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--frames", type=int, default=40)
    ap.add_argument("--seeds", default="0-15")
    ap.add_argument("--directional", action="store_true")
    ap.add_argument("--procs", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.seeds.split("-")) if "-" in a.seeds else (int(a.seeds), int(a.seeds))
    jobs = [(a.preset, a.res, a.frames, s, a.directional) for s in range(lo, hi + 1)]
    with mp.get_context("fork").Pool(min(a.procs, len(jobs))) as pool:
        res = pool.map(run, jobs)
    out = {"preset": a.preset, "res": a.res, "frames": a.frames, "directional": a.directional, "seeds": {}}
    for seed, ious, errs in res:
        out["seeds"][seed] = {"iou": ious, "vertex_error": errs}
        print(f"seed {seed:2d}: IoU min {min(ious):.3f} mean {sum(ious) / len(ious):.3f} last {ious[-1]:.3f}; "
              f"vertex err mean {1e3 * sum(errs) / len(errs):.1f} mm max {1e3 * max(errs):.1f} mm")
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main()
