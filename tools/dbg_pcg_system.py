"""Compare the tracker's compact Stage II normal system and PCG iterate with
the oracle's (reference layout) at the Stage II start surface of a bench
frame: gn_iterations = 1, so both assemble at v_init; PCG iterations 1..8.

  python tools/dbg_pcg_system.py [--frame 3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frame", type=int, default=3)
    a = ap.parse_args()
    from helpers import oracle_state_to_mirror, scene_bench
    from oracle import frame as OF
    from oracle import linsolve as LS
    from oracle.surface import normal_system, surface_evaluate
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene_bench("x5k", 1024, a.frame + 1, 0)
    cfg = SequenceConfig(directional=False)
    st = OF.State()
    for fr in frames[:a.frame]:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        st = OF.solve_frame(prep, actor, cam, cfg, st)[3]
    fr = frames[a.frame]
    prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
    trace = []
    xo = OF.solve_frame(prep, actor, cam, cfg, st, trace=trace)[0]
    pb = [t for t in trace if t[0] == "surface_problem"][0][1]
    prob, v0 = pb["problem"], pb["v_init"]
    ev = surface_evaluate(prob, v0, 0)
    diag, off, rows, cols, rhs = normal_system(prob, ev)

    def sym(m):
        return np.stack([m[:, 0, 0], m[:, 0, 1], m[:, 0, 2], m[:, 1, 1], m[:, 1, 2], m[:, 2, 2]], 1)

    for iters in (1, 2, 4, 8):
        c = SequenceConfig(directional=False)
        c.nonrigid.gn_iterations = 1
        c.nonrigid.pcg_iterations = iters
        c.enable_snapping = False
        B = Tracker(actor, cam, c, 1)
        B.set_state(0, oracle_state_to_mirror(st))
        B.set_frame(0, fr.image, fr.mask, fr.detections)
        B.set_pose(0, xo)
        B.step_stage(2)
        g = B.inspect_system(0)
        B.close()
        d_ref = LS.pcg(diag, off, rows, cols, rhs, iters)[0]
        dd = np.abs(g["diag"] - sym(diag)).max() / np.abs(diag).max()
        dr = np.abs(g["rhs"] - rhs).max() / np.abs(rhs).max()
        db = np.abs(g["best"] - d_ref).max() / np.abs(d_ref).max()
        worst = np.argsort(-np.abs(g["best"] - d_ref).max(1))[:5]
        print(f"pcg {iters}: diag rel {dd:.2e} rhs rel {dr:.2e} delta rel {db:.2e}; worst vertices "
              f"{worst.tolist()} deg {actor.mesh.degrees[worst].tolist()}", flush=True)
        if iters == 1:
            err = np.abs(g["diag"] - sym(diag)).max(1)
            wd = np.argsort(-err)[:5]
            print("   worst diag vertices", wd.tolist(), "deg", actor.mesh.degrees[wd].tolist(), err[wd].tolist())
            err = np.abs(g["rhs"] - rhs).max(1)
            wr = np.argsort(-err)[:5]
            print("   worst rhs vertices", wr.tolist(), "deg", actor.mesh.degrees[wr].tolist(), err[wr].tolist())


if __name__ == "__main__":
    main()
