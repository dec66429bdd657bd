"""Diagnostics for the bench-workload parity (no asserts): per frame, Stage I
and Stage II (per-stage teacher forced, as tests/test_gpu_bench_parity.py)
energies GPU vs oracle per GN iteration, set equality of the Stage II setup,
and the vertex error.

  python tools/dbg_bench_frames.py [--frames 8] [--preset x5k --res 1024]
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
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--preset", default="x5k")
    ap.add_argument("--res", type=int, default=1024)
    ap.add_argument("--pcg-iters", type=int, default=None)
    a = ap.parse_args()
    from helpers import bbox_diag, oracle_state_to_mirror, scene_bench
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene_bench(a.preset, a.res, a.frames, 0)
    cfg = SequenceConfig(directional=False)
    if a.pcg_iters:
        cfg.nonrigid.pcg_iterations = a.pcg_iters
    B = Tracker(actor, cam, cfg, 1)
    st = OF.State()
    diag = bbox_diag(actor)
    n = actor.mesh.n_vertices
    for fr in frames:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        trace = []
        xo, vo, _, st_new, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st, trace=trace)
        B.set_state(0, oracle_state_to_mirror(st))
        B.set_frame(0, fr.image, fr.mask, fr.detections)
        B.set_pose(0, xo)
        B.step_stage(2)
        _, vb, _, rep = B.result(0)
        ins = B.inspect(0)
        pb = [t for t in trace if t[0] == "surface_problem"][0][1]
        prob, v_init = pb["problem"], pb["v_init"]
        print(f"frame {fr.index}: vertex err/diag {np.abs(vb - vo).max() / diag:.3e}  "
              f"v_init err {np.abs(ins['v_init'] - v_init).max():.2e}  "
              f"sets equal: boundary {np.array_equal(ins['boundary'], prob.boundary_idx)} "
              f"enabled {np.array_equal(ins['enabled'], prob.enabled)} visible {np.array_equal(ins['visible'], prob.visible)}")
        R = rep.nonrigid
        for k, o in enumerate(slogs):
            g0, g1 = R.energy_before[k], R.energy_after[k]
            print(f"   it {k}: e0 {g0:.10e} vs {o['energy_before']:.10e} ({abs(g0 - o['energy_before']) / o['energy_before']:.1e})"
                  f"  e1 {g1:.10e} vs {o['energy_after']:.10e} ({abs(g1 - o['energy_after']) / o['energy_after']:.1e})"
                  f"  halv {R.halvings[k]}/{o['halvings']} brk {R.pcg_breakdown[k]}/{int(o['pcg_breakdown'])}")
            names = ("photo", "silhouette", "smooth", "edge", "velocity", "acceleration")
            print("        terms rel: " + " ".join(f"{nm[:5]} {abs(R.terms[k][j] - o['terms'].get(nm, 0.0)) / max(abs(o['terms'].get(nm, 0.0)), 1e-300):.1e}"
                                              for j, nm in enumerate(names)))
        print(f"   snap: walked {R.snap_walked} reached {R.snap_reached} stuck {R.snap_stuck}  pruned {R.pruned}")
        st = st_new


if __name__ == "__main__":
    main()
