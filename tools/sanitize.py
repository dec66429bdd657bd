"""compute-sanitizer target: one small tracker frame pair (smoke scene) and,
with --x5k, one bench-size frame (x5k @1024, 4 streams in one launch).

  compute-sanitizer --tool racecheck python tools/sanitize.py
  compute-sanitizer --tool memcheck  python tools/sanitize.py --x5k
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from helpers import scene, scene_bench
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    big = "--x5k" in sys.argv
    actor, cam, frames = scene_bench("x5k", 1024, 2) if big else scene("small", 128, 2)
    S = 4 if big else 2
    tr = Tracker(actor, cam, SequenceConfig(directional=False), S)
    for fr in frames:
        for s in range(S):
            tr.set_frame(s, fr.image, fr.mask, fr.detections)
        tr.step()
        x, v, _, _ = tr.result(0)
        print(f"frame {fr.index}: |x| {abs(x).max():.3f}")
    tr.close()
    print("sanitize target done")


if __name__ == "__main__":
    main()
