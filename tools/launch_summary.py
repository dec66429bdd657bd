"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.

  python tools/launch_summary.py launches.csv [--after k_prep --skip-first-frame]
Only launches after the first `--after` kernel are counted (skips input
generation); --frames-skip n drops the first n occurrences of that marker.
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui].strip().lower()
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        out.append((r[ki].split("(")[0], v * scale))
    return out


def main():
    path = sys.argv[1]
    marker = sys.argv[sys.argv.index("--after") + 1] if "--after" in sys.argv else None
    skip = int(sys.argv[sys.argv.index("--frames-skip") + 1]) if "--frames-skip" in sys.argv else 0
    launches = load(path)
    if marker:
        idx = [i for i, (k, _) in enumerate(launches) if k == marker]
        launches = launches[idx[min(skip, len(idx) - 1)]:] if idx else launches
    frames = max(1, sum(1 for k, _ in launches if k == marker)) if marker else 1
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in launches:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(launches)} launches, {tot / 1e3:.3f} ms kernel time, {frames} frame(s) -> "
          f"{tot / 1e3 / frames:.3f} ms/frame")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} n={n:5d} total={t / 1e3:9.3f} ms avg={t / n:9.1f} us share={t / tot:6.3f}")


if __name__ == "__main__":
    main()
