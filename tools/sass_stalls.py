"""Per-source-line stall-reason breakdown from an ncu SASS source page.

  ncu -i rep --page source --csv --print-source sass > sass.csv
  python tools/sass_stalls.py sass.csv path/to/obj.o mangled_kernel [file:lo-hi ...]
Prints, for the selected line ranges (default: the top lines), the samples
per stall reason, so a phase's critical path (long_sb = memory, wait =
fixed latency, barrier = idle at a barrier ...) can be read off.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def main():
    csv_path, obj, kname = sys.argv[1:4]
    ranges = []
    for a in sys.argv[4:]:
        f, r = a.split(":")
        lo, hi = (int(x) for x in r.split("-"))
        ranges.append((f, lo, hi))
    rows = list(csv.reader(open(csv_path)))
    hi_ = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi_]
    ai = h.index("Address")
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    names = [h[i][6:] for i in cols]
    by_off = {}
    addrs = []
    for r in rows[hi_ + 1:]:
        try:
            a = int(r[ai], 16)
        except (ValueError, IndexError):
            continue
        addrs.append(a)
        by_off[a] = [float(r[i] or 0) for i in cols]
    base = min(addrs)
    by_off = {a - base: v for a, v in by_off.items()}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    in_fn, line, agg = False, None, collections.defaultdict(lambda: [0.0] * len(cols))
    for l in out.splitlines():
        if l.startswith(".text.") or ".section" in l and ".text." in l:
            in_fn = kname in l
            continue
        if not in_fn:
            continue
        fm = re.search(r'File "([^"]+)", line (\d+)', l)
        if fm:
            line = (fm.group(1).split("/")[-1], int(fm.group(2)))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and line and int(m.group(1), 16) in by_off:
            v = by_off[int(m.group(1), 16)]
            acc = agg[line]
            for k in range(len(cols)):
                acc[k] += v[k]
    tot = sum(sum(v) for v in agg.values()) or 1.0
    sel = [(k, v) for k, v in agg.items()
           if not ranges or any(k[0] == f and lo <= k[1] <= hi for f, lo, hi in ranges)]
    sel.sort(key=lambda kv: -sum(kv[1]))
    grand = [0.0] * len(cols)
    for k, v in sel:
        for i in range(len(cols)):
            grand[i] += v[i]
    print(f"selected share of all samples: {sum(grand) / tot:.3f}")
    print("by reason: " + ", ".join(f"{n}={g / tot:.3f}" for n, g in sorted(zip(names, grand), key=lambda x: -x[1])[:8]))
    for (f, ln), v in sel[:30]:
        top = sorted(zip(names, v), key=lambda x: -x[1])[:3]
        print(f"{sum(v) / tot:6.3f} {f}:{ln} " + " ".join(f"{n}={x / tot:.3f}" for n, x in top))


if __name__ == "__main__":
    main()
