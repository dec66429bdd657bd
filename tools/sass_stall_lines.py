"""Per-source-line stall breakdown of an ncu SASS source page.

  ncu -i rep --page source --csv --print-source sass > sass.csv
  python tools/sass_stall_lines.py sass.csv obj.o mangled_kernel [file:first-last ...]
Prints, for each line range, the share of all samples and the top stall reasons.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, kname):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    in_fn, line, m_ = False, None, {}
    for l in out.splitlines():
        if l.startswith(".text.") or ".section" in l and ".text." in l:
            in_fn = kname in l
            continue
        if not in_fn:
            continue
        fm = re.search(r'File "([^"]+)", line (\d+)', l)
        if fm:
            line = (fm.group(1).split("/")[-1], int(fm.group(2)))
        mm = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if mm and line:
            m_[int(mm.group(1), 16)] = line
    return m_


def main():
    csv_path, obj, kname = sys.argv[1:4]
    ranges = []
    for a in sys.argv[4:]:
        f, r = a.split(":")
        lo, hi = (int(x) for x in r.split("-"))
        ranges.append((a, f, lo, hi))
    rows = list(csv.reader(open(csv_path)))
    hi_ = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi_]
    ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    recs = []
    for r in rows[hi_ + 1:]:
        try:
            recs.append((int(r[ai], 16), float(r[si]), {c: float(r[i] or 0) for i, c in stall_cols}))
        except (ValueError, IndexError):
            pass
    base = min(a for a, _, _ in recs)
    lm = line_map(obj, kname)
    tot = sum(s for _, s, _ in recs) or 1.0
    for name, f, lo, hi in ranges:
        agg = collections.Counter()
        n = 0.0
        for a, s, st in recs:
            ln = lm.get(a - base)
            if ln and ln[0] == f and lo <= ln[1] <= hi:
                n += s
                agg.update(st)
        top = ", ".join(f"{k[6:]} {v / max(n, 1):.2f}" for k, v in agg.most_common(5))
        print(f"{name:28s} {n / tot:6.3f}  {top}")


if __name__ == "__main__":
    main()
