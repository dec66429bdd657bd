"""Map ncu SASS-level stall samples to source lines.

  ncu -i rep --page source --csv --print-source sass --kernel-name regex:NAME > sass.csv
  python tools/sass_hotspots.py sass.csv path/to/obj.o mangled_kernel_name [top]
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
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    addrs, samples = [], []
    for r in rows[hi + 1:]:
        try:
            addrs.append(int(r[ai], 16))
            samples.append(float(r[si]))
        except (ValueError, IndexError):
            pass
    base = min(addrs)
    by_off = {a - base: s for a, s in zip(addrs, samples)}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    in_fn, line, agg = False, None, collections.Counter()
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
            agg[line] += by_off[int(m.group(1), 16)]
    tot = sum(agg.values()) or 1.0
    print(f"samples mapped {sum(agg.values()):.0f} of {sum(samples):.0f}")
    here = os.path.dirname(os.path.abspath(obj))
    src_dir = os.path.join(os.path.dirname(here), "csrc")
    for (f, ln), v in agg.most_common(top):
        try:
            src = open(os.path.join(src_dir, f)).read().splitlines()[ln - 1].strip()
        except OSError:
            src = ""
        print(f"{v / tot:6.3f} {f}:{ln} {src[:96]}")


if __name__ == "__main__":
    main()
