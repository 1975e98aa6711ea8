"""Bucket tools/ncu_lines.py output (stdin) by named line ranges of kernels_flat.cuh given as name:a-b args."""
import re
import sys

ranges = {}
for a in sys.argv[1:]:
    name, r = a.split(":")
    lo, hi = r.split("-")
    ranges[name] = (int(lo), int(hi))
b = {}
for line in sys.stdin:
    m = re.match(r"\('([^']+)', (\d+)\)\s+inst\s+([\d.]+)% lanes\s+([\d.]+) stall\s+([\d.]+)%", line)
    if not m:
        continue
    f, ln = m.group(1), int(m.group(2))
    k = f
    if f == "kernels_flat.cuh":
        k = "flat:other"
        for name, (lo, hi) in ranges.items():
            if lo <= ln <= hi:
                k = name
    x = b.setdefault(k, [0, 0])
    x[0] += float(m.group(3))
    x[1] += float(m.group(5))
for k, v in sorted(b.items(), key=lambda t: -t[1][0]):
    print(f"{k:28s} inst {v[0]:5.1f}%  stall {v[1]:5.1f}%")
