"""Per-source-line instruction / lane / stall attribution of one kernel in an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED_SUBSTRING [top]
Joins ncu's SASS page (per-instruction counts) with nvdisasm line info of the same .so.
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

rep, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
launch = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # which profiled launch of the report
tmp = Path(tempfile.mkdtemp())
subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=tmp, capture_output=True)
cubin = next(p for p in tmp.glob("*.cubin") if p.name.startswith("fmgpu.") or "fmgpu" in p.name)
sass = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//--------------------- .text.") and kname in l)
cur, idx2src = None, {}
for l in sass[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        idx2src[int(m.group(1), 16) // 16] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = rows[starts[launch]:starts[launch + 1]]
h, data = sec[1], [r for r in sec[2:] if len(r) == len(sec[1])]
ia, ta = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
sa = h.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for j, r in enumerate(data):
    a = agg[idx2src.get(j)]
    a[0] += float(r[ia] or 0)
    a[1] += float(r[ta] or 0)
    a[2] += float(r[sa] or 0)
tot = sum(a[0] for a in agg.values())
st = sum(a[2] for a in agg.values())
tt = sum(a[1] for a in agg.values())
print(f"warp insts {tot:.4g}, avg lanes {tt / tot:.2f}, stall samples {st:.0f}")
csrc = Path(__file__).resolve().parent.parent / "paper_1811_06127_b200" / "csrc"
files = {p.name: p.read_text().split("\n") for p in csrc.glob("*.cuh")}
key_i = 2 if "--by-stall" in sys.argv else 0
for s, (i, t, smp) in sorted(agg.items(), key=lambda x: -x[1][key_i])[:top]:
    txt = files.get(s[0], [""] * (s[1] if s else 1))[s[1] - 1].strip()[:70] if s else ""
    print(f"{str(s):30s} inst {100 * i / tot:5.1f}% lanes {t / max(i, 1):5.1f} stall {100 * smp / st:5.1f}%  {txt}")
