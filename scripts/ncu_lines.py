"""Aggregate ncu per-SASS stall samples of one kernel by CUDA source line.

    ncu -i rep --page source --csv --print-source sass > sass.csv
    python scripts/ncu_lines.py sass.csv build/finenv/<obj>.o <kernel-substring> [top]

Maps each sampled SASS instruction (offset from the kernel's first instruction) to
the source line nvdisasm -g reports for that offset in the locally built object
(the box builds the identical SASS from the same sources and nvcc).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

csv_path, obj, pat = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
if len(sys.argv) > 5 and sys.argv[5] == "inst":      # aggregate executed warp instructions instead
    i_s = hdr.index("Instructions Executed")
samples = []
base = None
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    s = int(r[i_s]) if r[i_s].isdigit() else 0
    samples.append((a - base, s, r[1].strip()))

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
full = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
names = [m for m in re.findall(r"\.section\t\.text\.([A-Za-z0-9_]+),", full) if pat in m]
name = names[0]
start = full.find(".section\t.text." + name + ",")
end = full.find(".section\t.text.", start + 1)
sec = full[start:end if end > 0 else None]
line_of = {}
cur = None
for line in sec.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
for off, s, src in samples:
    agg[line_of.get(off, ("?", 0))] += s
tot = sum(agg.values())
print("kernel", name[:120], "samples", tot)
byfile = collections.Counter()
for (f, _), s in agg.items():
    byfile[f] += s
print([(f, round(100 * s / tot, 1)) for f, s in byfile.most_common(10)])
for (f, l), s in agg.most_common(top):
    print(f"{100 * s / tot:5.1f}% {f}:{l}")
