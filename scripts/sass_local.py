"""Local-memory (STL / LDL) instructions of one kernel, by source line (-lineinfo builds).

    python scripts/sass_local.py <object> <kernel-substring> [--all-matches-index i]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
names = sorted(set(re.findall(r"_ZN[A-Za-z0-9_]+", subprocess.run(["cuobjdump", "-elf", cubin], capture_output=True,
                                                                      text=True).stdout)))
names = [n for n in names if all(p in n for p in pat.split(",")) and not n.endswith("_param_0")]
name = names[idx]
print("kernel:", subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()[:200])
full = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
start = full.find(".section\t.text." + name + ",")
end = full.find(".section\t.text.", start + 1)
sass = full[start:end if end > 0 else None]
cur = None
cnt = collections.Counter()
for line in sass.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"\b(STL|LDL)(\.\w+)*\b", line)
    if m and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        cnt[(cur, m.group(1))] += 1
for (loc, op), c in sorted(cnt.items(), key=lambda kv: (str(kv[0][0]), kv[0][1])):
    print(f"{op} {c:3d}  {loc}")
