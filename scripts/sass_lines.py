"""SASS instruction count per source line of one kernel (needs -lineinfo builds).

    python scripts/sass_lines.py build/finenv/rollout_stock.o <kernel-substring> [top]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
names = sorted(set(re.findall(r"_ZN[A-Za-z0-9_]+", subprocess.run(["cuobjdump", "-elf", cubin], capture_output=True,
                                                                      text=True).stdout)))
names = [n for n in names if pat in n and not n.endswith("_param_0")]
name = names[0]
print("kernel:", name[:160])
full = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
# keep the section of this function (".text.<name>:" up to the next ".text.")
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
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        cnt[cur] += 1
byfile = collections.Counter()
for (f, l), c in ((k if k else ("?", 0), v) for k, v in cnt.items()):
    byfile[f] += c
print("total", sum(cnt.values()))
print(byfile.most_common(12))
for k, c in cnt.most_common(top):
    print(c, k)
