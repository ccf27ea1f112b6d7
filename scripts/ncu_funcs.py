"""Per-function share of executed warp instructions of one kernel (ncu SASS page + nvdisasm line
info of the built object; the enclosing function is found by scanning the source upwards).

usage: python scripts/ncu_funcs.py <sass.csv> <object.o> <kernel-substring> <source.cu> [n_units]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

sass_csv, obj, kname, srcfile = sys.argv[1:5]
units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
               stdout=subprocess.DEVNULL)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(tmp, cubin)],
                     capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(txt) if re.match(r"^_ZN.*" + kname + r".*:$", l)][0]
end = next((i for i in range(start + 1, len(txt)) if txt[i].startswith(".text.")), len(txt))
base = os.path.basename(srcfile)
lines, cur = {}, None
for l in txt[start:end]:
    m = re.search(r'//## File ".*' + re.escape(base) + r'", line (\d+)', l)
    if m:
        cur = int(m.group(1))
        continue
    if "//## File" in l:
        cur = 0
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr, data = rows[1], []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
b0 = int(data[0][ia], 16)
E = Counter()
for r in data:
    E[lines.get(int(r[ia], 16) - b0, 0)] += int(r[iex] or 0)
src = open(srcfile).read().split("\n")


def fn_of(ln):
    for i in range(ln - 1, -1, -1):
        l = src[i]
        if l.startswith("__device__") or l.startswith("__global__") or re.match(r"^\w+_kernel\(", l):
            m = re.search(r"(\w+)\(", l + src[i + 1])
            return m.group(1) if m else l[:40]
    return "?"


F = Counter()
for ln, c in E.items():
    F[fn_of(ln) if ln > 0 else "(other file)"] += c
tot = sum(F.values())
for f, c in F.most_common():
    print(f"{f:30s} {100 * c / tot:5.1f}%  {c / units:9.1f} warp instructions per unit")
