"""Per-source-line share of ncu warp-stall samples and executed instructions for one kernel:
maps the SASS page of an ncu report (--page source --print-source sass --csv) to source lines
with nvdisasm --print-line-info of the built object.

usage: python scripts/ncu_lines.py <sass.csv> <object.o> <kernel-substring> <source.cu> [top]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

sass_csv, obj, kname, srcfile = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
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
for r in rows[2:]:  # the first kernel's section (a report may hold several)
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
b0 = int(data[0][ia], 16)
S, E = Counter(), Counter()
for r in data:
    ln = lines.get(int(r[ia], 16) - b0, 0)
    S[ln] += int(r[isamp] or 0)
    E[ln] += int(r[iex] or 0)
tot, totE = sum(S.values()), sum(E.values())
print(f"samples {tot}  warp instructions {totE}")
src = open(srcfile).read().split("\n")
for ln, s in S.most_common(top):
    print(f"{ln:5d} {100 * s / tot:5.1f}% samples {100 * E[ln] / totE:5.1f}% instr | "
          f"{src[ln - 1].strip()[:90] if ln > 0 else '(other file)'}")
