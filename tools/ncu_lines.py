"""Stall samples of an ncu --set full capture (--import-source on) aggregated by
CUDA source line: maps the SASS page onto nvdisasm -g line info of the
in-tree libocpgpu.so (which must be the build that was profiled).
usage: ncu_lines.py REPORT MANGLED_KERNEL_NAME [cubin-substring] [top]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
unit = sys.argv[3] if len(sys.argv) > 3 else "ocp_block"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_2411_00546_b200", "libocpgpu.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith(unit + ".") and f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if ".text." + kname in l and ("section" in l or l.startswith(".text")))
ins, cur, fname = [], None, None
for l in dis[start + 1:]:
    if ".section" in l and ins:
        break
    m = re.search(r'## File "(.*?)", line (\d+)', l)
    if m:
        fname, cur = os.path.basename(m.group(1)), int(m.group(2))
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m2:
        ins.append((int(m2.group(1), 16), (fname, cur)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.split("\n")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = []
for r in rows[hi + 1:]:
    if not r or r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
col = os.environ.get("NCU_COL", "Warp Stall Sampling (All Samples)")
i_s = hdr.index(col)
base = int(data[0][0], 16)
a2l = dict(ins)
byline = collections.Counter()
tot = 0
for r in data:
    ln = a2l.get(int(r[0], 16) - base)
    byline[ln] += int(r[i_s])
    tot += int(r[i_s])
srcs = {}
for (f, ln), v in byline.most_common(top):
    if f not in srcs:
        path = os.path.join(root, "paper_2411_00546_b200", "csrc", f)
        srcs[f] = open(path).read().split("\n") if os.path.exists(path) else []
    txt = srcs[f][ln - 1].strip()[:90] if ln and ln <= len(srcs[f]) else ""
    print(f"{v:7d} {100 * v / tot:5.1f}%  {f}:{ln}: {txt}")
