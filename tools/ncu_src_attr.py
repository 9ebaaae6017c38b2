"""Attribute ncu SASS-level stall samples to CUDA source lines: ncu --page source --print-source sass
CSV of one kernel + nvdisasm -g listing of the same function (offsets match the runtime addresses
minus the function start).  usage: ncu_src_attr.py <sass.csv> <nvdisasm.txt> <function-substring> [top]"""
import collections
import csv
import re
import sys

csvf, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(csvf)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
base = int(data[0]["Address"], 16)
key = "Warp Stall Sampling (All Samples)"
samp = {int(d["Address"], 16) - base: float(d[key] or 0) for d in data}
inst = {int(d["Address"], 16) - base: float(d["Instructions Executed"] or 0) for d in data}
# offset -> (file, line)
loc = {}
cur = None
infn = False
for line in open(dis):
    if line.startswith("//----") or line.startswith("\t.section"):
        infn = fn in line
        cur = None
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        loc[int(m.group(1), 16)] = cur
S = collections.Counter()
I = collections.Counter()
for off, s in samp.items():
    S[loc.get(off, ("?", 0))] += s
    I[loc.get(off, ("?", 0))] += inst.get(off, 0)
tot = sum(S.values())
print(f"total samples {tot:.0f}, instructions {sum(I.values()):.0f}, mapped {len(loc)} offsets")
for k, v in S.most_common(top):
    print(f"{100 * v / tot:5.1f}%  inst {I[k]:10.0f}  {k[0]}:{k[1]}")
