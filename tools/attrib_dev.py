"""Dev tool: dynamic instruction counts per inlined device function (glint_device.cuh)."""
import csv
import re
import sys
from collections import defaultdict

dis, srccsv, kern, npx = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kern}:"))
cur, order = None, []
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        op = m.group(2).split()
        order.append((cur, (op[1] if op[0].startswith("@") else op[0]).split(".")[0]))
rows = list(csv.reader(open(srccsv)))
hdr, data = rows[1], rows[2:]
ti = hdr.index("Thread Instructions Executed")
dev = open("paper_2306_05051_b200/csrc/glint_device.cuh").read().split("\n")
funcs = [(i + 1, re.search(r"(\w+)\(", l).group(1)) for i, l in enumerate(dev) if "__device__" in l]
agg = defaultdict(lambda: defaultdict(int))
for (c, op), r in zip(order, data):
    if c and c[0] != "glint_kernel.cu":
        name = c[0] if c[0] != "glint_device.cuh" else [f for i, f in funcs if i <= c[1]][-1]
        agg[name][op] += int(r[ti])
for k, ops in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    tot = sum(ops.values())
    print(f"{tot / npx:7.1f} {k:20s} " + " ".join(f"{o}:{c / npx:.0f}" for o, c in sorted(ops.items(), key=lambda kv: -kv[1])[:8]))
