"""Dev tool: attribute ncu per-SASS-instruction counts to kernel source lines.
usage: python tools/sass_lines.py <nvdisasm -g listing> <ncu --page source --print-source sass csv> <mangled kernel>"""
import csv
import re
import sys
from collections import defaultdict

dis, src, kern = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kern}:"))
cur = None
order = []
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        f, ln, rest = m.group(1).split("/")[-1], int(m.group(2)), m.group(3)
        m2 = re.findall(r'inlined at "([^"]+)", line (\d+)', rest)
        outer = (m2[-1][0].split("/")[-1], int(m2[-1][1])) if m2 else (f, ln)
        cur = (outer, (f, ln))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        order.append((cur, m.group(2).split()[0] if m.group(2).split()[0][0] != "@" else m.group(2).split()[1]))
rows = list(csv.reader(open(src)))
hdr = rows[1]
data = rows[2:]
ti = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
assert len(data) == len(order), (len(data), len(order))
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for (loc, op), r in zip(order, data):
    k = loc[0] if loc else ("?", 0)
    agg[k][0] += int(r[ti])
    agg[k][1] += int(r[ws])
    tot[0] += int(r[ti]); tot[1] += int(r[ws])
print(f"total thread inst {tot[0]:.4g}, stall samples {tot[1]}")
for k, (a, b) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"{k[0]}:{k[1]:4d}  inst {100*a/tot[0]:5.1f}%  samples {100*b/tot[1]:5.1f}%")
