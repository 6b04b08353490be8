"""Dev tool: per-stage dynamic instruction attribution of the glint kernel.
usage: python tools/attrib.py <nvdisasm -g listing> <ncu sass source csv> <mangled kernel> <pixels>"""
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
        cur = [(m.group(1).split("/")[-1], int(m.group(2)))] + [
            (a.split("/")[-1], int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        op = m.group(2).split()
        op = op[1] if op[0].startswith("@") else op[0]
        order.append((cur, op.split(".")[0]))
rows = list(csv.reader(open(srccsv)))
hdr, data = rows[1], rows[2:]
ti = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
assert len(data) == len(order), (len(data), len(order))
src = open("paper_2306_05051_b200/csrc/glint_kernel.cu").read().split("\n")
marks = []
for i, l in enumerate(src):
    m = re.search(r"// -{8,} (S[0-9][^:(]*|per-pixel shading frame)", l)
    if m:
        marks.append((i + 1, m.group(1).strip()))
    if "__device__ __forceinline__ void lattice(" in l:
        marks.append((i + 1, "S2 lattice fn"))
    if "fp32 Smith Lambda" in l:
        marks.append((i + 1, "smith fn"))
    if "// The kernel:" in l:
        marks.append((i + 1, "kernel loop"))
marks.sort()
bucket = defaultdict(lambda: [0, 0])
ops = defaultdict(lambda: defaultdict(int))
tot = [0, 0]
for (ch, op), r in zip(order, data):
    kl = -1
    for f, ln in (ch or []):
        if f == "glint_kernel.cu":
            kl = ln
    name = "?"
    for ln, nm in marks:
        if kl >= ln:
            name = nm
    if kl == -1:
        name = "no-line"
    bucket[name][0] += int(r[ti])
    bucket[name][1] += int(r[ws])
    ops[name][op] += int(r[ti])
    tot[0] += int(r[ti])
    tot[1] += int(r[ws])
for nm, (a, b) in sorted(bucket.items(), key=lambda kv: -kv[1][0]):
    top = sorted(ops[nm].items(), key=lambda kv: -kv[1])[:6]
    print(f"{nm:28s} {a / npx:7.1f} inst/px {100 * b / tot[1]:5.1f}% stalls | " + " ".join(f"{o}:{c / npx:.0f}" for o, c in top))
print(f"total {tot[0] / npx:.1f} thread-inst/px")
