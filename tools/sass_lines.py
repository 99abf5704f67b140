"""Join an ncu source page (--page source --csv --print-source sass) with the
line table of the same kernel's SASS (nvdisasm --print-line-info) and print
executed warp instructions per source line (and per opcode).

    python tools/sass_lines.py <page.csv> <nvdisasm.txt> <function-substring> [pixels]
"""
import collections
import csv
import re
import sys

page, dis, fn = sys.argv[1:4]
pixels = float(sys.argv[4]) if len(sys.argv) > 4 else None
rows = list(csv.reader(open(page)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
execd = [(r[src].strip(), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]

insts = []
cur = "?"
on = False
for l in open(dis):
    if l.strip().startswith(".text."):
        on = fn in l
        continue
    if not on:
        continue
    m = re.search(r'## File ".*?/([\w.]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", l)
    if m:
        insts.append((cur, m.group(1).strip()))
assert len(insts) == len(execd), (len(insts), len(execd))
by_line = collections.Counter()
by_op = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for (line, text), (t2, n) in zip(insts, execd):
    op = re.sub(r"^@!?U?P\w+\s+", "", text).split()[0].split(".")[0]
    by_line[line] += n
    by_op[op] += n
    ops[line][op] += n
tot = sum(by_line.values())
div = pixels / 32 if pixels else 1
print(f"total {tot} warp instr" + (f" = {tot / div:.1f} per pixel-warp" if pixels else ""))
for line, n in sorted(by_line.items(), key=lambda kv: -kv[1]):
    if n / tot < 0.002:
        continue
    print(f"{line:26s} {n / div:8.1f}  {dict(ops[line].most_common(6))}")
print("opcodes:", {k: round(v / div, 1) for k, v in by_op.most_common(25)})
