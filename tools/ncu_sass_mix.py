"""Instruction mix and stall samples per SASS opcode of an ncu report (first kernel)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
r = csv.reader(out)
next(r)
h = next(r)
ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
rows = list(r)
tot = sum(float(x[ie] or 0) for x in rows)
st = sum(float(x[ws] or 0) for x in rows)
print("total warp inst", tot, "stall samples", st, "sass lines", len(rows))
c, s = Counter(), Counter()
for x in rows:
    parts = x[1].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    op = op.split(".")[0]
    c[op] += float(x[ie] or 0)
    s[op] += float(x[ws] or 0)
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 22):
    print(f"{k:10s} {v / tot * 100:5.1f}% inst  {s[k] / st * 100:5.1f}% stall")
if len(sys.argv) > 3:  # hottest stall lines
    rows.sort(key=lambda x: -float(x[ws] or 0))
    for x in rows[:int(sys.argv[3])]:
        print(x[ws], x[1][:90])
