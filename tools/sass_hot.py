"""Hot instructions of an ncu SASS source page (--page source --csv
--print-source sass): per opcode and per region, executed warp instructions.

    python tools/sass_hot.py gpurun_out/sass_connect_four.csv [--top 40]
"""
import argparse
import collections
import csv

p = argparse.ArgumentParser()
p.add_argument("csv")
p.add_argument("--top", type=int, default=30)
p.add_argument("--dump", action="store_true", help="print every executed instruction")
a = p.parse_args()
rows = list(csv.reader(open(a.csv)))
head = rows[1]
ix = head.index("Instructions Executed")
isrc = head.index("Source")
ith = head.index("Thread Instructions Executed")
tot = 0
ops = collections.Counter()
lines = []
for r in rows[2:]:
    if len(r) <= ix or not r[ix].strip().isdigit():
        continue
    n = int(r[ix])
    src = r[isrc].strip()
    tot += n
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    ops[op.split(".")[0]] += n
    lines.append((n, int(r[ith]), src))
print(f"total warp inst {tot}")
for op, n in ops.most_common(a.top):
    print(f"{op:10s} {n:14d} {100 * n / tot:5.1f}%")
if a.dump:
    for n, t, src in lines:
        if n:
            print(f"{n:12d} {t / max(n, 1):5.1f} {src}")
