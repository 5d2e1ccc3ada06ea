"""Stall-reason totals of an `ncu --page source --csv` dump (first kernel),
overall and for the lines that wait on global loads (long_sb), plus the
instruction mix by opcode. Usage: ncu_regions.py src.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for h in stalls:
        tot[h] += float(r[col[h]] or 0)
S = sum(tot.values())
print("samples", int(S))
for h, v in tot.most_common(10):
    print(f"  {h:24s} {v / S:6.1%}")
ops = collections.Counter()
ie = col["Instructions Executed"]
I = sum(int(r[ie]) for r in data)
for r in data:
    op = r[col["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    ops[o.split(".")[0]] += int(r[ie])
print("warp instructions", I)
for o, v in ops.most_common(18):
    print(f"  {o:12s} {v / I:6.1%}")
