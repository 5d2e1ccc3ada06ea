"""Summarise an `ncu --page source --csv` dump: hottest SASS lines of the first kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
ie = hdr.index('Instructions Executed'); smp = hdr.index('Warp Stall Sampling (All Samples)')
src = hdr.index('Source'); at = hdr.index('Avg. Threads Executed')
tot = sum(int(r[ie]) for r in data); stot = sum(int(r[smp]) for r in data)
print('total inst', tot, 'samples', stot)
for r in data:
    if int(r[ie]) > tot * thr or int(r[smp]) > stot * thr:
        print(f"{int(r[ie])/tot:6.2%} smp={int(r[smp])/stot:6.2%} thr={r[at]:>5} {r[0][-5:]} {r[src].strip()[:100]}")
