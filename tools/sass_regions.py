"""Opcode mix and hottest regions of an `ncu --page source --print-source sass --csv` dump."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
ie = hdr.index('Instructions Executed'); src = hdr.index('Source'); smp = hdr.index('Warp Stall Sampling (All Samples)')
tot = sum(int(r[ie]) for r in data); st = sum(int(r[smp]) for r in data)
print('total warp-inst', tot)
op = collections.Counter()
for r in data:
    t = r[src].split()
    o = t[1] if t[0].startswith('@') else t[0]
    op[o.split('.')[0]] += int(r[ie])
print(' '.join(f'{k}:{v/tot:.1%}' for k, v in op.most_common(16)))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
win = [(sum(int(r[ie]) for r in data[i:i + W]), sum(int(r[smp]) for r in data[i:i + W]), i) for i in range(0, len(data), W)]
for s, ss, i in sorted(win, reverse=True)[:12]:
    print(f'idx {i:5d} addr {data[i][0][-5:]} inst {s/tot:6.2%} smp {ss/st:6.2%}')
