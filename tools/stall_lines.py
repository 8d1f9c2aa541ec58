"""Per-SASS-line stall attribution from `ncu --page source --csv --print-source sass` (first kernel)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out, started, hdr = [], False, None
for r in rows:
    if r and r[0] == 'Kernel Name':
        if started:
            break
        started = True
        continue
    if r and r[0] == 'Address':
        hdr = r
        continue
    if started and len(r) > 5:
        out.append(r)
iE = hdr.index('Instructions Executed')
iS = hdr.index('Warp Stall Sampling (All Samples)')
tot = sum(int(r[iE]) for r in out)
stall = sum(int(r[iS]) for r in out)
print('instr', tot, 'samples', stall)
cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
agg = {c: sum(int(r[hdr.index(c)]) for r in out) for c in cols}
for c, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f'{c:28s} {v / stall * 100:5.1f}%')
print('--- top lines')
for i, r in sorted(enumerate(out), key=lambda x: -int(x[1][iS]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    reasons = sorted(((int(r[hdr.index(c)]), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{int(r[iS]) / stall * 100:5.2f}% {i:5d} exec={int(r[iE]):>9d} {r[1].strip()[:58]:58s} {reasons}")
