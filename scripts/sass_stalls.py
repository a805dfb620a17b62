"""Top instructions by stall reason from an ncu SASS source page csv."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and '(Not' not in h]
tot = {r: sum(int(d[col[r]] or 0) for d in data) for r in reasons}
print({k: v for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
for r in sys.argv[2:]:
    print(f'--- top {r}')
    top = sorted(data, key=lambda d: -int(d[col[r]] or 0))[:12]
    for d in top:
        print(f"  {int(d[col[r]] or 0):6d}  {d[col['Address']][-5:]}  {d[col['Source']].strip()[:90]}")
