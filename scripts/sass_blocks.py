"""Group an ncu SASS source page (csv) into basic blocks by execution count; print hot blocks."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); src = hdr.index("Source"); st = hdr.index("Warp Stall Sampling (All Samples)")
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
tot = sum(int(r[ie] or 0) for r in data)
print('total warp inst', tot)
cur = None; blk = []
def flush():
    if blk and blk[0][0] > thr:
        c = blk[0][0]
        ops = {}
        for b in blk:
            t = b[2].split()
            op = t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '?')
            ops[op] = ops.get(op, 0) + 1
        print(f"count {c:>10d} x {len(blk):3d} = {c*len(blk)/1e6:8.1f}M ({100*c*len(blk)/tot:4.1f}%) stalls {sum(b[1] for b in blk):6d} "
              + " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:10]))
for r in data:
    c = int(r[ie] or 0); s = int(r[st] or 0)
    if cur is None or c != cur:
        flush(); blk = []; cur = c
    blk.append((c, s, r[src].strip()))
flush()
