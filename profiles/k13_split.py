"""K13 ncu SASS split: GEMM-warp barrier share, solver instructions per block, top solver stalls."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
blocks = int(sys.argv[2])
hdr = rows[1]; body = rows[2:]
isrc = hdr.index("Source"); iss = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed")
cols = [(j, h) for j, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
bars = [i for i, r in enumerate(body) if 'BAR.SYNC' in r[isrc]]
tot = sum(int(r[iss] or 0) for r in body)
gb = max(bars, key=lambda b: sum(int(body[x][iss] or 0) for x in range(b, b + 6)))
print("total samples", tot, "gemm barrier share %.1f%%" % (100 * sum(int(body[x][iss] or 0) for x in range(gb, gb + 6)) / tot))
lo = gb + 6
ex = sum(int(r[ie] or 0) for r in body[lo:])
c = collections.Counter()
for r in body[lo:]:
    for j, h in cols:
        try: c[h] += int(float(r[j] or 0))
        except ValueError: pass
print("solver instr/block %.0f" % (ex / blocks), "solver samples", sum(int(r[iss] or 0) for r in body[lo:]), c.most_common(5))
gex = sum(int(r[ie] or 0) for r in body[:gb])
print("gemm-side instr/block (all warps) %.0f" % (gex / blocks))
for h in sorted([(int(r[iss] or 0), i, r[isrc][:70]) for i, r in enumerate(body) if i >= lo], reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 10]:
    print("   ", h)
