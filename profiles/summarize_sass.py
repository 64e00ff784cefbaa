"""Top stall-sampled SASS lines of an ncu source-page CSV (--page source --csv --print-source=sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > iss and r[iss].strip().isdigit()]
tot = sum(int(r[iss]) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for r in sorted(body, key=lambda r: -int(r[iss]))[:n]:
    print(f"{int(r[iss]) / tot * 100:5.1f}%  {r[ia]:>6}  {r[isrc][:110]}")
