"""Opcode mix of one kernel from `ncu --page source --csv --print-source sass` (per point)."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
mix = Counter()
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    mix[o.split(".")[0]] += int(r[iex])
tot = sum(mix.values())
print(f"total warp-instr {tot}  per unit (x32 threads) {32 * tot / units:.0f}")
for o, c in mix.most_common(25):
    print(f"{o:10s} {c:12d} {100 * c / tot:5.1f}%  per unit {32 * c / units:8.1f}")
