"""Per-CUDA-source-line instruction counts from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, re
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, cur, iex = None, None, None
count = Counter(); text = {}; ops = defaultdict(Counter)
for r in rows:
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        iex = r.index("Instructions Executed"); continue
    if iex is None or len(r) <= iex:
        continue
    if r[0]:
        cur = (fname, int(r[0])); text[cur] = r[1].strip()[:90]
    elif cur and r[iex].isdigit():
        n = int(r[iex]); count[cur] += n
        op = r[3].strip().split()
        if op:
            o = op[1] if op[0].startswith("@") else op[0]
            ops[cur][o.split(".")[0]] += n
tot = sum(count.values())
print(f"total {tot} warp-instr; per unit {32 * tot / units:.0f} thread-instr")
for k, c in count.most_common(top):
    mix = ",".join(f"{o}:{32 * v / units:.0f}" for o, v in ops[k].most_common(4))
    print(f"{k[0]}:{k[1]:<5d} {32 * c / units:7.1f}/unit  {text[k][:70]:70s} [{mix}]")
