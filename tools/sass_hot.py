"""Per-opcode and per-instruction stall samples from an ncu source page
(SASS view).  Usage: ncu -i rep --page source --csv --print-source sass -k regex:K > x.csv;
python tools/sass_hot.py x.csv [top]"""
import csv
import sys
from collections import Counter


def num(s):
    try:
        return int(s)
    except ValueError:
        return 0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
tot = sum(num(r[i_s]) for r in data)
print("total samples", tot, "instructions", len(data))
cs, ce = Counter(), Counter()
for r in data:
    toks = r[i_src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    cs[op] += num(r[i_s])
    ce[op] += num(r[i_ex])
for op, v in cs.most_common(22):
    print(f"{op:10s} samples {v:8d} ({100 * v / max(tot, 1):5.1f} %)  executed {ce[op]}")
print("top instructions:")
for r in sorted(data, key=lambda r: -num(r[i_s]))[:top]:
    print(f"{num(r[i_s]):7d}  {r[0][-5:]}  {r[i_src][:100]}")
