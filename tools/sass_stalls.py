"""Per-instruction stall / bank-conflict view of one kernel in an ncu report.
usage: python tools/sass_stalls.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys, collections
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + rx,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows, _seen = [], set()
for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
    if r["Address"] in _seen or r["Address"] == "Address": continue
    _seen.add(r["Address"]); rows.append(r)
stalls = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
def f(r, k):
    try: return float(r[k].replace(",", ""))
    except Exception: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in rows)
ops = collections.Counter(); opsx = collections.Counter(); opn = collections.Counter()
for r in rows:
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"): op = r["Source"].split()[1]
    op = op.split(".")[0]
    ops[op] += f(r, "Warp Stall Sampling (All Samples)")
    opsx[op] += f(r, "L1 Wavefronts Shared Excessive")
    opn[op] += f(r, "Instructions Executed")
print(f"total samples {tot:.0f}; instructions {sum(opn.values()):.3g}")
print("by opcode: samples%  executed  smem-excess-wavefronts")
for op, v in ops.most_common(20):
    print(f"  {op:10s} {100*v/tot:5.1f}%  {opn[op]:.3g}  {opsx[op]:.3g}")
print("top instructions:")
rows.sort(key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))
for r in rows[:top]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    st = sorted(((f(r, k), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} exec={f(r,'Instructions Executed'):.3g} "
          f"xs={f(r,'L1 Wavefronts Shared Excessive'):.3g} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v))
