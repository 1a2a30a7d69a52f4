"""Aggregate ncu warp-stall samples per CUDA source line for one kernel.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
(needs a capture with --import-source on and -lineinfo builds)"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg, total, fname, src, hdr, why = {}, 0, "?", {}, None, {}
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if row[0] == "Function Name" or len(row) < 5:
        continue
    if row[0] != "-" and row[0].isdigit():  # a source line row: (line, text, address, sass, samples...)
        key = (fname, int(row[0]))
        src[key] = row[1].strip()[:90]
        try:
            s = int(row[4])
        except ValueError:
            continue
        agg[key] = agg.get(key, 0) + s
        total += s
        if hdr:
            reasons = why.setdefault(key, {})
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h and i < len(row):
                    try:
                        reasons[h[6:]] = reasons.get(h[6:], 0) + int(row[i])
                    except ValueError:
                        pass
print(f"total samples {total}")
for key, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    r = sorted(why.get(key, {}).items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{k}:{v}" for k, v in r if v)
    print(f"{100.0 * s / max(total, 1):5.1f}%  {key[0]}:{key[1]:<5} {src.get(key, '')[:70]}  [{rs}]")
