"""Writes profiles/traffic.json: DRAM bytes (read + write) per launch of the
spread / interpolation kernels from `ncu --set full` captures, keyed by bench
workload, for bench.py's roofline.traffic field.
  python tools/make_traffic.py config2=gpurun_out/r01_c2_full.ncu-rep config4=...
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
for arg in sys.argv[1:]:
    workload, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    entry = data.setdefault(workload, {})
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        kind = "spread" if "spread" in name else ("interp" if "interp" in name else None)
        if kind is None or kind in entry:
            continue
        try:
            b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
        except (ValueError, KeyError):
            continue
        if b != b:  # NaN: metric not collected
            continue
        entry[kind] = {"dram_bytes": b, "kernel": re.sub(r"\(.*", "", name), "source": os.path.basename(rep)}
json.dump(data, open(out_path, "w"), indent=1)
print(json.dumps(data, indent=1))
