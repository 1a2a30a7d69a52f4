"""Summarise ncu captures into profiles/ (markdown): per-kernel duration,
occupancy, pipe utilisation, DRAM traffic and stall breakdown, plus a
launch-list aggregate.  Usage:
  python tools/ncu_summary.py report.ncu-rep [launches.csv] > profiles/rNN_name.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, rows = raw(rep)
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    seen = set()
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        short = re.sub(r"\(.*", "", name)[:70]
        if short in seen:
            continue
        seen.add(short)
        print(f"## `{short}`\n")
        print("| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} | {r[i]} {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio", h)
            if m and r[i] not in ("", "0"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.05 and m.group(1) not in ("selected",):
                    stalls.append((v, m.group(1)))
        stalls.sort(reverse=True)
        print("| stalls per issued instr | " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:7]) + " |\n")
    if len(sys.argv) > 2:
        agg = defaultdict(list)
        for r in csv.reader(open(sys.argv[2])):
            if len(r) > 5 and r[0] != "ID":
                try:
                    agg[re.sub(r"\(.*", "", r[4])[:70]].append(float(r[-1]))
                except (ValueError, IndexError):
                    pass
        print("## launch list (cold-cache, serialised; compare shares)\n")
        print("| kernel | launches | avg us | total us |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} |")


if __name__ == "__main__":
    main()
