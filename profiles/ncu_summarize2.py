"""Summarise an ncu --set full report (raw page CSV) into a per-kernel table (tools, not product)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = {"kernel": "Kernel Name", "us": "gpu__time_duration.sum", "rdMB": "dram__bytes_read.sum",
        "wrMB": "dram__bytes_write.sum", "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm%": "sm__throughput.avg.pct_of_peak_sustained_elapsed", "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
        "grid": "launch__grid_size", "winst": "smsp__inst_executed.sum", "l2hit%": "lts__t_sector_hit_rate.pct"}
idx = {k: (hdr.index(v) if v in hdr else None) for k, v in want.items()}
units = rows[1]
print("| " + " | ".join(want) + " |")
print("|" + "---|" * len(want))
for r in rows[2:]:
    vals = []
    for k, i in idx.items():
        v = r[i] if i is not None else "-"
        if k == "kernel":
            v = v.split("(")[0].replace("void ", "")[:40]
        elif k in ("rdMB", "wrMB") and i is not None:
            u = units[i]
            x = float(v.replace(",", ""))
            v = f"{x / 1e6 if u == 'byte' else x * (1024 if u == 'Kbyte' else 1) if u == 'Mbyte' else x * 1e3 if u == 'Gbyte' else x:.1f}"
        elif k == "us" and i is not None:
            u = units[i]
            x = float(v.replace(",", ""))
            v = f"{x / 1e3 if u == 'nsecond' else x if u == 'usecond' else x * 1e3:.1f}"
        vals.append(v)
    print("| " + " | ".join(vals) + " |")
