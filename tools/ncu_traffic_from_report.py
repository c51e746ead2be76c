"""Writes profiles/ncu_traffic.json from an `ncu --set full` report of tools/profile_step.py (one
launch per op, in profile_step.ORDER).  Usage: python tools/ncu_traffic_from_report.py report.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from profile_step import ORDER  # noqa: E402

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    launches = rows[2:]
    assert len(launches) == len(ORDER), (len(launches), len(ORDER))
    f = lambda r, m: float(r[idx[m]].replace(",", "") or 0) * SCALE.get(units[idx[m]], 1)  # noqa: E731
    res = {"_about": "DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from one `ncu --set full "
                     "--clock-control none` capture of one serial pass of bench.py's step kernels plus the NEXT-row "
                     "kernels (tools/profile_step.py; summary profiles/r02_ncu_summary.md). ncu flushes caches "
                     "before each kernel; writes still resident in L2 when the kernel ends are not counted, so "
                     "traffic can be below the algorithmic bytes."}
    for op, r in zip(ORDER, launches):
        tp = M[3]
        res[op] = {"kernel": r[idx["Kernel Name"]].split("(")[0].split("<")[0],
                   "dram_bytes_per_launch": int(f(r, M[1]) + f(r, M[2])),
                   "ncu_us": round(f(r, M[0]), 1),
                   "tensor_pipe_active_pct": round(f(r, tp), 1) if tp in idx else None}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
