"""Summarise an ncu --set full report: per kernel time, DRAM bytes, throughput, occupancy, IPC.
Usage: python profiles/ncu_summarize.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    print("| kernel | us | DRAM rd MB | DRAM wr MB | DRAM % | SM % | IPC | warps % | regs | grid | warp-inst |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        v = [r[idx[m]] for m in M]
        f = lambda x: float(x.replace(",", "")) if x else 0.0  # noqa: E731
        mb = lambda m: f(r[idx[m]]) * scale.get(units[idx[m]], 1e-6) * 1e6  # noqa: E731
        v[1], v[2] = str(mb(M[1])), str(mb(M[2]))
        print(f"| {name} | {f(v[0]):.1f} | {f(v[1]) / 1e6:.1f} | {f(v[2]) / 1e6:.1f} | {f(v[3]):.1f} | {f(v[4]):.1f} | "
              f"{f(v[5]):.2f} | {f(v[6]):.1f} | {int(f(v[7]))} | {int(f(v[8]))} | {int(f(v[9]))} |")


if __name__ == "__main__":
    main(sys.argv[1])
