"""Per-kernel stall breakdown (pc sampling) and hottest SASS lines from an ncu report.
Usage: python profiles/ncu_stalls.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(path, kregex, top=15):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kregex}",
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    ops, st, lines = collections.Counter(), collections.Counter(), []
    tot = stt = 0
    for r in rows[2:]:
        try:
            n, s = int(float(r[i_ex] or 0)), int(float(r[i_st] or 0))
        except (ValueError, IndexError):
            continue
        p = r[i_src].split()
        if not p:
            continue
        op = (p[1] if p[0].startswith("@") else p[0]).split(".")[0]
        ops[op] += n
        st[op] += s
        tot += n
        stt += s
        lines.append((s, n, r[0], r[i_src]))
    print(f"instructions {tot}  stall samples {stt}")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n:10d} {100 * n / max(tot, 1):5.1f}%  stall {100 * st[op] / max(stt, 1):5.1f}%")
    print("hottest lines (stall samples, executions, sass):")
    for s, n, a, src in sorted(lines, reverse=True)[:top]:
        print(f"  {s:6d} {n:9d}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 15)
