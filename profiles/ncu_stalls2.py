"""Top stall sites of one kernel from `ncu -i rep --page source --csv --print-source sass -k ... -c 1`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
his = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r]
sec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = his[sec]
end = his[sec + 1] - 1 if sec + 1 < len(his) else len(rows)
hdr = rows[hi]
data = [r for r in rows[hi + 1:end] if len(r) == len(hdr)]
ia, iss, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
num = lambda x: int(float(x or 0))
tot = {h: sum(num(r[hdr.index(h)]) for r in data) for h in names}
allst = sum(tot.values())
print("kernel:", rows[hi - 1][1][:100])
print("stall totals:", [(k, round(v / allst, 3)) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]])
print("instructions executed:", sum(num(r[ie]) for r in data))
for r in sorted(data, key=lambda r: -num(r[iss]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    st = {h: num(r[hdr.index(h)]) for h in names}
    m = max(st, key=st.get)
    print(f"{num(r[iss]):6d} {num(r[ie]):9d}  {r[ia].strip()[:72]:72s} {m} {st[m]}")
