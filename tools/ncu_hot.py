"""Top SASS lines by warp-stall samples from an ncu source-page CSV.
    ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv; python tools/ncu_hot.py s.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
tot = sum(float(r[si] or 0) for r in body)
print("total samples", tot)
for r in sorted(body, key=lambda r: -float(r[si] or 0))[:n]:
    s = float(r[si] or 0)
    top = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{s/tot*100:5.1f}% {r[0]} {r[1][:70]:70s} " + " ".join(f"{h}={v:.0f}" for v, h in top))
