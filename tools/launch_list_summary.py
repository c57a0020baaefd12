"""Summarise an ncu launch list (``ncu --metrics gpu__time_duration.sum --csv --log-file X``)
into per-kernel launches / total time / share, the profiles/rN_launch_list_summary.csv format.
Set-up kernels (random weight init ``fill_uniform_kernel``, torch fills) are left out so the
shares are of the serving kernels.

    python tools/launch_list_summary.py gpurun_out/launches.csv "header line" > profiles/...csv
"""
import csv
import re
import sys
from collections import defaultdict

UNITS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def main():
    path, header = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", row["Kernel Name"]).replace("void ", "").strip()
        if "fill_uniform" in name or name.startswith("at::"):
            continue
        ms = float(row["Metric Value"].replace(",", "")) * UNITS.get(row.get("Metric Unit", "ns"), 1e-6)
        tot[name] += ms
        cnt[name] += 1
    all_ms = sum(tot.values()) or 1.0
    if header:
        for h in header.split("\\n"):
            print("# " + h)
    w = csv.writer(sys.stdout, lineterminator="\n")
    w.writerow(["kernel", "launches", "total_ms", "share", "avg_us"])
    for name in sorted(tot, key=lambda k: -tot[k]):
        w.writerow([name, cnt[name], f"{tot[name]:.3f}", f"{tot[name] / all_ms:.4f}",
                    f"{tot[name] / cnt[name] * 1e3:.2f}"])


if __name__ == "__main__":
    main()
