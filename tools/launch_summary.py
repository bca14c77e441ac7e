"""Average device time per kernel name from an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
head, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        head = r
        continue
    if head and len(r) == len(head):
        d = dict(zip(head, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(d.get("Metric Unit", "ns"), 1e-6)
            agg.setdefault(d["Kernel Name"][:70], []).append(float(d["Metric Value"].replace(",", "")) * scale)
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v):10.3f} ms  {k}")
