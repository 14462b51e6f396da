"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launches, total ms, share, average us.
    python tools/launch_summary.py gpurun_out/launches_cfg2_r1c.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            unit = d.get("Metric Unit", "nsecond")
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
            k = d["Kernel Name"].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {ms:.2f} | {ms / tot:.3f} | {ms / n * 1e3:.1f} |")
