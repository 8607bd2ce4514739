"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, avg and total time per kernel.

    python tools/launch_summary.py gpurun_out/<tag>/launches.csv > profiles/<tag>/launches_summary.json
"""

import csv
import io
import json
import sys


def summarize(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        name = r["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    out = [{"kernel": k, "launches": n, "avg_us": t / n, "total_us": t} for k, (n, t) in agg.items()]
    return sorted(out, key=lambda d: -d["total_us"])


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))
