"""Summarise an ncu --set full report: per kernel time, DRAM bytes, L2 hit rate, throughputs."""

import csv
import io
import json
import subprocess
import sys

WANT = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_read_sectors": "lts__t_sectors_srcunit_tex_op_read.sum",
}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, m in WANT.items():
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", "")) if r[i] else None
                u = units[i]
                if v is not None and u in SCALE:
                    v *= SCALE[u]
                d[k] = v
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    for d in res:
        print(json.dumps(d))
