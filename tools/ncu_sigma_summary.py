"""profiles/ncu_sigma_summary.json (read by bench.py's roofline object) from a sigma ncu_summary jsonl.

    python tools/ncu_sigma_summary.py profiles/<tag>/ncu_sigma_full.jsonl > profiles/ncu_sigma_summary.json
"""

import json
import sys


def main(path):
    per, tot = {}, 0.0
    for line in open(path):
        r = json.loads(line)
        b = r["dram_read"] + r["dram_write"]
        tot += b
        per[r["kernel"].split("(")[0]] = {"time_ms": r["time_ms"], "dram_bytes": b, "l2_hit_pct": r["l2_hit_pct"],
                                          "l2_pct": r["l2_pct"], "dram_pct": r["dram_pct"]}
    return {"source": f"{path} (ncu --set full, one launch of each sigma kernel, cfg2 1e8 dets)",
            "dram_bytes_per_sigma": tot, "per_kernel": per}


if __name__ == "__main__":
    print(json.dumps(main(sys.argv[1])))
