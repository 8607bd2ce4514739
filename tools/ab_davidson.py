"""Same-process A/B of environment knobs on the Davidson solve at the bench workload (cfg2, 1e8 dets).

    python tools/ab_davidson.py "SBD_RES_SPLIT=1" "SBD_RES_SPLIT=2" [--iters 60] [--rounds 2]

Each variant runs the native solve at reference defaults (max_iters --iters) alternately; prints the
mean s/iter after the first iteration, the iteration count and E0 per variant (one JSON line).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, SelectedBasis, davidson_solve

    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    table, a, b = bench._instance()
    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 26, 7, 7), table)
    out = {v: [] for v in args.variants}
    info = {}
    for _ in range(args.rounds):
        for v in args.variants:
            saved = dict(os.environ)
            for kv in filter(None, v.split(",")):
                k, val = kv.split("=", 1)
                os.environ[k] = val
            res = davidson_solve(app, app.diag_device, opts=DavidsonOptions(max_iters=args.iters), return_device=True)
            torch.cuda.synchronize()
            its = res.stats.iter_seconds
            out[v].append(statistics.mean(its[1:]))
            info[v] = {"iterations": res.stats.iterations, "energy": float(res.energies[0])}
            del res
            os.environ.clear()
            os.environ.update(saved)
    print(json.dumps({v: {"s_per_iter_best": min(t), **info[v]} for v, t in out.items()}), flush=True)


if __name__ == "__main__":
    main()
