"""Per-phase device time of the Davidson driver at the bench workload (tracing aid)."""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(iters: int = 40, roots: int = 1):
    import torch

    import bench
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, SelectedBasis, davidson_solve

    table, a, b = bench._instance()
    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 26, 7, 7), table)
    opts = DavidsonOptions(max_iters=iters, profile=True, n_roots=roots, restart_keep=max(4, roots))
    t0 = time.perf_counter()
    res = davidson_solve(app, app.diag_device, opts=opts, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    it = res.stats.iterations
    ph = {k: v / it for k, v in sorted(res.stats.phase_ms.items(), key=lambda kv: -kv[1])}
    out = {"iterations": it, "wall_ms_per_iter": wall * 1e3 / it, "device_ms_per_iter_by_phase": ph,
           "device_ms_per_iter_total": sum(ph.values())}
    # one steady-state iteration on the device clock: (phase, start ms, duration ms); gaps are idle time
    out["timeline_one_iteration"] = [(n, round(t0, 4), round(d, 4)) for n, t0, d in res.stats.timeline]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
