"""cfg4 (BASELINE configs[3]): 36 orbitals, 27a27b, 3e4 x 3e4 strings = 9e8 determinants, 3 lowest roots.

    python tools/cfg4_solve.py [--k-max 6] [--keep 4] [--check] > profiles/cfg4_solve_<tag>.json

BASELINE quotes cfg4 across 8 B200 (57.6 GB of Davidson basis per GPU at k_max = 32).  On
ONE B200 (180 GB) the operator scratch (diag, X^T, Y^T: 21.6 GB), the residual block (3 x 7.2 GB)
and the Ritz vectors (3 x 7.2 GB) leave room for 2 k_max <= 14 basis vectors of 7.2 GB, so
the solve runs at a reduced subspace (default k_max 6, keep 4 >= n_roots).  Output: energies,
residual norms (every root <= tol_residual certifies an eigenpair), iterations, s/iter.
--check re-solves with the reference algorithm (oracle.davidson_torch: two-pass MGS, vstack-free
Ritz vectors) driven by the same device sigma, at the same options, and reports the energy
differences (test infrastructure; a separate process-level run, not part of the timed solve).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, SelectedBasis, davidson_solve, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--k-max", type=int, default=6)
    ap.add_argument("--keep", type=int, default=4)
    ap.add_argument("--max-iters", type=int, default=2000)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    t0 = time.perf_counter()
    table = synth.random_integrals(36, seed=1)
    a, b = synth.random_product_strings(36, 27, 27, 30000, 30000, seed=2)
    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 36, 27, 27), table)
    setup_s = time.perf_counter() - t0
    diag = app.diag_device
    opts = DavidsonOptions(n_roots=3, max_subspace=args.k_max, restart_keep=args.keep, max_iters=args.max_iters)
    # device memory in use, sampled by NVML during the solve: the native solver's basis lives in
    # libsbd_b200 allocations that torch.cuda.max_memory_allocated does not see
    import threading

    import pynvml

    pynvml.nvmlInit()
    handle = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    peak = {"used": 0}
    done = threading.Event()

    def sample():
        while not done.is_set():
            peak["used"] = max(peak["used"], pynvml.nvmlDeviceGetMemoryInfo(handle).used)
            done.wait(0.05)

    sampler = threading.Thread(target=sample, daemon=True)
    sampler.start()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = davidson_solve(app, diag, opts=opts, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t1
    done.set()
    sampler.join()
    total_gb = pynvml.nvmlDeviceGetMemoryInfo(handle).total / 1e9
    its = res.stats.iter_seconds
    rec = {
        "config": "cfg4: 36 orbitals, 27a27b, 3e4 x 3e4 random strings (seed 2), integrals seed 1",
        "n_dets": app.n, "n_roots": 3, "options": {"max_subspace": args.k_max, "restart_keep": args.keep,
                                                    "tol_residual": opts.tol_residual, "max_iters": args.max_iters},
        "why_reduced_subspace": "one 180 GB B200: 21.6 GB operator scratch + 2 x 3 x 7.2 GB residual/Ritz blocks "
                                "leave room for 2 k_max <= 14 basis vectors; BASELINE runs this config on 8 GPUs",
        "energies": [float(e) for e in res.energies], "residual_norms": [float(r) for r in res.residual_norms],
        "converged": bool(res.converged), "iterations": res.stats.iterations, "restarts": res.stats.restarts,
        "wall_s": wall, "s_per_iter": float(np.mean(its[1:])) if len(its) > 1 else float(its[0]),
        "sigma_s_per_iter": float(np.mean(res.stats.apply_seconds[1:] or res.stats.apply_seconds)),
        "setup_s": setup_s, "torch_peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
        "device_mem_used_peak_gb": peak["used"] / 1e9, "device_mem_total_gb": total_gb,
    }
    e_b200 = np.array(rec["energies"])
    del res
    torch.cuda.empty_cache()
    print(json.dumps(rec), flush=True)
    if args.check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O  # checker only

        t2 = time.perf_counter()
        ref = O.davidson_torch(lambda v: app(v), diag, n_roots=3, max_subspace=args.k_max,
                               restart_keep=args.keep, max_iters=args.max_iters)
        chk = {"check": "oracle.davidson_torch (reference davidson.py:191-306, two-pass MGS) driven by the same "
                        "device sigma, same options",
               "energies": [float(e) for e in ref.energies], "converged": bool(ref.converged),
               "iterations": ref.iterations, "max_abs_de": float(np.abs(e_b200 - ref.energies).max()),
               "wall_s": time.perf_counter() - t2}
        print(json.dumps(chk), flush=True)


if __name__ == "__main__":
    main()
