"""Determinant-count sweep (BASELINE configs[4]): sigma dets/s and roofline fraction on one B200.

    python tools/sweep.py [--steps K] > profiles/sweep_<tag>.json

Each point samples uniform random strings (the restated reference generator,
integrals seed 1, strings seed 2), builds the device tables, and times K sigma
builds with CUDA events after 3 warm-ups.  The roofline numerator is the
algorithmic bytes of SURVEY section 8(d), B = 8 N (3 + c-bar_alpha), with
c-bar_alpha read from the actual tables.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POINTS = [  # norb, electrons per spin, strings per spin
    (12, 6, 924),    # cfg1: the full 12-orbital string set (dense: task 0 dominates)
    (16, 8, 1000),
    (20, 10, 3162),
    (26, 7, 10000),
    (32, 8, 17782),
    (36, 27, 30000),
    (40, 10, 31622),
]


def main():
    import torch

    import bench
    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    peak, peak_src = bench._peaks()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    out = []
    for norb, ne, ns in POINTS:
        t0 = time.perf_counter()
        table = synth.random_integrals(norb, seed=1)
        a, b = synth.random_product_strings(norb, ne, ne, ns, ns, seed=2)
        app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
        setup = time.perf_counter() - t0
        n = app.n
        x = torch.empty(n, dtype=torch.float64, device=dev).normal_(generator=torch.Generator(device=dev).manual_seed(1))
        y = torch.empty_like(x)
        for _ in range(3):
            app.sigma_device(x, out=y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            app.sigma_device(x, out=y)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = e0.elapsed_time(e1) / 1e3 / args.steps
        cbar, nbytes = app.sigma_model()
        rec = {"norb": norb, "n_elec_per_spin": ne, "strings_per_spin": ns, "n_dets": n, "cbar_alpha": cbar,
               "ms_per_sigma": t * 1e3, "dets_per_s": n / t, "algorithmic_bytes": nbytes,
               "achieved_gbs": nbytes / t / 1e9, "roofline_frac": nbytes / t / 1e9 / peak, "setup_s": setup}
        print(json.dumps(rec), file=sys.stderr, flush=True)
        out.append(rec)
        del app, x, y
        torch.cuda.empty_cache()
    print(json.dumps({"peak_gbs": peak, "peak_source": peak_src, "steps": args.steps, "points": out}, indent=1))


if __name__ == "__main__":
    main()
