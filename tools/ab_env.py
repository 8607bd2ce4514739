"""Same-process A/B of environment knobs on the sigma build, over sweep points.

    python tools/ab_env.py "SBD_CROSS_DCI=0" "SBD_CROSS_DCI=1" [--points cfg1,cfg2,cfg4,1e9] [--steps K]

Each point is built once; the variants are timed alternately (CUDA events over K
sigma builds after 2 warm-ups, best of 3 rounds) so box-to-box clock drift cancels.
The knobs are read by libsbd_b200.so at every launch.  Prints one JSON line per point.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

POINTS = {
    "cfg1": (12, 6, 0), "1e6": (16, 8, 1000), "1e7": (20, 10, 3162), "cfg2": (26, 7, 10000),
    "3e8": (32, 8, 17782), "cfg4": (36, 27, 30000), "1e9": (40, 10, 31622),
}


def _set(spec: str):
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=", 1)
        if v == "":
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def main():
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--points", default="cfg1,cfg2,cfg4,1e9")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    for name in args.points.split(","):
        norb, ne, ns = POINTS[name]
        table = synth.random_integrals(norb, seed=1)
        if ns == 0:
            app = HamiltonianApplier(synth.full_product_basis(norb, ne, ne), table)
        else:
            a, b = synth.random_product_strings(norb, ne, ne, ns, ns, seed=2)
            app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
        x = torch.empty(app.n, dtype=torch.float64, device="cuda").normal_(generator=torch.Generator("cuda").manual_seed(1))
        y = torch.empty_like(x)
        ref = None
        best = {v: float("inf") for v in args.variants}
        for _ in range(3):
            for v in args.variants:
                saved = dict(os.environ)
                _set(v)
                for _ in range(2):
                    app.sigma_device(x, out=y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(args.steps):
                    app.sigma_device(x, out=y)
                e1.record()
                torch.cuda.synchronize()
                best[v] = min(best[v], e0.elapsed_time(e1) / args.steps)
                if ref is None:
                    ref = y.clone()
                else:
                    err = float((y - ref).abs().max() / ref.abs().max())
                    assert err <= 1e-12, (name, v, err)
                os.environ.clear()
                os.environ.update(saved)
        cbar, bytes_ = app.sigma_model()
        print(json.dumps({"point": name, "n_dets": app.n, "cbar_alpha": cbar,
                          "ms": {v: round(t, 4) for v, t in best.items()},
                          "roofline_frac_fallback": {v: bytes_ / (t * 1e-3) / 6.55e12 for v, t in best.items()}}),
              flush=True)
        del app, x, y, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
