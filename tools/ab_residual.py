"""Per-k timing of the Davidson residual pass (sbd_residual_precond_target) at the bench size, per variant.

    python tools/ab_residual.py "SBD_RES_STREAM=0" "SBD_RES_STREAM=1" ["SBD_RES_STREAM=0,SBD_RES_SPLIT=2"] \
        [--n 100000000] [--ks 5,8,12,16,20,24,28,32]

CUDA events around 5 launches after 2 warm-ups, best of 3 rounds; variants alternate per k.  Reports ms and the
achieved HBM rate of the pass's (2k+1) reads + 1 write of n doubles.  One JSON line per k.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _set(spec: str):
    for kv in filter(None, spec.split(",")):
        key, val = kv.split("=", 1)
        os.environ[key] = val


def main():
    import torch

    from paper_2601_16637_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--ks", default="5,8,12,16,20,24,28,32")
    ap.add_argument("--m", type=int, default=1)
    args = ap.parse_args()
    n, m = args.n, args.m
    ks = [int(v) for v in args.ks.split(",")]
    kmax = max(ks)
    dev = torch.device("cuda", 0)
    g = torch.Generator("cuda").manual_seed(1)
    V = torch.empty((kmax, n), dtype=torch.float64, device=dev).normal_(generator=g)
    W = torch.empty((kmax, n), dtype=torch.float64, device=dev).normal_(generator=g)
    diag = torch.empty(n, dtype=torch.float64, device=dev).normal_(generator=g)
    T = torch.empty((m, n), dtype=torch.float64, device=dev)
    theta = torch.full((m,), 0.1, dtype=torch.float64, device=dev)
    res = torch.empty(kmax + 1 + m, dtype=torch.float64, device=dev)
    ctx = _lib.Context(0)
    ctx.bind_stream()
    p = _lib.ptr
    for k in ks:
        Y = torch.randn((k, m), dtype=torch.float64, device=dev, generator=g)
        best = {v: float("inf") for v in args.variants}
        for _ in range(3):
            for v in args.variants:
                saved = dict(os.environ)
                _set(v)

                def run():
                    ctx("sbd_residual_precond_target", p(V), p(W), k, n, n, p(Y), p(theta), m, 0, p(diag), 1e-3,
                        p(T), n, p(res))

                for _ in range(2):
                    run()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(5):
                    run()
                e1.record()
                torch.cuda.synchronize()
                best[v] = min(best[v], e0.elapsed_time(e1) / 5)
                os.environ.clear()
                os.environ.update(saved)
        gb = (2 * k + 1 + m) * 8 * n / 1e9
        print(json.dumps({"k": k, "m": m, "n": n, "gb": gb, "ms": {v: round(t, 4) for v, t in best.items()},
                          "tb_s": {v: round(gb / t, 3) for v, t in best.items()}}), flush=True)


if __name__ == "__main__":
    main()
