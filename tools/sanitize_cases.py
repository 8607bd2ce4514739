"""Small workloads that launch every kernel variant once, for compute-sanitizer runs.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_cases.py [variant]

variant = "all" (default) runs: tables, diag, every sigma variant (cluster multicast
task 0, TMA-staged, flat/unstaged, additive order, register streams, row Y^T, host
pipelined path), the explicit-basis sigma, device ingestion, the Davidson passes at
K = 8/16/24/32/64 with and without TMA, the native solver and the dense rows of verify.
Each case checks its result against the oracle, so a sanitizer run is also a parity run.
SAN_VARIANT=i restricts the sigma cases to SIGMA_ENVS[i] (one kernel variant per racecheck process).
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402  (checker)

SIGMA_ENVS = [{}, {"SBD_SIDE_LDG": "1"}, {"SBD_YT_BLOCKED": "0"}, {"SBD_CROSS_NO_CLUSTER": "1"},
              {"SBD_CROSS_UNSTAGED": "1"}, {"SBD_CROSS_ADD": "1"}, {"SBD_CROSS_DCI": "1"},
              {"SBD_CROSS_DCI": "1", "SBD_CROSS_ADD": "1"}, {"SBD_DENSE_GEMM": "1"},
              {"SBD_DENSE_GEMM": "1", "SBD_CROSS_DCI": "1"}]
DAV_ENVS = [{}, {"SBD_RES_STREAM": "0"}, {"SBD_DAV_TMA": "1"}, {"SBD_NO_TMA": "1"}]


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def sigma_cases():
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    for norb, ne, nsa, nsb, seed in ((12, 6, 300, 130, 8), (11, 4, 97, 77, 9)):
        a, b = random_product_strings(norb, ne, ne, nsa, nsb, seed=seed)
        table = random_integrals(norb, seed=seed)
        inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
        x = np.random.default_rng(seed).standard_normal(nsa * nsb)
        ref = O.sigma(inst, x)
        only = os.environ.get("SAN_VARIANT")  # one variant per process (racecheck runs)
        for vi, env in enumerate(SIGMA_ENVS):
            if only is not None and int(only) != vi:
                continue

            def run():
                app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
                assert np.array_equal(app.diag, O.diag(inst))
                yh = app(x)
                yd = app.sigma_device(torch.from_numpy(x).cuda()).cpu().numpy()
                for y in (yh, yd):
                    assert np.abs(y - ref).max() <= 1e-10 * np.abs(ref).max(), env
            _with_env(env, run)
            print("sigma ok", norb, ne, nsa, nsb, env, flush=True)


def explicit_case():
    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    a, b = random_product_strings(10, 4, 4, 40, 40, seed=3)
    rng = np.random.default_rng(4)
    pairs = {(int(a[i]), int(b[j])) for i, j in zip(rng.integers(0, 40, 900), rng.integers(0, 40, 900))}
    da = np.array([p[0] for p in pairs], dtype=np.uint64)
    db = np.array([p[1] for p in pairs], dtype=np.uint64)
    table = random_integrals(10, seed=3)
    app = HamiltonianApplier(SelectedBasis.explicit(list(zip(da.tolist(), db.tolist())), 10, 4, 4), table)
    inst = O.ExplicitInstance.make(10, table.h, table.eri, table.e_core, da, db)
    x = rng.standard_normal(app.n)
    ref = O.sigma_explicit(inst, x)
    assert np.abs(app(x) - ref).max() <= 1e-10 * np.abs(ref).max()
    print("explicit ok", flush=True)


def ingest_case():
    from paper_2601_16637_b200.ingest import ingest_sample_arrays

    rng = np.random.default_rng(5)
    a = rng.choice(np.array([0b0111, 0b1011, 0b1101, 0b1110, 0b10011], dtype=np.uint64), 500)
    b = rng.choice(np.array([0b0011, 0b0101, 0b1001, 0b11000], dtype=np.uint64), 500)
    ingest_sample_arrays(a, b, 6, 3, 2)
    print("ingest ok", flush=True)


def davidson_cases():
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, SelectedBasis, davidson_solve
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    a, b = random_product_strings(10, 5, 5, 60, 50, seed=2)
    table = random_integrals(10, seed=1)
    inst = O.Instance.make(10, table.h, table.eri, table.e_core, a, b)
    for k_max, keep, roots in ((8, 4, 1), (16, 4, 2), (24, 6, 1), (32, 4, 1), (64, 8, 3)):
        ref = O.davidson(lambda v: O.sigma(inst, v), O.diag(inst), n_roots=roots, max_subspace=k_max,
                         restart_keep=keep)
        for env in DAV_ENVS:
            for native in (True, False):
                def run():
                    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 10, 5, 5), table)
                    res = davidson_solve(app, app.diag, opts=DavidsonOptions(n_roots=roots, max_subspace=k_max,
                                                                             restart_keep=keep), native=native)
                    assert res.converged and np.abs(res.energies - ref.energies).max() <= 1e-8
                _with_env(env, run)
        print("davidson ok", k_max, flush=True)


def residual_case():
    """The streamed residual pass with several tiles per CTA (its stage ring wraps), odd n, k in each tile size."""
    import torch

    from paper_2601_16637_b200 import _lib

    n = 148 * 256 * 3 + 77
    ctx = _lib.Context(0)
    ctx.bind_stream()
    rng = np.random.default_rng(3)
    for k, m in ((5, 1), (16, 2), (28, 3)):
        V = torch.from_numpy(rng.standard_normal((k, n))).cuda()
        W = torch.from_numpy(rng.standard_normal((k, n))).cuda()
        Y = torch.from_numpy(rng.standard_normal((k, m))).cuda()
        th = torch.from_numpy(rng.standard_normal(m)).cuda()
        d = torch.from_numpy(rng.standard_normal(n)).cuda()
        T = torch.empty((m, n), dtype=torch.float64, device="cuda")
        out = torch.empty(k + 1 + m, dtype=torch.float64, device="cuda")
        p = _lib.ptr
        ctx("sbd_residual_precond_target", p(V), p(W), k, n, n, p(Y), p(th), m, m - 1, p(d), 1e-3, p(T), n, p(out))
        Vn, Wn, Yn, thn, dn = (t.cpu().numpy() for t in (V, W, Y, th, d))
        R = Yn.T @ Wn - thn[:, None] * (Yn.T @ Vn)
        dd = dn[None, :] - thn[:, None]
        Tn = R / (np.where(dd >= 0, 1.0, -1.0) * np.maximum(np.abs(dd), 1e-3))
        assert np.abs(T.cpu().numpy() - Tn).max() <= 1e-10 * np.abs(Tn).max()
        assert np.abs(out.cpu().numpy()[:k] - Vn @ Tn[m - 1]).max() <= 1e-9 * np.abs(Vn @ Tn[m - 1]).max()
    print("residual ok", flush=True)


def tables128_case():
    from paper_2601_16637_b200 import build_excitation_table128, sorted_strings128

    rng = np.random.default_rng(4)
    window = list(range(56, 72)) + list(range(120, 128))
    strings = sorted({sum(1 << int(o) for o in rng.choice(window, 4, replace=False)) for _ in range(3000)})
    rng.shuffle(strings)
    tab = build_excitation_table128(strings, 128)
    ref = O.build_table128(strings, 128)
    for f in O.TABLE_FIELDS:
        assert np.array_equal(getattr(tab, f), ref[f]), f
    w, perm = sorted_strings128(strings, 128)
    assert [int(lo) | int(hi) << 64 for lo, hi in w.tolist()] == sorted(strings)
    print("tables128 ok", flush=True)


def dense_case():
    from paper_2601_16637_b200 import SelectedBasis
    from paper_2601_16637_b200.dense import assemble_dense
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    a, b = random_product_strings(8, 3, 3, 20, 18, seed=5)
    table = random_integrals(8, seed=6)
    inst = O.Instance.make(8, table.h, table.eri, table.e_core, a, b)
    d = assemble_dense(SelectedBasis.product(a.tolist(), b.tolist(), 8, 3, 3), table)
    assert np.abs(d - O.dense(inst)).max() <= 1e-12 * np.abs(d).max()
    print("dense ok", flush=True)


CASES = {"sigma": sigma_cases, "explicit": explicit_case, "ingest": ingest_case, "davidson": davidson_cases,
         "dense": dense_case, "residual": residual_case, "tables128": tables128_case}

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in CASES.items():
        if which in ("all", name):
            fn()
    print("ALL OK")
