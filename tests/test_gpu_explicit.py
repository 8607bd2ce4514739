"""GPU parity for explicit (full-bitstring) bases (reference apply.py:320-458, 675-703).

Bars: diagonal bitwise; sigma within 1e-10 relative (inf-norm) of the reference
(golden, produced by the reference's _explicit_kernel) and of the oracle
restatement; lowest energies within 1e-8 Ha of the reference davidson_solve.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle as O
from test_oracle_golden import EXPLICIT, explicit_instance

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10


def _rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def _basis(g, meta, name):
    from paper_2601_16637_b200 import Determinant, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals

    m = meta[name]
    dets = [Determinant(int(a), int(b)) for a, b in zip(g[f"{name}/det_a"], g[f"{name}/det_b"])]
    return SelectedBasis.explicit(dets, m["norb"], m["na"], m["nb"]), random_integrals(m["norb"], seed=m["iseed"])


@pytest.mark.parametrize("name", EXPLICIT)
def test_explicit_vs_reference(explicit_golden, explicit_meta, name):
    import torch

    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, davidson_solve

    g = explicit_golden
    basis, table = _basis(g, explicit_meta, name)
    app = HamiltonianApplier(basis, table)
    assert app.tables is None and app.cache is None
    assert np.array_equal(app.diag, g[f"{name}/diag"])
    for x, y in zip(g[f"{name}/x"], g[f"{name}/y"]):
        assert _rel(app(x), y) <= SIGMA_RTOL                      # host protocol
        yd = app(torch.from_numpy(x).cuda()).cpu().numpy()        # device path
        assert _rel(yd, y) <= SIGMA_RTOL
    m = explicit_meta[name]
    n = basis.dimension
    opts = DavidsonOptions(n_roots=m["n_roots"], restart_keep=min(4, n), max_subspace=min(32, n))
    res = davidson_solve(app, app.diag, opts=opts)
    assert res.converged
    np.testing.assert_allclose(res.energies, g[f"{name}/energies"], atol=1e-8)
    assert abs(res.stats.iterations - m["iterations"]) <= 1


def test_explicit_random_vs_oracle():
    """Larger random explicit sets (one alpha string shared by many dets, and the converse)."""
    from paper_2601_16637_b200 import HamiltonianApplier
    from paper_2601_16637_b200.synth import random_explicit_basis, random_integrals

    for norb, na, nb, nd, seed in ((14, 5, 6, 60000, 3), (16, 4, 4, 30000, 4), (20, 3, 2, 20000, 5)):
        basis = random_explicit_basis(norb, na, nb, nd, seed)
        table = random_integrals(norb, seed)
        app = HamiltonianApplier(basis, table)
        inst = O.ExplicitInstance.make(norb, table.h, table.eri, table.e_core,
                                       [d.alpha for d in basis.dets], [d.beta for d in basis.dets])
        d = O.diag_explicit(inst)
        assert np.array_equal(app.diag, d)
        x = np.random.default_rng(seed).standard_normal(nd)
        assert _rel(app(x), O.sigma_explicit(inst, x, d)) <= SIGMA_RTOL, (norb, na, nb, nd)


def test_explicit_api_and_errors(explicit_golden, explicit_meta):
    from paper_2601_16637_b200 import HamiltonianApplier, _lib, apply_H_full, compute_diagonal

    g = explicit_golden
    basis, table = _basis(g, explicit_meta, "expl_6_3_3")
    x = g["expl_6_3_3/x"][0]
    assert _rel(apply_H_full(x, basis, table), g["expl_6_3_3/y"][0]) <= SIGMA_RTOL
    assert np.array_equal(compute_diagonal(basis, table), g["expl_6_3_3/diag"])
    with pytest.raises(ValueError):
        HamiltonianApplier(basis, table, row_window=(0, 1))
    app = HamiltonianApplier(basis, table)
    with pytest.raises(ValueError):
        app(np.zeros(basis.dimension + 1))
    # the C ABI rejects a duplicated determinant (SelectedBasis.explicit, basis.py:175)
    ctx = _lib.Context(0)
    h = np.ascontiguousarray(table.h)
    eri = np.ascontiguousarray(table.eri)
    ctx("sbd_set_integrals", table.norb, _lib.ptr(h), _lib.ptr(eri), eri.size, table.e_core)
    a = np.array([0b000111, 0b001011, 0b000111], dtype=np.uint64)
    b = np.array([0b000111, 0b000111, 0b000111], dtype=np.uint64)
    ctx("sbd_set_dets", _lib.ptr(a), _lib.ptr(b), 3, 3, 3)
    with pytest.raises(ValueError, match="duplicate"):
        ctx("sbd_build_tables")
    with pytest.raises(ValueError):
        ctx("sbd_sigma_local", ctypes.c_void_p(0))
