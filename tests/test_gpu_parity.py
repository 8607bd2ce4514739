"""GPU parity: device tables, diagonal and sigma vs the reference (golden) and the oracle.

Bars (north star): tables and indexing bit-exact; sigma within 1e-10 relative
(inf-norm) in fp64; diagonal bit-exact (same operation order).
All calls go through the C ABI (libsbd_b200.so) via the drop-in API.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import TABLE_FIELDS, big_instance, load_big, table_digests

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10
SMALL = ["full_4_2_2_s0", "full_4_2_2_s3", "full_5_2_3_s5", "partial_5_2_3", "partial_6_3_3",
         "partial_8_4_3", "full_6_3_2_s2", "single_det_3", "partial_10_5_5"]


def _rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def _basis(g, meta, name):
    from paper_2601_16637_b200 import SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals

    m = meta[name]
    basis = SelectedBasis.product(g[f"{name}/alpha"].tolist(), g[f"{name}/beta"].tolist(), m["norb"], m["na"],
                                  m["nb"])
    return basis, random_integrals(m["norb"], seed=m["iseed"])


@pytest.mark.parametrize("name", SMALL)
def test_small_tables_diag_sigma_vs_reference(small_golden, small_meta, name):
    from paper_2601_16637_b200 import HamiltonianApplier

    g = small_golden
    basis, table = _basis(g, small_meta, name)
    app = HamiltonianApplier(basis, table)
    for spin, tab in (("ta", app.tables.alpha), ("tb", app.tables.beta)):
        for f in TABLE_FIELDS:
            np.testing.assert_array_equal(getattr(tab, f), g[f"{name}/{spin}/{f}"], err_msg=f"{spin}.{f}")
    assert np.array_equal(app.diag, g[f"{name}/diag"])
    for x, y in zip(g[f"{name}/x"], g[f"{name}/y"]):
        assert _rel(app(x), y) <= SIGMA_RTOL


def test_hubbard_known_answers(small_golden):
    from paper_2601_16637_b200 import HamiltonianApplier, IntegralTable, SelectedBasis

    t = IntegralTable(2)
    t.set_h(0, 1, -1.0)
    t.set_eri(0, 0, 0, 0, 4.0)
    t.set_eri(1, 1, 1, 1, 4.0)
    b = SelectedBasis.product([0b01, 0b10], [0b01, 0b10], 2, 1, 1)
    app = HamiltonianApplier(b, t)
    assert np.array_equal(app.diag, [4.0, 0.0, 0.0, 4.0])  # test_apply.py:45-47
    assert np.allclose(app(np.array([1.0, 0, 0, 0])), [4.0, -1.0, -1.0, 0.0], atol=1e-14)  # :50-53
    dense = np.column_stack([app(np.eye(4)[:, j]) for j in range(4)])
    np.testing.assert_allclose(dense, small_golden["hubbard/dense"], atol=1e-14)


def test_sort_and_duplicates():
    from paper_2601_16637_b200 import build_excitation_table
    from paper_2601_16637_b200.synth import random_product_strings

    a, _ = random_product_strings(20, 6, 6, 3000, 10, seed=4)
    tab = build_excitation_table(a, 20)
    ref = O.build_table(a, 20)
    for f in TABLE_FIELDS:
        np.testing.assert_array_equal(getattr(tab, f), ref[f], err_msg=f)
    with pytest.raises(ValueError, match="dedup"):
        build_excitation_table(np.concatenate([a[:50], a[:1]]), 20)


@pytest.mark.parametrize("norb,ne,n", [(64, 3, 700), (40, 20, 4000), (8, 4, 70), (30, 1, 30), (16, 15, 16)])
def test_tables_edge_shapes_vs_oracle(norb, ne, n):
    """Full 64-bit strings, half filling, one electron / one hole, the whole string space."""
    from paper_2601_16637_b200 import build_excitation_table
    from paper_2601_16637_b200.synth import random_product_strings

    a, _ = random_product_strings(norb, ne, ne, n, 1, seed=n)
    tab = build_excitation_table(a, norb)
    ref = O.build_table(a, norb)
    for f in TABLE_FIELDS:
        np.testing.assert_array_equal(getattr(tab, f), ref[f], err_msg=f)


def test_empty_and_single_string_sectors():
    from paper_2601_16637_b200 import build_excitation_table

    t = build_excitation_table(np.array([0b1011], dtype=np.uint64), 5)
    assert t.s_off.tolist() == [0, 0] and t.d_off.tolist() == [0, 0]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg4"])
def test_big_config_tables_diag_sigma_windows(cfg):
    """Reference tables (SHA-256 of every column) and reference sigma on alpha-row windows.

    cfg4 is the 9e8-determinant Fe-S-like system (36 orbitals, 3e4 x 3e4 strings): its x rows (240 KB)
    exceed shared memory, so task 0 runs on the chunked sliced-ELL pipeline.
    """
    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis

    rec, arrays = load_big(cfg)
    table, a, b = big_instance(cfg)
    basis = SelectedBasis.product(a.tolist(), b.tolist(), rec["norb"], rec["na"], rec["nb"])
    app = HamiltonianApplier(basis, table)
    assert table_digests(app.tables.alpha) == rec["ta"]
    assert table_digests(app.tables.beta) == rec["tb"]
    import torch

    x = np.random.default_rng(12345).standard_normal(basis.dimension)
    y = app(torch.from_numpy(x).cuda()).cpu().numpy()
    nb = b.size
    for w in rec["windows"]:
        lo, hi = w["lo"], w["hi"]
        assert np.array_equal(app.diag[lo * nb:hi * nb], arrays[f"diag_{lo}_{hi}"])
        assert _rel(y[lo * nb:hi * nb], arrays[f"sigma_{lo}_{hi}"]) <= SIGMA_RTOL
    if cfg == "cfg1":  # full vector against the oracle (all 853,776 rows)
        inst = O.Instance.make(rec["norb"], table.h, table.eri, table.e_core, a, b)
        assert _rel(y, O.sigma(inst, x)) <= SIGMA_RTOL


def test_cfg2_full_size_properties():
    """1e8 determinants: linearity, adjoint symmetry, window reassembly, e2e == device path."""
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis

    table, a, b = big_instance("cfg2")
    basis = SelectedBasis.product(a.tolist(), b.tolist(), 26, 7, 7)
    app = HamiltonianApplier(basis, table)
    n = basis.dimension
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    z = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    hx, hz = app(x), app(z)
    lin = app(2.5 * x - 0.75 * z)
    assert float((lin - (2.5 * hx - 0.75 * hz)).abs().max() / hx.abs().max()) <= 1e-12
    lhs, rhs = float(z @ hx), float(hz @ x)
    assert abs(lhs - rhs) <= 1e-10 * (abs(lhs) + 1.0)
    # deterministic: repeated calls are bitwise equal
    assert torch.equal(app(x), hx)
    # windowed (one rank's rows) reassembles the full result
    nb = b.size
    lo, hi = 3333, 6667
    win = HamiltonianApplier(basis, table, row_window=(lo, hi))
    yw = win(x)
    assert torch.equal(yw, hx[lo * nb:hi * nb]) or float((yw - hx[lo * nb:hi * nb]).abs().max()) <= 1e-13 * float(
        hx.abs().max())
    del win
    # the numpy (host) protocol gives the same numbers
    xs = x[: n].cpu().numpy()
    ys = app(xs)
    assert np.array_equal(ys, hx.cpu().numpy())


@pytest.mark.parametrize("unstaged,order", [(False, "auto"), (True, "auto"), (False, "additive"), (True, "additive")])
def test_random_instances_vs_oracle(unstaged, order, monkeypatch):
    """Ragged random sets across shapes, incl. odd n_beta (scalar path) and 1-string sectors.

    ``unstaged`` forces the task-0 kernel variant that gathers through L1/L2
    (used when an x row does not fit shared memory); the (14, 2, 7) case has
    3432 beta strings, i.e. two column tiles of that variant.
    """
    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    if unstaged:
        monkeypatch.setenv("SBD_CROSS_UNSTAGED", "1")
    if order == "additive":  # task 0 added after the alpha side, whatever the single density
        monkeypatch.setenv("SBD_CROSS_ADD", "1")
    cases = [(10, 5, 4, 77, 131, 1), (14, 3, 4, 301, 257, 2), (16, 8, 8, 500, 1, 3), (16, 8, 8, 1, 499, 4),
             (12, 6, 6, 924, 129, 5), (20, 2, 9, 190, 600, 6), (14, 2, 7, 40, 3432, 7),
             (12, 6, 6, 924, 130, 8),   # 924 rows, even n_beta: pipelined host-buffer path
             (64, 2, 3, 300, 220, 9)]   # 64 orbitals: bit 63 in play, 2016 orbital pairs
    for norb, na, nb, nsa, nsb, seed in cases:
        a, _ = random_product_strings(norb, na, na, nsa, 1, seed)
        _, b = random_product_strings(norb, nb, nb, 1, nsb, seed + 100)
        table = random_integrals(norb, seed)
        basis = SelectedBasis.product(a.tolist(), b.tolist(), norb, na, nb)
        app = HamiltonianApplier(basis, table)
        inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
        assert np.array_equal(app.diag, O.diag(inst))
        x = np.random.default_rng(seed).standard_normal(basis.dimension)
        assert _rel(app(x), O.sigma(inst, x)) <= SIGMA_RTOL, (norb, na, nb, nsa, nsb)


def test_errors_follow_reference_conventions(small_golden, small_meta):
    from paper_2601_16637_b200 import HamiltonianApplier

    basis, table = _basis(small_golden, small_meta, "partial_5_2_3")
    with pytest.raises(ValueError, match="policy"):
        HamiltonianApplier(basis, table, exec_policy="speculative")
    app = HamiltonianApplier(basis, table)
    with pytest.raises(ValueError):
        app(np.zeros(5))
    assert app.apply_count == 0
    app(np.ones(basis.dimension))
    app(np.ones(basis.dimension))
    assert app.apply_count == 2
