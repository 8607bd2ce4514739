"""GPU parity of the 128-bit string path (norb 65..128): device radix sort/unique and excitation tables.

The reference's table builder (basis.py:62-103, 362-403) works on Python ints of any width, so
tests/golden/table128.npz holds its own output on norb 65..128 string lists; the bar is bit-exact.
Larger random sets are checked against the oracle (oracle/sbd_oracle.c orc_table128_*, itself pinned
to those fixtures by tests/test_oracle_golden.py).  All calls go through the C ABI
(sbd_table128_build / _counts / _export / _sorted).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import TABLE128_CASES, TABLE_FIELDS

pytestmark = pytest.mark.gpu


def _assert_tables_equal(tab, ref, label=""):
    for f in TABLE_FIELDS:
        got = np.asarray(getattr(tab, f)) if not isinstance(tab, dict) else tab[f]
        np.testing.assert_array_equal(got, ref[f], err_msg=f"{label} {f}")


def _walk(rng, norb, ne, n, window):
    """Connected random string set: single/double moves inside `window`, discovery order."""
    from math import comb

    assert comb(len(window), ne) >= n, "window too small for n distinct strings"
    window = np.asarray(window)
    start = 0
    for o in rng.choice(window, size=ne, replace=False):
        start |= 1 << int(o)
    out, seen = [start], {start}
    while len(out) < n:
        s = out[int(rng.integers(len(out)))]
        occ = [int(o) for o in window if (s >> int(o)) & 1]
        virt = [int(o) for o in window if not (s >> int(o)) & 1]
        k = 2 if rng.random() < 0.6 else 1
        for _ in range(k):
            p, r = occ[int(rng.integers(len(occ)))], virt[int(rng.integers(len(virt)))]
            s = (s & ~(1 << p)) | (1 << r)
            occ.remove(p), virt.remove(r)
            occ.append(r), virt.append(p)
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


@pytest.mark.parametrize("name", TABLE128_CASES)
def test_table128_bit_exact_vs_reference(table128_golden, name):
    from paper_2601_16637_b200 import build_excitation_table

    meta, g = table128_golden
    m = meta[name]
    words = g[f"{name}/words"]
    tab = build_excitation_table(words, m["norb"], m["n_elec"])
    assert tab.n_strings == m["n_strings"]
    _assert_tables_equal(tab, {f: g[f"{name}/{f}"] for f in TABLE_FIELDS}, name)
    # the same strings as Python ints take the same path
    ints = [int(lo) | (int(hi) << 64) for lo, hi in words.tolist()]
    tab2 = build_excitation_table(ints, m["norb"])
    _assert_tables_equal(tab2, {f: g[f"{name}/{f}"] for f in TABLE_FIELDS}, name + " ints")


@pytest.mark.parametrize("norb,ne,n,window", [
    (96, 6, 6000, list(range(50, 80)) + list(range(90, 96))),   # n > 4096: two-level lookup
    (128, 4, 3000, list(range(0, 8)) + list(range(60, 68)) + list(range(120, 128))),
    (80, 40, 1500, list(range(80))),                              # 40 electrons in both words
    (65, 1, 65, None),                                            # every one-electron string
])
def test_table128_random_vs_oracle(norb, ne, n, window):
    from paper_2601_16637_b200 import build_excitation_table128

    rng = np.random.default_rng(norb * 1000 + ne)
    if window is None:
        strings = [1 << int(o) for o in rng.permutation(norb)]
    else:
        strings = _walk(rng, norb, ne, n, window)
    ref = O.build_table128(strings, norb)
    assert ref["s_off"][-1] > 0
    tab = build_excitation_table128(strings, norb)
    _assert_tables_equal(tab, ref, f"norb{norb} ne{ne}")


def test_table128_equals_64bit_path_on_narrow_strings():
    """norb <= 64 strings through the two-word kernels give the one-word path's table."""
    from paper_2601_16637_b200 import build_excitation_table, build_excitation_table128, synth

    a, _ = synth.random_product_strings(26, 7, 7, 3000, 10, seed=2)
    t64 = build_excitation_table(a, 26, 7)
    t128 = build_excitation_table128(a.tolist(), 26, 7)
    for f in TABLE_FIELDS:
        np.testing.assert_array_equal(getattr(t64, f), getattr(t128, f), err_msg=f)
    full = synth.full_product_basis(64, 1, 1)  # bit 63, top of the low word
    t64 = build_excitation_table(full.alpha_array(), 64, 1)
    t128 = build_excitation_table128(full.alpha_strings, 64, 1)
    for f in TABLE_FIELDS:
        np.testing.assert_array_equal(getattr(t64, f), getattr(t128, f), err_msg=f)


def test_sorted_strings128_radix_order():
    """Device LSD radix sort over both words: sorted = words[perm], ascending as 128-bit integers."""
    from paper_2601_16637_b200 import sorted_strings128, string_words

    rng = np.random.default_rng(7)
    n = 100_000
    # 6 electrons over 128 orbitals, many strings equal in the high word (ties resolved by the low word)
    vals = set()
    while len(vals) < n:
        orbs = rng.choice(np.r_[0:8, 60:70, 120:128], size=6, replace=False)
        v = 0
        for o in orbs:
            v |= 1 << int(o)
        vals.add(v)
    strings = list(vals)
    rng.shuffle(strings)
    words = string_words(strings)
    got, perm = sorted_strings128(words, 128)
    np.testing.assert_array_equal(got, words[perm])
    keys = [int(lo) | (int(hi) << 64) for lo, hi in got.tolist()]
    assert keys == sorted(strings)
    assert np.array_equal(np.sort(perm), np.arange(n))


def test_table128_rejects_bad_input():
    from paper_2601_16637_b200 import build_excitation_table128, sorted_strings128

    with pytest.raises(ValueError, match="dedup"):
        build_excitation_table128([(1 << 70) | 1, (1 << 70) | 1], 72)
    with pytest.raises(ValueError, match="dedup"):
        sorted_strings128([3 << 100, 5 << 100, 3 << 100], 128)
    with pytest.raises(ValueError, match="above orbital"):
        build_excitation_table128([(1 << 80) | 1], 72)
    with pytest.raises(ValueError, match="electrons"):
        build_excitation_table128([(1 << 70) | 1, 7 << 64], 72, n_elec=2)
    with pytest.raises(ValueError, match="different electron counts"):
        build_excitation_table128([(1 << 70) | 1, 7 << 64], 72)
    with pytest.raises(ValueError):
        build_excitation_table128([1], 129)
    empty = build_excitation_table128([], 100, 3)
    assert empty.n_strings == 0 and empty.s_off.tolist() == [0] and empty.d_off.tolist() == [0]


def test_build_spin_tables_wide_product_basis():
    """build_spin_tables (reference apply.py:557-563) on a product basis of 100 orbitals."""
    from paper_2601_16637_b200 import SelectedBasis, build_spin_tables

    rng = np.random.default_rng(100)
    a = _walk(rng, 100, 5, 700, list(range(60, 72)) + list(range(94, 100)))
    b = _walk(rng, 100, 3, 400, list(range(0, 8)) + list(range(60, 70)))  # C(18, 3) = 816 >= 400
    tabs = build_spin_tables(SelectedBasis.product(a, b, 100, 5, 3))
    _assert_tables_equal(tabs.alpha, O.build_table128(a, 100), "alpha")
    _assert_tables_equal(tabs.beta, O.build_table128(b, 100), "beta")
