"""Seeded synthetic instances, bit-identical to the reference generators.

Restates reference ``synth.py:26-84`` so the GPU box (where the reference is
absent) builds *identical* integrals and string sets:

* ``random_integrals``: h ~ U(-1, 1) drawn over the lower triangle in
  row order, then (pq|rs) ~ eri_scale * U(0, 1) over the canonical
  tri-of-tri slots in storage order (reference ``synth.py:26-36``).  The
  draws are issued in the same order from the same ``default_rng(seed)``
  stream, vectorised.
* ``random_product_strings``: the reference materialises the whole
  C(norb, ne) pool and calls ``rng.choice(len(pool), n, replace=False)``
  (``synth.py:59-68``).  The choice only depends on the pool *size*, so we
  draw the same indices and *unrank* them into lexicographic combinations
  instead of enumerating the pool -- 9e8-det cfg4 strings in a second
  instead of 400 s / 7.5 GB.
"""

from __future__ import annotations

from itertools import combinations
from math import comb

import numpy as np

from .basis import Determinant, SelectedBasis
from .integrals import IntegralTable

__all__ = [
    "random_integrals",
    "all_strings",
    "unrank_combinations",
    "full_product_basis",
    "random_product_strings",
    "random_product_basis",
    "random_explicit_basis",
]


def random_integrals(norb: int, seed: int, eri_scale: float = 0.1) -> IntegralTable:
    rng = np.random.default_rng(seed)
    table = IntegralTable(norb)
    rows, cols = np.tril_indices(norb)          # (p, q<=p) in row order
    hv = rng.uniform(-1.0, 1.0, size=rows.size)
    table.h[rows, cols] = hv
    table.h[cols, rows] = hv
    table.eri[:] = eri_scale * rng.uniform(0.0, 1.0, size=table.eri.size)
    return table


def all_strings(norb: int, n_elec: int) -> list:
    return [sum(1 << p for p in c) for c in combinations(range(norb), n_elec)]


def unrank_combinations(idx: np.ndarray, norb: int, k: int) -> np.ndarray:
    """Lexicographic rank -> occupation mask, matching ``itertools.combinations`` order."""
    rem = np.asarray(idx, dtype=np.int64).copy()
    out = np.zeros(rem.shape, dtype=np.uint64)
    nxt = np.zeros(rem.shape, dtype=np.int64)  # smallest orbital still allowed
    for j in range(k):
        left = k - j - 1
        placed = np.zeros(rem.shape, dtype=bool)
        for c in range(norb):
            cnt = comb(norb - c - 1, left) if norb - c - 1 >= left else 0
            active = (~placed) & (nxt <= c)
            take = active & (rem < cnt)
            out[take] |= np.uint64(1) << np.uint64(c)
            nxt[take] = c + 1
            placed |= take
            skip = active & ~take
            rem[skip] -= cnt
        if not placed.all():
            raise ValueError("rank out of range")
    return out


def full_product_basis(norb: int, n_alpha: int, n_beta: int) -> SelectedBasis:
    return SelectedBasis.product(all_strings(norb, n_alpha), all_strings(norb, n_beta),
                                 norb, n_alpha, n_beta)


def random_product_strings(norb: int, n_alpha: int, n_beta: int, n_alpha_strings: int,
                           n_beta_strings: int, seed: int):
    """(alpha u64[], beta u64[]) of ``random_product_basis`` without building Python lists."""
    rng = np.random.default_rng(seed)
    pa, pb = comb(norb, n_alpha), comb(norb, n_beta)
    if n_alpha_strings > pa or n_beta_strings > pb:
        raise ValueError(f"requested {n_alpha_strings}x{n_beta_strings} strings but only "
                         f"{pa}x{pb} exist for norb={norb}")
    ia = rng.choice(pa, n_alpha_strings, replace=False)
    ib = rng.choice(pb, n_beta_strings, replace=False)
    return unrank_combinations(ia, norb, n_alpha), unrank_combinations(ib, norb, n_beta)


def random_product_basis(norb: int, n_alpha: int, n_beta: int, n_alpha_strings: int,
                         n_beta_strings: int, seed: int) -> SelectedBasis:
    a, b = random_product_strings(norb, n_alpha, n_beta, n_alpha_strings, n_beta_strings, seed)
    return SelectedBasis.product(a.tolist(), b.tolist(), norb, n_alpha, n_beta)


def random_explicit_basis(norb: int, n_alpha: int, n_beta: int, n_dets: int, seed: int) -> SelectedBasis:
    rng = np.random.default_rng(seed)
    pa, pb = comb(norb, n_alpha), comb(norb, n_beta)
    if n_dets > pa * pb:
        raise ValueError(f"requested {n_dets} determinants but only {pa * pb} exist")
    picks = rng.choice(pa * pb, n_dets, replace=False)
    ka, kb = np.divmod(np.asarray(picks, dtype=np.int64), pb)
    a = unrank_combinations(ka, norb, n_alpha)
    b = unrank_combinations(kb, norb, n_beta)
    return SelectedBasis.explicit([Determinant(int(x), int(y)) for x, y in zip(a, b)],
                                  norb, n_alpha, n_beta)
