"""Device ingestion against the reference's own ingest_samples (basis.py:251-313).

tests/golden/ingest.json holds the reference's outputs (make_golden.py ingest) on sample files with
comments, blank and padded lines, filtered lines and duplicates, in both modes, plus the reference
CLI's start vector (cli.py:117-128).  A numpy restatement (np.unique + first indices) checks a
2e6-sample set.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _samples(rng, norb, na, nb, n, pool, bad_frac=0.1):
    from paper_2601_16637_b200.synth import unrank_combinations
    from math import comb

    ia = rng.integers(0, min(pool, comb(norb, na)), n)
    ib = rng.integers(0, min(pool, comb(norb, nb)), n)
    a = unrank_combinations(ia, norb, na)
    b = unrank_combinations(ib, norb, nb)
    bad = rng.random(n) < bad_frac  # wrong electron count: filtered
    a[bad] = unrank_combinations(rng.integers(0, comb(norb, na - 1), int(bad.sum())), norb, na - 1)
    return a, b


def _golden_ingest():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "ingest.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", range(4))
@pytest.mark.parametrize("mode", ["product", "explicit"])
def test_ingest_matches_reference(case, mode):
    from paper_2601_16637_b200 import ingest_samples, start_vector

    g = _golden_ingest()[case]
    r = g["modes"][mode]
    basis, rep = ingest_samples(g["lines"], g["norb"], g["na"], g["nb"], mode=mode)
    assert (rep.n_lines, rep.n_filtered, rep.n_duplicates) == (r["n_lines"], r["n_filtered"], r["n_duplicates"])
    # multiplicities, in the reference Counter's first-seen order
    assert [[int(d.alpha), int(d.beta), int(c)] for d, c in rep.det_counts.items()] == r["det_counts"]
    assert basis.dimension == r["dimension"]
    if mode == "product":
        assert [int(v) for v in basis.alpha_strings] == r["alpha"]
        assert [int(v) for v in basis.beta_strings] == r["beta"]
    else:
        assert [[int(d.alpha), int(d.beta)] for d in basis.dets] == r["dets"]
    x0 = start_vector(basis, rep)
    want = np.zeros(basis.dimension)
    want[r["start_nz"]] = r["start_val"]
    np.testing.assert_array_equal(x0, want)


def test_ingest_large_vs_numpy():
    from paper_2601_16637_b200.ingest import ingest_arrays_raw

    rng = np.random.default_rng(11)
    norb, na, nb = 26, 7, 7
    a, b = _samples(rng, norb, na, nb, 2_000_000, pool=3000, bad_frac=0.05)
    r = ingest_arrays_raw(a, b, norb, na, nb)
    popa = np.unpackbits(a.view(np.uint8)).reshape(-1, 64).sum(1)
    popb = np.unpackbits(b.view(np.uint8)).reshape(-1, 64).sum(1)
    keep = (popa == na) & (popb == nb)
    ka, kb = a[keep], b[keep]
    assert r.n_filtered == int((~keep).sum())
    pairs = np.stack([ka, kb], 1)
    uniq, first, counts = np.unique(pairs, axis=0, return_index=True, return_counts=True)
    order = np.argsort(first, kind="stable")
    np.testing.assert_array_equal(r.det_alpha, uniq[order, 0])
    np.testing.assert_array_equal(r.det_beta, uniq[order, 1])
    np.testing.assert_array_equal(r.det_count, counts[order])
    for half, got in ((ka, r.alpha), (kb, r.beta)):
        u, f = np.unique(half, return_index=True)
        np.testing.assert_array_equal(got, u[np.argsort(f, kind="stable")])


def test_ingest_errors():
    from paper_2601_16637_b200 import ingest_sample_arrays

    with pytest.raises(ValueError):
        ingest_sample_arrays(np.array([0b1111], dtype=np.uint64), np.array([0b11], dtype=np.uint64), 3, 2, 2)
    with pytest.raises(ValueError):
        ingest_sample_arrays(np.array([0b11], dtype=np.uint64), np.array([0b11, 0b101], dtype=np.uint64), 3, 2, 2)
    with pytest.raises(ValueError, match="mode"):
        ingest_sample_arrays(np.array([0b11], dtype=np.uint64), np.array([0b11], dtype=np.uint64), 3, 2, 2,
                             mode="bogus")
    basis, rep = ingest_sample_arrays(np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint64), 3, 2, 2)
    assert basis.dimension == 0 and rep.n_lines == 0
