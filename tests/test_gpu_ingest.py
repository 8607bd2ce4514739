"""Device ingestion against the reference semantics of ingest_samples (basis.py:251-313).

The host ``ingest_samples`` (same contract, tested in test_host.py) is the checker for small
sample sets; a numpy restatement (np.unique + first indices) checks a 2e6-sample set.
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


@pytest.mark.parametrize("mode", ["product", "explicit"])
def test_ingest_matches_host_reference_semantics(mode):
    from paper_2601_16637_b200 import det_to_line, ingest_sample_arrays, ingest_samples, start_vector
    from paper_2601_16637_b200.basis import Determinant

    rng = np.random.default_rng(5)
    norb, na, nb = 10, 4, 3
    a, b = _samples(rng, norb, na, nb, 3000, pool=40)
    lines = [det_to_line(Determinant(int(x), int(y)), norb) for x, y in zip(a, b)]
    hb, hr = ingest_samples(lines, norb, na, nb, mode=mode)
    db, dr = ingest_sample_arrays(a, b, norb, na, nb, mode=mode)
    assert (dr.n_lines, dr.n_filtered, dr.n_duplicates) == (hr.n_lines, hr.n_filtered, hr.n_duplicates)
    assert dr.det_counts == hr.det_counts
    assert list(dr.det_counts) == list(hr.det_counts)  # first-seen order of the Counter too
    if mode == "product":
        assert db.alpha_strings == hb.alpha_strings and db.beta_strings == hb.beta_strings
    else:
        assert list(db.dets) == list(hb.dets)
    np.testing.assert_array_equal(start_vector(db, dr), start_vector(hb, hr))


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
