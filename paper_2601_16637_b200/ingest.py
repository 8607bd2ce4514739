"""Device ingestion of sampled configurations (SQD loop integration).

``ingest_sample_arrays(alpha, beta, norb, n_alpha, n_beta, mode)`` is the
array form of the reference's ``ingest_samples`` (``basis.py:251-313``):
filter by per-spin electron count, drop duplicate determinants keeping
first-seen order, count multiplicities, and collect the unique halves in
first-seen order -- all on the GPU (``sbd_ingest_samples``, radix sort +
segmented runs).  It returns the same ``(SelectedBasis, IngestReport)`` pair.

``start_vector(basis, report)`` is the reference CLI's sampling-informed
Davidson start (``cli.py:117-128``): determinant multiplicities as weights,
normalised.
"""

from __future__ import annotations

import ctypes
from collections import Counter
from typing import Optional

import numpy as np

from . import _lib
from .basis import Determinant, IngestReport, SelectedBasis

__all__ = ["ingest_sample_arrays", "start_vector", "IngestResult"]


class IngestResult:
    """Raw device-ingestion arrays (first-seen order), for callers that skip the Counter."""

    def __init__(self, det_alpha, det_beta, det_count, alpha, beta, n_samples, n_filtered):
        self.det_alpha = det_alpha
        self.det_beta = det_beta
        self.det_count = det_count
        self.alpha = alpha
        self.beta = beta
        self.n_samples = n_samples
        self.n_filtered = n_filtered


def ingest_arrays_raw(alpha, beta, norb: int, n_alpha_elec: int, n_beta_elec: int, device=None) -> IngestResult:
    import torch

    a = np.ascontiguousarray(np.asarray(alpha, dtype=np.uint64).reshape(-1))
    b = np.ascontiguousarray(np.asarray(beta, dtype=np.uint64).reshape(-1))
    if a.shape != b.shape:
        raise ValueError(f"alpha and beta sample arrays differ in length ({a.size} vs {b.size})")
    dev = torch.cuda.current_device() if device is None else int(device)
    ctx = _lib.Context(dev)
    try:
        nf, nd, na, nb = (ctypes.c_int64() for _ in range(4))
        ctx("sbd_ingest_samples", _lib.ptr(a), _lib.ptr(b), int(a.size), int(norb), int(n_alpha_elec),
            int(n_beta_elec), ctypes.byref(nf), ctypes.byref(nd), ctypes.byref(na), ctypes.byref(nb))
        da = np.empty(nd.value, dtype=np.uint64)
        db = np.empty(nd.value, dtype=np.uint64)
        dc = np.empty(nd.value, dtype=np.int64)
        ua = np.empty(na.value, dtype=np.uint64)
        ub = np.empty(nb.value, dtype=np.uint64)
        ctx("sbd_ingest_export", *(_lib.ptr(v) if v.size else None for v in (da, db, dc, ua, ub)))
    finally:
        ctx.close()
    return IngestResult(da, db, dc, ua, ub, int(a.size), int(nf.value))


def ingest_sample_arrays(alpha, beta, norb: int, n_alpha_elec: int, n_beta_elec: int, mode: str = "product",
                         device=None):
    """Sampled (alpha, beta) uint64 arrays -> (SelectedBasis, IngestReport), reference semantics."""
    mode = mode.lower()
    if mode not in ("product", "explicit"):
        raise ValueError(f"mode must be 'product' or 'explicit', got {mode!r}")
    r = ingest_arrays_raw(alpha, beta, norb, n_alpha_elec, n_beta_elec, device)
    dets = [Determinant(int(x), int(y)) for x, y in zip(r.det_alpha, r.det_beta)]
    counts = Counter(dict(zip(dets, (int(c) for c in r.det_count))))
    n_kept = r.n_samples - r.n_filtered
    report = IngestReport(n_lines=r.n_samples, n_filtered=r.n_filtered, n_duplicates=n_kept - len(dets),
                          det_counts=counts)
    if mode == "product":
        basis = SelectedBasis.product(r.alpha.tolist(), r.beta.tolist(), norb, n_alpha_elec, n_beta_elec)
    else:
        basis = SelectedBasis.explicit(dets, norb, n_alpha_elec, n_beta_elec)
    return basis, report


def start_vector(basis: SelectedBasis, report: IngestReport) -> Optional[np.ndarray]:
    """Determinant multiplicities as Davidson start weights (reference cli.py:117-128)."""
    if not report.det_counts:
        return None
    x0 = np.zeros(basis.dimension)
    for det, count in report.det_counts.items():
        try:
            x0[basis.index_of(det)] = float(count)
        except KeyError:
            continue
    norm = np.linalg.norm(x0)
    return x0 / norm if norm > 0 else None
