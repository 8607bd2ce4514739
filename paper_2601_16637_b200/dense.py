"""Dense brute-force check matrix (reference ``oracle.py``: ``assemble_dense``, ``dense_eigensolve``).

``assemble_dense`` evaluates every element <det_i|H|det_j> on the GPU from the
two determinants' occupation words (``sbd_dense_rows``, csrc/sbd_dense.cu: a
restatement of ``_hij_words``, apply.py:152-177), sharing none of the sigma
path's tables, coefficients or kernels -- the same independence the
reference's matelem-based assembly has (oracle.py:34-45).  Capped to small
dimensions: it checks answers, it does not produce them.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .basis import SelectedBasis
from .integrals import IntegralTable

__all__ = ["DEFAULT_CAP", "assemble_dense", "dense_eigensolve"]

DEFAULT_CAP = 4096


def _check_cap(n: int, cap: int) -> None:
    if n > cap:
        raise ValueError(f"dense assembly refused: dimension {n} exceeds cap {cap}; shrink the instance (fewer "
                         "sampled strings or orbitals) or pass a larger cap explicitly")


def assemble_dense(basis: SelectedBasis, table: IntegralTable, cap: int = DEFAULT_CAP, device=None) -> np.ndarray:
    """M[i, j] = <det_i|H|det_j> for every pair, evaluated per element on the device."""
    import torch

    from .apply import _device_index

    n = basis.dimension
    _check_cap(n, cap)
    dev = _device_index(device)
    ctx = _lib.Context(dev)
    try:
        h = np.ascontiguousarray(table.h, dtype=np.float64)
        eri = np.ascontiguousarray(table.eri, dtype=np.float64)
        ctx("sbd_set_integrals", int(table.norb), _lib.ptr(h), _lib.ptr(eri), int(eri.size), float(table.e_core))
        if basis.mode == "product":
            a = np.ascontiguousarray(basis.alpha_array(), dtype=np.uint64)
            b = np.ascontiguousarray(basis.beta_array(), dtype=np.uint64)
            ctx("sbd_set_strings", 0, _lib.ptr(a), int(a.size), int(basis.n_alpha_elec))
            ctx("sbd_set_strings", 1, _lib.ptr(b), int(b.size), int(basis.n_beta_elec))
        else:
            da = np.ascontiguousarray([d.alpha for d in basis.dets], dtype=np.uint64)
            db = np.ascontiguousarray([d.beta for d in basis.dets], dtype=np.uint64)
            ctx("sbd_set_dets", _lib.ptr(da), _lib.ptr(db), int(n), int(basis.n_alpha_elec), int(basis.n_beta_elec))
        out = torch.empty((n, n), dtype=torch.float64, device=torch.device("cuda", dev))
        ctx.bind_stream()
        if n:
            ctx("sbd_dense_rows", 0, n, _lib.ptr(out))
        return out.cpu().numpy()
    finally:
        ctx.close()


def dense_eigensolve(mat: np.ndarray, cap: int = DEFAULT_CAP):
    """Full spectrum (ascending) and orthonormal eigenvector columns (LAPACK eigh on the host)."""
    mat = np.asarray(mat, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {mat.shape}")
    _check_cap(mat.shape[0], cap)
    return np.linalg.eigh(mat)
