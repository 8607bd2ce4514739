"""Drop-in matrix-free operator y = H x on the B200 (reference ``apply.py``).

``HamiltonianApplier`` keeps the reference constructor and call protocol
(``apply.py:651-704``): ``applier(x) -> y`` with ``.diag``, ``.n``,
``.apply_count``, ``.tables``.  Everything behind it runs on the GPU through
the C ABI (``include/sbd.h``): string sort/unique and excitation tables
(``sbd_build_tables``), the diagonal (``sbd_diag``) and the sigma build
(``sbd_sigma``).  There is no CPU path -- without the CUDA extension or a
device, construction raises.

Accepted vectors:

* numpy float64 (the reference protocol): copied to the device and back
  inside the call (``sbd_sigma_host``);
* torch CUDA float64 tensors: stay on the device (``sbd_sigma``), which is
  what the device-resident ``davidson_solve`` uses.

Both ``exec_policy`` values of the reference are accepted; the GPU kernel is
row-owned without atomics, so every call is deterministic.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .basis import ExcitationTable, SelectedBasis
from .integrals import IntegralTable

__all__ = [
    "SpinTables",
    "HamiltonianApplier",
    "apply_H",
    "apply_H_full",
    "compute_diagonal",
    "build_spin_tables",
    "build_excitation_table",
    "check_policy",
]

_POLICIES = ("parallel", "deterministic")


def check_policy(exec_policy: str) -> str:
    if exec_policy not in _POLICIES:
        raise ValueError(f"exec_policy must be 'parallel' or 'deterministic', got {exec_policy!r}")
    return exec_policy


@dataclass
class SpinTables:
    alpha: ExcitationTable
    beta: ExcitationTable


def _device_index(device) -> int:
    import torch

    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


def _upload_instance(ctx: _lib.Context, table: IntegralTable, alpha: np.ndarray, beta: Optional[np.ndarray],
                     na: int, nb: int) -> None:
    h = np.ascontiguousarray(table.h, dtype=np.float64)
    eri = np.ascontiguousarray(table.eri, dtype=np.float64)
    ctx("sbd_set_integrals", int(table.norb), _lib.ptr(h), _lib.ptr(eri), int(eri.size), float(table.e_core))
    a = np.ascontiguousarray(alpha, dtype=np.uint64)
    ctx("sbd_set_strings", 0, _lib.ptr(a), int(a.size), int(na))
    if beta is not None:
        b = np.ascontiguousarray(beta, dtype=np.uint64)
        ctx("sbd_set_strings", 1, _lib.ptr(b), int(b.size), int(nb))
    ctx("sbd_build_tables")


_TABLE_ORDER = ("s_off", "s_tgt", "s_hole", "s_part", "s_phase", "d_off", "d_tgt", "d_hole1", "d_hole2",
                "d_part1", "d_part2", "d_phase")


def _table_columns(n: int, ns: int, nd: int) -> dict:
    return dict(
        s_off=np.zeros(n + 1, np.int64), s_tgt=np.zeros(ns, np.int64), s_hole=np.zeros(ns, np.int16),
        s_part=np.zeros(ns, np.int16), s_phase=np.zeros(ns, np.int8),
        d_off=np.zeros(n + 1, np.int64), d_tgt=np.zeros(nd, np.int64), d_hole1=np.zeros(nd, np.int16),
        d_hole2=np.zeros(nd, np.int16), d_part1=np.zeros(nd, np.int16), d_part2=np.zeros(nd, np.int16),
        d_phase=np.zeros(nd, np.int8),
    )


def _export_table(ctx: _lib.Context, spin: int, norb: int) -> ExcitationTable:
    n, ns, nd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    ctx("sbd_table_counts", spin, ctypes.byref(n), ctypes.byref(ns), ctypes.byref(nd))
    cols = _table_columns(n.value, ns.value, nd.value)
    ctx("sbd_export_table", spin, *[_lib.ptr(cols[k]) if cols[k].size else None for k in _TABLE_ORDER])
    return ExcitationTable(n_strings=n.value, norb=norb, **cols)


def string_words(strings) -> np.ndarray:
    """Strings of up to 128 orbitals (Python ints, or an (n, 2) uint64 array) -> (n, 2) uint64 (lo, hi)."""
    if isinstance(strings, np.ndarray) and strings.ndim == 2:
        if strings.shape[1] != 2:
            raise ValueError("a word array must have shape (n, 2)")
        return np.ascontiguousarray(strings, dtype=np.uint64)
    vals = [int(v) for v in strings]
    if any(v < 0 or v >> 128 for v in vals):
        raise ValueError("strings must be non-negative and below 2**128")
    return np.array([[v & 0xFFFFFFFFFFFFFFFF, v >> 64] for v in vals], dtype=np.uint64).reshape(-1, 2)


def build_excitation_table128(strings, norb: int, n_elec: Optional[int] = None, device=None) -> ExcitationTable:
    """``build_excitation_table`` for strings of up to 128 orbitals (two-word masks), built on the GPU.

    The reference's table builder (``basis.py:62-103,362-403``) works on Python ints of any width; its
    integrals stop at 64 orbitals (``integrals.py:67-68``), so wide strings get tables (and the sorted
    order, ``sorted_strings128``) but no Hamiltonian.  ``strings``: Python ints or (n, 2) uint64 words.
    """
    if not 1 <= norb <= 128:
        raise ValueError(f"norb must be in [1, 128], got {norb}")
    w = string_words(strings)
    n = w.shape[0]
    counts = [int(a).bit_count() + int(b).bit_count() for a, b in w.tolist()]
    if n_elec is None:
        n_elec = counts[0] if n else 0
        if any(c != n_elec for c in counts):
            raise ValueError("strings have different electron counts")
    ctx = _lib.Context(_device_index(device))
    try:
        ctx("sbd_table128_build", int(norb), _lib.ptr(w) if n else None, int(n), int(n_elec))
        nn, ns, nd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ctx("sbd_table128_counts", ctypes.byref(nn), ctypes.byref(ns), ctypes.byref(nd))
        cols = _table_columns(nn.value, ns.value, nd.value)
        ctx("sbd_table128_export", *[_lib.ptr(cols[k]) if cols[k].size else None for k in _TABLE_ORDER])
        return ExcitationTable(n_strings=nn.value, norb=norb, **cols)
    finally:
        ctx.close()


def sorted_strings128(strings, norb: int, device=None):
    """Device radix sort of up to 128-bit strings: (sorted (n, 2) uint64 words, perm int64), sorted = words[perm].

    Rejects duplicates (the uniqueness check of ``basis.py:364-366``)."""
    w = string_words(strings)
    n = w.shape[0]
    n_elec = int(w[0, 0]).bit_count() + int(w[0, 1]).bit_count() if n else 0
    ctx = _lib.Context(_device_index(device))
    try:
        ctx("sbd_table128_build", int(norb), _lib.ptr(w) if n else None, int(n), n_elec)
        out, perm = np.zeros((n, 2), np.uint64), np.zeros(n, np.int64)
        if n:
            ctx("sbd_table128_sorted", _lib.ptr(out), _lib.ptr(perm))
        return out, perm
    finally:
        ctx.close()


def build_excitation_table(strings, norb: int, n_elec: Optional[int] = None, device=None) -> ExcitationTable:
    """In-set CSR singles/doubles of one string list, built on the GPU.

    Same contract as reference ``basis.py:362-403`` (caller-order rows and
    targets, enumeration order within a row, ValueError on duplicates).
    ``norb`` > 64 takes the two-word path (:func:`build_excitation_table128`).
    """
    from .integrals import IntegralTable as _IT

    if norb > 64:
        return build_excitation_table128(strings, norb, n_elec, device)
    arr = np.ascontiguousarray(np.asarray(list(strings) if not isinstance(strings, np.ndarray) else strings,
                                          dtype=np.uint64))
    if n_elec is None:
        n_elec = int(arr[0]).bit_count() if arr.size else 0
        if arr.size and any(int(s).bit_count() != n_elec for s in arr.tolist()):
            raise ValueError("strings have different electron counts")
    ctx = _lib.Context(_device_index(device))
    try:
        _upload_instance(ctx, _IT(norb), arr, None, n_elec, 0)
        return _export_table(ctx, 0, norb)
    finally:
        ctx.close()


def build_spin_tables(basis: SelectedBasis, device=None) -> SpinTables:
    """Both sectors' tables (reference ``apply.py:557-563``), built on the GPU."""
    if basis.mode != "product":
        raise ValueError("spin-sector tables apply to product-mode bases only")
    wide = basis.norb > 64  # two-word strings: tables only (build_excitation_table128)
    return SpinTables(
        alpha=build_excitation_table(basis.alpha_strings if wide else basis.alpha_array(), basis.norb,
                                     basis.n_alpha_elec, device),
        beta=build_excitation_table(basis.beta_strings if wide else basis.beta_array(), basis.norb,
                                    basis.n_beta_elec, device),
    )


class HamiltonianApplier:
    """Reusable y = H x over a product or explicit basis, resident on one GPU.

    ``tables`` (reference-built SpinTables) is accepted for signature
    compatibility; the device always builds its own, bit-identical tables.
    ``row_window=(lo, hi)`` restricts the owned (output) alpha rows, the
    contract of the reference's windowed apply (``apply.py:501-546``) and of
    one rank of the distributed applier (product mode only).  Explicit bases
    follow the reference's explicit branch (``apply.py:675-683,696-703``):
    ``tables`` and ``cache`` are None, y is indexed by determinant order.
    """

    def __init__(self, basis: SelectedBasis, table: IntegralTable, tables: Optional[SpinTables] = None,
                 exec_policy: str = "parallel", device=None, row_window=None):
        check_policy(exec_policy)
        import torch

        if basis.mode == "explicit":
            self._init_explicit(basis, table, exec_policy, device, row_window)
            return

        self.basis = basis
        self.table = table
        self.exec_policy = exec_policy
        self.n = basis.dimension
        self.apply_count = 0
        self.device = _device_index(device)
        self._torch_device = torch.device("cuda", self.device)
        self._ctx = _lib.Context(self.device)
        with torch.cuda.device(self.device):
            _upload_instance(self._ctx, table, basis.alpha_array(), basis.beta_array(), basis.n_alpha_elec,
                             basis.n_beta_elec)
        self.n_alpha = len(basis.alpha_strings)
        self.n_beta = len(basis.beta_strings)
        lo, hi = (0, self.n_alpha) if row_window is None else (int(row_window[0]), int(row_window[1]))
        self.row_window = (lo, hi)
        if row_window is not None:
            self._ctx("sbd_set_row_window", lo, hi)
        self.n_own = (hi - lo) * self.n_beta
        self._tables = None
        self._diag_dev = None
        self._diag_host = None
        self._ctx.bind_stream()
        self._ctx("sbd_diag", None)  # built on the device now (the sigma reads it); copies are lazy

    def _init_explicit(self, basis, table, exec_policy, device, row_window):
        import torch

        if row_window is not None:
            raise ValueError("row windows apply to product-mode bases only")
        self.basis = basis
        self.table = table
        self.exec_policy = exec_policy
        self.n = basis.dimension
        self.apply_count = 0
        self.cache = None
        self.device = _device_index(device)
        self._torch_device = torch.device("cuda", self.device)
        self._ctx = _lib.Context(self.device)
        da = np.ascontiguousarray([d.alpha for d in basis.dets], dtype=np.uint64)
        db = np.ascontiguousarray([d.beta for d in basis.dets], dtype=np.uint64)
        with torch.cuda.device(self.device):
            h = np.ascontiguousarray(table.h, dtype=np.float64)
            eri = np.ascontiguousarray(table.eri, dtype=np.float64)
            self._ctx("sbd_set_integrals", int(table.norb), _lib.ptr(h), _lib.ptr(eri), int(eri.size),
                      float(table.e_core))
            self._ctx("sbd_set_dets", _lib.ptr(da), _lib.ptr(db), int(self.n), int(basis.n_alpha_elec),
                      int(basis.n_beta_elec))
            self._ctx("sbd_build_tables")
        self.row_window = None
        self.n_own = self.n
        self._tables = None
        self._diag_dev = None
        self._diag_host = None
        self._ctx.bind_stream()
        self._ctx("sbd_diag", None)

    # -- reference attributes -------------------------------------------------
    @property
    def diag_device(self):
        """Diagonal of the owned rows as a torch CUDA tensor (copied out of the context once)."""
        if self._diag_dev is None:
            import torch

            d = torch.empty(self.n_own, dtype=torch.float64, device=self._torch_device)
            self._ctx.bind_stream()
            if self.n_own:
                self._ctx("sbd_diag", _lib.ptr(d))
            torch.cuda.synchronize(self.device)
            self._diag_dev = d
        return self._diag_dev

    @property
    def diag(self):
        """Reference attribute (apply.py:651-704): the diagonal as a numpy array, copied on first use."""
        if self._diag_host is None:
            self._diag_host = self.diag_device.cpu().numpy()
        return self._diag_host

    @property
    def tables(self):
        if self.basis.mode != "product":
            return None  # reference: explicit appliers carry no spin tables (apply.py:680)
        if self._tables is None:
            self._tables = SpinTables(alpha=_export_table(self._ctx, 0, self.basis.norb),
                                      beta=_export_table(self._ctx, 1, self.basis.norb))
        return self._tables

    @property
    def context(self) -> _lib.Context:
        return self._ctx

    def task0_kernel(self) -> str:
        """The task-0 kernel the last sigma ran (B200 introspection: "sell-cluster", "sell-tma",
        "sell-flat", "direct-ci" or "none")."""
        k = ctypes.c_int()
        self._ctx("sbd_last_task0", ctypes.byref(k))
        return {0: "none", 1: "sell-cluster", 2: "sell-tma", 3: "sell-flat", 4: "direct-ci"}[k.value]

    def sigma_model(self):
        """(c-bar_alpha, algorithmic bytes per sigma) -- BASELINE.md section 4."""
        cb, by = ctypes.c_double(), ctypes.c_double()
        self._ctx("sbd_sigma_model", ctypes.byref(cb), ctypes.byref(by))
        return cb.value, by.value

    # -- application ------------------------------------------------------------
    def sigma_device(self, x, out=None):
        """Device path: x (all rows, torch CUDA f64) -> y (owned rows)."""
        import torch

        if x.dtype != torch.float64 or not x.is_cuda or x.numel() != self.n:
            raise ValueError(f"expected a CUDA float64 vector of length {self.n}")
        if x.device != self._torch_device:
            raise ValueError(f"x is on {x.device}, the applier on {self._torch_device}")
        if out is not None and (out.dtype != torch.float64 or out.device != self._torch_device
                                or out.numel() != self.n_own or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous float64 tensor of {self.n_own} elements on "
                             f"{self._torch_device}")
        self.apply_count += 1
        x = x.contiguous()
        y = torch.empty(self.n_own, dtype=torch.float64, device=x.device) if out is None else out
        self._ctx.bind_stream()
        if self.n_own:
            self._ctx("sbd_sigma", _lib.ptr(x), _lib.ptr(y))
        return y

    def __call__(self, x, out=None):
        try:
            import torch

            if isinstance(x, torch.Tensor) and x.is_cuda:
                return self.sigma_device(x.reshape(-1), out=out)
        except ImportError:  # pragma: no cover
            pass
        xa = np.asarray(x, dtype=np.float64)
        if xa.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {xa.shape}")
        xa = np.ascontiguousarray(xa)
        self.apply_count += 1
        y = np.empty(self.n_own, dtype=np.float64) if out is None else out
        if y.shape != (self.n_own,) or y.dtype != np.float64 or not y.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of the owned length")
        self._ctx.bind_stream()
        if self.n_own:
            self._ctx("sbd_sigma_host", _lib.ptr(xa), _lib.ptr(y))
        return y


def compute_diagonal(basis: SelectedBasis, table: IntegralTable, cache=None, device=None) -> np.ndarray:
    """d_i = <det_i|H|det_i> (reference ``apply.py:573-586``; bitwise equal), either basis mode."""
    return HamiltonianApplier(basis, table, device=device).diag


def apply_H(x, basis: SelectedBasis, table: IntegralTable, tables: Optional[SpinTables] = None, cache=None,
            exec_policy: str = "parallel", device=None):
    """One full product-basis application (reference ``apply.py:589-605``)."""
    if basis.mode != "product":
        raise ValueError("apply_H serves product-mode bases; see apply_H_full")
    n = basis.dimension
    xa = x if not isinstance(x, (list, tuple)) else np.asarray(x, dtype=np.float64)
    if isinstance(xa, np.ndarray) and xa.shape != (n,):
        raise ValueError(f"expected vector of length {n}, got shape {xa.shape}")
    return HamiltonianApplier(basis, table, tables, exec_policy, device=device)(xa)


def apply_H_full(x, basis: SelectedBasis, table: IntegralTable, exec_policy: str = "parallel", device=None):
    """y = H x over an explicit determinant list (reference ``apply.py:626-648``)."""
    if basis.mode != "explicit":
        raise ValueError("apply_H_full serves explicit-mode bases; see apply_H")
    return HamiltonianApplier(basis, table, exec_policy=exec_policy, device=device)(x)
