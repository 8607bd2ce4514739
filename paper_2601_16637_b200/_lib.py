"""ctypes binding of ``include/sbd.h`` (libsbd_b200.so, built in-tree for sm_100a).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  Status codes map to the reference's
exception types: SBD_EINVAL -> ValueError, SBD_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

# SBD_LIB overrides the in-tree library (A/B measurements of two builds on one box)
LIB_PATH = os.environ.get("SBD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsbd_b200.so")

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "sbd_abi_version": [],
    "sbd_last_error": [_vp],
    "sbd_create": [_c_int, ctypes.POINTER(_vp)],
    "sbd_destroy": [_vp],
    "sbd_set_stream": [_vp, _vp],
    "sbd_set_integrals": [_vp, _c_int, _vp, _vp, _c_i64, _c_dbl],
    "sbd_set_strings": [_vp, _c_int, _vp, _c_i64, _c_int],
    "sbd_set_dets": [_vp, _vp, _vp, _c_i64, _c_int, _c_int],
    "sbd_ingest_samples": [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "sbd_ingest_export": [_vp, _vp, _vp, _vp, _vp, _vp],
    "sbd_build_tables": [_vp],
    "sbd_table_counts": [_vp, _c_int, _vp, _vp, _vp],
    "sbd_export_table": [_vp, _c_int] + [_vp] * 12,
    "sbd_export_sorted": [_vp, _c_int, _vp, _vp],
    "sbd_table128_build": [_vp, _c_int, _vp, _c_i64, _c_int],
    "sbd_table128_counts": [_vp, _vp, _vp, _vp],
    "sbd_table128_export": [_vp] + [_vp] * 12,
    "sbd_table128_sorted": [_vp, _vp, _vp],
    "sbd_set_row_window": [_vp, _c_i64, _c_i64],
    "sbd_diag": [_vp, _vp],
    "sbd_sigma": [_vp, _vp, _vp],
    "sbd_sigma_local": [_vp, _vp],
    "sbd_sigma_remote": [_vp, _vp, _vp],
    "sbd_sigma_host": [_vp, _vp, _vp],
    "sbd_sigma_model": [_vp, _vp, _vp],
    "sbd_last_task0": [_vp, _vp],
    "sbd_sigma_multi": [_vp, _vp, _c_i64, _vp, _c_i64, _c_int],
    "sbd_vdots": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp],
    "sbd_vdots2": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _vp],
    "sbd_residual_precond": [_vp, _vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _c_int, _vp, _c_dbl, _vp,
                             _c_i64, _vp, _vp],
    "sbd_residual_precond_target": [_vp, _vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _c_int, _c_int, _vp,
                                    _c_dbl, _vp, _c_i64, _vp],
    "sbd_gs_update": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _vp],
    "sbd_gs_update_nodots": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _vp],
    "sbd_gs_finalize": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp],
    "sbd_scale_copy": [_vp, _vp, _vp, _c_i64, _vp],
    "sbd_rotate": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _c_int],
    "sbd_combine": [_vp, _vp, _c_int, _c_i64, _c_i64, _vp, _c_int, _vp, _c_i64],
    "sbd_jacobi": [_vp, _vp, _c_int, _c_int, _vp, _vp, _c_int, _vp],
    "sbd_dense_rows": [_vp, _c_i64, _c_i64, _vp],
    "sbd_nccl_unique_id": [_vp],
    "sbd_dist_init": [_vp, _c_int, _c_int, _vp, _vp],
    "sbd_dist_plan": [_vp, _c_int, _c_dbl, _c_int],
    "sbd_sigma_dist": [_vp, _vp, _vp],
    "sbd_dist_allreduce": [_vp, _vp, _c_i64, _c_int],
    "sbd_dist_check": [_vp],
    "sbd_dist_info": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sbd_dist_set_profiling": [_vp, _c_int],
    "sbd_dist_stats": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sbd_davidson_default_opts": [_vp],
    "sbd_davidson": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _vp],
}


class DavidsonOptsC(ctypes.Structure):
    """``sbd_davidson_opts`` (include/sbd.h)."""
    _fields_ = [("n_roots", _c_int), ("tol_residual", _c_dbl), ("max_iters", _c_int), ("max_subspace", _c_int),
                ("restart_keep", _c_int), ("precond_delta", _c_dbl), ("reorthogonalize", _c_int),
                ("track_orthogonality", _c_int), ("selective_reorth", _c_int)]


class DavidsonStatsC(ctypes.Structure):
    """``sbd_davidson_stats`` (include/sbd.h); history pointers are caller-owned host arrays."""
    _fields_ = [("iterations", _c_int), ("converged", _c_int), ("n_applies", _c_int), ("restarts", _c_int),
                ("breakdowns", _c_int), ("n_found", _c_int), ("sigma_ms", _c_dbl), ("theta_hist", _vp),
                ("res_hist", _vp), ("ortho_hist", _vp), ("apply_ms_hist", _vp), ("iter_ms_hist", _vp), ("restart_iters", _vp)]


_RESTYPE = {"sbd_last_error": ctypes.c_char_p}

EXPORTED = tuple(_SIGS)

_lib: Optional[ctypes.CDLL] = None


class ExtensionMissing(ImportError):
    pass


def load() -> ctypes.CDLL:
    """Load libsbd_b200.so (raises ExtensionMissing if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} not found: build the sm_100a extension first "
                "(python -m paper_2601_16637_b200._build or __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, _c_int)
        _lib = lib
    return _lib


def last_error(ctx=None) -> str:
    msg = load().sbd_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None, what: str = "") -> None:
    if rc == 0:
        return
    msg = last_error(ctx)
    if rc == 1:
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def ptr(x) -> int:
    """Raw address of a numpy array or torch tensor (no copies)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (``sbd_nccl_unique_id``) for ``sbd_dist_init``."""
    buf = ctypes.create_string_buffer(128)
    check(load().sbd_nccl_unique_id(buf), None, "sbd_nccl_unique_id")
    return buf.raw


def call(name: str, *args, ctx=None):
    rc = getattr(load(), name)(*args)
    check(rc, ctx, name)


class Context:
    """Owns one ``sbd_ctx`` on one CUDA device (HamiltonianApplier state)."""

    def __init__(self, device: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2601_16637_b200 needs a CUDA device (no CPU fallback)")
        self.device = int(device)
        h = _vp()
        check(load().sbd_create(self.device, ctypes.byref(h)), None, "sbd_create")
        self._h = h
        self.bind_stream()

    @property
    def handle(self):
        return self._h

    def bind_stream(self, stream=None) -> None:
        import torch

        s = torch.cuda.current_stream(self.device) if stream is None else stream
        self(("sbd_set_stream"), _vp(s.cuda_stream))

    def __call__(self, name: str, *args):
        rc = getattr(load(), name)(self._h, *args)
        check(rc, self._h, name)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            load().sbd_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
