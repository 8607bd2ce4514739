"""Device-resident Davidson driver (reference ``davidson.py``), same API.

``davidson_solve(apply_h, diag, x0=None, opts=None) -> DavidsonResult`` keeps
the reference's algorithm step for step -- single-vector expansion with
cached images W, Jacobi Rayleigh-Ritz, residuals from W (no extra
applications), damped diagonal preconditioner, reorthogonalised
Gram-Schmidt, thick restart by rotating V and W, random-direction breakdown
recovery, honest non-convergence -- and its defaults, so iteration counts
are like-for-like.  What changes is where the data lives: V, W, the
residual/correction vectors and the projected matrix stay on the GPU; every
pass over the subspace is one fused CUDA kernel (``csrc/sbd_davidson.cu``);
the host reads back only O(k) scalars per iteration (residual norms, the
breakdown test).

Numerical note: the reference's modified Gram-Schmidt (two sequential
sweeps) is replaced by classical Gram-Schmidt applied twice (CGS2), which
needs 2 passes over V instead of 2k; in exact arithmetic both produce the
same vector, and CGS2 is orthogonal to working precision.

``apply_h`` may be this package's ``HamiltonianApplier`` (the operator stays
on the device: x and y are CUDA tensors), a ``DistributedApplier`` rank, or
any numpy callable (its input/output cross the host link each iteration).
"""

from __future__ import annotations

import math

import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib

__all__ = [
    "DavidsonOptions",
    "DavidsonStats",
    "DavidsonResult",
    "davidson_solve",
    "jacobi_eigh",
    "projected_eigensolve",
    "precondition",
    "orthogonalize",
]


@dataclass
class DavidsonOptions:
    n_roots: int = 1
    tol_residual: float = 1e-8
    max_iters: int = 200
    max_subspace: int = 32
    restart_keep: int = 4
    precond_delta: float = 1e-6
    reorthogonalize: bool = True
    # B200 extension: record ||V V^T - I||_F per iteration from the Gram row
    # fused into the V^T w pass (no extra pass over V).
    track_orthogonality: bool = True
    # B200 extension: per-phase CUDA-event timing in stats.phase_ms (tracing)
    profile: bool = False
    # B200 extension (off = reference): skip the second Gram-Schmidt pass when the first kept
    # |t1| >= |t0| / sqrt(2) ("twice is enough"), saving one pass over V in most iterations
    selective_reorth: bool = False

    def __post_init__(self):
        if not 1 <= self.n_roots <= self.restart_keep <= self.max_subspace:
            raise ValueError(
                "need 1 <= n_roots <= restart_keep <= max_subspace, got "
                f"{self.n_roots}/{self.restart_keep}/{self.max_subspace}")
        if self.tol_residual <= 0:
            raise ValueError("tol_residual must be positive")
        if self.precond_delta <= 0:
            raise ValueError("precond_delta must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.max_subspace > 64:
            raise ValueError("max_subspace must be <= 64 on the B200 path")
        if self.n_roots > 8:
            raise ValueError("n_roots must be <= 8 on the B200 path")


@dataclass
class DavidsonStats:
    iterations: int = 0
    converged: bool = False
    n_applies: int = 0
    restarts: int = 0
    breakdowns: int = 0
    theta_history: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    theta_deltas: list = field(default_factory=list)
    ortho_history: list = field(default_factory=list)
    apply_seconds: list = field(default_factory=list)
    restart_iters: list = field(default_factory=list)
    iter_seconds: list = field(default_factory=list)  # B200 extension: wall time per iteration
    phase_ms: dict = field(default_factory=dict)  # B200 extension: summed device time per phase
    host_ms: dict = field(default_factory=dict)  # B200 extension: host time per section (enqueue / wait)
    timeline: list = field(default_factory=list)  # B200 extension (profile): one iteration on the device clock


@dataclass
class DavidsonResult:
    energies: np.ndarray
    vectors: np.ndarray  # (n_roots, N); torch CUDA tensor when return_device=True
    residual_norms: np.ndarray
    stats: DavidsonStats

    @property
    def converged(self) -> bool:
        return self.stats.converged


class _Engine:
    """Kernel launcher bound to one device (any context can drive the vector kernels)."""

    def __init__(self, device: int, ctx: Optional[_lib.Context] = None, profile: bool = False):
        self.ctx = ctx if ctx is not None else _lib.Context(device)
        self.own_ctx = ctx is None
        self.profile = profile
        self._events = []  # (name, start, end)

    def __call__(self, name, *args):
        self.ctx.bind_stream()
        if self.profile:
            with self.phase(name):
                self.ctx(name, *args)
        else:
            self.ctx(name, *args)

    def phase(self, name):
        import contextlib

        import torch

        if not self.profile:
            return contextlib.nullcontext()
        eng = self

        class _P:
            def __enter__(self):
                self.s = torch.cuda.Event(enable_timing=True)
                self.e = torch.cuda.Event(enable_timing=True)
                self.s.record()

            def __exit__(self, *exc):
                self.e.record()
                eng._events.append((name, self.s, self.e))
        return _P()

    def summary(self) -> dict:
        import torch

        torch.cuda.synchronize()
        out = {}
        for name, s, e in self._events:
            out[name] = out.get(name, 0.0) + s.elapsed_time(e)
        return out

    def timeline(self, first: int, count: int) -> list:
        """(name, start, duration) in ms, relative to event `first` (profile mode; gaps = idle device)."""
        ev = self._events[first:first + count]
        if not ev:
            return []
        t0 = ev[0][1]
        return [(n, t0.elapsed_time(s), s.elapsed_time(e)) for n, s, e in ev]


def _p(t):
    return _lib.ptr(t)


def jacobi_eigh(mat, max_sweeps: int = 64, device=None):
    """Full spectrum of a symmetric matrix by the device cyclic-Jacobi kernel.

    Reference ``davidson.py:127-148``: symmetrise, sweep to off-norm
    <= 1e-14 ||A||_F, ascending stable order.  Returns numpy arrays.
    """
    import torch

    mat = np.asarray(mat, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {mat.shape}")
    if not np.isfinite(mat).all():
        raise ValueError("matrix contains non-finite entries")
    n = mat.shape[0]
    if n > 64:
        raise ValueError("device Jacobi handles n <= 64")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    eng = _Engine(dev.index)
    a = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    v = torch.empty((n, n), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    eng("sbd_jacobi", _p(a), n, n, _p(w), _p(v), max_sweeps, _p(info))
    if int(info.item()) >= max_sweeps:
        raise RuntimeError(f"Jacobi sweep limit {max_sweeps} reached without convergence")
    return w.cpu().numpy(), v.cpu().numpy()


def projected_eigensolve(t_mat):
    return jacobi_eigh(t_mat)


def precondition(r, diag, theta: float, delta: float):
    """t_i = r_i / (sign(d_i - theta) max(|d_i - theta|, delta)); sign(0) = +1 (davidson.py:159-163)."""
    d = diag - theta
    sign = np.where(d >= 0.0, 1.0, -1.0)
    return r / (sign * np.maximum(np.abs(d), delta))


def orthogonalize(t, vset, reorthogonalize: bool = True):
    """Host helper with the reference contract (davidson.py:166-185), CGS form."""
    v = np.array(t, dtype=np.float64)
    norm0 = np.linalg.norm(v)
    if norm0 == 0.0:
        return None
    if len(vset):
        basis = np.vstack(vset)
        for _ in range(2 if reorthogonalize else 1):
            v -= basis.T @ (basis @ v)
    norm = np.linalg.norm(v)
    return None if norm < 1e-12 * norm0 else v / norm


def _operator(apply_h, n: int, device):
    """Return f(x_dev, y_dev) writing H x into y (device tensors)."""
    import torch

    if hasattr(apply_h, "sigma_device"):
        n_own = getattr(apply_h, "n_own", n)
        if n_own != n:
            raise ValueError("distributed operators go through DistributedApplier.davidson")

        def f(x, y):
            apply_h.sigma_device(x, out=y)
        return f, getattr(apply_h, "context", None)

    def g(x, y):
        out = apply_h(x.cpu().numpy())
        out = torch.as_tensor(np.asarray(out, dtype=np.float64))
        if out.shape != (n,):
            raise ValueError(f"apply_h returned shape {tuple(out.shape)}, expected ({n},)")
        y.copy_(out.to(y.device, non_blocking=False))
    return g, None


def davidson_solve(apply_h: Callable, diag, x0=None, opts: Optional[DavidsonOptions] = None,
                   device=None, return_device: bool = False, allreduce=None,
                   rank_offset: int = 0, ctx=None, native: Optional[bool] = None) -> DavidsonResult:
    """Lowest ``opts.n_roots`` eigenpairs (reference ``davidson.py:191-306``).

    ``allreduce(tensor)`` (optional) sums a small CUDA tensor over ranks in
    place; the row-partitioned multi-GPU driver passes an NCCL all-reduce,
    its ``apply_h(x_dev, y_dev)`` on the rank's rows, and ``rank_offset`` =
    global index of the rank's first amplitude.

    ``native``: run the control loop in C++ (``sbd_davidson``, same algorithm
    and kernels, no Python between the passes).  Default: on for a
    single-GPU ``HamiltonianApplier`` unless ``opts.profile`` is set or
    ``SBD_DAV_PYTHON=1``; ``True`` raises ValueError where it cannot apply.
    """
    import torch

    opts = DavidsonOptions() if opts is None else opts
    if isinstance(diag, torch.Tensor):
        diag_dev = diag.to(torch.float64)
    else:
        diag_np = np.asarray(diag, dtype=np.float64)
        diag_dev = None
    n_loc = int(diag.numel()) if isinstance(diag, torch.Tensor) else int(diag_np.shape[0])
    n = n_loc
    if allreduce is not None:
        nt = torch.tensor([float(n_loc)], dtype=torch.float64, device=diag.device)
        allreduce(nt)
        n = int(nt.item())
    if n < 1:
        raise ValueError("empty problem")
    if n < opts.n_roots:
        raise ValueError(f"cannot extract {opts.n_roots} roots from dimension {n}")

    if device is None:
        device = getattr(apply_h, "device", None)
        if device is None and isinstance(diag, torch.Tensor) and diag.is_cuda:
            device = diag.device.index
        if device is None:
            device = torch.cuda.current_device()
    dev = torch.device("cuda", int(device))
    if _use_native(apply_h, allreduce, opts, native):
        with torch.cuda.device(dev):
            dd = diag if isinstance(diag, torch.Tensor) else torch.from_numpy(diag_np)
            res = _solve_native(apply_h.context, n, dd.to(dev, torch.float64).contiguous(), x0, opts, dev,
                                return_device)
            apply_h.apply_count += res.stats.n_applies
            return res
    with torch.cuda.device(dev):
        return _solve(apply_h, diag_dev if diag_dev is not None else torch.from_numpy(diag_np).to(dev),
                      x0, opts, n, n_loc, dev, return_device, allreduce, rank_offset, ctx)


def _use_native(apply_h, allreduce, opts, native) -> bool:
    import os

    from .apply import HamiltonianApplier

    ok = (allreduce is None and isinstance(apply_h, HamiltonianApplier) and apply_h.n_own == apply_h.n
          and not opts.profile)
    if native is None:
        return ok and os.environ.get("SBD_DAV_PYTHON", "0") != "1"
    if native and not ok:
        raise ValueError("native=True needs a single-GPU HamiltonianApplier owning all rows and profile=False")
    return bool(native)


def _solve_native(ctx, n, diag_dev, x0, opts, dev, return_device):
    """C++ control loop (``sbd_davidson``, csrc/sbd_solver.cu) over a context.

    ``n`` is the context's own length: all rows for a single-GPU applier, the
    rank's rows for a partitioned context (sbd_dist_init), whose dot products
    the library all-reduces.
    """
    import ctypes

    import torch

    f64 = dict(dtype=torch.float64, device=dev)
    if diag_dev.numel() != n:
        raise ValueError(f"diag has {diag_dev.numel()} entries, expected {n}")
    v0 = None
    if x0 is not None:
        v0 = (x0.to(**f64) if isinstance(x0, torch.Tensor)
              else torch.from_numpy(np.asarray(x0, dtype=np.float64).copy()).to(dev)).reshape(-1).contiguous()
        if v0.numel() != n:
            raise ValueError(f"x0 has {v0.numel()} entries, expected {n}")
    m, mi = opts.n_roots, opts.max_iters
    hist = {name: np.full(mi * (m if name in ("theta", "res") else 1), np.nan)
            for name in ("theta", "res", "ortho", "apply", "iter")}
    restart_iters = np.zeros(mi, dtype=np.int32)
    o = _lib.DavidsonOptsC(n_roots=m, tol_residual=float(opts.tol_residual), max_iters=mi,
                           max_subspace=opts.max_subspace, restart_keep=opts.restart_keep,
                           precond_delta=float(opts.precond_delta), reorthogonalize=int(opts.reorthogonalize),
                           track_orthogonality=int(opts.track_orthogonality),
                           selective_reorth=int(opts.selective_reorth))
    st = _lib.DavidsonStatsC(theta_hist=hist["theta"].ctypes.data, res_hist=hist["res"].ctypes.data,
                             ortho_hist=hist["ortho"].ctypes.data, apply_ms_hist=hist["apply"].ctypes.data,
                             iter_ms_hist=hist["iter"].ctypes.data, restart_iters=restart_iters.ctypes.data)
    evals = np.full(m, np.nan)
    res = np.full(m, np.nan)
    U = torch.empty((m, n), **f64)
    ctx.bind_stream()
    ctx("sbd_davidson", ctypes.byref(o), _p(diag_dev), _p(v0), evals.ctypes.data, res.ctypes.data, _p(U), n,
        ctypes.byref(st))
    it, nf = st.iterations, st.n_found
    stats = DavidsonStats(iterations=it, converged=bool(st.converged), n_applies=st.n_applies,
                          restarts=st.restarts, breakdowns=st.breakdowns)
    th = hist["theta"].reshape(mi, m)[:it]
    rs = hist["res"].reshape(mi, m)[:it]
    prev = None
    for i in range(it):
        row = th[i][~np.isnan(th[i])]
        stats.theta_history.append(row.copy())
        stats.residual_history.append(rs[i][~np.isnan(rs[i])].copy())
        stats.theta_deltas.append(abs(row[0] - prev) if prev is not None else np.inf)
        prev = row[0]
    stats.ortho_history = [float(v) for v in hist["ortho"][:it]]
    stats.apply_seconds = [float(v) / 1e3 for v in hist["apply"][:it]]
    stats.iter_seconds = [float(v) / 1e3 for v in hist["iter"][:it]]
    stats.restart_iters = [int(v) for v in restart_iters[:st.restarts]]
    stats.host_ms = {"native": float(np.nansum(hist["iter"][:it]))}
    U = U[:nf]
    vectors = U if return_device else U.cpu().numpy()
    return DavidsonResult(energies=evals[:nf].copy(), vectors=vectors, residual_norms=res[:nf].copy(), stats=stats)


def _solve(apply_h, diag_dev, x0, opts, n, n_loc, dev, return_device, allreduce, rank_offset, ctx):
    """Driver loop.  The projected matrix T = V^T H V and the Gram matrix G stay
    on the device next to V and W; the Rayleigh-Ritz eigensolve reads T in
    place.  The host sees one packed read-back per iteration (Ritz values,
    residual norms, |t|^2, Jacobi sweep count, orthogonality loss) for the
    control decisions, plus one for the CGS2 branch test."""
    import torch

    f64 = dict(dtype=torch.float64, device=dev)
    diag_dev = diag_dev.to(dev).contiguous()
    if allreduce is None:
        apply_fn, op_ctx = _operator(apply_h, n_loc, dev)
        ctx = ctx if ctx is not None else op_ctx
    else:
        apply_fn = apply_h
    eng = _Engine(dev.index, ctx, profile=opts.profile)
    reduce = allreduce if allreduce is not None else (lambda t: None)
    stream = torch.cuda.current_stream(dev)

    m = opts.n_roots
    k_max = min(opts.max_subspace, n)
    keep = min(opts.restart_keep, k_max)
    stats = DavidsonStats()
    rng = np.random.default_rng(0x5BD1A6)

    # leading dimension padded to a multiple of 32 doubles: 16-byte aligned rows
    # for the 128-bit kernels; vectors are the [:n_loc] views
    ld = max(32, (n_loc + 31) // 32 * 32)
    V = torch.zeros((k_max, ld), **f64)[:, :n_loc]
    W = torch.zeros((k_max, ld), **f64)[:, :n_loc]
    Tv = torch.zeros((m, ld), **f64)[:, :n_loc]   # preconditioned residuals (one per root)
    small = torch.zeros(2 * 64 + 16, **f64)       # device scratch for dot products
    small2 = torch.zeros(2 * 64 + 16, **f64)      # CGS outputs (never aliases its input c)
    scale = torch.zeros(1, **f64)
    T = torch.zeros((k_max, k_max), **f64)        # projected matrix, device-resident
    G = torch.zeros((k_max, k_max), **f64)        # Gram matrix of V (orthogonality stats)
    eye = torch.eye(k_max, **f64)
    Y_dev = torch.zeros((k_max * 8,), **f64)
    Yk_dev = torch.zeros((k_max * 8,), **f64)
    th_dev = torch.zeros(8, **f64)
    jac_w = torch.zeros(k_max, **f64)
    jac_v = torch.zeros((k_max * k_max,), **f64)
    jac_info = torch.zeros(1, dtype=torch.int32, device=dev)
    c_dev = torch.zeros(64, **f64)
    pack = torch.zeros(2 * 64 + 32, **f64)
    host = torch.zeros(2 * 64 + 32, dtype=torch.float64, pin_memory=True)

    # start vector (davidson.py:219-227)
    if x0 is None:
        if allreduce is not None:
            raise ValueError("distributed solves pass x0 (DistributedApplier computes the global argmin)")
        V[0].zero_()
        V[0, int(torch.argmin(diag_dev).item())] = 1.0
    else:
        if isinstance(x0, torch.Tensor):
            v0 = x0.to(**f64).reshape(-1)
        else:
            v0 = torch.from_numpy(np.asarray(x0, dtype=np.float64).reshape(-1).copy()).to(dev)
        if v0.numel() != n_loc:
            raise ValueError(f"x0 has {v0.numel()} entries, expected {n_loc}")
        # the native driver's normalisation (sbd_solver.cu setup): sbd_vdots, then x0 * (1 / |x0|), so both
        # control loops start from the same bits
        v0 = v0.contiguous()
        nrm2 = torch.zeros(1, **f64)
        ld_native = max(32, (n_loc + 31) // 32 * 32)  # the native basis' leading dimension (same kernel choice)
        eng("sbd_vdots", _lib.ptr(v0), 1, ld_native, n_loc, _lib.ptr(v0), _lib.ptr(nrm2))
        reduce(nrm2)
        norm = math.sqrt(max(float(nrm2.item()), 0.0))
        if not norm > 0.0 or not math.isfinite(norm):
            raise ValueError("x0 must be nonzero")
        V[0].copy_(v0 * (1.0 / norm))

    k = 1
    theta = np.zeros(m)
    mk = 1
    res_norms = np.full(m, np.inf)
    prev_theta0 = None
    jp = 0  # root whose correction the fused kernel projects
    ritz_rotated = False
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    host_ms = {}
    _tick = [time.perf_counter()]

    def hp(name):  # host-side time per section (perf_counter only: always on, reported in stats.host_ms)
        t = time.perf_counter()
        host_ms[name] = host_ms.get(name, 0.0) + (t - _tick[0]) * 1e3
        _tick[0] = t

    def readback(t_dev, cnt):
        with eng.phase("readback"):
            host[:cnt].copy_(t_dev[:cnt], non_blocking=True)
        hp("enqueue")
        stream.synchronize()
        hp("sync_wait")
        return host[:cnt].numpy().copy()

    for iteration in range(1, opts.max_iters + 1):
        t_iter = time.perf_counter()
        stats.iterations = iteration
        # image of the newest direction (davidson.py:241-245)
        ev0.record(stream)
        with eng.phase("sigma"):
            apply_fn(V[k - 1], W[k - 1])
        ev1.record(stream)
        stats.n_applies += 1

        # T[:, k-1] = V^T w and the Gram row of v_{k-1}: one pass over V
        eng("sbd_vdots2", _p(V), k, ld, n_loc, _p(W[k - 1]), _p(V[k - 1]), _p(small))
        reduce(small[: 2 * k])
        with eng.phase("torch:T"):
            T[:k, k - 1] = small[:k]
            T[k - 1, :k] = small[:k]
            G[:k, k - 1] = small[k:2 * k]
            G[k - 1, :k] = small[k:2 * k]

        # Rayleigh-Ritz on the device, in place on T (davidson.py:251)
        eng("sbd_jacobi", _p(T), k, k_max, _p(jac_w), _p(jac_v), 64, _p(jac_info))
        # numpy slicing in the reference keeps min(m, k) roots while k < m
        mk = min(m, k)
        evecs = jac_v[: k * k].view(k, k)
        with eng.phase("torch:ritz"):
            Y_dev[: k * mk].copy_(evecs[:, :mk].reshape(-1))
            th_dev[:mk].copy_(jac_w[:mk])
        ritz_rotated = False

        # residuals, preconditioned corrections and V^T t in one pass
        jp = min(jp, mk - 1)
        eng("sbd_residual_precond_target", _p(V), _p(W), k, ld, n_loc, _p(Y_dev), _p(th_dev), mk, jp,
            _p(diag_dev), float(opts.precond_delta), _p(Tv), ld, _p(small))
        reduce(small[: k + 1 + mk])
        c_dev[:k].copy_(small[:k])

        # one packed read-back: theta | residual^2 | |t|^2 | sweeps | ortho
        with eng.phase("torch:pack"):
            pack[:mk].copy_(jac_w[:mk])
            pack[mk:2 * mk].copy_(small[k + 1:k + 1 + mk])
            pack[2 * mk] = small[k]
            pack[2 * mk + 1] = jac_info[0].to(torch.float64)
            if opts.track_orthogonality:
                pack[2 * mk + 2] = torch.linalg.norm(G[:k, :k] - eye[:k, :k])
        # speculative CGS pass 1 on the projected root (the usual next step: not
        # converged, same target root, no restart), read back with the pack, so an
        # iteration costs one host round trip instead of two
        spec = opts.reorthogonalize and k < k_max and iteration < opts.max_iters
        npk = 2 * mk + 3
        if spec:
            eng("sbd_gs_update", _p(V), k, ld, n_loc, _p(c_dev), _p(Tv[jp]), _p(small2))
            reduce(small2[: k + 1])
            pack[npk:npk + k + 1].copy_(small2[: k + 1])
        hv = readback(pack, npk + (k + 1 if spec else 0))
        stats.apply_seconds.append(ev0.elapsed_time(ev1) / 1e3)
        if hv[2 * mk + 1] >= 64:
            raise RuntimeError("Jacobi sweep limit 64 reached without convergence")
        theta = hv[:mk].copy()
        res_norms = np.sqrt(np.maximum(hv[mk:2 * mk], 0.0))
        t_norm2 = float(hv[2 * mk])

        stats.ortho_history.append(float(hv[2 * mk + 2]) if opts.track_orthogonality else float("nan"))
        stats.theta_history.append(theta.copy())
        stats.residual_history.append(res_norms.copy())
        stats.theta_deltas.append(abs(theta[0] - prev_theta0) if prev_theta0 is not None else np.inf)
        prev_theta0 = theta[0]
        hp("control")

        if bool(np.all(res_norms <= opts.tol_residual)):
            stats.converged = True
            stats.iter_seconds.append(time.perf_counter() - t_iter)
            break
        if iteration == opts.max_iters:
            stats.iter_seconds.append(time.perf_counter() - t_iter)
            break

        target = int(np.argmax(res_norms > opts.tol_residual))
        t_vec = Tv[target]
        pre = (hv[npk:npk + k].copy(), float(hv[npk + k])) if spec and target == jp else None
        if target != jp:
            # the fused projection used another root: one extra pass
            eng("sbd_vdots2", _p(V), k, ld, n_loc, _p(t_vec), _p(t_vec), _p(small))
            reduce(small[: 2 * k])
            c_dev[:k].copy_(small[:k])
            nn = (t_vec @ t_vec).reshape(1)
            reduce(nn)
            t_norm2 = float(nn.item())
            jp = target

        if k == k_max:
            # thick restart (davidson.py:280-289): rotate V and W in place
            yk = evecs[:, :keep]
            Yk_dev[: k * keep].copy_(yk.reshape(-1))
            eng("sbd_rotate", _p(V), k, ld, n_loc, _p(Yk_dev), keep)
            eng("sbd_rotate", _p(W), k, ld, n_loc, _p(Yk_dev), keep)
            # the k x k bookkeeping on the host (a few microseconds; no cuBLAS on the path)
            yk_h = yk.cpu().numpy()
            G_new = yk_h.T @ G[:k, :k].cpu().numpy() @ yk_h
            c_new = yk_h.T @ c_dev[:k].cpu().numpy()
            T.zero_()
            T[:keep, :keep] = torch.diag(jac_w[:keep])
            G.zero_()
            G[:keep, :keep] = torch.from_numpy(G_new).to(dev)
            c_dev[:keep].copy_(torch.from_numpy(c_new).to(dev))
            stats.restarts += 1
            stats.restart_iters.append(iteration)
            k = keep
            ritz_rotated = True

        v_ok = _orthogonalize_device(eng, V, k, ld, n_loc, t_vec, c_dev, t_norm2, opts, small2, scale, reduce,
                                     readback, pre)
        attempts = 0
        while not v_ok and attempts < 3:
            stats.breakdowns += 1
            rv = rng.standard_normal(n)  # same stream as the reference (davidson.py:295)
            lo = rank_offset
            t_vec.copy_(torch.from_numpy(rv[lo:lo + n_loc]))
            eng("sbd_vdots2", _p(V), k, ld, n_loc, _p(t_vec), _p(t_vec), _p(small))
            reduce(small[: 2 * k])
            c_dev[:k].copy_(small[:k])
            nn = (t_vec @ t_vec).reshape(1)
            reduce(nn)
            v_ok = _orthogonalize_device(eng, V, k, ld, n_loc, t_vec, c_dev, float(nn.item()), opts, small2, scale,
                                         reduce, readback)
            attempts += 1
        if not v_ok:
            stats.iter_seconds.append(time.perf_counter() - t_iter)
            break
        k += 1
        stats.iter_seconds.append(time.perf_counter() - t_iter)

    # Ritz vectors of the last Rayleigh-Ritz (davidson.py:256), computed once
    if ritz_rotated:
        Yr = torch.zeros((k, mk), **f64)
        Yr[:mk, :mk] = torch.eye(mk, **f64)
    else:
        Yr = jac_v[: k * k].view(k, k)[:, :mk]
    kk = Yr.shape[0]
    Y_dev[: kk * mk].copy_(Yr.reshape(-1))
    U = torch.empty((mk, n_loc), **f64)
    eng("sbd_combine", _p(V), kk, ld, n_loc, _p(Y_dev), mk, _p(U), n_loc)
    del V, W, Tv
    torch.cuda.current_stream(dev).synchronize()
    stats.host_ms = host_ms
    if opts.profile:
        stats.phase_ms = eng.summary()
        sig = [i for i, ev in enumerate(eng._events) if ev[0] == "sigma"]
        if len(sig) >= 3:
            a, b = sig[len(sig) // 2], sig[len(sig) // 2 + 1]
            stats.timeline = eng.timeline(a, b - a + 1)
        stats.phase_ms.update({"host:" + k_: v for k_, v in host_ms.items()})
    vectors = U if return_device else U.cpu().numpy()
    if eng.own_ctx:
        eng.ctx.close()
    return DavidsonResult(energies=theta.copy(), vectors=vectors, residual_norms=res_norms.copy(), stats=stats)


def _orthogonalize_device(eng, V, k, ld, n_loc, t, c, t_norm2, opts, small, scale, reduce, readback,
                          pre=None) -> bool:
    """CGS2 of t against V[:k] given c = V^T t (device); writes the normalised V[k] on success.

    ``pre = (c2, |t'|^2)``: CGS pass 1 already ran (speculatively, output in ``small``).

    Rejection rule of the reference orthogonalize (davidson.py:166-185): the
    remainder norm must stay >= 1e-12 of the input norm.
    """
    norm0 = float(np.sqrt(max(t_norm2, 0.0)))
    if norm0 == 0.0:
        return False
    if opts.reorthogonalize:
        # CGS pass 1: t' = t - V c ; c2 = V^T t' ; |t'|^2
        if pre is None:
            eng("sbd_gs_update", _p(V), k, ld, n_loc, _p(c), _p(t), _p(small))
            reduce(small[: k + 1])
            hv = readback(small, k + 1)
            c2, n2p = hv[:k], float(hv[k])
        else:
            c2, n2p = pre
        if opts.selective_reorth and n2p >= 0.5 * t_norm2:  # |t'| >= |t| / sqrt(2): one pass is enough
            norm = float(np.sqrt(max(n2p, 0.0)))
            if norm < 1e-12 * norm0 or norm == 0.0:
                return False
            scale.fill_(1.0 / norm)
            eng("sbd_scale_copy", _p(t), _p(V[k]), n_loc, _p(scale))
            return True
        n2 = n2p - float(c2 @ c2)  # |t' - V c2|^2 for orthonormal V
        c2d = small[:k].clone()
        if n2p > 0.0 and n2 > 0.5 * n2p:
            # pass 2 fused with the normalisation, written straight into V[k]
            if np.sqrt(n2) < 1e-12 * norm0:
                return False
            scale.fill_(1.0 / np.sqrt(n2))
            eng("sbd_gs_finalize", _p(V), k, ld, n_loc, _p(c2d), _p(t), _p(V[k]), _p(scale), _p(small))
            return True
        eng("sbd_gs_update_nodots", _p(V), k, ld, n_loc, _p(c2d), _p(t), _p(small))
    else:
        eng("sbd_gs_update_nodots", _p(V), k, ld, n_loc, _p(c), _p(t), _p(small))
    reduce(small[:1])
    norm = float(np.sqrt(max(float(readback(small, 1)[0]), 0.0)))
    if norm < 1e-12 * norm0 or norm == 0.0:
        return False
    scale.fill_(1.0 / norm)
    eng("sbd_scale_copy", _p(t), _p(V[k]), n_loc, _p(scale))
    return True
