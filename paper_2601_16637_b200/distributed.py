"""Alpha-block partitioned sigma and Davidson over GPUs (reference ``distsim.py``).

The reference simulates P workers with Python threads passing ket blocks
around a ring (``distsim.py:200-259``).  Here each rank is one process on one
GPU and the whole partitioned operator lives in ``libsbd_b200.so``
(``csrc/sbd_dist.cu``, NCCL over NVLink/NVSwitch inside the library):

* partition: contiguous alpha blocks, the first ``rem`` blocks one row longer
  (``make_partition``, ``distsim.py:63-77``); rank r owns x, sigma, diag, V and
  W rows ``[lo_r, hi_r) x n_beta``;
* per sigma, the reference ring's exchange pattern -- at step s rank r sends to
  (r + s) mod P and receives the block of (r - s) mod P -- on an exchange
  stream, while the compute stream runs the beta-beta part and the alpha
  pass over the rank's own rows, then one alpha pass per group of landed
  steps (``y +=``), then task 0.  Only the last group's transfer can be
  exposed (``sbd_dist_stats`` measures it: ``overlap_stats``);
* sparse exchange: when the referenced remote rows are a
  minority (cfg4: ~40%), only those rows travel, packed by the sender;
* Davidson: vectors stay row-partitioned; the native control loop
  (``sbd_davidson``) all-reduces the O(k) dot products of every fused pass.

``DistributedApplier(...).apply(x)`` keeps the reference signature (full
numpy x on every rank in, full y out).  The device-resident path is
``apply_device`` / ``davidson``.

``_rank_engine`` replaces the CUDA rank (tests on CPU): the same ring then
runs over ``torch.distributed`` (gloo) in Python, block by block, as the
CPU twin of the native schedule.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = ["Partition", "PartitionError", "make_partition", "DistributedApplier", "Comm", "OverlapReport",
           "overlap_stats"]


class PartitionError(ValueError):
    pass


@dataclass(frozen=True)
class Partition:
    n_workers: int
    alpha_blocks: tuple

    def block_of(self, w: int):
        return self.alpha_blocks[w]


def make_partition(n_alpha: int, n_workers: int) -> Partition:
    """Contiguous alpha blocks whose sizes differ by at most one (reference distsim.py:63-77)."""
    if n_workers < 1:
        raise PartitionError(f"need at least one worker, got {n_workers}")
    if n_workers > n_alpha:
        raise PartitionError(f"cannot split {n_alpha} alpha strings over {n_workers} workers")
    base, rem = divmod(n_alpha, n_workers)
    edges = np.cumsum([0] + [base + (1 if w < rem else 0) for w in range(n_workers)])
    return Partition(n_workers, tuple((int(edges[w]), int(edges[w + 1])) for w in range(n_workers)))


@dataclass
class OverlapReport:
    """Per-step overlap of one or more partitioned sigmas (reference ``OverlapReport``, distsim.py:81-88).

    Step 0 is the rank-local work (beta side + the alpha pass over the own
    rows); step g >= 1 is ring-step group g.  Times are device seconds per
    sigma, averaged over ranks: ``compute`` the passes, ``transfer`` the
    group's NCCL transfer, ``exposed`` the compute stream's wait for it.
    """
    n_workers: int
    n_steps: int
    overlap: bool
    transfer_delay: float
    per_step: list  # rows: (step, mean compute, mean transfer, mean exposed, ratio)
    total_compute_s: float
    total_transfer_s: float
    total_exposed_s: float
    overlap_ratio: float
    sigma_s: float = 0.0           # mean device time of one sigma (first exchange launch -> last pass), max over ranks
    n_sigma: int = 0
    per_rank: list = field(default_factory=list)


def overlap_stats(records, overlap: bool = True) -> OverlapReport:
    """Aggregate per-rank step records (``DistributedApplier.step_records``) like distsim.py:340-367."""
    p = len(records)
    n_steps = max(len(r["compute_ms"]) for r in records)
    per_step = []
    for s in range(n_steps):
        rows = [r for r in records if s < len(r["compute_ms"])]
        ns = [max(r["n_sigma"], 1) for r in rows]
        compute = float(np.mean([r["compute_ms"][s] / n for r, n in zip(rows, ns)])) / 1e3
        transfer = float(np.mean([r["transfer_ms"][s] / n for r, n in zip(rows, ns)])) / 1e3
        exposed = float(np.mean([r["exposed_ms"][s] / n for r, n in zip(rows, ns)])) / 1e3
        total = compute + exposed
        per_step.append((s, compute, transfer, exposed, 1.0 - (exposed / total if total > 0 else 0.0)))
    tc, tt, te = (sum(row[i] for row in per_step) for i in (1, 2, 3))
    denom = tc + te
    sig = max(r["total_ms"] / max(r["n_sigma"], 1) for r in records) / 1e3
    return OverlapReport(n_workers=p, n_steps=n_steps, overlap=overlap, transfer_delay=0.0, per_step=per_step,
                         total_compute_s=tc, total_transfer_s=tt, total_exposed_s=te,
                         overlap_ratio=1.0 - (te / denom if denom > 0 else 0.0), sigma_s=sig,
                         n_sigma=int(min(r["n_sigma"] for r in records)), per_rank=list(records))


class Comm:
    """torch.distributed plumbing: object exchange at setup, the reference-protocol gathers, the CPU twin."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _staged(self, t) -> bool:
        return self.backend == "gloo" and t.is_cuda

    def allreduce(self, t, op=None) -> None:
        if self.world == 1:
            return
        op = self.dist.ReduceOp.SUM if op is None else op
        if self._staged(t):
            h = t.cpu()
            self.dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=op, group=self.group)

    def allgather_blocks(self, out, local, blocks, row) -> None:
        """Gather every rank's ``local`` (its rows of ``blocks``, ``row`` elements each) into ``out``.

        One padded ``all_gather_into_tensor`` (blocks differ by at most one row), unpadded into ``out``.
        """
        import torch

        if self.world == 1:
            out.copy_(local)
            return
        mx = max(b - a for a, b in blocks) * row
        dev = torch.device("cpu") if self.backend == "gloo" else local.device
        send = torch.zeros(mx, dtype=local.dtype, device=dev)
        send[: local.numel()] = local.to(dev)
        recv = torch.empty(self.world * mx, dtype=local.dtype, device=dev)
        if self.backend == "gloo":
            parts = list(recv.view(self.world, mx).unbind(0))
            self.dist.all_gather(parts, send, group=self.group)
        else:
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
        rv = recv.view(self.world, mx)
        for q, (a, b) in enumerate(blocks):
            out[a * row:b * row].copy_(rv[q, :(b - a) * row])

    def barrier(self) -> None:
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def broadcast_object(self, obj, src: int = 0):
        lst = [obj]
        self.dist.broadcast_object_list(lst, src=self._global(src), group=self.group)
        return lst[0]

    def sendrecv(self, send, to: int, recv, frm: int) -> None:
        """Blocking ring step (CPU twin)."""
        ops = [self.dist.P2POp(self.dist.isend, send, self._global(to), group=self.group),
               self.dist.P2POp(self.dist.irecv, recv, self._global(frm), group=self.group)]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()

    def _global(self, rank: int) -> int:
        return rank if self.group is None else self.dist.get_global_rank(self.group, rank)


_EXCHANGE = {"auto": 0, "allgather": 1, "dense": 1, "sparse": 2}


class _NativeRank:
    """This rank's partitioned context: tables, plan and NCCL inside libsbd_b200.so (sbd_dist_*)."""

    def __init__(self, basis, table, comm: Comm, partition: Partition, device, exchange: str,
                 sparse_threshold: float, group_steps: int):
        import torch

        from . import _lib

        self.device = torch.device("cuda", int(device))
        self.ctx = ctx = _lib.Context(self.device.index)
        h = np.ascontiguousarray(table.h, dtype=np.float64)
        eri = np.ascontiguousarray(table.eri, dtype=np.float64)
        a = np.ascontiguousarray(basis.alpha_array(), dtype=np.uint64)
        b = np.ascontiguousarray(basis.beta_array(), dtype=np.uint64)
        with torch.cuda.device(self.device):
            ctx("sbd_set_integrals", int(table.norb), _lib.ptr(h), _lib.ptr(eri), int(eri.size), float(table.e_core))
            ctx("sbd_set_strings", 0, _lib.ptr(a), int(a.size), int(basis.n_alpha_elec))
            ctx("sbd_set_strings", 1, _lib.ptr(b), int(b.size), int(basis.n_beta_elec))
            uid = _lib.nccl_unique_id() if (comm.rank == 0 and comm.world > 1) else None
            uid = comm.broadcast_object(uid) if comm.world > 1 else None
            edges = np.array([lo for lo, _ in partition.alpha_blocks] + [partition.alpha_blocks[-1][1]],
                             dtype=np.int64)
            ctx("sbd_dist_init", comm.rank, comm.world, uid, _lib.ptr(edges))
            ctx("sbd_build_tables")
            ctx.bind_stream()
            ctx("sbd_dist_plan", _EXCHANGE[exchange], float(sparse_threshold), int(group_steps))
            lo, hi = partition.block_of(comm.rank)
            self.n_own = (hi - lo) * b.size
            self.diag = torch.empty(self.n_own, dtype=torch.float64, device=self.device)
            ctx("sbd_diag", _lib.ptr(self.diag))
            torch.cuda.synchronize(self.device)
        self.n_alpha, self.n_beta = int(a.size), int(b.size)

    @property
    def context(self):
        return self.ctx

    def sigma(self, x_own, y_own) -> None:
        from . import _lib

        self.ctx.bind_stream()
        self.ctx("sbd_sigma_dist", _lib.ptr(x_own), _lib.ptr(y_own))

    def info(self) -> dict:
        vals = [ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(),
                ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()]
        self.ctx("sbd_dist_info", *[ctypes.byref(v) for v in vals])
        keys = ("rank", "nranks", "alpha_lo", "alpha_hi", "sparse", "needed_fraction", "recv_rows", "send_rows",
                "n_groups")
        return {k: v.value for k, v in zip(keys, vals)}

    def set_profiling(self, on: bool) -> None:
        self.ctx("sbd_dist_set_profiling", int(bool(on)))

    def step_record(self) -> dict:
        n_sigma, n_steps, total = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double()
        buf = [np.zeros(64) for _ in range(3)]
        self.ctx("sbd_dist_stats", ctypes.byref(n_sigma), ctypes.byref(n_steps), *[b.ctypes.data for b in buf],
                 ctypes.byref(total))
        k = n_steps.value
        return {"n_sigma": n_sigma.value, "compute_ms": buf[0][:k].tolist(), "transfer_ms": buf[1][:k].tolist(),
                "exposed_ms": buf[2][:k].tolist(), "total_ms": total.value}


class DistributedApplier:
    """One rank of the alpha-block partitioned y = H x (reference ``distsim.py:130-316``).

    Call on every rank of an initialised ``torch.distributed`` group (any
    backend: it only carries the NCCL unique id at setup and the
    reference-protocol gathers; the per-sigma traffic is the library's own
    NCCL communicator).  ``overlap=False`` makes every alpha pass wait for
    the whole exchange (one group); ``transfer_delay`` has no device analogue
    and must be 0.  ``exchange``: "auto" (sparse when the referenced fraction
    of remote rows is at most ``sparse_threshold``), "allgather"/"dense" or
    "sparse"; ``group_steps``: ring steps per pipelined alpha pass.
    """

    def __init__(self, basis, table, tables=None, partition: Optional[Partition] = None, n_workers: Optional[int] = None,
                 overlap: bool = True, transfer_delay: float = 0.0, group=None, device=None, _rank_engine=None,
                 exchange: str = "auto", sparse_threshold: float = 0.6, group_steps: int = 2):
        import torch

        if basis.mode != "product":
            raise ValueError("distributed application requires a product-mode basis")
        if transfer_delay < 0:
            raise ValueError("transfer_delay must be >= 0")
        if transfer_delay:
            raise ValueError("transfer_delay is a simulation knob; the B200 path uses real NVLink transfers")
        if exchange not in _EXCHANGE:
            raise ValueError(f"exchange must be 'auto', 'allgather', 'dense' or 'sparse', got {exchange!r}")
        if group_steps < 1:
            raise ValueError("group_steps must be >= 1")
        self.comm = Comm(group)
        world = self.comm.world
        if n_workers is not None and n_workers != world:
            raise PartitionError(f"n_workers={n_workers} but the process group has {world} ranks")
        self.partition = make_partition(len(basis.alpha_strings), world) if partition is None else partition
        if self.partition.n_workers != world:
            raise PartitionError("partition size must equal the number of ranks")
        self.basis, self.table, self.overlap = basis, table, overlap
        self.n = basis.dimension
        self.n_beta = len(basis.beta_strings)
        self.rank = self.comm.rank
        self.lo, self.hi = self.partition.block_of(self.rank)
        self.n_own = (self.hi - self.lo) * self.n_beta
        self.apply_count = 0
        self.group_steps = group_steps if overlap else max(world - 1, 1)
        if _rank_engine is not None:  # CPU twin of the schedule (tests): torch.distributed ring in Python
            self.native = False
            self.engine = _rank_engine(basis, table, self.lo, self.hi)
            self.device = self.engine.device
            self.diag_local = self.engine.diag
            self.exchange = "dense"
            return
        self.native = True
        if device is None:
            device = torch.cuda.current_device()
        self.engine = _NativeRank(basis, table, self.comm, self.partition, device, exchange, sparse_threshold,
                                  self.group_steps)
        self.device = self.engine.device
        self.diag_local = self.engine.diag
        info = self.engine.info() if world > 1 else {"sparse": 0, "needed_fraction": 1.0, "recv_rows": 0}
        self.exchange = "sparse" if info["sparse"] == 1 else "dense"
        self.sparse_fraction = float(info["needed_fraction"])
        self.remote_rows_needed = int(info["recv_rows"])
        self.remote_rows_total = int(self.partition.alpha_blocks[-1][1] - (self.hi - self.lo))

    # -- device-resident path -----------------------------------------------------
    def apply_device(self, x_own, y_own=None):
        """sigma rows of this rank from this rank's rows of x (both device tensors)."""
        import torch

        if x_own.numel() != self.n_own:
            raise ValueError(f"expected {self.n_own} local amplitudes, got {x_own.numel()}")
        y = torch.empty(self.n_own, dtype=torch.float64, device=self.device) if y_own is None else y_own
        if y.numel() != self.n_own or y.dtype != torch.float64:
            raise ValueError(f"out must be a float64 tensor of {self.n_own} elements")
        self.apply_count += 1
        if self.native:
            x_own = x_own.contiguous()
            self.engine.sigma(x_own, y)
        else:
            self._ring_twin(x_own, y)
        return y

    def _ring_twin(self, x_own, y):
        """CPU twin of sbd_sigma_dist: own block first, then ring step s brings the block of (r - s) mod P."""
        import torch

        P, r, nb = self.comm.world, self.rank, self.n_beta
        blocks = self.partition.alpha_blocks
        self.engine.sigma_block(x_own, self.rank, y, first=True)
        held = x_own
        for s in range(1, P):
            frm = (r - s) % P
            a, b = blocks[frm]
            recv = torch.empty((b - a) * nb, dtype=torch.float64, device=self.device)
            self.comm.sendrecv(x_own, (r + s) % P, recv, frm)
            held = recv
            self.engine.sigma_block(held, frm, y, first=False)

    # -- reference protocol ---------------------------------------------------------
    def apply(self, x) -> np.ndarray:
        import torch

        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {x.shape}")
        nb = self.n_beta
        x_own = torch.from_numpy(np.ascontiguousarray(x[self.lo * nb:self.hi * nb])).to(self.device)
        y_own = self.apply_device(x_own)
        y_full = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self.comm.allgather_blocks(y_full, y_own, self.partition.alpha_blocks, nb)
        return y_full.cpu().numpy()

    __call__ = apply

    # -- overlap accounting (reference overlap_stats) ------------------------------
    def profile(self, on: bool = True) -> None:
        """Record per-step compute / transfer / exposed device times of every following sigma."""
        if self.native and self.comm.world > 1:
            self.engine.set_profiling(on)

    def step_records(self) -> dict:
        return self.engine.step_record() if (self.native and self.comm.world > 1) else {
            "n_sigma": 0, "compute_ms": [], "transfer_ms": [], "exposed_ms": [], "total_ms": 0.0}

    def overlap_report(self) -> OverlapReport:
        """Collective: every rank's step records, aggregated (reference ``overlap_stats``)."""
        recs = self.comm.allgather_object(self.step_records())
        recs = [r for r in recs if r["compute_ms"]]
        if not recs:
            return OverlapReport(self.comm.world, 0, self.overlap, 0.0, [], 0.0, 0.0, 0.0, 1.0)
        return overlap_stats(recs, self.overlap)

    # -- partitioned Davidson -------------------------------------------------------
    def global_argmin_start(self):
        """x0 = e_{argmin diag} over all ranks (reference davidson.py:219-221), local slice."""
        import torch

        d = self.diag_local
        loc_min = float(torch.min(d).item()) if d.numel() else float("inf")
        loc_idx = int(torch.argmin(d).item()) + self.lo * self.n_beta if d.numel() else self.n
        t = torch.tensor([loc_min], dtype=torch.float64, device=self.device)
        self.comm.allreduce(t, self.comm.dist.ReduceOp.MIN)
        gmin = float(t.item())
        cand = torch.tensor([float(loc_idx if loc_min == gmin else self.n)], dtype=torch.float64, device=self.device)
        self.comm.allreduce(cand, self.comm.dist.ReduceOp.MIN)
        gidx = int(cand.item())
        x0 = torch.zeros(self.n_own, dtype=torch.float64, device=self.device)
        if self.lo * self.n_beta <= gidx < self.hi * self.n_beta:
            x0[gidx - self.lo * self.n_beta] = 1.0
        return x0

    def davidson(self, x0=None, opts=None):
        """Lowest eigenpairs with V/W row-partitioned across ranks; vectors returned as local slices.

        Native ranks run the C++ control loop (``sbd_davidson`` on the partitioned context, NCCL
        all-reduces inside the library); the CPU twin runs the Python loop with torch all-reduces.
        """
        import torch

        from .davidson import DavidsonOptions, _solve_native, davidson_solve

        x0_local = None
        if x0 is not None:
            xa = x0 if isinstance(x0, torch.Tensor) else torch.from_numpy(np.asarray(x0, dtype=np.float64))
            xa = xa.reshape(-1)
            nb = self.n_beta
            x0_local = xa[self.lo * nb:self.hi * nb] if xa.numel() == self.n else xa
            x0_local = x0_local.to(self.device, dtype=torch.float64)
        if self.native:
            opts = DavidsonOptions() if opts is None else opts
            if opts.n_roots > self.n:
                raise ValueError(f"cannot extract {opts.n_roots} roots from dimension {self.n}")
            with torch.cuda.device(self.device):
                res = _solve_native(self.engine.context, self.n_own, self.diag_local, x0_local, opts, self.device,
                                    True)
            self.apply_count += res.stats.n_applies
            return res
        if x0_local is None:
            x0_local = self.global_argmin_start()

        def op(x_dev, y_dev):
            self.apply_device(x_dev, y_dev)

        return davidson_solve(op, self.diag_local, x0=x0_local, opts=opts, device=self.device.index,
                              return_device=True, allreduce=self.comm.allreduce,
                              rank_offset=self.lo * self.n_beta, ctx=getattr(self.engine, "context", None))
