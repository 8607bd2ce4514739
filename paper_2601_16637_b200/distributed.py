"""Alpha-block partitioned sigma and Davidson over GPUs (reference ``distsim.py``).

The reference simulates P workers with Python threads passing ket blocks
around a ring (``distsim.py:200-259``).  Here each rank is one process on one
GPU (``torch.distributed``, NCCL over NVLink/NVSwitch):

* partition: contiguous alpha blocks, the first ``rem`` blocks one row longer
  (``make_partition``, ``distsim.py:63-77``); rank r owns x, sigma, diag, V and
  W rows ``[lo_r, hi_r) x n_beta``;
* per sigma, ONE exchange: an all-gather of the trial vector's blocks
  (NVSwitch gives every peer full bandwidth, so no ring is needed), launched
  first on NCCL's stream while the compute stream runs the beta-beta part
  from the rank's own rows (``sbd_sigma_local``); the alpha-alpha and
  alpha-beta parts (``sbd_sigma_remote``) start once the gather lands;
* Davidson: vectors stay row-partitioned; the O(k) dot products of every
  fused pass are all-reduced (a few hundred bytes per iteration).
* sparse exchange (the successor of the reference ring): a rank
  only reads the x rows its own rows connect to.  When those are a minority
  of the remote rows (cfg4: ~40%), the all-gather is replaced by grouped
  point-to-point transfers of exactly the referenced rows (request lists are
  exchanged once at construction; each sigma packs, sends, receives and
  scatters rows), cutting the per-sigma NVLink volume in proportion.

``DistributedApplier(...).apply(x)`` keeps the reference signature (full
numpy x on every rank in, full y out).  The device-resident path is
``apply_device`` / ``davidson``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = ["Partition", "PartitionError", "make_partition", "DistributedApplier", "Comm"]


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


class Comm:
    """Collectives used by the partitioned path; NCCL native, gloo staged through host."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _staged(self, t) -> bool:
        return self.backend == "gloo" and t.is_cuda

    def allreduce(self, t) -> None:
        if self.world == 1:
            return
        if self._staged(t):
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)

    def allgather_start(self, views, local):
        """Start gathering ``local`` of every rank into ``views``; returns a waitable."""
        if self.world == 1:
            views[0].copy_(local)
            return None
        if self.backend == "gloo":
            # gloo all_gather needs equal sizes: pad every block to the longest
            import torch

            mx = max(v.numel() for v in views)
            send = torch.zeros(mx, dtype=local.dtype)
            send[: local.numel()] = local.cpu()
            recv = [torch.empty(mx, dtype=local.dtype) for _ in views]
            self.dist.all_gather(recv, send, group=self.group)
            for v, h in zip(views, recv):
                v.copy_(h[: v.numel()])
            return None
        return self.dist.all_gather(views, local, group=self.group, async_op=True)

    def barrier(self) -> None:
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange_rows(self, sends: dict, recvs: dict):
        """Point-to-point transfers {peer: tensor}; returns a list of waitables (empty when staged)."""
        if self.backend == "gloo":  # gloo: host-staged, blocking
            import torch

            ops, host_recv = [], {}
            for p, t in sends.items():
                ops.append(self.dist.isend(t.cpu(), self._global(p), group=self.group))
            for p, t in recvs.items():
                host_recv[p] = torch.empty(t.shape, dtype=t.dtype)
                ops.append(self.dist.irecv(host_recv[p], self._global(p), group=self.group))
            for op in ops:
                op.wait()
            for p, t in recvs.items():
                t.copy_(host_recv[p])
            return []
        ops = [self.dist.P2POp(self.dist.isend, t, self._global(p), group=self.group) for p, t in sends.items()]
        ops += [self.dist.P2POp(self.dist.irecv, t, self._global(p), group=self.group) for p, t in recvs.items()]
        return self.dist.batch_isend_irecv(ops) if ops else []

    def _global(self, rank: int) -> int:
        return rank if self.group is None else self.dist.get_global_rank(self.group, rank)


class _CudaRank:
    """This rank's slice of the operator on its GPU (a row-windowed HamiltonianApplier)."""

    def __init__(self, basis, table, lo, hi, device):
        from .apply import HamiltonianApplier

        self.app = HamiltonianApplier(basis, table, row_window=(lo, hi), device=device)
        self.device = self.app._torch_device
        self.diag = self.app.diag_device

    def sigma_local(self, x_own):
        from . import _lib

        self.app.context.bind_stream()
        self.app.context("sbd_sigma_local", _lib.ptr(x_own))

    def sigma_remote(self, x_full, y_own):
        from . import _lib

        self.app.context.bind_stream()
        self.app.context("sbd_sigma_remote", _lib.ptr(x_full), _lib.ptr(y_own))

    @property
    def context(self):
        return self.app.context

    def alpha_targets(self, lo, hi):
        """Alpha rows that rows [lo, hi) connect to (singles and doubles, in-set)."""
        t = self.app.tables.alpha
        parts = [t.s_tgt[t.s_off[lo]:t.s_off[hi]], t.d_tgt[t.d_off[lo]:t.d_off[hi]]]
        return np.unique(np.concatenate(parts).astype(np.int64))


class DistributedApplier:
    """One rank of the alpha-block partitioned y = H x (reference ``distsim.py:130-316``).

    Call on every rank of an initialised ``torch.distributed`` group.
    ``overlap`` keeps its reference meaning (communication overlapped with
    local work); ``transfer_delay`` has no device analogue and must be 0.
    """

    def __init__(self, basis, table, tables=None, partition: Optional[Partition] = None, n_workers: Optional[int] = None,
                 overlap: bool = True, transfer_delay: float = 0.0, group=None, device=None, _rank_engine=None,
                 exchange: str = "auto", sparse_threshold: float = 0.6):
        import torch

        if basis.mode != "product":
            raise ValueError("distributed application requires a product-mode basis")
        if transfer_delay < 0:
            raise ValueError("transfer_delay must be >= 0")
        if transfer_delay:
            raise ValueError("transfer_delay is a simulation knob; the B200 path uses real NVLink transfers")
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
        if _rank_engine is not None:
            self.engine = _rank_engine(basis, table, self.lo, self.hi)
        else:
            if device is None:
                device = torch.cuda.current_device()
            self.engine = _CudaRank(basis, table, self.lo, self.hi, device)
        self.device = self.engine.device
        self.diag_local = self.engine.diag
        self._x_full = torch.empty(self.n, dtype=torch.float64, device=self.device)
        nb = self.n_beta
        self._views = [self._x_full[a * nb:b * nb] for a, b in self.partition.alpha_blocks]
        self.apply_count = 0
        if exchange not in ("auto", "allgather", "sparse"):
            raise ValueError(f"exchange must be 'auto', 'allgather' or 'sparse', got {exchange!r}")
        self.exchange = "allgather"
        self.remote_rows_needed = 0
        if world > 1 and exchange != "allgather":
            self._plan_sparse(exchange, sparse_threshold)

    # -- sparse row exchange ------------------------------------------
    def _plan_sparse(self, exchange, threshold):
        import torch

        blocks = self.partition.alpha_blocks
        need = self.engine.alpha_targets(self.lo, self.hi)
        need = need[(need < self.lo) | (need >= self.hi)]
        owner = np.searchsorted(np.array([b for _, b in blocks]), need, side="right")
        req = {int(p): need[owner == p] for p in np.unique(owner)}
        everyone = self.comm.allgather_object(req)  # setup only: who needs which of my rows
        n_alpha = blocks[-1][1]
        # the decision must be the same on every rank: the largest needed fraction decides
        frac = max(sum(v.size for v in r.values()) / max(n_alpha - (b - a), 1) for r, (a, b) in zip(everyone, blocks))
        self.remote_rows_needed = int(need.size)
        self.remote_rows_total = int(n_alpha - (self.hi - self.lo))
        self.sparse_fraction = float(frac)
        if exchange == "auto" and frac > threshold:
            return  # dense enough: the all-gather moves about as much and is one collective
        dev = self.device
        nb = self.n_beta
        self._recv_rows = {p: torch.from_numpy(rows).to(dev) for p, rows in req.items() if rows.size}
        self._recv_buf = {p: torch.empty((rows.numel(), nb), dtype=torch.float64, device=dev)
                          for p, rows in self._recv_rows.items()}
        self._send_rows = {}
        for q, r in enumerate(everyone):
            if q != self.rank and self.rank in r and r[self.rank].size:
                self._send_rows[q] = torch.from_numpy(r[self.rank] - self.lo).to(dev)
        self._send_buf = {q: torch.empty((rows.numel(), nb), dtype=torch.float64, device=dev)
                          for q, rows in self._send_rows.items()}
        self.exchange = "sparse"

    def _sparse_start(self, x_own):
        nb = self.n_beta
        xo = x_own.view(-1, nb)
        for q, rows in self._send_rows.items():
            self._send_buf[q].copy_(xo.index_select(0, rows))
        return self.comm.exchange_rows(self._send_buf, self._recv_buf)

    def _sparse_finish(self, x_own, works):
        for w in works:
            w.wait()
        xf = self._x_full.view(-1, self.n_beta)
        for p, rows in self._recv_rows.items():
            xf.index_copy_(0, rows, self._recv_buf[p])
        self._views[self.rank].copy_(x_own)

    # -- device-resident path -----------------------------------------------------
    def apply_device(self, x_own, y_own=None):
        """sigma rows of this rank from this rank's rows of x (both device tensors)."""
        import torch

        if x_own.numel() != self.n_own:
            raise ValueError(f"expected {self.n_own} local amplitudes, got {x_own.numel()}")
        y = torch.empty(self.n_own, dtype=torch.float64, device=self.device) if y_own is None else y_own
        self.apply_count += 1
        if self.exchange == "sparse":
            works = self._sparse_start(x_own)                      # NCCL p2p, referenced rows only
            if self.overlap:
                self.engine.sigma_local(x_own)                     # compute stream, concurrently
                self._sparse_finish(x_own, works)
            else:
                self._sparse_finish(x_own, works)
                self.engine.sigma_local(x_own)
            self.engine.sigma_remote(self._x_full, y)
            return y
        if self.overlap:
            work = self.comm.allgather_start(self._views, x_own)  # NCCL stream
            self.engine.sigma_local(x_own)                         # compute stream, concurrently
            if work is not None:
                work.wait()
        else:
            work = self.comm.allgather_start(self._views, x_own)
            if work is not None:
                work.wait()
            self.engine.sigma_local(x_own)
        self.engine.sigma_remote(self._x_full, y)
        return y

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
        views = [y_full[a * nb:b * nb] for a, b in self.partition.alpha_blocks]
        w = self.comm.allgather_start(views, y_own)
        if w is not None:
            w.wait()
        return y_full.cpu().numpy()

    __call__ = apply

    # -- partitioned Davidson -------------------------------------------------------
    def global_argmin_start(self):
        """x0 = e_{argmin diag} over all ranks (reference davidson.py:219-221), local slice."""
        import torch

        d = self.diag_local
        loc_min = float(torch.min(d).item()) if d.numel() else float("inf")
        loc_idx = int(torch.argmin(d).item()) + self.lo * self.n_beta if d.numel() else self.n
        # lexicographic (value, global index) minimum via two all-reduces
        t = torch.tensor([loc_min], dtype=torch.float64, device=self.device)
        neg = -t
        self._allreduce_max(neg)
        gmin = -float(neg.item())
        cand = torch.tensor([float(loc_idx if loc_min == gmin else self.n)], dtype=torch.float64, device=self.device)
        negc = -cand
        self._allreduce_max(negc)
        gidx = int(-negc.item())
        x0 = torch.zeros(self.n_own, dtype=torch.float64, device=self.device)
        if self.lo * self.n_beta <= gidx < self.hi * self.n_beta:
            x0[gidx - self.lo * self.n_beta] = 1.0
        return x0

    def _allreduce_max(self, t):
        if self.comm.world == 1:
            return
        if self.comm._staged(t):
            h = t.cpu()
            self.comm.dist.all_reduce(h, op=self.comm.dist.ReduceOp.MAX, group=self.comm.group)
            t.copy_(h)
        else:
            self.comm.dist.all_reduce(t, op=self.comm.dist.ReduceOp.MAX, group=self.comm.group)

    def davidson(self, x0=None, opts=None):
        """Lowest eigenpairs with V/W row-partitioned across ranks; vectors returned as local slices."""
        from .davidson import davidson_solve

        if x0 is None:
            x0_local = self.global_argmin_start()
        else:
            import torch

            xa = x0 if isinstance(x0, torch.Tensor) else torch.from_numpy(np.asarray(x0, dtype=np.float64))
            xa = xa.reshape(-1)
            nb = self.n_beta
            x0_local = xa[self.lo * nb:self.hi * nb] if xa.numel() == self.n else xa
            x0_local = x0_local.to(self.device, dtype=torch.float64)

        def op(x_dev, y_dev):
            self.apply_device(x_dev, y_dev)

        return davidson_solve(op, self.diag_local, x0=x0_local, opts=opts, device=self.device.index,
                              return_device=True, allreduce=self.comm.allreduce,
                              rank_offset=self.lo * self.n_beta, ctx=getattr(self.engine, "context", None))
