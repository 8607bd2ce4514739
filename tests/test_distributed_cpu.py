"""Multi-process (gloo, CPU) tests of the alpha-block partitioned path's host logic.

Each rank's device engine is replaced by the CPU oracle (test infrastructure),
which makes DistributedApplier run the CPU twin of the native schedule: the
own block first (diag, beta side, alpha terms into the own rows), then ring
step s brings the block of (r - s) mod P and its alpha terms are added
(y +=), exactly the pass order of sbd_sigma_dist.  Everything else --
make_partition, the ring's neighbour pattern, the padded all_gather of the
y blocks for the reference-protocol apply(), the global argmin start vector --
is the product code (paper_2601_16637_b200/distributed.py).  Mirrors the
reference's P-invariance tests (test_distsim.py:69-81).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleRank:
    """Stand-in for _CudaRank: the same sigma rows, computed by the CPU oracle."""

    def __init__(self, basis, table, lo, hi):
        import oracle as O

        self.O = O
        self.inst = O.Instance.make(basis.norb, table.h, table.eri, table.e_core, basis.alpha_array(),
                                    basis.beta_array())
        self.lo, self.hi = lo, hi
        self.device = torch.device("cpu")
        self.diag = torch.from_numpy(O.diag(self.inst, (lo, hi)))
        self.local_calls = 0

    def sigma_block(self, x_block, q, y_own, first):
        """Contribution of ket block q (the reference ring's per-step product, ket window = block q)."""
        from paper_2601_16637_b200.distributed import make_partition

        a, b = make_partition(self.inst.alpha.size, self.world).block_of(q)
        part = self.O.sigma(self.inst, x_block.numpy(), bra=(self.lo, self.hi), ket=(a, b))
        if first:
            self.local_calls += 1
            y_own.copy_(torch.from_numpy(part))
        else:
            y_own.add_(torch.from_numpy(part))


def _worker(rank, world, port, case, q):
    try:
        import sys

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "oracle"))
        sys.path.insert(0, os.path.join(root, "tests"))
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from paper_2601_16637_b200.distributed import DistributedApplier
        from paper_2601_16637_b200.synth import random_integrals, random_product_basis

        norb, na, nb, nsa, nsb, seed = case
        table = random_integrals(norb, seed)
        basis = random_product_basis(norb, na, nb, nsa, nsb, seed + 1)
        OracleRank.world = world
        dapp = DistributedApplier(basis, table, _rank_engine=OracleRank)
        x = np.random.default_rng(seed).standard_normal(basis.dimension)
        y = dapp(x)
        assert dapp.exchange == "dense" and not dapp.native
        x0 = dapp.global_argmin_start()
        dist.barrier()
        q.put((rank, dapp.lo, dapp.hi, y, x0.numpy(), dapp.engine.local_calls))
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        import traceback

        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case", [
    (2, (8, 4, 3, 30, 25, 3)),   # even-ish split
    (3, (8, 4, 4, 31, 20, 5)),   # uneven alpha blocks (11, 10, 10)
    (2, (6, 3, 3, 3, 20, 7)),    # tiny alpha sector
    (4, (12, 4, 4, 60, 20, 9)),  # sparse connectivity: ranks need a fraction of the remote rows
])
def test_partitioned_apply_matches_serial(world, case):
    import oracle as O

    from paper_2601_16637_b200.distributed import make_partition
    from paper_2601_16637_b200.synth import random_integrals, random_product_basis

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for o in out:
        assert not isinstance(o[1], str), o[2]
    norb, na, nb, nsa, nsb, seed = case
    table = random_integrals(norb, seed)
    basis = random_product_basis(norb, na, nb, nsa, nsb, seed + 1)
    inst = O.Instance.make(norb, table.h, table.eri, table.e_core, basis.alpha_array(), basis.beta_array())
    x = np.random.default_rng(seed).standard_normal(basis.dimension)
    ref = O.sigma(inst, x)
    part = make_partition(nsa, world)
    d = O.diag(inst)
    gidx = int(np.argmin(d))
    nbeta = nsb
    for rank, lo, hi, y, x0, local_calls in out:
        assert (lo, hi) == part.block_of(rank)
        # every rank returns the full, gathered y (reference DistributedApplier.apply contract)
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
        assert local_calls == 1  # the own block (diag + beta side) is applied once per sigma
        # start vector: e_{global argmin diag}, sliced to the rank's rows
        want = np.zeros((hi - lo) * nbeta)
        if lo * nbeta <= gidx < hi * nbeta:
            want[gidx - lo * nbeta] = 1.0
        assert np.array_equal(x0, want)


def test_make_partition_semantics():
    from paper_2601_16637_b200.distributed import PartitionError, make_partition

    p = make_partition(10, 3)
    assert p.alpha_blocks == ((0, 4), (4, 7), (7, 10))  # first rem blocks one longer (distsim.py:63-77)
    assert make_partition(8, 8).alpha_blocks[-1] == (7, 8)
    with pytest.raises(PartitionError):
        make_partition(3, 4)
    with pytest.raises(PartitionError):
        make_partition(3, 0)
