"""Partitioned path with the real CUDA kernels: 2-3 ranks sharing one GPU (gloo).

Only one GPU is available per test box, so ranks share cuda:0 and talk over
gloo (CUDA tensors are staged through host by distributed.Comm).  This
exercises everything rank-specific on the device: row windows, the split
sbd_sigma_local / sbd_sigma_remote, the all-gather into x_full, and the
row-partitioned Davidson with all-reduced dot products.  Mirrors the
reference's P-invariance contract (test_distsim.py:76-81, test_cli.py:131-140).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q, exchange="auto"):
    try:
        import sys

        import torch
        import torch.distributed as dist

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from paper_2601_16637_b200 import DavidsonOptions
        from paper_2601_16637_b200.distributed import DistributedApplier
        from paper_2601_16637_b200.synth import random_integrals, random_product_basis

        norb, na, nb, nsa, nsb, seed, nroots = case
        table = random_integrals(norb, seed)
        basis = random_product_basis(norb, na, nb, nsa, nsb, seed + 1)
        dapp = DistributedApplier(basis, table, device=0, exchange=exchange)
        if exchange == "sparse":  # rows a rank does not receive must never be read
            assert dapp.exchange == "sparse"
            dapp._x_full.fill_(float("nan"))
        x = np.random.default_rng(seed).standard_normal(basis.dimension)
        y = dapp(x)
        res = dapp.davidson(opts=DavidsonOptions(n_roots=nroots, max_subspace=16, restart_keep=4))
        q.put((rank, y, res.energies, res.stats.iterations, res.converged, dapp.lo, dapp.hi,
               res.vectors.cpu().numpy()))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world,case,exchange,order", [(2, (10, 5, 5, 60, 50, 3, 1), "allgather", "auto"),
                                                       (3, (12, 4, 5, 100, 91, 4, 2), "allgather", "auto"),
                                                       (3, (12, 4, 5, 100, 91, 4, 2), "sparse", "auto"),
                                                       (2, (16, 4, 4, 300, 40, 5, 1), "sparse", "auto"),
                                                       (3, (12, 4, 5, 100, 91, 4, 2), "allgather", "additive")])
def test_partitioned_sigma_and_davidson_match_single_gpu(world, case, exchange, order, monkeypatch):
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, davidson_solve
    from paper_2601_16637_b200.synth import random_integrals, random_product_basis

    if order == "additive":  # task 0 added after the alpha side on every rank's row window
        monkeypatch.setenv("SBD_CROSS_ADD", "1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert not isinstance(o[1], str), o[2]
    norb, na, nb, nsa, nsb, seed, nroots = case
    table = random_integrals(norb, seed)
    basis = random_product_basis(norb, na, nb, nsa, nsb, seed + 1)
    app = HamiltonianApplier(basis, table)
    x = np.random.default_rng(seed).standard_normal(basis.dimension)
    ref = app(x)
    single = davidson_solve(app, app.diag, opts=DavidsonOptions(n_roots=nroots, max_subspace=16, restart_keep=4))
    vec = np.zeros((len(single.energies), basis.dimension))
    for rank, y, e, it, conv, lo, hi, v in out:
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()   # P-invariance
        assert conv
        np.testing.assert_allclose(e, single.energies, atol=1e-10)
        assert abs(it - single.stats.iterations) <= 1
        vec[:, lo * nsb:hi * nsb] = v
    for j in range(len(single.energies)):  # gathered Ritz vectors are eigenvectors
        u = vec[j]
        assert np.linalg.norm(u) == pytest.approx(1.0, abs=1e-9)
        assert np.linalg.norm(app(u) - single.energies[j] * u) <= 1e-7
