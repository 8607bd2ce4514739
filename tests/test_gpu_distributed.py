"""Partitioned path with the real CUDA kernels and the library's own NCCL: 2-4 ranks on ONE GPU.

Only one GPU is available per test box, so the ranks share cuda:0.  NCCL
refuses two ranks on one device of one host, so every rank claims its own
NCCL_HOSTID: NCCL then sees separate hosts and runs its socket transport over
loopback (slow, but the same communicator calls, grouped send/recv ring steps,
all-reduces and stream/event ordering as on NVLink).  This exercises the
native partitioned sigma (sbd_dist_init / sbd_dist_plan / sbd_sigma_dist:
exchange plan, x_work remap, pipelined alpha passes, additive task 0) and the
native partitioned Davidson (sbd_davidson with all-reduced dot products).
torch.distributed (gloo) only carries the NCCL unique id and the
reference-protocol gathers.  Mirrors the reference's P-invariance contract
(test_distsim.py:76-81, test_cli.py:131-140).
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


def share_gpu_nccl_env(rank: int) -> None:
    """Let several NCCL ranks share one GPU (test boxes have one): distinct host ids, socket transport."""
    os.environ.update(NCCL_HOSTID=f"sbd-test-rank-{rank}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")


def _worker(rank, world, port, case, q, kw, env):
    try:
        import sys

        import torch
        import torch.distributed as dist

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        os.environ.update(env)
        share_gpu_nccl_env(rank)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from paper_2601_16637_b200 import DavidsonOptions
        from paper_2601_16637_b200.distributed import DistributedApplier
        from paper_2601_16637_b200.synth import random_integrals, random_product_basis

        norb, na, nb, nsa, nsb, seed, nroots = case
        table = random_integrals(norb, seed)
        basis = random_product_basis(norb, na, nb, nsa, nsb, seed + 1)
        dapp = DistributedApplier(basis, table, device=0, **kw)
        assert dapp.native
        dapp.profile(True)
        x = np.random.default_rng(seed).standard_normal(basis.dimension)
        y = dapp(x)
        y2 = dapp(x)
        rep = dapp.overlap_report()
        res = dapp.davidson(opts=DavidsonOptions(n_roots=nroots, max_subspace=16, restart_keep=4))
        info = dapp.engine.info()
        q.put((rank, y, res.energies, res.stats.iterations, res.converged, dapp.lo, dapp.hi,
               res.vectors.cpu().numpy(), np.array_equal(y, y2), dapp.exchange, info, rep))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, "error", traceback.format_exc()))


CASES = [
    # world, (norb, na, nb, n_alpha, n_beta, seed, n_roots), applier kwargs, env
    (2, (10, 5, 5, 60, 50, 3, 1), dict(exchange="dense"), {}),
    (3, (12, 4, 5, 100, 91, 4, 2), dict(exchange="dense", group_steps=1), {}),   # odd n_beta: scalar kernels
    (3, (12, 4, 5, 100, 91, 4, 2), dict(exchange="sparse"), {}),
    (2, (16, 4, 4, 300, 40, 5, 1), dict(exchange="auto"), {}),                      # auto -> sparse
    (4, (12, 5, 5, 120, 64, 6, 1), dict(exchange="dense", group_steps=2), {}),     # groups {1,2},{3}
    (4, (12, 5, 5, 120, 64, 6, 1), dict(exchange="sparse", overlap=False), {}),    # one group
    (3, (12, 4, 5, 100, 92, 4, 2), dict(exchange="dense"), {"SBD_CROSS_UNSTAGED": "1"}),  # flat task-0 kernel
]


@pytest.mark.parametrize("world,case,kw,env", CASES)
def test_partitioned_sigma_and_davidson_match_single_gpu(world, case, kw, env, monkeypatch):
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, davidson_solve
    from paper_2601_16637_b200.synth import random_integrals, random_product_basis

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, kw, env)) for r in range(world)]
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
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    app = HamiltonianApplier(basis, table)
    x = np.random.default_rng(seed).standard_normal(basis.dimension)
    ref = app(x)
    import oracle as O  # the gathered partitioned sigma against the CPU restatement too, not only the 1-GPU path

    inst = O.Instance.make(norb, table.h, table.eri, table.e_core, basis.alpha_array(), basis.beta_array())
    ref_o = O.sigma(inst, x)
    assert np.abs(ref - ref_o).max() <= 1e-10 * np.abs(ref_o).max()
    single = davidson_solve(app, app.diag, opts=DavidsonOptions(n_roots=nroots, max_subspace=16, restart_keep=4))
    vec = np.zeros((len(single.energies), basis.dimension))
    for rank, y, e, it, conv, lo, hi, v, determ, exch, info, rep in out:
        want_sparse = kw.get("exchange") == "sparse" or (kw.get("exchange") == "auto"
                                                          and info["needed_fraction"] <= 0.6)
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()   # P-invariance
        assert np.abs(y - ref_o).max() <= 1e-10 * np.abs(ref_o).max()  # parity with the oracle
        assert determ                                               # repeated sigma: bitwise equal
        assert exch == ("sparse" if want_sparse else "dense")
        assert info["nranks"] == world and (info["alpha_lo"], info["alpha_hi"]) == (lo, hi)
        if not want_sparse:  # dense plans receive every remote row
            assert info["recv_rows"] == nsa - (hi - lo)
        else:
            assert info["recv_rows"] <= nsa - (hi - lo)
        assert conv
        np.testing.assert_allclose(e, single.energies, atol=1e-10)
        assert abs(it - single.stats.iterations) <= 1
        vec[:, lo * nsb:hi * nsb] = v
        # overlap accounting: local step + one row per group, two profiled sigmas
        ng = 1 if kw.get("overlap") is False else -(-(world - 1) // kw.get("group_steps", 2))
        assert rep.n_steps == ng + 1 and rep.n_sigma == 2
        assert all(row[1] >= 0 and row[2] >= 0 and row[3] >= 0 for row in rep.per_step)
        assert 0.0 <= rep.overlap_ratio <= 1.0 and rep.sigma_s > 0
    for j in range(len(single.energies)):  # gathered Ritz vectors are eigenvectors
        u = vec[j]
        assert np.linalg.norm(u) == pytest.approx(1.0, abs=1e-9)
        assert np.linalg.norm(app(u) - single.energies[j] * u) <= 1e-7
