"""Every dispatch variant of the Davidson passes and of the sigma kernels, against numpy / the oracle.

The passes (csrc/sbd_davidson.cu) pick a kernel by subspace size, alignment
and three knobs read per launch (register passes for k <= 32, TMA-staged
passes for k > 32 or SBD_DAV_TMA=1, tile/generic passes with SBD_NO_TMA=1 or
unaligned vectors; the streamed residual pass, or the register one with
SBD_RES_STREAM=0; lane splits SBD_RES_SPLIT / SBD_GS_SPLIT and L2 prefetch
SBD_RES_PF / SBD_GS_PF).  Each is checked here against a float64 numpy
restatement of the reference step it fuses (davidson.py:159-185,248-289).
The sigma variants (SBD_SIDE_LDG, SBD_YT_BLOCKED, SBD_CROSS_NO_CLUSTER,
SBD_CROSS_UNSTAGED, SBD_CROSS_ADD) are checked against the oracle and
against each other.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

VARIANTS = [
    {},
    {"SBD_DAV_TMA": "1"},
    {"SBD_NO_TMA": "1"},
    {"SBD_RES_STREAM": "0"},
    {"SBD_RES_SPLIT": "1", "SBD_GS_SPLIT": "1", "SBD_RES_STREAM": "0"},
    {"SBD_RES_SPLIT": "2", "SBD_GS_SPLIT": "2", "SBD_RES_STREAM": "0"},
    {"SBD_RES_SPLIT": "4", "SBD_RES_STREAM": "0"},
    {"SBD_RES_PF": "1", "SBD_GS_PF": "1", "SBD_RES_STREAM": "0"},
    {"SBD_GS_PF": "0"},
]


def _ctx():
    from paper_2601_16637_b200 import _lib

    return _lib.Context(0)


def _setup(k, m, n, seed, offset):
    """V, W (k x ld) with ld even; `offset` doubles shift the base pointers (offset 1: unaligned)."""
    import torch

    rng = np.random.default_rng(seed)
    ld = (n + 31) // 32 * 32
    dev = torch.device("cuda", 0)

    def mat(rows):
        buf = torch.zeros(rows * ld + 2, dtype=torch.float64, device=dev)
        view = buf[offset:offset + rows * ld].view(rows, ld)
        view[:, :n] = torch.from_numpy(rng.standard_normal((rows, n)))
        return buf, view

    vb, V = mat(k)
    wb, W = mat(k)
    Y = torch.from_numpy(rng.standard_normal((k, m))).to(dev)
    theta = torch.from_numpy(rng.standard_normal(m)).to(dev)
    diag = torch.zeros(n + 2, dtype=torch.float64, device=dev)
    dview = diag[offset:offset + n]
    dview.copy_(torch.from_numpy(rng.standard_normal(n) * 2.0))
    dview[::97] = theta[0]  # d - theta == 0 exactly: the sign(0) = +1 branch with the delta floor
    return ld, vb, V, wb, W, Y, theta, diag, dview


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("k,m,n,offset", [(1, 1, 1000, 0), (5, 2, 999, 0), (17, 3, 4097, 0), (24, 1, 3000, 0),
                                          (32, 5, 2048, 0), (40, 2, 1500, 0), (64, 8, 1200, 0), (20, 2, 777, 1),
                                          # several tiles per CTA: the streamed residual's stage ring wraps
                                          (16, 2, 300_001, 0), (12, 4, 200_003, 0), (3, 3, 1_000_001, 0)])
def test_davidson_passes_match_numpy(env, k, m, n, offset, monkeypatch):
    import torch

    from paper_2601_16637_b200 import _lib

    for key, val in env.items():
        monkeypatch.setenv(key, val)
    ctx = _ctx()
    ld, vb, V, wb, W, Y, theta, diag, dview = _setup(k, m, n, 11 * k + m, offset)
    Vn, Wn = _np(V)[:, :n], _np(W)[:, :n]
    Yn, thn, dn = _np(Y), _np(theta), _np(dview)
    dev = V.device
    p = _lib.ptr
    delta = 1e-3
    rtol = 1e-12

    def close(a, b, what):
        scale = max(np.abs(b).max(), 1e-300)
        assert np.abs(a - b).max() <= rtol * scale * 10, (what, np.abs(a - b).max() / scale)

    # vdots2: <V_i, w> and <V_i, u>
    w, u = Wn[0].copy(), Vn[k - 1].copy()
    wt = torch.from_numpy(w).to(dev)
    ut = torch.from_numpy(u).to(dev)
    out = torch.zeros(2 * k, dtype=torch.float64, device=dev)
    ctx("sbd_vdots2", p(V), k, ld, n, p(wt), p(ut), p(out))
    close(_np(out), np.concatenate([Vn @ w, Vn @ u]), "vdots2")

    # residual + preconditioner + projection of target root jp (davidson.py:252-258, 159-163)
    T = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    res = torch.zeros(k + 1 + m, dtype=torch.float64, device=dev)
    jp = m - 1
    ctx("sbd_residual_precond_target", p(V), p(W), k, ld, n, p(Y), p(theta), m, jp, p(dview), delta, p(T), ld,
        p(res))
    R = Yn.T @ Wn - thn[:, None] * (Yn.T @ Vn)
    dd = dn[None, :] - thn[:, None]
    den = np.where(dd >= 0, 1.0, -1.0) * np.maximum(np.abs(dd), delta)
    Tn = R / den
    close(_np(T)[:, :n], Tn, "residual t")
    resn = _np(res)
    close(resn[:k], Vn @ Tn[jp], "V^T t")
    close(resn[k:k + 1], np.array([Tn[jp] @ Tn[jp]]), "|t|^2")
    close(resn[k + 1:], (R * R).sum(axis=1), "|r|^2")

    # CGS pass with dots, pass without, fused finalize (davidson.py:166-185)
    c = torch.from_numpy(Vn @ Tn[jp]).to(dev)
    t = T[jp].clone()
    o2 = torch.zeros(k + 1, dtype=torch.float64, device=dev)
    ctx("sbd_gs_update", p(V), k, ld, n, p(c), p(t), p(o2))
    t1 = Tn[jp] - Vn.T @ _np(c)
    close(_np(t)[:n], t1, "gs t")
    close(_np(o2), np.concatenate([Vn @ t1, [t1 @ t1]]), "gs dots")
    c2 = torch.from_numpy(Vn @ t1).to(dev)
    t2 = t.clone()
    o1 = torch.zeros(1, dtype=torch.float64, device=dev)
    ctx("sbd_gs_update_nodots", p(V), k, ld, n, p(c2), p(t2), p(o1))
    t2n = t1 - Vn.T @ _np(c2)
    close(_np(t2)[:n], t2n, "gs nodots t")
    close(_np(o1), np.array([t2n @ t2n]), "gs nodots norm")
    scale = torch.tensor([0.5], dtype=torch.float64, device=dev)
    vout = torch.zeros(ld, dtype=torch.float64, device=dev)
    t3 = t.clone()
    ctx("sbd_gs_finalize", p(V), k, ld, n, p(c2), p(t3), p(vout), p(scale), p(o1))
    close(_np(vout)[:n], 0.5 * t2n, "finalize v")
    close(_np(o1), np.array([t2n @ t2n]), "finalize norm")

    # combine (Ritz vectors, davidson.py:256) and in-place thick-restart rotation (davidson.py:280-289)
    U = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    ctx("sbd_combine", p(V), k, ld, n, p(Y), m, p(U), ld)
    close(_np(U)[:, :n], Yn.T @ Vn, "combine")
    keep = min(k, 4)
    Yk = torch.from_numpy(np.ascontiguousarray(Yn[:, :1].repeat(keep, axis=1) + np.arange(keep))).to(dev)
    ctx("sbd_rotate", p(V), k, ld, n, p(Yk), keep)
    close(_np(V)[:keep, :n], _np(Yk).T @ Vn, "rotate")
    torch.cuda.synchronize()
    ctx.close()


@pytest.mark.parametrize("max_subspace", [48, 64])
def test_davidson_large_subspace_vs_oracle(max_subspace):
    """k in (32, 64]: the TMA-staged passes inside the full solver (native and Python control loops)."""
    from paper_2601_16637_b200 import DavidsonOptions, HamiltonianApplier, SelectedBasis, davidson_solve
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    norb, ne = 12, 5
    a, b = random_product_strings(norb, ne, ne, 300, 260, seed=3)
    table = random_integrals(norb, seed=4)
    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
    inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
    opts = DavidsonOptions(n_roots=3, max_subspace=max_subspace, restart_keep=6)
    ref = O.davidson(lambda v: O.sigma(inst, v), O.diag(inst), n_roots=3, max_subspace=max_subspace,
                     restart_keep=6)
    for native in (True, False):
        res = davidson_solve(app, app.diag, opts=opts, native=native)
        assert res.converged
        np.testing.assert_allclose(res.energies, ref.energies, atol=1e-8)
        assert abs(res.stats.iterations - ref.iterations) <= 2
        assert max(res.stats.ortho_history) <= 1e-10


SIGMA_VARIANTS = [
    {},
    {"SBD_SIDE_LDG": "1"},
    {"SBD_YT_BLOCKED": "0"},
    {"SBD_CROSS_NO_CLUSTER": "1"},
    {"SBD_CROSS_UNSTAGED": "1"},
    {"SBD_CROSS_ADD": "1"},
    {"SBD_CROSS_ADD": "0", "SBD_YT_BLOCKED": "0"},
    {"SBD_DENSE_GEMM": "1"},
    {"SBD_DENSE_GEMM": "1", "SBD_CROSS_ADD": "1"},
    {"SBD_DENSE_GEMM": "0"},
]


@pytest.mark.parametrize("env", SIGMA_VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_sigma_variants_vs_oracle(env, monkeypatch):
    """Each sigma kernel variant, device and host-buffer (pipelined) paths, even and odd n_beta."""
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    for key, val in env.items():
        monkeypatch.setenv(key, val)
    for norb, ne, nsa, nsb, seed in ((12, 6, 924, 130, 8), (12, 5, 600, 77, 9), (14, 4, 520, 1001, 10)):
        a, b = random_product_strings(norb, ne, ne, nsa, nsb, seed=seed)
        table = random_integrals(norb, seed=seed)
        app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
        inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
        x = np.random.default_rng(seed).standard_normal(app.n)
        ref = O.sigma(inst, x)
        yh = app(x)  # host buffers: pipelined chunks when eligible
        yd = app.sigma_device(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.abs(yh - ref).max() <= 1e-10 * np.abs(ref).max(), (norb, ne, nsa, nsb)
        assert np.abs(yd - ref).max() <= 1e-10 * np.abs(ref).max(), (norb, ne, nsa, nsb)


def test_dense_rows_match_oracle_elements():
    """sbd_dense_rows (verify's independent matrix) element by element against the oracle's _hij_words."""
    from paper_2601_16637_b200 import SelectedBasis
    from paper_2601_16637_b200.dense import assemble_dense
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    norb, ne = 10, 4
    a, b = random_product_strings(norb, ne, ne, 30, 25, seed=5)
    table = random_integrals(norb, seed=6)
    basis = SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne)
    dense = assemble_dense(basis, table)
    inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
    ref = O.dense(inst)
    assert np.abs(dense - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(dense, dense.T) or np.abs(dense - dense.T).max() <= 1e-14 * np.abs(dense).max()


@pytest.mark.parametrize("env", [{"SBD_CROSS_DCI": "1"}, {"SBD_CROSS_DCI": "1", "SBD_CROSS_ADD": "1"}],
                         ids=["dci", "dci-additive"])
def test_direct_ci_task0_vs_oracle(env, monkeypatch):
    """Task 0 as the fp64 tensor-core contraction (sbd_dci.cu), forced on every shape it serves:
    K not a multiple of 4, 1-8 beta positions per thread, 5-12 row fragments (norb 9-14), 4 and 9
    k-steps, partial last column tile, row windows, host (pipelined) and device paths."""
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    for key, val in env.items():
        monkeypatch.setenv(key, val)
    # (14, 7, 3), (16, 3, 8) and the 3000-string beta sectors are outside the shapes the kernel serves (49
    # alpha singles; 15 row fragments; gather block too wide for shared memory): the forced knob then
    # falls back to the SELL kernels, which must still agree
    cases = [(12, 6, 6, 924, 924, 1), (12, 5, 6, 500, 862, 2), (13, 4, 5, 300, 1286, 3), (14, 7, 3, 400, 364, 4),
             (16, 3, 8, 200, 3000, 5), (14, 3, 7, 200, 3000, 8), (9, 2, 3, 36, 84, 6), (12, 1, 11, 12, 12, 7),
             (10, 3, 3, 120, 120, 9), (11, 2, 2, 55, 54, 10)]
    for norb, na, nb, nsa, nsb, seed in cases:
        a, _ = random_product_strings(norb, na, na, nsa, 1, seed)
        _, b = random_product_strings(norb, nb, nb, 1, nsb, seed + 50)
        table = random_integrals(norb, seed)
        basis = SelectedBasis.product(a.tolist(), b.tolist(), norb, na, nb)
        inst = O.Instance.make(norb, table.h, table.eri, table.e_core, a, b)
        x = np.random.default_rng(seed).standard_normal(basis.dimension)
        ref = O.sigma(inst, x)
        app = HamiltonianApplier(basis, table)
        yh = app(x)
        yd = app.sigma_device(torch.from_numpy(x).cuda()).cpu().numpy()
        if nsb <= 1300 and (norb, na, nb) != (14, 7, 3):  # shapes whose buffers fit must run the DMMA kernel
            assert app.task0_kernel() == "direct-ci", (norb, na, nb)
        for y in (yh, yd):
            assert np.abs(y - ref).max() <= 1e-10 * np.abs(ref).max(), (norb, na, nb, nsa, nsb)
        assert np.array_equal(app.sigma_device(torch.from_numpy(x).cuda()).cpu().numpy(), yd)  # reproducible
        lo, hi = nsa // 3, nsa // 3 + max(1, nsa // 4)
        win = HamiltonianApplier(basis, table, row_window=(lo, hi))
        yw = win(x)
        assert np.abs(yw - ref[lo * nsb:hi * nsb]).max() <= 1e-10 * np.abs(ref).max()
