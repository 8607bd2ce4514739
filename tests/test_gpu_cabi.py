"""A pure-C consumer of include/sbd.h (examples/c_solve.c): sigma and the native Davidson vs the oracle.

This is the drop-in boundary without Python in the loop: gcc links the program
against libsbd_b200.so, it reads a numpy-written instance, and its outputs are
compared here with the C oracle.
"""

from __future__ import annotations

import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib = os.path.join(ROOT, "paper_2601_16637_b200")
    exe = str(tmp_path / "c_solve")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
                    os.path.join(ROOT, "examples", "c_solve.c"), "-L", lib, "-lsbd_b200", f"-Wl,-rpath,{lib}",
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("norb,ne_a,ne_b,nsa,nsb,n_roots", [(10, 5, 5, 60, 50, 1), (12, 4, 5, 200, 150, 2)])
def test_c_program_sigma_and_davidson_vs_oracle(tmp_path, norb, ne_a, ne_b, nsa, nsb, n_roots):
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    exe = _build(tmp_path)
    a, _ = random_product_strings(norb, ne_a, ne_a, nsa, 1, seed=4)
    _, b = random_product_strings(norb, ne_b, ne_b, 1, nsb, seed=5)
    t = random_integrals(norb, seed=6)
    n = a.size * b.size
    x = np.random.default_rng(7).standard_normal(n)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        np.array([norb, ne_a, ne_b], np.int32).tofile(f)
        np.array([a.size, b.size, t.eri.size], np.int64).tofile(f)
        np.array([t.e_core], np.float64).tofile(f)
        for arr, dt in ((t.h, np.float64), (t.eri, np.float64), (a, np.uint64), (b, np.uint64), (x, np.float64)):
            np.ascontiguousarray(arr, dtype=dt).tofile(f)
    r = subprocess.run([exe, str(inp), str(out), str(n_roots)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    y = np.frombuffer(raw[:8 * n], np.float64)
    it, conv, nfound = np.frombuffer(raw[8 * n:8 * n + 12], np.int32)
    e = np.frombuffer(raw[8 * n + 12:8 * n + 12 + 8 * n_roots], np.float64)

    inst = O.Instance.make(norb, t.h, t.eri, t.e_core, a, b)
    ref_y = O.sigma(inst, x)
    assert np.abs(y - ref_y).max() <= 1e-10 * np.abs(ref_y).max()
    ref = O.davidson(lambda v: O.sigma(inst, v), O.diag(inst), n_roots=n_roots)
    assert conv == 1 and nfound == n_roots
    np.testing.assert_allclose(e, ref.energies, atol=1e-8, rtol=0)


def test_sigma_multi_equals_single_calls():
    """sbd_sigma_multi (the block form of SURVEY 8(b)) against nvec single sbd_sigma calls, and its argument checks."""
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis, _lib
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    a, b = random_product_strings(11, 4, 4, 120, 90, seed=5)
    app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 11, 4, 4), random_integrals(11, seed=5))
    n, nvec, ld = app.n, 3, app.n + 6
    X = torch.randn(nvec, ld, dtype=torch.float64, device="cuda")
    Y = torch.zeros(nvec, ld, dtype=torch.float64, device="cuda")
    app._ctx("sbd_sigma_multi", _lib.ptr(X), ld, _lib.ptr(Y), ld, nvec)
    for v in range(nvec):
        assert torch.equal(Y[v, :n], app.sigma_device(X[v, :n].contiguous()))
    with pytest.raises(ValueError):
        app._ctx("sbd_sigma_multi", _lib.ptr(X), n - 1, _lib.ptr(Y), ld, 2)
