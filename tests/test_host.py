"""Host-side data model and plumbing (no GPU): generators, integrals, bases, C-ABI exports."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import BIG_CONFIGS, ROOT, big_instance, digest, load_big


@pytest.mark.parametrize("cfg", list(BIG_CONFIGS))
def test_synth_restatement_is_bit_identical(cfg):
    rec, _ = load_big(cfg)
    table, a, b = big_instance(cfg)
    assert digest(table.h, np.float64) == rec["h_digest"]
    assert digest(table.eri, np.float64) == rec["eri_digest"]
    assert digest(a, np.uint64) == rec["alpha_digest"]
    assert digest(b, np.uint64) == rec["beta_digest"]


def test_small_synth_matches_golden(small_golden, small_meta):
    from paper_2601_16637_b200 import synth

    for name, m in small_meta.items():
        if m["nsa"] is None:
            basis = synth.full_product_basis(m["norb"], m["na"], m["nb"])
        else:
            basis = synth.random_product_basis(m["norb"], m["na"], m["nb"], m["nsa"], m["nsb"], m["bseed"])
        assert basis.alpha_strings == small_golden[f"{name}/alpha"].tolist()
        assert basis.beta_strings == small_golden[f"{name}/beta"].tolist()


def test_unrank_matches_itertools():
    from paper_2601_16637_b200.synth import all_strings, unrank_combinations

    for norb, k in ((6, 3), (9, 2), (12, 6), (7, 7), (5, 1)):
        pool = all_strings(norb, k)
        got = unrank_combinations(np.arange(len(pool)), norb, k)
        assert got.tolist() == pool


def test_integrals_folding_and_fcidump_roundtrip():
    from paper_2601_16637_b200 import parse_fcidump, write_fcidump
    from paper_2601_16637_b200.synth import random_integrals

    t = random_integrals(5, seed=3)
    t.e_core = 1.25
    for p, q, r, s in ((0, 1, 2, 3), (4, 2, 1, 0), (3, 3, 1, 2)):
        v = t.get_eri(p, q, r, s)
        for perm in ((q, p, r, s), (p, q, s, r), (r, s, p, q), (s, r, q, p)):
            assert t.get_eri(*perm) == v
    t2 = parse_fcidump(write_fcidump(t, nelec=4, ms2=0))
    assert np.array_equal(t2.h, t.h) and np.array_equal(t2.eri, t.eri) and t2.e_core == t.e_core
    assert (t2.nelec, t2.ms2) == (4, 0)


def test_fcidump_errors_carry_line_numbers():
    from paper_2601_16637_b200 import FcidumpError, parse_fcidump

    with pytest.raises(FcidumpError, match="line 3"):
        parse_fcidump("&FCI NORB=2,NELEC=2,MS2=0,\n/\n1.0 1 1 x 0\n")
    with pytest.raises(FcidumpError):
        parse_fcidump("NORB=2\n")
    t = parse_fcidump("&FCI NORB=2,NELEC=2,MS2=0\n&END\n1.0 1 1 0 0\n2.0 1 1 0 0\n")
    assert t.n_conflicts == 1 and t.h[0, 0] == 2.0


def test_basis_validation_and_index():
    from paper_2601_16637_b200 import Determinant, SelectedBasis

    b = SelectedBasis.product([0b011, 0b101], [0b01, 0b10, 0b11][:2], 3, 2, 1)
    assert b.dimension == 4
    assert b.index_of(Determinant(0b101, 0b10)) == 3 and b.det_at(3) == Determinant(0b101, 0b10)
    with pytest.raises(ValueError, match="electrons"):
        SelectedBasis.product([0b111], [0b1], 3, 2, 1)
    with pytest.raises(ValueError, match="bits above"):
        SelectedBasis.product([0b1001], [0b1], 3, 2, 1)
    with pytest.raises(ValueError, match="duplicate"):
        SelectedBasis.explicit([(1, 1), (1, 1)], 2, 1, 1)


def test_sample_line_parser():
    """Host text layer of ingest_samples (reference basis.py:231-248): bit order, skips, error lines."""
    from paper_2601_16637_b200.basis import SampleFormatError, parse_sample_lines

    lines = ["# comment", "1100" + "0011", "  1010" + "0101  ", "", "1100" + "0011", "1110" + "0011"]
    a, b = parse_sample_lines(lines, 4)
    assert a.tolist() == [0b0011, 0b0101, 0b0011, 0b0111] and b.tolist() == [0b1100, 0b1010, 0b1100, 0b1100]
    a, b = parse_sample_lines("\n".join(["1" * 32 + "0" * 32, "0" * 63 + "1"]), 32)
    assert a.tolist() == [(1 << 32) - 1, 0] and b.tolist() == [0, 1 << 31]
    with pytest.raises(SampleFormatError, match="line 3"):
        parse_sample_lines(["11000011", "#", "1100001"], 4)
    with pytest.raises(SampleFormatError, match="line 2.*'2'"):
        parse_sample_lines(["11000011", "11002011", "110"], 4)  # the earlier line's error wins
    with pytest.raises(SampleFormatError, match="line 1"):
        parse_sample_lines(["1100001\u00e9"], 4)
    with pytest.raises(ValueError, match="norb in \\[1, 64\\]"):
        parse_sample_lines(["0" * 140], 70)  # wide strings: tables only (build_excitation_table128)


def test_host_enumerators_match_golden(small_golden):
    from paper_2601_16637_b200 import enumerate_doubles, enumerate_singles, single_phase

    assert sorted(enumerate_singles(0b0011, 3)) == sorted(map(tuple, small_golden["enum/singles_0b0011_3"].tolist()))
    assert [list(t) for t in enumerate_doubles(0b0011, 4)] == small_golden["enum/doubles_0b0011_4"].tolist()
    # test_basis.py:166-170
    assert single_phase(0b0011, 1, 2) == +1
    assert single_phase(0b0011, 0, 2) == -1
    assert single_phase(0b0101, 0, 4) == -1
    assert single_phase(0b0101, 2, 0) == single_phase(0b0101, 0, 2)


def test_davidson_options_validation():
    from paper_2601_16637_b200 import DavidsonOptions

    DavidsonOptions()
    for bad in (dict(n_roots=0), dict(n_roots=5), dict(tol_residual=0), dict(precond_delta=-1),
                dict(max_iters=0), dict(restart_keep=40)):
        with pytest.raises(ValueError):
            DavidsonOptions(**bad)


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "sbd.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(sbd_\w+)\s*\(", txt, re.M)))


def test_cabi_library_exports_every_header_symbol():
    from paper_2601_16637_b200 import _lib

    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.sbd_abi_version() == 1


@pytest.mark.skipif(__import__("conftest").gpu_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    from paper_2601_16637_b200 import HamiltonianApplier
    from paper_2601_16637_b200.synth import full_product_basis, random_integrals

    with pytest.raises(RuntimeError):
        HamiltonianApplier(full_product_basis(4, 2, 2), random_integrals(4, seed=0))


def test_native_davidson_default_options_match_reference_defaults():
    """sbd_davidson_default_opts (C) == DavidsonOptions() (davidson.py:33-40); struct layout via ctypes."""
    import ctypes

    from paper_2601_16637_b200 import DavidsonOptions, _lib

    o = _lib.DavidsonOptsC()
    assert _lib.load().sbd_davidson_default_opts(ctypes.byref(o)) == 0
    d = DavidsonOptions()
    for f in ("n_roots", "tol_residual", "max_iters", "max_subspace", "restart_keep", "precond_delta",
              "reorthogonalize", "track_orthogonality", "selective_reorth"):
        assert getattr(o, f) == getattr(d, f), f
    assert _lib.load().sbd_davidson_default_opts(None) == 1


def test_bench_gpus_flag_starts_that_many_ranks():
    """bench.py --gpus N (no torchrun env) re-launches itself as N ranks; rank 0 reports n_gpus = N."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--backend", "gloo", "--dry-run"], cwd=root,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # only rank 0 prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["rank_sum"] == 1


def test_string_words_host_conversion():
    """Host side of the 128-bit path: Python ints <-> (lo, hi) uint64 word pairs, the layout sbd_table128_build takes."""
    from paper_2601_16637_b200 import string_words

    vals = [0, 1, (1 << 63), (1 << 64), (1 << 127) | 5, (1 << 128) - 1]
    w = string_words(vals)
    assert w.dtype == np.uint64 and w.shape == (len(vals), 2)
    assert [int(lo) | (int(hi) << 64) for lo, hi in w.tolist()] == vals
    assert string_words(w) is not None and np.array_equal(string_words(w), w)  # (n, 2) arrays pass through
    assert string_words([]).shape == (0, 2)
    with pytest.raises(ValueError):
        string_words([1 << 128])
    with pytest.raises(ValueError):
        string_words([-1])
    with pytest.raises(ValueError):
        string_words(np.zeros((3, 3), dtype=np.uint64))
