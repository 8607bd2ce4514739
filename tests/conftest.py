"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # test infrastructure: the CPU oracle


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def small_golden():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def explicit_golden():
    return dict(np.load(os.path.join(GOLDEN, "explicit.npz")))


@pytest.fixture(scope="session")
def explicit_meta():
    with open(os.path.join(GOLDEN, "explicit_meta.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def table128_golden():
    """Reference build_excitation_table on norb 65..128 string lists (make_golden.py table128)."""
    with open(os.path.join(GOLDEN, "table128_meta.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(GOLDEN, "table128.npz")))


TABLE128_CASES = ("w72_e4", "w100_e3", "w128_e2_all", "w128_e5", "w128_e127", "w128_e126", "w65_e3")


@pytest.fixture(scope="session")
def small_meta():
    with open(os.path.join(GOLDEN, "small_meta.json")) as f:
        return json.load(f)


def load_big(name):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    with open(path) as f:
        rec = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return rec, arrays


TABLE_FIELDS = ("s_off", "s_tgt", "s_hole", "s_part", "s_phase",
                "d_off", "d_tgt", "d_hole1", "d_hole2", "d_part1", "d_part2", "d_phase")
TABLE_DTYPES = dict(s_off=np.int64, s_tgt=np.int64, s_hole=np.int16, s_part=np.int16, s_phase=np.int8,
                    d_off=np.int64, d_tgt=np.int64, d_hole1=np.int16, d_hole2=np.int16,
                    d_part1=np.int16, d_part2=np.int16, d_phase=np.int8)


def digest(arr, dtype) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=dtype)).tobytes()).hexdigest()


def table_digests(tab) -> dict:
    get = (lambda f: tab[f]) if isinstance(tab, dict) else (lambda f: getattr(tab, f))
    return {f: digest(get(f), TABLE_DTYPES[f]) for f in TABLE_FIELDS}


BIG_CONFIGS = {
    # name: (norb, na, nb, n_strings or None for the full set)
    "cfg1": (12, 6, 6, None),
    "cfg2": (26, 7, 7, 10000),
    "cfg4": (36, 27, 27, 30000),
}


def big_instance(name):
    """Integrals (seed 1) and strings (seed 2) of a BASELINE config, via the restated generators."""
    from paper_2601_16637_b200 import synth

    norb, na, nb, ns = BIG_CONFIGS[name]
    table = synth.random_integrals(norb, seed=1)
    if ns is None:
        a = np.asarray(synth.all_strings(norb, na), dtype=np.uint64)
        b = np.asarray(synth.all_strings(norb, nb), dtype=np.uint64)
    else:
        a, b = synth.random_product_strings(norb, na, nb, ns, ns, seed=2)
    return table, a, b


def small_cases(small_meta):
    return sorted(small_meta)


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
