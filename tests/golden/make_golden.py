"""Generate golden fixtures by running the REFERENCE (sbdiag) in this container.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py small cfg1 cfg2 [cfg1-davidson] [cfg4] [table128]

The reference is not present on the GPU box, so its outputs are committed as
small fixtures here: full arrays for the small instances, and for cfg1/cfg2/
cfg4 SHA-256 digests of every excitation-table column plus sigma/diagonal
values on windows of alpha rows (the reference's own windowed apply,
``apply.py:501-546,608-623``, as used by ``test_apply.py:238-255``).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from sbdiag import synth  # noqa: E402
from sbdiag.apply import (  # noqa: E402
    HamiltonianApplier,
    _apply_product,
    build_det_cache,
    build_spin_tables,
    compute_diagonal,
)
from sbdiag.basis import build_excitation_table, enumerate_doubles, enumerate_singles  # noqa: E402
from sbdiag.davidson import DavidsonOptions, davidson_solve  # noqa: E402

FIELDS = ("s_off", "s_tgt", "s_hole", "s_part", "s_phase",
          "d_off", "d_tgt", "d_hole1", "d_hole2", "d_part1", "d_part2", "d_phase")
DTYPES = dict(s_off=np.int64, s_tgt=np.int64, s_hole=np.int16, s_part=np.int16, s_phase=np.int8,
              d_off=np.int64, d_tgt=np.int64, d_hole1=np.int16, d_hole2=np.int16,
              d_part1=np.int16, d_part2=np.int16, d_phase=np.int8)


def digest(arr, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=dtype)).tobytes()).hexdigest()


def table_digests(tab) -> dict:
    return {f: digest(getattr(tab, f), DTYPES[f]) for f in FIELDS}


def strings_digest(strings) -> str:
    return digest(np.asarray(strings, dtype=np.uint64), np.uint64)


def _hubbard():
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import hubbard_dimer_basis, hubbard_dimer_table
    return hubbard_dimer_basis(), hubbard_dimer_table()


SMALL_CASES = [
    # name, norb, na, nb, n_alpha_strings (None = full), n_beta_strings, integral seed, basis seed
    ("full_4_2_2_s0", 4, 2, 2, None, None, 0, None),
    ("full_4_2_2_s3", 4, 2, 2, None, None, 3, None),
    ("full_5_2_3_s5", 5, 2, 3, None, None, 5, None),
    ("partial_5_2_3", 5, 2, 3, 6, 7, 9, 1),
    ("partial_6_3_3", 6, 3, 3, 8, 8, 21, 5),
    ("partial_8_4_3", 8, 4, 3, 30, 25, 7, 11),
    ("full_6_3_2_s2", 6, 3, 2, None, None, 2, None),
    ("single_det_3", 3, 2, 2, 1, 1, 42, 0),
    ("partial_10_5_5", 10, 5, 5, 60, 50, 13, 17),
]


def make_small():
    out = {}
    meta = {}
    for name, norb, na, nb, nsa, nsb, iseed, bseed in SMALL_CASES:
        table = synth.random_integrals(norb, seed=iseed)
        if nsa is None:
            basis = synth.full_product_basis(norb, na, nb)
        else:
            basis = synth.random_product_basis(norb, na, nb, nsa, nsb, seed=bseed)
        tabs = build_spin_tables(basis)
        app = HamiltonianApplier(basis, table, tables=tabs, exec_policy="deterministic")
        rng = np.random.default_rng(1000 + iseed)
        xs = rng.standard_normal((3, basis.dimension))
        ys = np.stack([app(x) for x in xs])
        opts = DavidsonOptions(n_roots=min(2, basis.dimension), restart_keep=min(4, basis.dimension),
                               max_subspace=min(32, basis.dimension)) if basis.dimension >= 2 else \
            DavidsonOptions(n_roots=1, restart_keep=1, max_subspace=1)
        res = davidson_solve(app, app.diag, opts=opts)
        out[f"{name}/alpha"] = np.asarray(basis.alpha_strings, dtype=np.uint64)
        out[f"{name}/beta"] = np.asarray(basis.beta_strings, dtype=np.uint64)
        out[f"{name}/diag"] = app.diag
        out[f"{name}/x"] = xs
        out[f"{name}/y"] = ys
        out[f"{name}/energies"] = res.energies
        for spin, tab in (("ta", tabs.alpha), ("tb", tabs.beta)):
            for f in FIELDS:
                out[f"{name}/{spin}/{f}"] = np.asarray(getattr(tab, f), dtype=DTYPES[f])
        meta[name] = dict(norb=norb, na=na, nb=nb, nsa=nsa, nsb=nsb, iseed=iseed, bseed=bseed,
                          iterations=res.stats.iterations, converged=res.stats.converged,
                          n_roots=opts.n_roots)
    hb, ht = _hubbard()
    happ = HamiltonianApplier(hb, ht)
    out["hubbard/diag"] = happ.diag
    out["hubbard/col0"] = happ(np.array([1.0, 0.0, 0.0, 0.0]))
    out["hubbard/dense"] = np.column_stack([happ(np.eye(4)[:, j]) for j in range(4)])
    out["hubbard/energy"] = davidson_solve(happ, happ.diag, opts=DavidsonOptions(max_subspace=4)).energies
    # worked enumeration examples (test_basis.py:107-122)
    out["enum/singles_0b0011_3"] = np.array(enumerate_singles(0b0011, 3), dtype=np.int64)
    out["enum/doubles_0b0011_4"] = np.array(enumerate_doubles(0b0011, 4), dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    with open(os.path.join(HERE, "small_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("small: wrote", len(out), "arrays")


def _big(name, norb, na, nb, ns, windows, strings=None):
    t0 = time.time()
    table = synth.random_integrals(norb, seed=1)
    if strings is None:
        basis = synth.full_product_basis(norb, na, nb) if ns is None else \
            synth.random_product_basis(norb, na, nb, ns, ns, seed=2)
    else:
        from sbdiag.basis import SelectedBasis
        basis = SelectedBasis.product(strings[0], strings[1], norb, na, nb)
    t_basis = time.time() - t0
    t0 = time.time()
    tabs = build_spin_tables(basis)
    t_tab = time.time() - t0
    nbeta = len(basis.beta_strings)
    rec = dict(norb=norb, na=na, nb=nb, n_alpha=len(basis.alpha_strings), n_beta=nbeta,
               alpha_digest=strings_digest(basis.alpha_strings),
               beta_digest=strings_digest(basis.beta_strings),
               h_digest=digest(table.h, np.float64), eri_digest=digest(table.eri, np.float64),
               ta=table_digests(tabs.alpha), tb=table_digests(tabs.beta),
               ta_counts=[int(tabs.alpha.s_off[-1]), int(tabs.alpha.d_off[-1])],
               tb_counts=[int(tabs.beta.s_off[-1]), int(tabs.beta.d_off[-1])],
               seconds_basis=t_basis, seconds_tables=t_tab, windows=[])
    arrays = {}
    if windows:
        x = np.random.default_rng(12345).standard_normal(basis.dimension)
        cache = None
        for lo, hi in windows:
            cache = build_det_cache(basis, ((lo, hi), (0, nbeta)), None, cache)
            d = compute_diagonal(basis, table, cache)
            t0 = time.time()
            y = _apply_product(x, basis, table, tabs, cache, d, "parallel")
            rec["windows"].append(dict(lo=lo, hi=hi, seconds=time.time() - t0))
            arrays[f"diag_{lo}_{hi}"] = d
            arrays[f"sigma_{lo}_{hi}"] = y
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    print(name, "done", {k: rec[k] for k in ("ta_counts", "tb_counts", "seconds_basis", "seconds_tables")})
    return basis, table, tabs


def make_cfg1():
    _big("cfg1", 12, 6, 6, None, [(0, 8), (457, 461), (916, 924)])


def make_cfg1_davidson():
    table = synth.random_integrals(12, seed=1)
    basis = synth.full_product_basis(12, 6, 6)
    app = HamiltonianApplier(basis, table)
    t0 = time.time()
    res = davidson_solve(app, app.diag)
    rec = dict(energy=float(res.energies[0]), iterations=res.stats.iterations,
               restarts=res.stats.restarts, converged=res.stats.converged,
               seconds=time.time() - t0, mean_apply=float(np.mean(res.stats.apply_seconds)),
               threads=int(os.environ.get("NUMBA_NUM_THREADS", os.cpu_count())))
    with open(os.path.join(HERE, "cfg1_davidson.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print("cfg1 davidson", rec)


def make_cfg2():
    _big("cfg2", 26, 7, 7, 10000, [(0, 2), (5000, 5001), (9998, 10000)])


def make_cfg4():
    # the reference generator enumerates C(36,27)=94M strings (~400 s, 7.5 GB)
    _big("cfg4", 36, 27, 27, 30000, [(0, 1)])


EXPLICIT_CASES = [
    # name, norb, na, nb, n_dets, integral seed, basis seed
    ("expl_4_2_2_all", 4, 2, 2, 36, 0, 3),
    ("expl_5_2_3_some", 5, 2, 3, 40, 9, 1),
    ("expl_6_3_3", 6, 3, 3, 150, 21, 5),
    ("expl_8_4_3", 8, 4, 3, 900, 7, 11),
    ("expl_single", 3, 2, 2, 1, 42, 0),
    ("expl_10_5_5", 10, 5, 5, 4000, 13, 17),
    ("expl_12_6_6", 12, 6, 6, 20000, 1, 2),
]


def make_explicit():
    """Explicit (full-bitstring) bases: the reference's _explicit_kernel (apply.py:320-458)."""
    out, meta = {}, {}
    for name, norb, na, nb, nd, iseed, bseed in EXPLICIT_CASES:
        table = synth.random_integrals(norb, seed=iseed)
        basis = synth.random_explicit_basis(norb, na, nb, nd, seed=bseed)
        app = HamiltonianApplier(basis, table, exec_policy="deterministic")
        rng = np.random.default_rng(2000 + iseed)
        xs = rng.standard_normal((2, basis.dimension))
        ys = np.stack([app(x) for x in xs])
        n = basis.dimension
        opts = DavidsonOptions(n_roots=min(2, n), restart_keep=min(4, n), max_subspace=min(32, n))
        res = davidson_solve(app, app.diag, opts=opts)
        out[f"{name}/det_a"] = np.array([d.alpha for d in basis.dets], dtype=np.uint64)
        out[f"{name}/det_b"] = np.array([d.beta for d in basis.dets], dtype=np.uint64)
        out[f"{name}/diag"] = app.diag
        out[f"{name}/x"] = xs
        out[f"{name}/y"] = ys
        out[f"{name}/energies"] = res.energies
        meta[name] = dict(norb=norb, na=na, nb=nb, n_dets=nd, iseed=iseed, bseed=bseed,
                          iterations=res.stats.iterations, converged=res.stats.converged, n_roots=opts.n_roots)
        print(name, n, res.energies, res.stats.iterations)
    np.savez_compressed(os.path.join(HERE, "explicit.npz"), **out)
    with open(os.path.join(HERE, "explicit_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def _sample_lines(rng, norb, na, nb, n, pool, seed):
    """Sample-file lines with the reference format's corner cases: '#' comments, blank and padded lines,
    wrong electron counts (filtered) and heavy duplication (a small pool of strings)."""
    from sbdiag.synth import random_product_basis

    basis = random_product_basis(norb, na, nb, pool, pool, seed)
    A, B = list(basis.alpha_strings), list(basis.beta_strings)
    bits = lambda w: "".join("1" if w >> p & 1 else "0" for p in range(norb))  # noqa: E731
    lines = ["# sampled configurations", ""]
    for i in range(n):
        r = rng.random()
        if r < 0.03:
            lines.append("# comment " + str(i))
        elif r < 0.05:
            lines.append("   ")
        elif r < 0.12:  # one electron short in alpha or beta: filtered
            a = A[rng.integers(len(A))] if rng.random() < 0.5 else (A[rng.integers(len(A))] & ~(1 << (A[0].bit_length() - 1)))
            b = B[rng.integers(len(B))]
            if bin(a).count("1") == na:
                b = b & (b - 1)
            lines.append(bits(a) + bits(b))
        else:
            pad = "  " if r > 0.95 else ""
            lines.append(pad + bits(A[rng.integers(len(A))]) + bits(B[rng.integers(len(B))]) + pad)
    return lines


INGEST_CASES = [(6, 3, 3, 200, 4, 1), (10, 4, 3, 1500, 25, 2), (12, 6, 6, 2500, 120, 3), (20, 5, 5, 2000, 900, 4)]


def make_ingest():
    """Reference ingest_samples (basis.py:251-313) + the CLI start vector (cli.py:117-128) on sample files."""
    from sbdiag.basis import ingest_samples
    from sbdiag.cli import _start_vector

    rng = np.random.default_rng(2024)
    out = []
    for norb, na, nb, n, pool, seed in INGEST_CASES:
        lines = _sample_lines(rng, norb, na, nb, n, pool, seed)
        case = dict(norb=norb, na=na, nb=nb, lines=lines, modes={})
        out.append(case)
        for mode in ("product", "explicit"):
            basis, rep = ingest_samples(lines, norb, na, nb, mode)
            x0 = _start_vector(basis, rep.det_counts)
            nz = np.nonzero(x0)[0]
            rec = dict(n_lines=rep.n_lines,
                       n_filtered=rep.n_filtered, n_duplicates=rep.n_duplicates,
                       det_counts=[[int(d.alpha), int(d.beta), int(c)] for d, c in rep.det_counts.items()],
                       start_nz=nz.tolist(), start_val=x0[nz].tolist(), dimension=basis.dimension)
            if mode == "product":
                rec.update(alpha=[int(v) for v in basis.alpha_strings], beta=[int(v) for v in basis.beta_strings])
            else:
                rec.update(dets=[[int(d.alpha), int(d.beta)] for d in basis.dets])
            case["modes"][mode] = rec
    with open(os.path.join(HERE, "ingest.json"), "w") as f:
        json.dump(out, f)
    # files for the CLI --fcidump/--samples cases
    from sbdiag.integrals import write_fcidump

    table = synth.random_integrals(8, seed=11)
    with open(os.path.join(HERE, "cli_case.fcidump"), "w") as f:
        f.write(write_fcidump(table, nelec=7, ms2=1))
    with open(os.path.join(HERE, "cli_case.samples"), "w") as f:
        f.write("\n".join(_sample_lines(np.random.default_rng(5), 8, 4, 3, 400, 14, 12)) + "\n")


CLI_CASES = [
    ["solve", "--gen-random", "8,4,4,3", "--strings", "30", "--json"],
    ["solve", "--gen-random", "10,5,4,7", "--strings", "60", "--nroots", "2", "--json"],
    ["solve", "--gen-random", "8,3,3,5", "--strings", "200", "--mode", "explicit", "--json"],
    ["verify", "--gen-random", "6,3,3,2", "--strings", "20", "--json"],
    ["solve", "--fcidump", "{golden}/cli_case.fcidump", "--samples", "{golden}/cli_case.samples", "--nroots", "2",
     "--json"],
    ["solve", "--fcidump", "{golden}/cli_case.fcidump", "--samples", "{golden}/cli_case.samples", "--mode",
     "explicit", "--json"],
    ["verify", "--fcidump", "{golden}/cli_case.fcidump", "--samples", "{golden}/cli_case.samples", "--json"],
]


def make_cli():
    """Reports of the reference CLI (cli.py) on --gen-random instances."""
    import contextlib
    import io

    from sbdiag.cli import main

    out = []
    for argv in CLI_CASES:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = main([a.format(golden=HERE) for a in argv])
        rep = json.loads(buf.getvalue())
        for k in ("solve_seconds", "apply_seconds"):
            rep.pop(k, None)
        out.append(dict(argv=argv, rc=rc, report=rep))
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def _walk_strings(rng, norb, ne, n, seeds, window):
    """A connected in-set string list for norb > 64: random single/double moves from seed strings,
    orbitals drawn from `window` (so the set has many in-set excitations), caller order = discovery order."""
    window = list(window)
    out, seen = [], set()
    for s in seeds:
        assert bin(s).count("1") == ne and s not in seen
        out.append(s)
        seen.add(s)
    while len(out) < n:
        s = out[int(rng.integers(len(out)))]
        occ = [p for p in window if (s >> p) & 1]
        virt = [p for p in window if not (s >> p) & 1]
        k = 1 if (len(occ) < 2 or len(virt) < 2 or rng.random() < 0.5) else 2
        if not occ or not virt:
            continue
        holes = rng.choice(occ, size=min(k, len(occ)), replace=False)
        parts = rng.choice(virt, size=len(holes), replace=False)
        t = s
        for p, r in zip(holes, parts):
            t = (t & ~(1 << int(p))) | (1 << int(r))
        if t not in seen:
            seen.add(t)
            out.append(t)
    return out


def _mask(orbs):
    m = 0
    for o in orbs:
        m |= 1 << o
    return m


# name, norb, n_elec, string-list builder (rng -> list of Python ints)
TABLE128_CASES = [
    # electrons straddling the 64-bit word boundary
    ("w72_e4", 72, 4, lambda rng: _walk_strings(rng, 72, 4, 300, [_mask([60, 62, 64, 66])], range(52, 72))),
    ("w100_e3", 100, 3, lambda rng: _walk_strings(rng, 100, 3, 200, [_mask([1, 63, 99]), _mask([62, 64, 65])],
                                                  list(range(0, 4)) + list(range(58, 70)) + list(range(95, 100)))),
    # every string of 2 electrons in 24 orbitals around bit 64 and at the top (bit 127)
    ("w128_e2_all", 128, 2, lambda rng: [a | b for a, b in (
        (1 << i, 1 << j) for i, j in __import__("itertools").combinations(list(range(56, 72)) + list(range(120, 128)), 2))]),
    ("w128_e5", 128, 5, lambda rng: _walk_strings(rng, 128, 5, 100, [_mask([0, 63, 64, 100, 127])],
                                                  list(range(0, 3)) + list(range(61, 67)) + list(range(124, 128)))),
    # one hole: nv = 1 (no doubles), 8001 hole pairs
    ("w128_e127", 128, 127, lambda rng: [((1 << 128) - 1) & ~(1 << h) for h in rng.permutation(128).tolist()]),
    # two holes inside a 24-orbital window: 7875 hole pairs, 1 particle pair
    ("w128_e126", 128, 126, lambda rng: [((1 << 128) - 1) & ~((1 << i) | (1 << j)) for i, j in
                                         __import__("itertools").combinations(list(range(52, 70)) + list(range(122, 128)), 2)]),
    # 65 orbitals, the smallest two-word case
    ("w65_e3", 65, 3, lambda rng: _walk_strings(rng, 65, 3, 250, [_mask([0, 32, 64])], range(65))),
]


def make_table128():
    """Reference build_excitation_table (basis.py:362-403) on norb > 64 string lists.

    The reference caps norb at 64 for integrals (integrals.py:67-68), but its table builder works on
    Python ints of any width; these fixtures pin the 128-bit table path to it.  Strings are stored as
    (lo, hi) uint64 word pairs."""
    rng = np.random.default_rng(128)
    out, meta = {}, {}
    for name, norb, ne, make in TABLE128_CASES:
        strings = [int(s) for s in make(rng)]
        assert len(set(strings)) == len(strings) and all(bin(s).count("1") == ne for s in strings)
        t0 = time.perf_counter()
        tab = build_excitation_table(strings, norb)
        out[f"{name}/words"] = np.array([[s & (2**64 - 1), s >> 64] for s in strings], dtype=np.uint64)
        for f in FIELDS:
            out[f"{name}/{f}"] = np.asarray(getattr(tab, f), dtype=DTYPES[f])
        meta[name] = dict(norb=norb, n_elec=ne, n_strings=len(strings), n_singles=int(tab.s_off[-1]),
                          n_doubles=int(tab.d_off[-1]))
        print(name, meta[name], f"{time.perf_counter() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "table128.npz"), **out)
    with open(os.path.join(HERE, "table128_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    jobs = dict(small=make_small, cli=make_cli, ingest=make_ingest, cfg1=make_cfg1, cfg2=make_cfg2, cfg4=make_cfg4, explicit=make_explicit,
                table128=make_table128,
                **{"cfg1-davidson": make_cfg1_davidson})
    for arg in sys.argv[1:]:
        jobs[arg]()
