"""CLI parity (reference cli.py): commands, flags, exit codes and report schema.

CPU tests cover argument handling and exit codes (usage/input errors exit 1
before any device work); GPU tests compare reports against the reference
CLI's own reports (tests/golden/cli.json, made by make_golden.py cli).
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2601_16637_b200.cli import EXIT_INPUT_ERROR, build_parser, main

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cli.json")


@pytest.mark.parametrize("argv", [[], ["bogus"], ["solve"], ["solve", "--gen-random", "3,2"],
                                  ["solve", "--gen-random", "99,2,2,1"], ["bench", "--gen-random", "x"],
                                  ["solve", "--fcidump", "/nonexistent", "--samples", "/nonexistent"]])
def test_usage_and_input_errors_exit_1(argv, capsys):
    assert main(argv) == EXIT_INPUT_ERROR
    assert "error:" in capsys.readouterr().err


def test_parser_matches_reference_flags():
    p = build_parser()
    a = p.parse_args(["solve", "--gen-random", "8,4,4,3", "--strings", "30", "--nroots", "2", "--tol", "1e-9",
                      "--max-iter", "50", "--max-subspace", "16", "--restart-keep", "3", "--delta", "1e-5",
                      "--json", "--mode", "explicit", "--workers", "1", "--overlap", "off", "--deterministic"])
    assert (a.nroots, a.tol, a.max_iter, a.max_subspace, a.restart_keep, a.delta) == (2, 1e-9, 50, 16, 3, 1e-5)
    v = p.parse_args(["verify", "--gen-random", "6,3,3,2", "--tol-match", "1e-7", "--oracle-cap", "100"])
    assert (v.tol_match, v.oracle_cap) == (1e-7, 100)
    b = p.parse_args(["bench", "--gen-random", "6,3,3,2", "--workers", "1", "--repeats", "2"])
    assert (b.workers_list, b.repeats) == ("1", 2)


def _n_cli_cases():
    with open(GOLDEN) as f:
        return len(json.load(f))


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(_n_cli_cases()))
def test_reports_match_reference_cli(case, capsys):
    """Reference CLI reports: --gen-random instances and an FCIDUMP + sample-file instance (device ingestion)."""
    with open(GOLDEN) as f:
        ref = json.load(f)[case]
    rc = main([a.format(golden=os.path.dirname(GOLDEN)) for a in ref["argv"]])
    rep = json.loads(capsys.readouterr().out)
    assert rc == ref["rc"]
    r = ref["report"]
    assert rep["schema_version"] == r["schema_version"] and rep["command"] == r["command"]
    assert rep["basis"] == r["basis"]
    assert rep.get("ingest") == r.get("ingest")  # n_lines / n_filtered / n_duplicates of the sample file
    if r["command"] == "solve":
        np.testing.assert_allclose(rep["energies"], r["energies"], atol=1e-8)
        assert rep["converged"] == r["converged"]
        assert abs(rep["iterations"] - r["iterations"]) <= 1
        assert set(r) - {"solve_seconds", "apply_seconds"} <= set(rep)
    else:
        assert abs(rep["davidson_energy"] - r["davidson_energy"]) <= 1e-8
        assert abs(rep["oracle_energy"] - r["oracle_energy"]) <= 1e-8
        assert rep["passed"] == r["passed"]


@pytest.mark.gpu
def test_bench_and_text_report(capsys, tmp_path):
    out = tmp_path / "rep.txt"
    assert main(["bench", "--gen-random", "8,4,4,3", "--strings", "30", "--repeats", "2", "--out", str(out)]) == 0
    text = out.read_text()
    assert "mult timing over 2 repeats" in text and "speedup" in text
    assert main(["solve", "--gen-random", "8,4,4,3", "--strings", "30"]) == 0
    assert "energies = [" in capsys.readouterr().out


@pytest.mark.gpu
def test_solve_from_fcidump_and_samples(tmp_path, capsys):
    """The file path: FCIDUMP + sample lines -> ingest -> multiplicity start vector -> Davidson."""
    from paper_2601_16637_b200 import (DavidsonOptions, Determinant, HamiltonianApplier, davidson_solve,
                                       det_to_line, ingest_samples, start_vector, write_fcidump)
    from paper_2601_16637_b200.synth import random_integrals, random_product_strings

    norb, na, nb = 8, 3, 2
    table = random_integrals(norb, seed=4)
    table.nelec, table.ms2 = na + nb, na - nb
    fcid = tmp_path / "FCIDUMP"
    fcid.write_text(write_fcidump(table))
    a, b = random_product_strings(norb, na, nb, 12, 9, seed=6)
    rng = np.random.default_rng(2)
    lines = [det_to_line(Determinant(int(a[i]), int(b[j])), norb)
             for i, j in zip(rng.integers(0, a.size, 400), rng.integers(0, b.size, 400))]
    lines += ["# comment", "", det_to_line(Determinant(0b1111, 0b11), norb)]  # filtered (4 alpha electrons)
    samples = tmp_path / "samples.txt"
    samples.write_text("\n".join(lines) + "\n")
    assert main(["solve", "--fcidump", str(fcid), "--samples", str(samples), "--json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    basis, report = ingest_samples(lines, norb, na, nb)
    assert rep["ingest"] == {"n_lines": report.n_lines, "n_filtered": report.n_filtered,
                             "n_duplicates": report.n_duplicates}
    app = HamiltonianApplier(basis, table)
    res = davidson_solve(app, app.diag, x0=start_vector(basis, report), opts=DavidsonOptions())
    np.testing.assert_allclose(rep["energies"], res.energies, atol=1e-10)


@pytest.mark.gpu
def test_solve_workers_2_under_torchrun_matches_one_worker(tmp_path):
    """`solve --workers 2` under torchrun: each rank binds its GPU, joins the group and runs the
    partitioned native solve; rank 0's report equals the one-worker report (reference test_cli.py:131-140).
    SBD_SHARE_GPU=1 puts both ranks on the one GPU of the test box."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = ["solve", "--gen-random", "10,5,5,3", "--strings", "40", "--nroots", "2", "--json"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["SBD_SHARE_GPU"] = "1"
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", "--master-port=29533", "-m", "paper_2601_16637_b200", *args,
                          "--workers", "2"], cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    reps = [json.loads(out.stdout)]  # one report: rank 0's
    assert reps[0]["workers"] == 2
    one = subprocess.run([sys.executable, "-m", "paper_2601_16637_b200", *args], cwd=root, capture_output=True,
                         text=True, timeout=600, env={k: v for k, v in env.items() if k != "SBD_SHARE_GPU"})
    ref = json.loads(one.stdout)
    np.testing.assert_allclose(reps[0]["energies"], ref["energies"], atol=1e-10)
    assert abs(reps[0]["iterations"] - ref["iterations"]) <= 1
