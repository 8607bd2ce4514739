#!/usr/bin/env python
"""Sigma-build dets/s and s per Davidson iteration (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1: one rank per GPU, NCCL)

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset), bench.py
re-launches itself under ``python -m torch.distributed.run`` with N ranks on
127.0.0.1 and forwards rank 0's line.  --share-gpu puts every rank on cuda:0
(functional runs on a one-GPU box: NCCL then uses its socket transport, so
the numbers are not NVLink numbers).

A *step* is one sigma build y = H x over the whole determinant space of the
workload (BASELINE configs[1]: 26 orbitals, 7a7b, 1e4 x 1e4 random strings =
1e8 determinants).  At N > 1 the same 1e8-det system is partitioned by alpha
blocks (configs[2], strong scaling): every step runs the reference ring's
exchange pattern over NCCL (libsbd_b200's own communicator), overlapped with
the local beta-beta work and the alpha passes over blocks that have landed.  x (800 MB) is larger than L2, so
no flush is needed between steps.

Printed: one JSON line (rank 0) with the device-timed value, the roofline of
the sigma build, the end-to-end number through the public API (pinned host
x in, host y out, copies inside the timed region), clocks sampled during the
timed region, the CPU baseline (the oracle port on this host's cores) and the
device-resident Davidson seconds per iteration.

--impl reference times the reference algorithm's CPU implementation (the C
oracle port of pkg/src/sbdiag/apply.py, all host threads) on a bounded
alpha-row window of the same workload; it never touches the GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sigma-build dets/s and s per Davidson iter at 1/2/4/8 B200 vs CPU ref"
WORKLOAD = dict(norb=26, n_alpha=7, n_beta=7, n_strings=10000, integral_seed=1, basis_seed=2)
WORKLOAD_NAME = "cfg2/cfg3: synthetic N2-like 26 orbitals (7a,7b), 1e4 x 1e4 sampled strings = 1e8 dets"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _instance():
    from paper_2601_16637_b200 import synth

    w = WORKLOAD
    table = synth.random_integrals(w["norb"], seed=w["integral_seed"])
    a, b = synth.random_product_strings(w["norb"], w["n_alpha"], w["n_beta"], w["n_strings"], w["n_strings"],
                                        seed=w["basis_seed"])
    return table, a, b


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.start = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def running(self) -> bool:
        """True once nvidia-smi has produced a sample (or when it is unavailable)."""
        return self.proc is None or len(self.lines) > 0

    def mark(self):
        """Start of the timed region: summary() only uses samples taken after this."""
        self.start = len(self.lines)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[self.start:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn(args) -> int:
    """--gpus N without a torchrun environment: re-run this script as N ranks (rank 0 prints)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def _share_gpu_env(rank: int) -> None:
    """Several NCCL ranks on one GPU: distinct host ids make NCCL use its socket transport."""
    os.environ.update(NCCL_HOSTID=f"sbd-bench-rank-{rank}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(v: float, world: int, device) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _traffic():
    """Per-sigma DRAM bytes of the sigma kernels from the committed ncu capture, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_sigma_summary.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        rec = json.load(f)
    return rec.get("dram_bytes_per_sigma"), rec


# -- CPU baseline / reference arm -----------------------------------------------------


def _cpu_oracle_setup(table, a, b):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # the checker / CPU baseline, never the measured GPU path

    inst = O.Instance.make(WORKLOAD["norb"], table.h, table.eri, table.e_core, a, b)
    x = np.random.default_rng(12345).standard_normal(a.size * b.size)
    return O, inst, x


def _cpu_window_rate(O, inst, x, rows: int, reps: int, warm: int = 1):
    nb = inst.beta.size
    d = O.diag(inst, (0, rows))
    for _ in range(warm):
        O.sigma(inst, x, d, bra=(0, rows))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.sigma(inst, x, d, bra=(0, rows))
        ts.append(time.perf_counter() - t0)
    return rows * nb / statistics.median(ts), ts


def cpu_baseline(table, a, b, budget_s: float = 12.0):
    O, inst, x = _cpu_oracle_setup(table, a, b)
    threads = O.max_threads()
    rate, _ = _cpu_window_rate(O, inst, x, 4, 1, 0)
    rows = int(max(4, min(a.size, rate * budget_s / 3 / b.size)))
    rate, ts = _cpu_window_rate(O, inst, x, rows, 3, 0)
    return {"value": rate, "unit": "dets/s", "cores": threads, "kind": "port",
            "sample": f"oracle C port of apply.py _product_kernel (all {threads} host threads) on alpha rows "
                      f"[0,{rows}) x {b.size} beta = {rows * b.size} dets, median of 3 "
                      f"({statistics.median(ts):.2f} s each); full sigma extrapolates to "
                      f"{a.size * b.size / rate:.1f} s"}


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    table, a, b = _instance()
    O, inst, x = _cpu_oracle_setup(table, a, b)
    threads = O.max_threads()
    rate, _ = _cpu_window_rate(O, inst, x, 4, 1, 0)
    rows = int(max(4, min(a.size, rate * 1.5 / b.size)))  # ~1.5 s per step
    nb = b.size
    d = O.diag(inst, (0, rows))
    for _ in range(args.warmup):
        O.sigma(inst, x, d, bra=(0, rows))
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.sigma(inst, x, d, bra=(0, rows))
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    value = rows * nb / t
    sample = (f"alpha rows [0,{rows}) x {nb} beta = {rows * nb} dets per step of the 1e8-det workload "
              f"(oracle C port of the reference numba kernel, {threads} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "dets/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAME, "n_dets": int(a.size * nb), "sample_rows": rows,
                   "parallelism": f"{threads} CPU threads"},
        "cpu_baseline": {"value": value, "unit": "dets/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "dets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# -- explicit-basis section ---------------------------------------------------------------

EXPLICIT_STRINGS = 1000  # per spin: the first 1000 cfg2 strings, all pairs, shuffled = 1e6 dets


def explicit_bench(table, a, b, dev, stream, args, with_cpu=True):
    """Explicit-mode sigma (explicit_sigma_kernel) on 1e6 determinants: device-timed dets/s,
    parity against the product kernel on the same determinants, and the oracle port of the
    reference's _explicit_kernel on a bounded row sample."""
    import torch

    from paper_2601_16637_b200 import Determinant, HamiltonianApplier, SelectedBasis

    w = WORKLOAD
    sa, sb = a[:EXPLICIT_STRINGS], b[:EXPLICIT_STRINGS]
    pairs = np.random.default_rng(7).permutation(sa.size * sb.size)
    da, db = sa[pairs // sb.size], sb[pairs % sb.size]
    basis = SelectedBasis.explicit([Determinant(int(x), int(y)) for x, y in zip(da, db)], w["norb"], w["n_alpha"],
                                   w["n_beta"])
    app = HamiltonianApplier(basis, table, device=dev.index)
    n = basis.dimension
    x = torch.empty(n, dtype=torch.float64, device=dev).normal_(generator=torch.Generator(device=dev).manual_seed(3))
    y = torch.empty_like(x)
    for _ in range(3):
        app.sigma_device(x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(10, args.steps)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(reps):
        app.sigma_device(x, out=y)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3 / reps
    # same determinants through the product kernel
    prod = HamiltonianApplier(SelectedBasis.product(sa.tolist(), sb.tolist(), w["norb"], w["n_alpha"], w["n_beta"]),
                              table, device=dev.index)
    xp = torch.empty_like(x)
    xp[torch.from_numpy(pairs).to(dev)] = x
    yp = prod.sigma_device(xp)[torch.from_numpy(pairs).to(dev)]
    parity = float((yp - y).abs().max() / y.abs().max())
    out = {"workload": f"explicit list: all {sa.size} x {sb.size} pairs of the first cfg2 strings, shuffled",
           "n_dets": int(n), "value": n / t, "unit": "dets/s", "ms_per_step": t * 1e3,
           "parity_vs_product_kernel": parity, "kernel": "explicit_sigma_kernel"}
    if with_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        inst = O.ExplicitInstance.make(w["norb"], table.h, table.eri, table.e_core, da, db)
        xh = x.cpu().numpy()
        d = np.zeros(n)

        def run(rows):
            d[:rows] = [O.lib().orc_hdiag(int(p), int(q), inst.h, inst.norb, inst.eri, inst.e_core)
                        for p, q in zip(da[:rows], db[:rows])]
            t0 = time.perf_counter()
            yc = O.sigma_explicit(inst, xh, d, rows=(0, rows))
            return yc, time.perf_counter() - t0

        _, dt = run(64)  # probe, then a ~8 s sample
        rows = int(min(n, max(64, 64 * 8.0 / max(dt, 1e-4))))
        yc, dt = run(rows)
        err = float(np.abs(yc - y[:rows].cpu().numpy()).max() / max(np.abs(yc).max(), 1e-300))
        out["cpu_baseline"] = {"value": rows / dt, "unit": "dets/s", "cores": O.max_threads(), "kind": "port",
                               "sample": f"oracle C port of _explicit_kernel on determinants [0,{rows}) "
                                         f"({dt:.2f} s), all host threads; max rel diff vs GPU {err:.1e}"}
    del app, prod
    return out


# -- GPU arm -----------------------------------------------------------------------------


def run_ours(args):
    import torch

    world, rank, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist

        if args.share_gpu:
            local = 0
            _share_gpu_env(rank)
        torch.cuda.set_device(local)
        # torch's group carries the NCCL id and the max-over-ranks timings; the per-sigma
        # traffic is libsbd_b200's own NCCL communicator
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local) if args.backend == "nccl" else None)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
    from paper_2601_16637_b200.davidson import DavidsonOptions, davidson_solve
    from paper_2601_16637_b200.distributed import DistributedApplier

    table, a, b = _instance()
    basis = SelectedBasis.product(a.tolist(), b.tolist(), WORKLOAD["norb"], WORKLOAD["n_alpha"], WORKLOAD["n_beta"])
    n = basis.dimension
    nb = b.size
    t_setup = time.perf_counter()
    if world == 1:
        app = HamiltonianApplier(basis, table, device=dev.index)
        n_own = n
        lo = 0
        x_own = torch.empty(n, dtype=torch.float64, device=dev)
        y_own = torch.empty(n, dtype=torch.float64, device=dev)

        def step():
            app.sigma_device(x_own, out=y_own)

        cbar, bytes_total = app.sigma_model()
        ctx = app.context
    else:
        dapp = DistributedApplier(basis, table, device=dev.index, exchange=args.exchange, group_steps=args.group_steps)
        app = None
        n_own = dapp.n_own
        lo = dapp.lo
        x_own = torch.empty(n_own, dtype=torch.float64, device=dev)
        y_own = torch.empty(n_own, dtype=torch.float64, device=dev)

        def step():
            dapp.apply_device(x_own, y_own)

        import ctypes

        cb, by = ctypes.c_double(), ctypes.c_double()
        dapp.engine.context("sbd_sigma_model", ctypes.byref(cb), ctypes.byref(by))
        cbar = cb.value
        bytes_total = 8.0 * n * (3.0 + cbar)
        ctx = dapp.engine.context
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup
    gen = torch.Generator(device=dev).manual_seed(12345 + rank)
    x_own.normal_(generator=gen)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # ---- device-timed sigma (value) --------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        # keep the GPU busy (untimed) until the sampler is live, so every sample it
        # reports below lies inside the timed region
        t_wait = time.perf_counter()
        while True:
            live = clk.running() or time.perf_counter() - t_wait > 5.0
            if world > 1:  # every rank runs the same number of (collective) steps
                import torch.distributed as dist

                flag = torch.tensor([0.0 if live else 1.0], device=dev)
                dist.all_reduce(flag)
                live = float(flag.item()) == 0.0
            if live:
                break
            step()
            torch.cuda.synchronize(dev)
        barrier()
        clk.mark()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    t_step = _max_over_ranks(t_step, world, dev)
    value = n / t_step
    clocks = clk.summary()

    # ---- roofline of the sigma build (this rank's share) -------------------------------
    peak, peak_src = _peaks()
    bytes_rank = 8.0 * n_own * (3.0 + cbar)
    achieved = bytes_rank / t_step / 1e9
    traffic, traffic_rec = _traffic()
    kernels = {}
    overlap = None
    if world > 1:  # a separate profiled pass (events per ring-step group): exposed communication
        dapp.profile(True)
        for _ in range(max(3, min(args.steps, 10))):
            step()
        torch.cuda.synchronize(dev)
        rep_ = dapp.overlap_report()
        dapp.profile(False)
        info = dapp.engine.info()
        overlap = {"sigma_ms": rep_.sigma_s * 1e3, "overlap_ratio": rep_.overlap_ratio,
                   "exposed_ms_per_sigma": rep_.total_exposed_s * 1e3,
                   "transfer_ms_per_sigma": rep_.total_transfer_s * 1e3,
                   "compute_ms_per_sigma": rep_.total_compute_s * 1e3,
                   "per_step_ms": [[st, c * 1e3, t * 1e3, e * 1e3, r] for st, c, t, e, r in rep_.per_step],
                   "per_step_columns": ["step (0 = local, g = ring-step group)", "compute", "transfer", "exposed",
                                        "ratio"],
                   "exchange": dapp.exchange, "group_steps": args.group_steps,
                   "recv_bytes_per_sigma_rank0": 8 * info["recv_rows"] * nb,
                   "needed_fraction": info["needed_fraction"], "sigmas_profiled": rep_.n_sigma,
                   "note": "profiled run, separate from the timed region"}
    if world == 1:
        from paper_2601_16637_b200 import _lib

        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tl, tr = [], []
        for _ in range(args.steps):
            ev[0].record(stream)
            ctx("sbd_sigma_local", _lib.ptr(x_own))
            ev[1].record(stream)
            ctx("sbd_sigma_remote", _lib.ptr(x_own), _lib.ptr(y_own))
            ev[2].record(stream)
            torch.cuda.synchronize(dev)
            tl.append(ev[0].elapsed_time(ev[1]))
            tr.append(ev[1].elapsed_time(ev[2]))
        kernels = {"beta_side_incl_transpose_ms": statistics.median(tl), "alpha_side_ms": statistics.median(tr)}

    # ---- end to end through the public API -----------------------------------------------
    e2e = None
    if args.no_e2e:
        pass
    elif world == 1:
        xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
        yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
        xh.copy_(x_own.cpu())
        xn, yn = xh.numpy(), yh.numpy()
        app(xn, out=yn)  # warm (allocates the staging buffers)
        reps = max(3, min(args.steps, 10))
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(reps):
            app(xn, out=yn)  # H2D of x, sigma, D2H of y: HamiltonianApplier.__call__ (numpy protocol)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_e2e = e0.elapsed_time(e1) / 1e3 / reps
        e2e = {"value": n / t_e2e, "unit": "dets/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "ms_per_step": t_e2e * 1e3, "path": "HamiltonianApplier.__call__(numpy x in pinned memory)"}
        del xh, yh
    else:
        xh = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
        yh = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
        xh.copy_(x_own.cpu())
        reps = max(3, min(args.steps, 10))
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(reps):
            x_own.copy_(xh, non_blocking=True)
            dapp.apply_device(x_own, y_own)
            yh.copy_(y_own, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_e2e = _max_over_ranks(e0.elapsed_time(e1) / 1e3 / reps, world, dev)
        e2e = {"value": n / t_e2e, "unit": "dets/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "h2d_bytes_per_rank": 8 * n_own, "d2h_bytes_per_rank": 8 * n_own,
               "ms_per_step": t_e2e * 1e3,
               "path": "DistributedApplier.apply_device, each rank copying its own rows (pinned H2D/D2H); "
                       "bytes_per_step are whole-job totals"}

    # ---- device-resident Davidson, reference defaults ------------------------------------
    dav = None

    def run_davidson(opts):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        if world == 1:
            res = davidson_solve(app, app.diag_device, opts=opts, return_device=True)
        else:
            res = dapp.davidson(opts=opts)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        its = res.stats.iter_seconds
        s_iter = statistics.mean(its[1:]) if len(its) > 1 else its[0]
        s_iter = _max_over_ranks(s_iter, world, dev)
        out = {"s_per_iter": s_iter, "iterations": res.stats.iterations, "converged": res.stats.converged,
               "restarts": res.stats.restarts, "energy": float(res.energies[0]),
               "sigma_s_per_iter": statistics.mean(res.stats.apply_seconds[1:] or res.stats.apply_seconds),
               "wall_s": wall,
               "host_ms_per_iter": {k: v / res.stats.iterations for k, v in res.stats.host_ms.items()}}
        del res
        return out

    if not args.no_davidson:
        dav = run_davidson(DavidsonOptions(max_iters=args.davidson_iters))
        dav["options"] = ("reference defaults (tol 1e-8, k_max 32, keep 4)"
                          + (f", max_iters={args.davidson_iters}" if args.davidson_iters != 200 else ""))
        # reported separately, not the headline: skip the second Gram-Schmidt pass when the first kept
        # |t1| >= |t0|/sqrt(2) (B200 extension DavidsonOptions.selective_reorth)
        sel = run_davidson(DavidsonOptions(max_iters=args.davidson_iters, selective_reorth=True))
        sel["options"] = "reference defaults + selective_reorth (second CGS pass only when |t1| < |t0|/sqrt(2))"
        dav["selective_reorth"] = sel

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(table, a, b)

    # ---- explicit (full-bitstring) basis: SURVEY section 8(f)2 ---------------------------
    expl = None
    if rank == 0 and world == 1 and not args.no_explicit:
        expl = explicit_bench(table, a, b, dev, stream, args, with_cpu=not args.no_cpu)

    if world == 1:
        launches_per_step = 4  # transpose, beta side, task-0 cross, alpha side
    else:  # transpose, beta side, own-rows alpha pass, one pass per ring-step group, task 0 (+ sparse packs)
        ng = -(-(world - 1) // max(1, args.group_steps))
        launches_per_step = 4 + ng + ((world - 1) if dapp.exchange == "sparse" else 0)
    line = {
        "metric": METRIC, "value": value, "unit": "dets/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAME, "n_dets": int(n), "n_alpha": int(a.size), "n_beta": int(nb),
                   "cbar_alpha": cbar, "parallelism": f"alpha-block x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (x = 800 MB); no flush", "setup_s": setup_s},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "kernel": "sigma build (transpose + beta-side + task-0 + alpha-side kernels)",
                     "algorithmic_bytes": "8*N_own*(3 + cbar_alpha) per sigma (BASELINE.md section 4)",
                     "bytes_per_launch": bytes_rank,
                     "per_kernel_ncu": (traffic_rec or {}).get("per_kernel"),
                     "ncu_source": (traffic_rec or {}).get("source")},
        "kernels": kernels,
        "overlap": overlap,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "davidson": dav,
        "cpu_baseline": cpu,
        "explicit": expl,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-davidson", action="store_true")
    ap.add_argument("--davidson-iters", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-explicit", action="store_true")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend for setup and timing reductions (N > 1)")
    ap.add_argument("--share-gpu", action="store_true", help="all ranks on cuda:0 (functional runs on one GPU)")
    ap.add_argument("--exchange", choices=["auto", "dense", "sparse"], default="auto")
    ap.add_argument("--group-steps", type=int, default=2, help="ring steps per pipelined alpha pass")
    ap.add_argument("--dry-run", action="store_true", help="start the ranks and report them, no GPU work")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def run_dry(args):
    """Launch check: every rank joins the group; rank 0 prints the world it saw."""
    world, rank, _ = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ranks = [0]
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group(args.backend)
        t = torch.tensor([float(rank)])
        dist.all_reduce(t)
        ranks = [int(t.item())]
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "dry_run": True, "rank_sum": ranks[0],
                          "backend": args.backend}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
