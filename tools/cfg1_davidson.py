"""cfg1 (12 orbitals, full 924 x 924 string set) Davidson on the device vs the reference run.

The reference's own davidson_solve at defaults took 744 s on 8 container cores
(tests/golden/cfg1_davidson.json, E0 = -20.91738303).
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, davidson_solve, synth

    table = synth.random_integrals(12, seed=1)
    basis = synth.full_product_basis(12, 6, 6)
    app = HamiltonianApplier(basis, table)
    x = torch.randn(app.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        app.sigma_device(x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        app.sigma_device(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    sig_ms = e0.elapsed_time(e1) / 50
    # first solve: includes the one-time loading of the Davidson kernels (CUDA lazy
    # module loading); the second is the steady-state figure
    t0 = time.perf_counter()
    davidson_solve(app, app.diag_device)
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = davidson_solve(app, app.diag_device)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg1_davidson.json")))
    print(json.dumps({"n_dets": app.n, "sigma_ms": sig_ms, "sigma_dets_per_s": app.n / sig_ms * 1e3,
                      "davidson_s": wall, "davidson_first_call_s": first, "iterations": res.stats.iterations, "energy": float(res.energies[0]),
                      "reference_energy": ref["energy"], "abs_diff": abs(float(res.energies[0]) - ref["energy"]),
                      "reference_s": ref["seconds"], "reference_iterations": ref["iterations"]}, indent=1))


if __name__ == "__main__":
    main()
