"""One sweep point, a few sigma builds (for ncu per-kernel captures of the sparse regime).

    python tools/sigma_probe.py NORB NE NS [STEPS]     (NS = 0: the full string set in combinations order)
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis, synth

    norb, ne, ns = (int(v) for v in sys.argv[1:4])
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    table = synth.random_integrals(norb, seed=1)
    if ns == 0:
        app = HamiltonianApplier(synth.full_product_basis(norb, ne, ne), table)
    else:
        a, b = synth.random_product_strings(norb, ne, ne, ns, ns, seed=2)
        app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
    x = torch.empty(app.n, dtype=torch.float64, device="cuda").normal_()
    y = torch.empty_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        app.sigma_device(x, out=y)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        app.sigma_device(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    print(f"norb {norb} N {app.n}: {e0.elapsed_time(e1) / steps:.3f} ms per sigma")


if __name__ == "__main__":
    main()
