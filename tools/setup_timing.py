"""Setup (configuration processing + tables + coefficients) wall time at the sparse configs, twice each,
and the 128-bit table builder on the same alpha strings (its tables must equal the 64-bit path's).

    python tools/setup_timing.py
"""

from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2601_16637_b200 import (HamiltonianApplier, SelectedBasis, build_excitation_table,
                                       build_excitation_table128, synth)

    for norb, ne, ns in [(36, 27, 30000), (40, 10, 31622)]:
        table = synth.random_integrals(norb, seed=1)
        a, b = synth.random_product_strings(norb, ne, ne, ns, ns, seed=2)
        for _ in range(2):
            t = time.perf_counter()
            app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), norb, ne, ne), table)
            torch.cuda.synchronize()
            print(norb, "setup_s", round(time.perf_counter() - t, 3), flush=True)
            del app
        t = time.perf_counter()
        t64 = build_excitation_table(a, norb, ne)
        t1 = time.perf_counter()
        t128 = build_excitation_table128(a.tolist(), norb, ne)
        t2 = time.perf_counter()
        same = all(np.array_equal(getattr(t64, f), getattr(t128, f)) for f in ("s_off", "s_tgt", "s_phase",
                                                                               "d_off", "d_tgt", "d_phase"))
        print(norb, "table64_s", round(t1 - t, 3), "table128_s", round(t2 - t1, 3), "equal", same,
              int(t64.s_off[-1]), int(t64.d_off[-1]), flush=True)


if __name__ == "__main__":
    main()
