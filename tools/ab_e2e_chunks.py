"""Same-process e2e A/B of the pipelined host-buffer sigma chunk count (SBD_HOST_CHUNKS) at the bench workload."""
import os, sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2601_16637_b200 import HamiltonianApplier, SelectedBasis
table, a, b = bench._instance()
app = HamiltonianApplier(SelectedBasis.product(a.tolist(), b.tolist(), 26, 7, 7), table)
x = torch.empty(app.n, dtype=torch.float64).pin_memory(); x.normal_()
y = torch.empty(app.n, dtype=torch.float64).pin_memory()
xn, yn = x.numpy(), y.numpy()
res = {}
for rnd in range(3):
    for ch in ("8", "24", "40"):
        os.environ["SBD_HOST_CHUNKS"] = ch
        app(xn, out=yn)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5): app(xn, out=yn)
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / 5 * 1e3
        res[ch] = min(res.get(ch, 1e9), t)
print(json.dumps(res))
