"""Probe: can N ranks share ONE GPU over NCCL?  Each rank claims a distinct NCCL_HOSTID,
so NCCL sees N hosts and uses its socket transport (loopback) instead of refusing the
duplicate GPU.  Used by the one-GPU multi-rank tests (functional only, not a bandwidth figure).

    python tools/nccl_probe.py [N]
"""
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def run(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_HOSTID=f"sbd-rank-{rank}",
                      NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    n = 1 << 20
    x = torch.full((n,), float(rank + 1), dtype=torch.float64, device="cuda")
    out = torch.empty(world * n, dtype=torch.float64, device="cuda")
    dist.all_gather_into_tensor(out, x)
    ok = all(float(out[r * n]) == r + 1 for r in range(world))
    r = torch.tensor([rank + 1.0], dtype=torch.float64, device="cuda")
    dist.all_reduce(r)
    ok &= float(r) == world * (world + 1) / 2
    buf = torch.empty(n, dtype=torch.float64, device="cuda")
    ops = [dist.P2POp(dist.isend, x, (rank + 1) % world), dist.P2POp(dist.irecv, buf, (rank - 1) % world)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    ok &= float(buf[0]) == (rank - 1) % world + 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dist.all_gather_into_tensor(out, x)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"rank {rank}: ok={ok} allgather {world * n * 8 / dt / 1e9:.2f} GB/s", flush=True)
    dist.destroy_process_group()
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    mp.spawn(run, args=(world, 29511), nprocs=world, join=True)
