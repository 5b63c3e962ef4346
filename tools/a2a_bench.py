"""NVLink all-to-all microbenchmark ("measure the achieved NCCL
all-to-all bus bandwidth on the box"): one rank per GPU under torchrun, the
slab exchange's message sizes (C/P bytes per rank at n^3), NCCL grouped
send/recv (torch all_to_all_single) timed with CUDA events, max over ranks.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/a2a_bench.py [--n 1024]

Prints one JSON line per size: bytes sent per rank, time, algorithm bandwidth
(bytes sent per rank / time) and bus bandwidth (x (P-1)/P), against the
NVLink 5 900 GB/s per direction."""
import argparse
import json
import os

import torch
import torch.distributed as dist

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = a.n
spec_bytes = n * n * ((n // 2 + 1 + 7) // 8 * 8) * 16  # the half-spectrum workspace (fp64)
for frac in (1, 4, 16):  # whole exchange, and the chunked exchange's sub-steps
    per_rank = spec_bytes // world // frac
    x = torch.empty(per_rank // 8, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    s.record()
    for _ in range(a.iters):
        dist.all_to_all_single(y, x)
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / a.iters], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    sent = per_rank * (world - 1) / world
    if rank == 0:
        print(json.dumps({"n": n, "ranks": world, "bytes_per_rank": per_rank, "bytes_sent_per_rank": sent,
                          "ms": ms, "algbw_gbs": per_rank / ms / 1e6, "busbw_gbs": sent / ms / 1e6,
                          "nvlink_spec_gbs": 900.0, "sub_step": frac}), flush=True)
dist.destroy_process_group()
