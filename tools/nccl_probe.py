"""NCCL transport / bandwidth probe (torchrun, one process per GPU)."""
import os
import time

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
for mb in (0.0625, 1, 16, 64, 256):
    n = int(mb * 1024 * 1024 / 4)
    x = torch.ones(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        dist.all_reduce(x, op=dist.ReduceOp.MIN)
    torch.cuda.synchronize()
    t = time.perf_counter()
    iters = 20
    for _ in range(iters):
        dist.all_reduce(x, op=dist.ReduceOp.MIN)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / iters
    if rank == 0:
        print(f"allreduce(min) {mb:8.4f} MB: {dt * 1e6:9.1f} us  algbw {mb / 1024 / dt:7.1f} GB/s",
              flush=True)
dist.destroy_process_group()

# broadcast 64 KB in place from alternating roots, like the FW diagonal tile
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
x = torch.ones(16384, dtype=torch.int32, device="cuda")
for _ in range(5):
    dist.broadcast(x, src=0)
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(100):
    dist.broadcast(x, src=i % world)
torch.cuda.synchronize()
if rank == 0:
    print(f"broadcast 64 KB alternating roots: {(time.perf_counter() - t) / 100 * 1e6:.1f} us",
          flush=True)
dist.destroy_process_group()
