"""Small-message NCCL latency check (torchrun, 2+ GPUs): torch.distributed's
communicator vs a raw ncclAllReduce on a private stream (libstg's pattern)."""
import os
import time

import torch
import torch.distributed as dist

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
x = torch.ones(1024, dtype=torch.int32, device="cuda")
for it in range(20):
    dist.all_reduce(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(200):
    dist.all_reduce(x)
    torch.cuda.synchronize()
t1 = time.perf_counter()
if rank == 0:
    print(f"torch all_reduce 4 KB + sync: {1e6 * (t1 - t0) / 200:.1f} us")
dist.barrier()
dist.destroy_process_group()
