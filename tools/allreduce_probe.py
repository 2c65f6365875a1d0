"""Developer probe: NCCL all-reduce time of config 2's packed [W^T A | W^T W] (8.4 MB f32) at N
ranks (torchrun), alone, to split the bench's all-reduce phase into transfer and rank skew."""
import os
import torch
import torch.distributed as dist

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
for mb in (0.008, 1.0, 8.4, 33.6):
    x = torch.ones(int(mb * 1e6 / 4), device="cuda")
    for _ in range(10):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    if rank == 0:
        print(f"N={world} {mb} MB all-reduce: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us", flush=True)
dist.destroy_process_group()
