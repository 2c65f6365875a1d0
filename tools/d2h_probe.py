"""Developer probe: pageable (fresh / touched) vs pinned 16 MB device-to-host copies in every rank at
once (torchrun --nproc-per-node N tools/d2h_probe.py) — sizing the direct copy-out path."""
import os, time, numpy as np, torch, torch.distributed as dist
r = int(os.environ.get("LOCAL_RANK", 0)); torch.cuda.set_device(r)
dist.init_process_group("gloo")
d = torch.rand(4 << 20, device="cuda")
for trial in range(3):
    dist.barrier()
    h = np.empty(4 << 20, np.float32)
    t = time.perf_counter(); torch.from_numpy(h).copy_(d); torch.cuda.synchronize(); a = time.perf_counter() - t
    h2 = np.ones(4 << 20, np.float32)
    t = time.perf_counter(); torch.from_numpy(h2).copy_(d); torch.cuda.synchronize(); b = time.perf_counter() - t
    p = torch.empty(4 << 20, pin_memory=True)
    t = time.perf_counter(); p.copy_(d); torch.cuda.synchronize(); c = time.perf_counter() - t
    print(f"rank {r} trial {trial}: fresh {a*1e3:.1f} ms, touched {b*1e3:.1f} ms, pinned {c*1e3:.1f} ms", flush=True)
