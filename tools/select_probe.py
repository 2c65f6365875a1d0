"""Developer probe: MU solve rate at config-5 shape (32768 x 16384) for a few k, eta 0 vs 1e-6,
and the per-k host time of one select_k sweep step."""
import time
import numpy as np
import torch
import paper_2202_09518_b200 as nmf
from paper_2202_09518_b200.nmf import _select_on

m, n = 32768, 16384
ctx = nmf.Context(0)
ctx.set_problem(m, n, 9, 0, m)
ctx.generate_dense_uniform(42, 99)
for k in (4, 9, 16):
    ctx.set_rank(k)
    for eta in (0.0, 1e-6):
        cfg = nmf.NmfConfig(k=k, max_iters=500, error_check_interval=10, eta=eta, seed=1)
        ctx.solve(cfg)
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.solve(cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"k={k} eta={eta}: {500 / dt:.0f} it/s", flush=True)
for k in (4, 16):
    cfg = nmf.SelectionConfig(k_min=k, k_max=k, n_perturbations=4, seed=0,
                              nmf=nmf.NmfConfig(max_iters=100, error_check_interval=10, eta=1e-6))
    t = time.perf_counter()
    rep = _select_on(ctx, m, cfg)
    dt = time.perf_counter() - t
    it = sum(r.iterations for r in rep.records)
    print(f"select k={k} P=4 100 it: {dt:.2f} s, {it} iterations, {it / dt:.0f} it/s", flush=True)
