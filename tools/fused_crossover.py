"""Developer probe: MU iteration rate of the one-pass fused kernel vs the two streaming passes
over a grid of dense shapes (m, n, k), to place the fused kernel's dispatch threshold.
Prints one JSON line per (m, n, k)."""
import json
import os
import sys
import time

import torch
import paper_2202_09518_b200 as nmf

ITERS = 200
shapes = [(m, n) for m in (16384, 32768, 65536) for n in (8192, 16384, 32768, 65536)]
lags = ["1"]  # OOCNMF_FUSED_D values to try for the fused kernel
ks = (8, 16, 32)
args = sys.argv[1:]
if args and args[0].startswith("--d="):
    lags = args.pop(0)[4:].split(",")
if args and args[0].startswith("--k="):
    ks = tuple(int(x) for x in args.pop(0)[4:].split(","))
if args:
    shapes = [tuple(int(x) for x in s.split("x")) for s in args]
for m, n in shapes:
    ctx = nmf.Context(0)
    ctx.set_problem(m, n, 16, 0, m)
    ctx.generate_dense_uniform(42, 99)
    for k in ks:
        rec = {"m": m, "n": n, "k": k}
        for mode in ["1:" + d for d in lags] + ["0"]:
            os.environ["OOCNMF_FUSED"] = mode[0]
            if mode != "0":
                os.environ["OOCNMF_FUSED_D"] = mode[2:]
            ctx.set_rank(k)
            cfg = nmf.NmfConfig(k=k, max_iters=ITERS, error_check_interval=ITERS, eta=0.0, seed=1)
            ctx.solve(cfg)
            torch.cuda.synchronize()
            t = time.perf_counter()
            _, info = ctx.solve(cfg)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            rec["split" if mode == "0" else "fused_D" + mode[2:]] = round(ITERS / dt, 1)
            assert (info["fused_pass_launches"] > 0) == (mode != "0")
        print(json.dumps(rec), flush=True)
    ctx.close()
