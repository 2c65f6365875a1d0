"""Small solves through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): the one-pass dense kernel (kp 16, 32), the two tensor-core passes (kp 64, and the
one-pass kernel disabled), the CSR SpMM path, the out-of-core path and a CNMF solve.
    compute-sanitizer --tool memcheck python tools/sanitize_solve.py
Not part of the product."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2202_09518_b200 as nmf  # noqa: E402


def dense(m, n, seed):
    return (np.arange(m * n, dtype=np.float64).reshape(m, n) * 0.618 % 1.0 + 0.01 * seed).astype(np.float32)


def solve(a, k, **kw):
    cfg = nmf.NmfConfig(k=k, max_iters=4, error_check_interval=2, eta=0.0, seed=1, **kw)
    r = nmf.nmf_serial(a, cfg)
    print(f"{type(a).__name__} k={k} err={r.error_trace[-1][1]:.6f}", flush=True)


a = dense(300, 700, 1)
solve(a, 16)  # one-pass kernel, kp 16
solve(a, 32)  # one-pass kernel, kp 32
solve(a, 48)  # two passes, kp 64
os.environ["OOCNMF_FUSED"] = "0"
solve(a, 32)  # two passes, kp 32
del os.environ["OOCNMF_FUSED"]
d = dense(400, 300, 2).astype(np.float64)
d[d < 0.7] = 0.0
solve(nmf.CsrMatrix.from_dense(d), 32)  # CSR: fused SpMM + updates
with nmf.Context(0) as ctx:  # out-of-core: host slab in 3 row batches
    ctx.set_problem(300, 700, 16)
    ctx.attach_host(np.ascontiguousarray(a), 128)
    tr, _ = ctx.solve(nmf.NmfConfig(k=16, max_iters=3, error_check_interval=3, eta=0.0, seed=1))
    print("ooc", tr[-1][1], flush=True)
comm = nmf.DistComm(0, 1, 0)
r = nmf.nmf_distributed(a, nmf.NmfConfig(k=8, max_iters=3, error_check_interval=3, eta=0.0, seed=1),
                        nmf.make_plan(300, 700, 8, 1, 1, nmf.Strategy.cnmf), comm)
comm.close()
print("cnmf", r.error_trace[-1][1], flush=True)
