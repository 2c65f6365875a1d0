"""Developer probe: the dense e2e call of bench.py repeated in one process after a resident
config-2 context (as the bench runs it), with per-phase times and the copy-in/out internals
(OOCNMF_PROFILE_IO=1): where do the 0.1-1 s hiccups of the e2e phases come from."""
import gc
import time

import numpy as np
import torch

import paper_2202_09518_b200 as nmf

m = n = 65536
k = 32
main = nmf.Context(0)
main.set_problem(m, n, k)
main.generate_dense_uniform(42, 99)
main.solve(nmf.NmfConfig(k=k, max_iters=20, error_check_interval=10, eta=0.0, seed=0))
host = np.empty((m, n), np.float32)
main.download_dense(host)
nmf.check(nmf._capi.lib().oocnmf_host_register(host.ctypes.data, host.nbytes))
for rep in range(4):
    gc.collect()
    ph = {}
    t = time.perf_counter()

    def mark(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        ph[name] = round(now - t, 4)
        t = now

    c = nmf.Context(0)
    mark("create")
    c.set_problem(m, n, k)
    mark("set_problem")
    c.load_dense(host)
    mark("upload")
    c.solve(nmf.NmfConfig(k=k, max_iters=50, error_check_interval=10, eta=0.0, seed=0))
    mark("solve")
    w, h = c.get_factors()
    mark("download")
    c.close()
    mark("destroy")
    print(rep, ph, flush=True)
