"""Developer probe: phases of the config-2 end-to-end call as bench.py's e2e runs it (pinned f32
A, create, load_dense, solve, get_factors, close), twice in one process — run with PYTHONPATH=.
and OOCNMF_PROFILE_IO=1 to see the copy-out internals."""
import time
import numpy as np
import torch
import paper_2202_09518_b200 as nmf

m = n = 65536
k = 32
host = np.empty((m, n), np.float32)
with nmf.Context(0) as g:
    g.set_problem(m, n, k)
    g.generate_dense_uniform(42, 99)
    g.download_dense(host)
nmf.check(nmf._capi.lib().oocnmf_host_register(host.ctypes.data, host.nbytes))
for rep in range(3):
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
    c.load_dense(host)
    mark("upload")
    c.solve(nmf.NmfConfig(k=k, max_iters=50, error_check_interval=10, eta=0.0, seed=0))
    mark("solve")
    w, h = c.get_factors()
    mark("download")
    c.close()
    mark("destroy")
    print(rep, ph, flush=True)
