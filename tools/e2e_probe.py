"""Developer probe: phases of the config-3 end-to-end call (CSR generation, download, set_problem,
load_csr, solve, get_factors) — run with PYTHONPATH=. and OOCNMF_PROFILE_IO=1."""
import time, numpy as np, torch
import paper_2202_09518_b200 as nmf
m=n=4194304; k=32
ctx=nmf.Context(0); ctx.set_problem(m,n,k)
t=time.perf_counter(); ctx.generate_csr_uniform(1e-5,1); print("gen",time.perf_counter()-t)
t=time.perf_counter(); host=ctx.download_csr(); print("download+validate",time.perf_counter()-t, host.nnz)
for rep in range(2):
    T=time.perf_counter()
    t=time.perf_counter(); ctx.set_problem(m,n,k); print("set_problem",time.perf_counter()-t)
    t=time.perf_counter(); ctx.load_csr(host); print("load_csr",time.perf_counter()-t)
    t=time.perf_counter(); ctx.solve(nmf.NmfConfig(k=k,max_iters=20,error_check_interval=10,eta=0.0,seed=0,device=0)); print("solve",time.perf_counter()-t)
    t=time.perf_counter(); ctx.get_factors(); print("get_factors",time.perf_counter()-t)
    print("total", time.perf_counter()-T)
