"""Worker for tests/test_multi_gpu.py — launched with torch.distributed.run, one rank per GPU.

Runs the row-partitioned solve through the public API (nmf_distributed over NCCL) on dense,
CSR and out-of-core sources and writes rank 0's results to the JSON path in argv[1].
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2202_09518_b200 as nmf  # noqa: E402


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def main(out_path):
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = nmf.DistComm(rank, world, local)
    port = oracle.port
    results = {}

    def run(name, a, m, n, k, iters, interval, host_slab=None, batch_rows=0, strategy=nmf.Strategy.rnmf, **kw):
        plan = nmf.make_plan(m, n, k, world, 1, strategy)
        w0, h0 = port.init_factors(m, n, k, 0)
        cfg = nmf.NmfConfig(k=k, max_iters=iters, error_check_interval=interval, eta=0.0,
                            init=nmf.FactorInit.from_files, init_w=f32(w0), init_h=f32(h0), device=local, **kw)
        slab = None
        if host_slab is not None:
            (r0, r1), _ = plan.slabs[rank]
            slab = np.ascontiguousarray(host_slab[r0:r1])
        comm.reset_stats()
        res = nmf.nmf_distributed(a, cfg, plan, comm, host_slab=slab, batch_rows=batch_rows)
        h_calls = comm.stats().calls[nmf.PhaseTag.h_update]
        results[name] = {"trace": [e for _, e in res.error_trace], "iters": [i for i, _ in res.error_trace],
                         "h_calls": h_calls,
                         "w_fro": float(np.linalg.norm(res.w)), "h_fro": float(np.linalg.norm(res.h)),
                         "w_sum": float(res.w.sum()), "h_sum": float(res.h.sum()),
                         "allreduce_s": res.counters.allreduce_s, "w_shape": list(res.w.shape)}

    a = port.uniform_dense(1100, 900, 42, 99).astype(np.float32)
    run("dense_k16", a, 1100, 900, 16, 30, 10)
    run("dense_k32", a, 1100, 900, 32, 30, 10)
    rp, ci, v, (m, n) = port.gen_sparse(1500, 1200, 0.02, 3)
    run("csr_k16", nmf.CsrMatrix(m, n, rp, ci, f32(v)), m, n, 16, 20, 10)
    # n = 2048: whole 128-row H tiles per rank up to N = 16 -> the sharded H update path
    rp3, ci3, v3, (m3, n3) = port.gen_sparse(1100, 2048, 0.02, 8)
    run("csr_shard_k16", nmf.CsrMatrix(m3, n3, rp3, ci3, f32(v3)), m3, n3, 16, 20, 10)
    run("ooc_k32", None, 1100, 900, 32, 20, 10, host_slab=a, batch_rows=128)
    # config 3 scaled (2^15 x 2^15, density 4e-3, the reference generator on this rank's GPU)
    # against the compiled reference's serial run (tests/golden): the sharded H update over
    # NCCL, or over NVLS multicast from 4 ranks / with OOCNMF_NVLS=1
    g3 = np.load(os.path.join(ROOT, "tests", "golden", "csr_config3_scaled_32768_d4e-3_k32.npz"))
    m3g, n3g, seed3 = g3["gen"].tolist()
    with nmf.Context(local) as gctx:
        gctx.set_problem(m3g, n3g, 32)
        gctx.generate_csr_uniform(float(g3["density"]), seed3)
        c3 = gctx.download_csr()
    run("csr_cfg3_k32", c3, m3g, n3g, 32, int(g3["iters"]), int(g3["interval"]))
    # column partition (CNMF) on wide inputs: W replicated, H column slabs
    wide = port.uniform_dense(700, 1300, 7, 99).astype(np.float32)
    run("cnmf_dense_k16", wide, 700, 1300, 16, 30, 10, strategy=nmf.Strategy.cnmf)
    run("cnmf_dense_k32", wide, 700, 1300, 32, 30, 10, strategy=nmf.Strategy.cnmf)
    rp2, ci2, v2, (m2, n2) = port.gen_sparse(900, 1600, 0.02, 5)
    run("cnmf_csr_k16", nmf.CsrMatrix(m2, n2, rp2, ci2, f32(v2)), m2, n2, 16, 20, 10, strategy=nmf.Strategy.cnmf)
    # model selection: the P runs of each k spread over the ranks as replicas
    lr = oracle.ref.gen_lowrank(96, 64, 3, 0.01, 5)[0] if oracle.ref.available else port.uniform_dense(96, 64, 5, 1)
    scfg = nmf.SelectionConfig(k_min=1, k_max=4, n_perturbations=5, seed=3,
                               nmf=nmf.NmfConfig(max_iters=120, error_check_interval=20, eta=0.0, device=local))
    rep = nmf.select_k_distributed(lr.astype(np.float32), scfg, comm)
    results["select"] = {"chosen": rep.chosen_k, "rationale": rep.rationale,
                         "records": [[r.k, r.valid, r.runs_used, r.min_silhouette, r.mean_silhouette,
                                      r.mean_relative_error] for r in rep.records],
                         "medians_sum": [float(r.medians.sum()) for r in rep.records]}
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(results, f)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
