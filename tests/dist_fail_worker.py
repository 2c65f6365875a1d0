"""Worker for tests/test_multi_gpu.py::test_dead_rank_raises_comm_error — two ranks (processes,
one GPU each). Rank 1 joins the NCCL group and dies; rank 0's solve must raise CommError
within the collective timeout (src/comm.cpp:89-111 semantics) instead of hanging, and every
later collective on its context must fail (the group is poisoned). Rank 0 writes a JSON verdict
to argv[1].
"""
import json
import os
import sys
import time

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2202_09518_b200 as nmf  # noqa: E402


def main(out_path):
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dist.init_process_group("gloo")  # only ships the NCCL unique id
    comm = nmf.DistComm(rank, world, local, timeout_s=5.0)
    if rank == 1:
        os._exit(0)  # a rank that dies after joining the group
    m, n, k = 512, 384, 8
    a = (np.arange(m * n, dtype=np.float64).reshape(m, n) % 7 + 1).astype(np.float32)
    cfg = nmf.NmfConfig(k=k, max_iters=20, error_check_interval=10, eta=0.0, device=local)
    plan = nmf.make_plan(m, n, k, world, 1, nmf.Strategy.rnmf)
    verdict = {}
    t0 = time.time()
    try:
        nmf.nmf_distributed(a, cfg, plan, comm)
        verdict["first"] = "returned"
    except nmf.CommError as e:
        verdict["first"] = "CommError"
        verdict["message"] = str(e)
    verdict["seconds"] = time.time() - t0
    try:
        comm.barrier()
        verdict["second"] = "returned"
    except nmf.CommError as e:
        verdict["second"] = "CommError"
        verdict["second_message"] = str(e)
    with open(out_path, "w") as f:
        json.dump(verdict, f)
    os._exit(0)


if __name__ == "__main__":
    main(sys.argv[1])
