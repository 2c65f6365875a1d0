"""CPU (gloo, world_size 2) tests of the row-partitioned path's host logic and decomposition.

The GPU RNMF iteration per rank is: local W update (H replicated), local partial
[W^T A | W^T W] packed into one buffer, ONE all-reduce, replicated H update, trace-form error
from the reduced terms (no extra collective). Here each gloo rank runs that exact schedule in
f64 numpy on its row slab; the result must equal the serial oracle (1e-8 trace,
1e-6 factors). The NCCL unique-id exchange is exercised through the same helper the
product uses.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2202_09518_b200 as nmf
from paper_2202_09518_b200.nmf import exchange_unique_id


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_schedule(rank, world, a, k, w0, h0, iters, interval, eps=1e-12):
    """What one rank of the device path computes, restated in f64 numpy + gloo all-reduce."""
    import torch

    m, n = a.shape
    plan = nmf.make_plan(m, n, k, world, 1, nmf.Strategy.rnmf)
    (r0, r1), _ = plan.slabs[rank]
    A = a[r0:r1]
    W = w0[r0:r1].copy()
    H = h0.copy()
    nA2 = torch.tensor([float((A * A).sum())], dtype=torch.float64)
    dist.all_reduce(nA2)
    trace = []
    for it in range(1, iters + 1):
        hht = H @ H.T
        W *= (A @ H.T) / (W @ hht + eps)                      # local W update
        packed = np.concatenate([(W.T @ A).ravel(), (W.T @ W).ravel()])
        t = torch.from_numpy(packed)
        dist.all_reduce(t)                                    # the single collective
        wta = t[: k * n].numpy().reshape(k, n)
        wtw = t[k * n:].numpy().reshape(k, k)
        H *= wta / (wtw @ H + eps)                            # replicated H update
        if it % interval == 0 or it == iters:
            res = nA2.item() - 2 * float((wta * H).sum()) + float((wtw * (H @ H.T)).sum())
            trace.append(np.sqrt(max(res, 0.0) / nA2.item()))
    wfull = [torch.zeros(0)] * world
    dist.all_gather_object(wfull, W)
    return np.vstack(wfull), H, np.array(trace)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = exchange_unique_id(rank, lambda: bytes(range(128)))
        a = oracle.port.uniform_dense(90, 70, 5, 99)
        w0, h0 = oracle.port.init_factors(90, 70, 6, 1)
        w, h, tr = _rank_schedule(rank, world, a, 6, w0, h0, iters=20, interval=5)
        out[rank] = (uid, w, h, tr)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_schedule_matches_serial_oracle():
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == bytes(range(128))          # unique-id exchange
    a = oracle.port.uniform_dense(90, 70, 5, 99)
    w0, h0 = oracle.port.init_factors(90, 70, 6, 1)
    ser = oracle.port.nmf_serial(a, 6, w0, h0, max_iters=20, interval=5)
    for r in range(world):
        _, w, h, tr = out[r]
        np.testing.assert_allclose(tr, ser.trace_err, rtol=1e-8)
        np.testing.assert_allclose(w, ser.w, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(h, ser.h, rtol=1e-6, atol=1e-12)
    # and the reference's own row-partitioned run agrees
    d = oracle.port.nmf_rnmf(a, 6, w0, h0, world, 1, max_iters=20, interval=5)
    np.testing.assert_allclose(d.trace_err, out[0][3], rtol=1e-8)


@pytest.mark.parametrize("m,world", [(10, 3), (65536, 8), (7, 7)])
def test_rank_slabs_tile_rows_exactly(m, world):
    plan = nmf.make_plan(m, 5, 2, world, 1, nmf.Strategy.rnmf)
    rows = [s[0] for s in plan.slabs]
    assert rows[0][0] == 0 and rows[-1][1] == m
    assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    sizes = [r1 - r0 for r0, r1 in rows]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
