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


def _cnmf_schedule(rank, world, a, k, w0, h0, iters, interval, eps=1e-12):
    """The column-partitioned (CNMF) device schedule restated in f64 numpy + gloo: W replicated,
    H column slab, per W update the all-reduced A·H^T and HH^T; H update local; trace-form error
    with the slab cross terms summed (src/nmf_distributed.cpp:112-149)."""
    import torch

    m, n = a.shape
    plan = nmf.make_plan(m, n, k, world, 1, nmf.Strategy.cnmf)
    _, (c0, c1) = plan.slabs[rank]
    A, W, H = a[:, c0:c1], w0.copy(), h0[:, c0:c1].copy()
    nA2 = torch.tensor([float((A * A).sum())], dtype=torch.float64)
    dist.all_reduce(nA2)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    hht = allreduce(H @ H.T)
    trace = []
    for it in range(1, iters + 1):
        aht = allreduce(A @ H.T)
        W *= aht / (W @ hht + eps)                         # replicated W update
        wta, wtw = W.T @ A, W.T @ W
        H *= wta / (wtw @ H + eps)                         # local H update
        hht = allreduce(H @ H.T)                           # next W update's Gram
        if it % interval == 0 or it == iters:
            cross = allreduce(np.array([float((wta * H).sum())]))[0]
            res = nA2.item() - 2 * cross + float((wtw * hht).sum())
            trace.append(np.sqrt(max(res, 0.0) / nA2.item()))
    parts = [None] * world
    dist.all_gather_object(parts, (c0, H))
    hfull = np.zeros((k, n))
    for cs, hs in parts:
        hfull[:, cs:cs + hs.shape[1]] = hs
    return W, hfull, np.array(trace)


def _cnmf_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = oracle.port.uniform_dense(60, 110, 7, 99)
        w0, h0 = oracle.port.init_factors(60, 110, 5, 2)
        out[rank] = _cnmf_schedule(rank, world, a, 5, w0, h0, iters=20, interval=5)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not oracle.ref.available, reason="needs oracle/_ref (reference CNMF worker)")
def test_two_rank_gloo_cnmf_schedule_matches_reference():
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_cnmf_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    a = oracle.port.uniform_dense(60, 110, 7, 99)
    w0, h0 = oracle.port.init_factors(60, 110, 5, 2)
    ref = oracle.ref.nmf_distributed(a, 5, world, 1, strategy=1, w0=w0, h0=h0, max_iters=20, interval=5)
    ser = oracle.port.nmf_serial(a, 5, w0, h0, max_iters=20, interval=5)
    for r in range(world):
        w, h, tr = out[r]
        np.testing.assert_allclose(tr, ref.trace_err, rtol=1e-8)
        np.testing.assert_allclose(w, ref.w, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(h, ref.h, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(tr, ser.trace_err, rtol=1e-8)   # CNMF is the serial iteration


@pytest.mark.parametrize("n,world", [(110, 2), (1300, 4), (9, 9)])
def test_cnmf_slabs_and_csr_column_windows_tile_exactly(n, world):
    plan = nmf.make_plan(6, n, 2, world, 1, nmf.Strategy.cnmf)
    cols = [s[1] for s in plan.slabs]
    assert cols[0][0] == 0 and cols[-1][1] == n and all(cols[i][1] == cols[i + 1][0] for i in range(world - 1))
    d = oracle.port.uniform_dense(6, n, 3, 1)
    d[d < 0.5] = 0
    c = nmf.CsrMatrix.from_dense(d)
    back = np.hstack([c.col_window(c0, c1).to_dense() for c0, c1 in cols])
    assert np.array_equal(back, c.to_dense())
