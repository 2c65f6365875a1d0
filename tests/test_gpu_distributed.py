"""The distributed drop-in boundary on the GPU: a reference-style C++ caller of
run_distributed_threads / spawn_group / CommHandle (tests/cpp/dist_demo.cpp, compiled unchanged
against the reference header names) and the Python mirror, against the CPU oracle's
row-partitioned run (oracle/mu_oracle.c, pinned to src/nmf_distributed.cpp:151-289).

One rank per visible GPU (up to 4); on a one-GPU box the group is the loopback backend.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
port = oracle.port


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def _workers():
    return max(1, min(nmf.device_count(), 4))


def test_cpp_run_distributed_threads_is_a_drop_in(gpu):
    workers = _workers()
    m, n, k = 700, 500, 8
    exe = os.path.join(ROOT, "paper_2202_09518_b200", "lib", "dist_demo")
    out = subprocess.run([exe, str(workers), str(m), str(n), str(k)], capture_output=True, text=True, check=True,
                         timeout=300).stdout
    lines = [json.loads(x) for x in out.strip().splitlines() if x.startswith("{")]  # (NCCL may print a banner)
    trace = [d["err"] for d in lines if "err" in d]
    a = f32(port.uniform_dense(m, n, 42, 99))
    w0, h0 = port.init_factors(m, n, k, 0)
    ref = port.nmf_rnmf(a, k, f32(w0), f32(h0), n_workers=workers, max_iters=30, interval=10)
    np.testing.assert_allclose(trace, ref.trace_err, rtol=1e-4)
    norms = [d for d in lines if "w_fro" in d][0]
    assert norms["ranks"] == workers and norms["identical"]
    assert norms["w_fro"] == pytest.approx(np.linalg.norm(ref.w), rel=1e-3)
    assert norms["h_fro"] == pytest.approx(np.linalg.norm(ref.h), rel=1e-3)
    st = [d for d in lines if "h_update_calls" in d][0]
    if workers > 1:
        # per iteration one grouped all-reduce of [W^T A | W^T W], or (sharded H, OOCNMF_SHARD_H=1)
        # a grouped reduce-scatter + Gram all-reduce and an H all-gather; one W gather;
        # ||A||^2 and per check the residual (+ the sharded cross term) all-reduce
        # (CollectiveStats per PhaseTag, comm.hpp:28-43)
        sharded = os.environ.get("OOCNMF_SHARD_H") == "1" and 512 % (128 * workers) == 0
        assert st["h_update_calls"] == (60 if sharded else 30) and st["gather_calls"] == 1
        assert st["error_check_calls"] == 1 + 3 * (2 if sharded else 1)
        assert st["h_update_bytes"] > 30 * (512 * 8 * 4)
    grp = [d for d in lines if "allreduce_last" in d][0]
    assert grp["allreduce_last"] == 6.0 * workers * (workers + 1) / 2
    assert grp["generic_calls"] == 1 and grp["barrier_calls"] == 1
    assert any(d.get("shape_error") for d in lines)


def test_python_run_distributed_threads_matches_oracle(gpu):
    workers = _workers()
    m, n, k = 640, 480, 16
    a = port.uniform_dense(m, n, 3, 99).astype(np.float32)
    w0, h0 = port.init_factors(m, n, k, 0)
    cfg = nmf.NmfConfig(k=k, max_iters=20, error_check_interval=10, eta=0.0, init=nmf.FactorInit.from_files,
                        init_w=f32(w0), init_h=f32(h0))
    plan = nmf.make_plan(m, n, k, workers, 1, nmf.Strategy.rnmf)
    stats = []
    res = nmf.run_distributed_threads(a, cfg, plan, stats_out=stats)
    ref = port.nmf_rnmf(f32(a), k, f32(w0), f32(h0), n_workers=workers, max_iters=20, interval=10)
    assert len(res) == workers and len(stats) == workers
    for r in res:
        np.testing.assert_allclose([e for _, e in r.error_trace], ref.trace_err, rtol=1e-4)
        assert np.linalg.norm(r.w - ref.w) <= 1e-3 * np.linalg.norm(ref.w)
        assert np.array_equal(r.w, res[0].w) and np.array_equal(r.h, res[0].h)
    if workers > 1:
        sharded = os.environ.get("OOCNMF_SHARD_H") == "1" and 512 % (128 * workers) == 0
        assert stats[0].calls[nmf.PhaseTag.h_update] == (40 if sharded else 20)
        assert stats[0].seconds[nmf.PhaseTag.h_update] > 0


def test_group_collectives_and_stats(gpu):
    import threading

    workers = _workers()
    group = nmf.spawn_group(workers)
    out = [None] * workers

    def work(r):
        buf = np.arange(6, dtype=np.float64) * (r + 1)
        group[r].all_reduce_sum(buf, nmf.PhaseTag.gather)
        group[r].barrier()
        out[r] = buf

    ts = [threading.Thread(target=work, args=(r,)) for r in range(workers)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    want = np.arange(6, dtype=np.float64) * workers * (workers + 1) / 2
    for r in range(workers):
        assert np.array_equal(out[r], want)
        s = group[r].stats()
        assert s.calls[nmf.PhaseTag.gather] == 1 and s.bytes[nmf.PhaseTag.gather] == 48
        assert s.calls[nmf.PhaseTag.barrier] == 1
        group[r].reset_stats()
        assert group[r].stats().total_calls() == 0
    for g in group:
        g.close()
    with pytest.raises(nmf.ShapeError):
        nmf.spawn_group(nmf.device_count() + 1)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_file_source_over_budget_streams_out_of_core(gpu, tmp_path, dtype):
    """ASource::file with a StoreConfig budget the rank's dense window exceeds (the reference's
    ChunkStore over a PDN1 file, src/chunk_store.cpp:106-168): the window is read once into
    page-locked host memory and streamed in budget-sized row batches every iteration; the result
    equals the in-HBM solve and StoreCounters report the loads / bytes / residency."""
    m, n, k = 1000, 700, 8
    d = f32(port.uniform_dense(m, n, 9, 99))
    nmf.write_pdn1(tmp_path / "a.pdn1", d, dtype=dtype)
    cfg = nmf.NmfConfig(k=k, max_iters=20, error_check_interval=10, eta=0.0, seed=4, device=gpu)
    plan = nmf.make_plan(m, n, k, 1, 1, nmf.Strategy.rnmf)
    budget = 2 * 256 * 768 * 4  # two 256-row staging batches of the padded 768-column layout
    comm = nmf.DistComm(0, 1, gpu)
    try:
        sc = nmf.StoreCounters()
        ooc = nmf.nmf_distributed(str(tmp_path / "a.pdn1"), cfg, plan, comm,
                                  store_cfg=nmf.StoreConfig(budget_bytes=budget), store_counters=sc)
        sc_mem = nmf.StoreCounters()
        mem = nmf.nmf_distributed(str(tmp_path / "a.pdn1"), cfg, plan, comm, store_counters=sc_mem)
    finally:
        comm.close()
    np.testing.assert_allclose([e for _, e in ooc.error_trace], [e for _, e in mem.error_trace], rtol=5e-6)
    assert np.linalg.norm(ooc.w - mem.w) <= 1e-5 * np.linalg.norm(mem.w)
    assert sc.loads == 20 * 4 and sc.evictions == sc.loads - 2  # 4 batches of <= 256 rows per iteration
    assert sc.bytes_read == m * n * (4 if dtype == "f32" else 8) and sc.io_seconds > 0
    assert sc.peak_resident_bytes == 2 * 256 * 768 * 4 <= budget
    assert sc_mem.loads == 1 and sc_mem.peak_resident_bytes == m * 768 * 4


_NVLS_THREADS = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle, paper_2202_09518_b200 as nmf
workers = int(sys.argv[2])
rp, ci, v, (m, n) = oracle.port.gen_sparse(1100, 2048, 0.02, 8)
a = nmf.CsrMatrix(m, n, rp, ci, v.astype(np.float32).astype(np.float64))
w0, h0 = oracle.port.init_factors(m, n, 16, 0)
f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
cfg = nmf.NmfConfig(k=16, max_iters=20, error_check_interval=10, eta=0.0, init=nmf.FactorInit.from_files,
                    init_w=f32(w0), init_h=f32(h0))
stats = []
res = nmf.run_distributed_threads(a, cfg, nmf.make_plan(m, n, 16, workers, 1, nmf.Strategy.rnmf), stats_out=stats)
print(json.dumps({"trace": [[e for _, e in r.error_trace] for r in res],
                  "w": [float(np.linalg.norm(r.w)) for r in res], "h": [float(np.linalg.norm(r.h)) for r in res],
                  "h_calls": stats[0].calls[nmf.PhaseTag.h_update]}))
"""


@pytest.mark.parametrize("nvls", ["1", "0"])
def test_threads_backend_sharded_csr_nvls(gpu, nvls):
    """The sharded CSR H update over the threads backend (one process, ncclCommInitAll), with the
    NVLS kernel (kernels_nvls.cu) forced on and off: both match the oracle's row-partitioned run."""
    workers = _workers()
    if workers < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, OOCNMF_NVLS=nvls)
    out = subprocess.run([sys.executable, "-c", _NVLS_THREADS, ROOT, str(workers)], capture_output=True, text=True,
                         env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    rp, ci, v, shape = port.gen_sparse(1100, 2048, 0.02, 8)
    w0, h0 = port.init_factors(1100, 2048, 16, 0)
    ref = port.nmf_rnmf((rp, ci, f32(v), shape), 16, f32(w0), f32(h0), workers, 1, max_iters=20, interval=10)
    for tr in d["trace"]:
        np.testing.assert_allclose(tr, ref.trace_err, rtol=1e-4)
    assert d["w"][0] == pytest.approx(np.linalg.norm(ref.w), rel=1e-3)
    assert d["h"][0] == pytest.approx(np.linalg.norm(ref.h), rel=1e-3)
    # NVLS: 2 h_update collectives on the 18 non-check iterations (W^T W + the fused kernel) and
    # the NCCL path's 6 (4 reduce-scatter chunks, W^T W, all-gather) on the 2 check iterations
    assert d["h_calls"] == (18 * 2 + 2 * 6 if nvls == "1" else 20 * 6)
