"""GPU parity at the BASELINE configs' real k and K (fixtures: tests/golden/make_golden_r2.py).

Same bar as tests/test_gpu_parity.py (BASELINE.json north_star): objective trajectory within
1e-4 relative, final W and H within 1e-3 relative Frobenius, the GPU's fp32 against the
reference's f64 on the same f32-rounded inputs and seeded init. Every fixture was produced by
the compiled reference (oracle/_ref); inputs are regenerated on the device with the generators
that tests/test_gpu_parity.py pins bit-for-bit against the reference's (src/synth.cpp:60-86,
bench/kernels_bench.cpp:12-18).
"""
import os

import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
port = oracle.port

TRACE_TOL = 1e-4
FACTOR_TOL = 1e-3


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def rel_fro(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def golden(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def check_trace(trace, g):
    got_it = np.array([i for i, _ in trace])
    got = np.array([e for _, e in trace])
    ref = np.asarray(g["trace_err"])
    assert np.array_equal(got_it, np.asarray(g["trace_iters"])), (got_it, g["trace_iters"])
    assert np.all(np.abs(got - ref) <= TRACE_TOL * ref), (got, ref)
    return float(np.max(np.abs(got - ref) / ref))


def check_factors(w, h, g):
    ws, hs = int(g["w_stride"]), int(g["h_stride"])
    assert rel_fro(w[::ws], g["w"]) <= FACTOR_TOL, rel_fro(w[::ws], g["w"])
    assert rel_fro(h[:, ::hs], g["h"]) <= FACTOR_TOL, rel_fro(h[:, ::hs], g["h"])
    assert abs(np.linalg.norm(w) / float(g["w_fro"]) - 1) <= FACTOR_TOL
    assert abs(np.linalg.norm(h) / float(g["h_fro"]) - 1) <= FACTOR_TOL


def cfg_from(g, m, n, **kw):
    k = int(g["k"])
    w0, h0 = port.init_factors(m, n, k, int(g["seed"]))
    return nmf.NmfConfig(k=k, max_iters=int(g["iters"]), error_check_interval=int(g["interval"]), eta=0.0,
                         init=nmf.FactorInit.from_files, init_w=f32(w0), init_h=f32(h0), **kw)


# ------------------------------------------------------------------ CSR at config 3's kp
CSR_MODES = {
    "fused": {},
    "split": {"OOCNMF_FUSE_W": "0", "OOCNMF_FUSE_H": "0"},
    "chunked": {"OOCNMF_SPMM_CHUNK_MB": "0.01", "OOCNMF_SPMM_CHUNK_FORCE": "1"},
}


@pytest.mark.parametrize("name", ["csr_3000x2500_d001_k32", "csr_3000x2500_d001_k48"])
@pytest.mark.parametrize("mode", list(CSR_MODES))
def test_csr_kp32_kp64_match_reference(gpu, monkeypatch, name, mode):
    """k = 32 runs the kp = 32 SpMMs (k_spmm_v4<32>, k_spmm_mu<32>: 8 lanes per row), k = 48 the
    kp = 64 ones, in the fused (default), split and column-chunked configurations."""
    for key, val in CSR_MODES[mode].items():
        monkeypatch.setenv(key, val)
    base = golden("csr_3000x2500_d001_k16")
    g = golden(name)
    m, n = base["shape"].tolist()
    a = nmf.CsrMatrix(m, n, base["rp"], base["ci"], base["v"])
    res = nmf.nmf_serial(a, cfg_from(g, m, n))
    check_trace(res.error_trace, g)
    check_factors(res.w, res.h, g)


@pytest.mark.parametrize("mode", ["fused", "split"])
def test_config3_scaled_matches_reference(gpu, monkeypatch, mode):
    """Config 3 scaled to 2^15 x 2^15 at density 4e-3 (4.3 M entries, ~131 per row), k = 32,
    20 iterations, the reference generator evaluated on the device."""
    for key, val in CSR_MODES[mode].items():
        monkeypatch.setenv(key, val)
    g = golden("csr_config3_scaled_32768_d4e-3_k32")
    m, n, seed = g["gen"].tolist()
    cfg = cfg_from(g, m, n)
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(m, n, cfg.k)
        ctx.generate_csr_uniform(float(g["density"]), seed)
        nnz = ctx.download_csr().nnz
        assert nnz == int(g["nnz"])
        ctx.set_factors(cfg.init_w, cfg.init_h)
        trace, info = ctx.solve(cfg)
        w, h = ctx.get_factors()
    check_trace(trace, g)
    check_factors(w, h, g)


# ------------------------------------------------------------------ dense: config 2's K
@pytest.mark.parametrize("name,m,n", [("longk_1024x65536_k32", 1024, 65536), ("longk_65536x1024_k32", 65536, 1024)])
def test_long_k_matches_reference(gpu, name, m, n):
    """65536-deep passes: 1024 K steps per tile in pass 1 (1024 x 65536) / pass 2
    (65536 x 1024), i.e. 512 drained two-step chains summed in f32 registers per tile."""
    g = golden(name)
    cfg = cfg_from(g, m, n)
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(m, n, cfg.k)
        ctx.generate_dense_uniform(42, 99)
        ctx.set_factors(cfg.init_w, cfg.init_h)
        trace, info = ctx.solve(cfg)
        w, h = ctx.get_factors()
    check_trace(trace, g)
    check_factors(w, h, g)


def test_config2_two_iterations_match_reference(gpu):
    """Config 2 itself (65536 x 65536, k = 32), an error check after each of 2 iterations, against
    the reference run on the same f32-rounded A (0.502504328195 at iteration
    2 on the f64 A)."""
    g = golden("config2_65536_k32_2it")
    m = n = 65536
    cfg = cfg_from(g, m, n)
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(m, n, cfg.k)
        ctx.generate_dense_uniform(42, 99)
        ctx.set_factors(cfg.init_w, cfg.init_h)
        trace, info = ctx.solve(cfg)
        w, h = ctx.get_factors()
    check_trace(trace, g)
    check_factors(w, h, g)
    assert abs(trace[-1][1] - 0.502504328195) <= 1e-4 * 0.502504328195
