"""GPU parity at the BASELINE configs' real k and K (fixtures: tests/golden/make_golden_r2.py).

Same bar as tests/test_gpu_parity.py (BASELINE.json north_star): objective trajectory within
1e-4 relative, final W and H within 1e-3 relative Frobenius, the GPU's fp32 against the
reference's f64 on the same f32-rounded inputs and seeded init. Every fixture was produced by
the compiled reference (oracle/_ref); inputs are regenerated on the device with the generators
that tests/test_gpu_parity.py pins bit-for-bit against the reference's (src/synth.cpp:60-86,
bench/kernels_bench.cpp:12-18).
"""
import json
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


# ------------------------------------------------------------------ the one-pass kernel
@pytest.mark.parametrize("m,n,k,lookahead", [
    (4096, 2048, 16, "2"),     # config 1 shape, kp 16
    (1536, 1024, 32, "1"),     # NQ = 16 < 148 CTAs: most CTAs publish no P1 partial
    (333, 517, 7, "2"),        # ragged, one tile of padding each way
    (2048, 18944, 32, "3"),    # 148 column tiles: one owned tile per CTA
    (640, 40960, 32, "2"),     # 320 tiles: 2-3 owned tiles per CTA, 5 row blocks
    (128, 256, 32, "2"),       # one row block (D capped at 1), two column tiles
])
def test_fused_pass_matches_two_pass_kernels(gpu, monkeypatch, m, n, k, lookahead):
    """kernels_fused.cu (A read once per iteration: P1, the distributed W update, P2 from L2)
    against the two streaming passes + factor-update kernel (OOCNMF_FUSED=0) and the f64
    reference arithmetic (oracle port) on the same f32 inputs."""
    a = port.uniform_dense(m, n, 7, 99).astype(np.float32)
    w0, h0 = port.init_factors(m, n, k, 3)
    cfg = nmf.NmfConfig(k=k, max_iters=30, error_check_interval=10, eta=0.0, init=nmf.FactorInit.from_files,
                        init_w=f32(w0), init_h=f32(h0))
    monkeypatch.setenv("OOCNMF_FUSED", "1")  # these shapes are below the automatic threshold
    monkeypatch.setenv("OOCNMF_FUSED_D", lookahead)
    fused = nmf.nmf_serial(a, cfg)
    assert fused.info["fused_pass_launches"] == 30
    monkeypatch.setenv("OOCNMF_FUSED", "0")
    split = nmf.nmf_serial(a, cfg)
    assert split.info["fused_pass_launches"] == 0
    ref = port.nmf_serial(f32(a), k, f32(w0), f32(h0), max_iters=30, interval=10)
    ef = np.array([e for _, e in fused.error_trace])
    es = np.array([e for _, e in split.error_trace])
    np.testing.assert_allclose(ef, es, rtol=2e-6)
    assert np.all(np.abs(ef - ref.trace_err) <= TRACE_TOL * ref.trace_err)
    assert rel_fro(fused.w, ref.w) <= FACTOR_TOL and rel_fro(fused.h, ref.h) <= FACTOR_TOL
    assert rel_fro(fused.w, split.w) <= 1e-4 and rel_fro(fused.h, split.h) <= 1e-4


def test_fused_pass_is_deterministic(gpu, monkeypatch):
    monkeypatch.setenv("OOCNMF_FUSED", "1")
    a = port.uniform_dense(1024, 4096, 5, 99).astype(np.float32)
    w0, h0 = port.init_factors(1024, 4096, 32, 1)
    cfg = nmf.NmfConfig(k=32, max_iters=12, error_check_interval=4, eta=0.0, init=nmf.FactorInit.from_files,
                        init_w=f32(w0), init_h=f32(h0))
    r1, r2 = nmf.nmf_serial(a, cfg), nmf.nmf_serial(a, cfg)
    assert r1.info["fused_pass_launches"] == 12
    assert np.array_equal(r1.w, r2.w) and np.array_equal(r1.h, r2.h)
    assert [e for _, e in r1.error_trace] == [e for _, e in r2.error_trace]


# ------------------------------------------------------------------ k > 64 (wide factors)
def _wide_input(name):
    if name == "wide_lowrank_1024x768_k96":
        if not oracle.ref.available:
            pytest.skip("low-rank input regeneration needs oracle/_ref")
        return oracle.ref.gen_lowrank(1024, 768, 12, 0.01, 3)[0].astype(np.float32)
    return port.uniform_dense(512, 640, 42, 99).astype(np.float32)


@pytest.mark.parametrize("name", ["wide_lowrank_1024x768_k96", "wide_uniform_512x640_k200"])
@pytest.mark.parametrize("mode", ["in_core", "out_of_core", "cnmf"])
def test_wide_k_matches_reference(gpu, name, mode):
    """k > 64 (kp 128 / 256): the kp = 64 tensor-core passes per 64-column group, the wide factor /
    Gram / residual kernels (kernels_wide.cu), in core, streamed from host memory in row batches,
    and column-partitioned, against the compiled reference."""
    g = golden(name)
    a = _wide_input(name)
    m, n = a.shape
    cfg = cfg_from(g, m, n)
    if mode == "in_core":
        res = nmf.nmf_serial(a, cfg)
        trace, w, h = res.error_trace, res.w, res.h
    elif mode == "out_of_core":
        with nmf.Context(gpu) as ctx:
            ctx.set_problem(m, n, cfg.k)
            ctx.attach_host(np.ascontiguousarray(a), 256)
            ctx.set_factors(cfg.init_w, cfg.init_h)
            trace, _ = ctx.solve(cfg)
            w, h = ctx.get_factors()
    else:
        comm = nmf.DistComm(0, 1, gpu)
        try:
            res = nmf.nmf_distributed(a, cfg, nmf.make_plan(m, n, cfg.k, 1, 1, nmf.Strategy.cnmf), comm)
        finally:
            comm.close()
        trace, w, h = res.error_trace, res.w, res.h
    check_trace(trace, g)
    check_factors(w, h, g)


def test_wide_k_csr_matches_reference(gpu):
    base = golden("csr_3000x2500_d001_k16")
    g = golden("wide_csr_3000x2500_d001_k80")
    m, n = base["shape"].tolist()
    a = nmf.CsrMatrix(m, n, base["rp"], base["ci"], base["v"])
    res = nmf.nmf_serial(a, cfg_from(g, m, n))
    check_trace(res.error_trace, g)
    check_factors(res.w, res.h, g)


def test_wide_k_products_match_f64(gpu):
    m, n, k = 300, 520, 130  # kp 192: three groups, ragged k
    rng = np.random.default_rng(7)
    a = rng.random((m, n)).astype(np.float32)
    w = f32(rng.random((m, k)))
    h = f32(rng.random((k, n)))
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(m, n, k)
        ctx.load_dense(a)
        ctx.set_factors(w, h)
        aht, wta, hht, wtw = ctx.products()
    a64 = a.astype(np.float64)
    assert rel_fro(aht, a64 @ h.T) < 3e-6 and rel_fro(wta, w.T @ a64) < 3e-6
    assert rel_fro(hht, h @ h.T) < 3e-6 and rel_fro(wtw, w.T @ w) < 3e-6
    assert np.array_equal(hht, hht.T) and np.array_equal(wtw, wtw.T)


@pytest.mark.parametrize("fused", ["1", "0"])
def test_eta_exit_restores_the_factors_of_the_stopping_check(gpu, monkeypatch, fused):
    """eta > 0: the early exit (src/nmf_serial.cpp:111) is taken one block late so the device never
    waits on the host; the factors must still be those of the stopping check (snapshot
    restore), the trace must end there and iterations_run must match the reference."""
    g = golden("uniform_1536x1024_k32") if os.path.exists(os.path.join(GOLD, "uniform_1536x1024_k32.npz")) else None
    a = port.uniform_dense(1536, 1024, 42, 99).astype(np.float32)
    w0, h0 = port.init_factors(1536, 1024, 32, 0)
    full = port.nmf_serial(f32(a), 32, f32(w0), f32(h0), max_iters=50, interval=10)
    eta = 0.5 * (full.trace_err[2] + full.trace_err[3])  # between the checks at 30 and 40
    ref = port.nmf_serial(f32(a), 32, f32(w0), f32(h0), max_iters=50, interval=10, eta=eta)
    assert ref.converged and ref.iterations_run == 40
    cfg = nmf.NmfConfig(k=32, max_iters=50, error_check_interval=10, eta=eta, init=nmf.FactorInit.from_files,
                        init_w=f32(w0), init_h=f32(h0))
    monkeypatch.setenv("OOCNMF_FUSED", fused)
    r = nmf.nmf_serial(a, cfg)
    assert (r.info["fused_pass_launches"] > 0) == (fused == "1")
    assert r.converged and r.iterations_run == 40 and [i for i, _ in r.error_trace] == [10, 20, 30, 40]
    assert rel_fro(r.w, ref.w) <= FACTOR_TOL and rel_fro(r.h, ref.h) <= FACTOR_TOL
    assert rel_fro(r.w, full.w) > 10 * rel_fro(r.w, ref.w)  # not the factors of iteration 50
    if g is not None:
        np.testing.assert_allclose([e for _, e in r.error_trace], g["trace_err"][:4], rtol=TRACE_TOL)


_WGRAM = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle, paper_2202_09518_b200 as nmf
a = oracle.port.uniform_dense(1024, 4096, 5, 99).astype(np.float32)
w0, h0 = oracle.port.init_factors(1024, 4096, 32, 1)
f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
cfg = nmf.NmfConfig(k=32, max_iters=30, error_check_interval=10, eta=0.0, init=nmf.FactorInit.from_files,
                    init_w=f32(w0), init_h=f32(h0))
r = nmf.nmf_serial(a, cfg)
print(json.dumps({"trace": [e for _, e in r.error_trace], "w": float(np.linalg.norm(r.w)),
                  "h": float(np.linalg.norm(r.h)), "fused": r.info["fused_pass_launches"]}))
"""


def test_in_kernel_w_gram_matches_the_gram_pass(gpu):
    """The one-pass kernel's updaters accumulate W^T W of the new rows (f64 slots per CTA); the
    separate Gram pass (OOCNMF_FUSED_WGRAM=0) gives the same trajectory to f32 rounding."""
    import subprocess
    import sys

    out = {}
    for w in ("1", "0"):
        env = dict(os.environ, OOCNMF_FUSED="1", OOCNMF_FUSED_WGRAM=w)
        r = subprocess.run([sys.executable, "-c", _WGRAM, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))],
                           capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[w] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["1"]["fused"] == out["0"]["fused"] == 30
    np.testing.assert_allclose(out["1"]["trace"], out["0"]["trace"], rtol=1e-6)
    assert out["1"]["w"] == pytest.approx(out["0"]["w"], rel=1e-5)
    assert out["1"]["h"] == pytest.approx(out["0"]["h"], rel=1e-5)


def test_fused_pass_is_deterministic_at_scale(gpu):
    """The one-pass kernel at a config-2 row width (8192 x 65536: 64 row blocks, every slot of
    the partial ring reused 21 times, 3-4 owned tiles per CTA): two solves are bit-identical
    (fixed-order sums everywhere; a race in the publish / gather / discard / W-stage reuse
    paths would show up here as a difference)."""
    m, n, k = 8192, 65536, 32
    cfg = nmf.NmfConfig(k=k, max_iters=20, error_check_interval=10, eta=0.0, seed=3)
    outs = []
    for _ in range(2):
        with nmf.Context(gpu) as ctx:
            ctx.set_problem(m, n, k)
            ctx.generate_dense_uniform(42, 99)
            trace, info = ctx.solve(cfg)
            assert info["fused_pass_launches"] == 20
            outs.append((trace, *ctx.get_factors()))
    (t1, w1, h1), (t2, w2, h2) = outs
    assert [e for _, e in t1] == [e for _, e in t2]
    assert np.array_equal(w1, w2) and np.array_equal(h1, h2)


def test_context_reports_its_paths(gpu, monkeypatch):
    """Context.paths() (C-ABI oocnmf_ctx_paths): the shape dispatch between the one-pass kernel
    and the two streaming passes, and the CSR path."""
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(1024, 2048, 32)
        ctx.generate_dense_uniform(42, 99)
        p = ctx.paths()
        assert p["two_pass_tc"] and not p["one_pass"] and not p["csr"]
        monkeypatch.setenv("OOCNMF_FUSED", "1")
        ctx.set_rank(32)  # re-plans
        p = ctx.paths()
        assert p["one_pass"] and not p["two_pass_tc"]
    with nmf.Context(gpu) as ctx:
        ctx.set_problem(1000, 900, 16)
        ctx.generate_csr_uniform(0.01, 3)
        p = ctx.paths()
        assert p["csr"] and not p["one_pass"] and not p["nvls_h_update"]
