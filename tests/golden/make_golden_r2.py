"""Round-2 golden fixtures: the BASELINE configs' real k and K, made by the reference itself.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden_r2.py [name ...]

Like make_golden.py, every value comes from the compiled reference library (oracle/_ref, built
from /root/reference/proj/src by oracle/Makefile) on f32-rounded inputs and init, so the GPU
parity tests compare arithmetic precision only. The fixtures pin the cases round 1 left open:

* CSR at k = 32 and k = 48 (the kp = 32 / kp = 64 SpMM instantiations config 3 runs);
* config 3 scaled to 2^15 x 2^15 at density 4e-3 with the reference generator
  (src/synth.cpp:60-86), k = 32, 20 iterations;
* long-K dense shapes (1024 x 65536 and 65536 x 1024, k = 32, 10 iterations): config 2's
  65536-deep passes;
* config 2 itself (65536 x 65536, k = 32) for 2 iterations with an error check after each;
* k > 64 (96, 200 dense; 80 CSR): the wide-factor path.

Large factors are stored as strided samples (rows of W, columns of H) plus their full
Frobenius norms and sums; the tests compare the same samples (relative Frobenius on the sample).
Inputs are not stored: the tests regenerate them with the oracle's generators (pinned
bit-for-bit against the reference in tests/test_oracle.py) or the device generators.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

ref = oracle.ref


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def run_case(name, a, shape, k, iters, interval, seed=0, w_stride=1, h_stride=1, extra=None):
    m, n = shape
    t = time.time()
    w0, h0 = ref.init_factors(m, n, k, seed)
    w0, h0 = f32(w0), f32(h0)
    r = ref.nmf_serial(a, k, w0, h0, max_iters=iters, interval=interval, eta=0.0)
    out = dict(k=k, iters=iters, interval=interval, seed=seed, trace_iters=r.trace_iters, trace_err=r.trace_err,
               w_stride=w_stride, h_stride=h_stride,
               w=r.w[::w_stride].astype(np.float32), h=r.h[:, ::h_stride].astype(np.float32),
               w_fro=np.linalg.norm(r.w), h_fro=np.linalg.norm(r.h), w_sum=r.w.sum(), h_sum=r.h.sum(),
               iterations_run=r.iterations_run)
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: {r.trace_err.tolist()} ({time.time() - t:.1f} s)", flush=True)


def csr_k32_k48():
    g = np.load(os.path.join(HERE, "csr_3000x2500_d001_k16.npz"))
    m, n = g["shape"].tolist()
    a = (g["rp"], g["ci"], g["v"].astype(np.float64), (m, n))
    run_case("csr_3000x2500_d001_k32", a, (m, n), 32, 40, 10)
    run_case("csr_3000x2500_d001_k48", a, (m, n), 48, 30, 10)


def csr_config3_scaled():
    m = n = 1 << 15
    rp, ci, v, shape = ref.gen_sparse(m, n, 4e-3, 3)
    a = (rp, ci, f32(v), shape)
    run_case("csr_config3_scaled_32768_d4e-3_k32", a, (m, n), 32, 20, 10, w_stride=8, h_stride=8,
             extra=dict(nnz=len(ci), gen=np.array([m, n, 3]), density=4e-3))


def long_k():
    a = f32(ref.uniform_dense(1024, 65536, 42, 99))
    run_case("longk_1024x65536_k32", a, a.shape, 32, 10, 2, h_stride=16)
    del a
    a = f32(ref.uniform_dense(65536, 1024, 42, 99))
    run_case("longk_65536x1024_k32", a, a.shape, 32, 10, 2, w_stride=16)


def config2():
    m = n = 65536
    k, iters, interval = 32, 2, 1
    t = time.time()
    hnd = ref.dense_uniform_handle(m, n, 42, 99, round_f32=True)  # 34 GB, built in place
    w0, h0 = ref.init_factors(m, n, k, 0)
    w0, h0 = f32(w0), f32(h0)
    r = ref.nmf_serial_handle(hnd, m, n, k, w0, h0, max_iters=iters, interval=interval, eta=0.0)
    ref.dense_free(hnd)
    ws = hs = 64
    np.savez_compressed(os.path.join(HERE, "config2_65536_k32_2it.npz"), k=k, iters=iters, interval=interval, seed=0,
                        trace_iters=r.trace_iters, trace_err=r.trace_err, w_stride=ws, h_stride=hs,
                        w=r.w[::ws].astype(np.float32), h=r.h[:, ::hs].astype(np.float32),
                        w_fro=np.linalg.norm(r.w), h_fro=np.linalg.norm(r.h), w_sum=r.w.sum(), h_sum=r.h.sum(),
                        iterations_run=r.iterations_run)
    print(f"config2_65536_k32_2it: {r.trace_err.tolist()} ({time.time() - t:.1f} s)", flush=True)


def wide():
    # k > 64 (kp 128 / 256: the paper's scaling study runs k = 128 and 256)
    a, _, _ = ref.gen_lowrank(1024, 768, 12, 0.01, 3)
    run_case("wide_lowrank_1024x768_k96", f32(a), a.shape, 96, 30, 10)
    a = f32(ref.uniform_dense(512, 640, 42, 99))
    run_case("wide_uniform_512x640_k200", a, a.shape, 200, 20, 10)
    g = np.load(os.path.join(HERE, "csr_3000x2500_d001_k16.npz"))
    m, n = g["shape"].tolist()
    run_case("wide_csr_3000x2500_d001_k80", (g["rp"], g["ci"], g["v"].astype(np.float64), (m, n)), (m, n), 80, 20, 10)


CASES = {"csr": csr_k32_k48, "config3": csr_config3_scaled, "longk": long_k, "config2": config2, "wide": wide}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
