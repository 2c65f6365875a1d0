"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py

Every fixture is produced by the compiled reference library (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile) through oracle/ref_shim.cpp. Inputs and the
initial factors are rounded to float32 first (SURVEY.md §7 hard part 7), so the reference's
f64 arithmetic runs on exactly the values the B200 backend sees and only the arithmetic
precision differs. The GPU parity tests compare against these files; the CPU tests pin the
C restatement (oracle/mu_oracle.c) against them bit-for-bit.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

ref = oracle.ref


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def run_case(name, a, k, iters, interval, seed=0, extra=None):
    m, n = a.shape if not isinstance(a, tuple) else a[3]
    w0, h0 = ref.init_factors(m, n, k, seed)
    w0, h0 = f32(w0), f32(h0)
    r = ref.nmf_serial(a, k, w0, h0, max_iters=iters, interval=interval, eta=0.0)
    out = dict(k=k, iters=iters, interval=interval, seed=seed, trace_iters=r.trace_iters,
               trace_err=r.trace_err, w=r.w.astype(np.float32), h=r.h.astype(np.float32),
               w_fro=np.linalg.norm(r.w), h_fro=np.linalg.norm(r.h), w_sum=r.w.sum(), h_sum=r.h.sum())
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, r.trace_err[-1])


def main():
    # the reference on f64 inputs (no rounding) — pinned by the CPU tests.
    a = ref.uniform_dense(4096, 2048, 42, 99)
    r = ref.nmf_serial(a, 16, max_iters=100, interval=10, eta=0.0, seed=0)
    a_lr, _, _ = ref.gen_lowrank(4096, 2048, 16, 0.01, 7)
    r2 = ref.nmf_serial(a_lr, 16, max_iters=100, interval=10, eta=0.0, seed=0)
    w0, h0 = ref.init_factors(4096, 2048, 16, 0)
    appendix = {
        "config": "4096x2048, k=16, 100 it, interval 10, seed 0, eps 1e-12, eta 0, f64 inputs",
        "init": {"w0_00_02": w0[0, :3].tolist(), "h0_00_02": h0[0, :3].tolist()},
        "uniform": {"norm_a": float(np.sqrt((a * a).sum())), "trace": r.trace_err.tolist()},
        "lowrank": {"norm_a": float(np.sqrt((a_lr * a_lr).sum())), "trace": r2.trace_err.tolist()},
    }
    with open(os.path.join(HERE, "appendix_f64.json"), "w") as f:
        json.dump(appendix, f, indent=1)

    # Config 1 (BASELINE.json configs[0]) on f32-rounded inputs: uniform and low-rank A.
    run_case("config1_uniform_f32in", f32(a), 16, 100, 10)
    run_case("config1_lowrank_f32in", f32(a_lr), 16, 100, 10)
    # k = 32 / 64 and a non-power-of-two k (padding path), smaller shapes.
    a3 = f32(ref.uniform_dense(1536, 1024, 42, 99))
    run_case("uniform_1536x1024_k32", a3, 32, 50, 10)
    a4, _, _ = ref.gen_lowrank(1024, 768, 12, 0.0, 3)
    run_case("lowrank_1024x768_k64", f32(a4), 64, 30, 10)
    run_case("lowrank_1024x768_k5", f32(a4), 5, 40, 10)
    # Ragged, non-multiple-of-128 shape.
    a5, _, _ = ref.gen_lowrank(333, 517, 4, 0.05, 11)
    run_case("lowrank_333x517_k7", f32(a5), 7, 60, 7)
    # CSR: reference generator, values rounded to f32.
    rp, ci, v, shape = ref.gen_sparse(3000, 2500, 0.01, 5)
    run_case("csr_3000x2500_d001_k16", (rp, ci, f32(v), shape), 16, 40, 10,
             extra=dict(rp=rp, ci=ci, v=f32(v), shape=np.array(shape)))


if __name__ == "__main__":
    main()
