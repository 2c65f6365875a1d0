"""TEST INFRASTRUCTURE ONLY — CPU parity oracle for the MU-NMF hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker; the product
(``paper_2202_09518_b200``) never imports it.

Two checkers, both f64:

* :data:`port` — ``oracle/mu_oracle.c``, a plain-C restatement of the reference's
  ``nmf_serial`` (src/nmf_serial.cpp:56-121) and row-partitioned ``nmf_distributed``
  (src/nmf_distributed.cpp:151-289) keeping the reference's summation order.
* :data:`ref` — ``oracle/_ref/libref_oocnmf.so``, the reference library compiled from its
  own sources (oracle/Makefile) behind ``oracle/ref_shim.cpp``. Absent on a box that never
  had /root/reference unless the prebuilt .so travelled with the snapshot.

tests/test_oracle.py pins ``port`` bit-for-bit against ``ref`` and both against the golden
vectors in tests/golden/ (SURVEY.md Appendix + fixtures made by tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "_build", "libmu_oracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libref_oocnmf.so")

_u64 = C.c_uint64
_dbl = C.c_double
_pd = C.POINTER(C.c_double)
_pu = C.POINTER(C.c_uint64)
_pi = C.POINTER(C.c_int)


def _ptr(a, t=_pd):
    return None if a is None else a.ctypes.data_as(t)


def build() -> None:
    """Compile the oracle libraries (make -f oracle/Makefile)."""
    import subprocess

    subprocess.run(["make", "-s", "-f", os.path.join(_HERE, "Makefile"), "-j8"], check=True)


@dataclass
class Result:
    w: np.ndarray
    h: np.ndarray
    trace_iters: np.ndarray
    trace_err: np.ndarray
    iterations_run: int
    converged: bool
    counters: dict = field(default_factory=dict)

    @property
    def error_trace(self):
        return list(zip(self.trace_iters.tolist(), self.trace_err.tolist()))


class _Lib:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self._lib = None

    @property
    def available(self) -> bool:
        return os.path.exists(self.path)

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(self.path):
                raise FileNotFoundError(f"oracle library {self.path} not built (make -f oracle/Makefile)")
            self._lib = C.CDLL(self.path)
        return self._lib


class Port(_Lib):
    """ctypes front-end of oracle/mu_oracle.c."""

    def __init__(self):
        super().__init__(PORT_PATH, "mo_")

    def uniform_dense(self, rows, n, seed, stream, row0=0):
        out = np.empty((rows, n), np.float64)
        f = self.lib.mo_uniform_dense
        f.argtypes = [_u64, _u64, _u64, _u64, _u64, _pd]
        f(row0, rows, n, seed, stream, _ptr(out))
        return out

    def init_factors(self, m, n, k, seed):
        w = np.empty((m, k), np.float64)
        h = np.empty((k, n), np.float64)
        f = self.lib.mo_init_factors
        f.argtypes = [_u64, _u64, _u64, _u64, _pd, _pd]
        f(m, n, k, seed, _ptr(w), _ptr(h))
        return w, h

    def _run(self, fn, pre_args, m, n, k, w0, h0, max_iters, interval, eta, eps, post_args=()):
        w = np.ascontiguousarray(w0, np.float64).copy()
        h = np.ascontiguousarray(h0, np.float64).copy()
        cap = max_iters // interval + 2
        ti = np.zeros(cap, np.uint64)
        te = np.zeros(cap, np.float64)
        nt, run, conv = _u64(), _u64(), C.c_int()
        st = fn(*pre_args, *post_args, max_iters, interval, eta, eps, _ptr(w), _ptr(h), _ptr(ti, _pu),
                _ptr(te), cap, C.byref(nt), C.byref(run), C.byref(conv))
        if st == 1:
            raise ValueError("oracle: invalid shape/config")
        if st == 2:
            raise ArithmeticError("oracle: zero-norm A or non-finite factors")
        ntr = min(nt.value, cap)
        return Result(w, h, ti[:ntr].astype(np.int64), te[:ntr], run.value, bool(conv.value))

    def nmf_serial(self, a, k, w0, h0, max_iters=100, interval=10, eta=0.0, eps=1e-12):
        """Dense ``a`` (m x n ndarray) or CSR triple ``(row_ptr, col_idx, vals, (m, n))``."""
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp = np.ascontiguousarray(rp, np.uint64)
            ci = np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            f = self.lib.mo_nmf_serial_csr
            f.argtypes = [_pu, _pu, _pd, _u64, _u64, _u64, _u64, _u64, _dbl, _dbl, _pd, _pd, _pu, _pd,
                          _u64, _pu, _pu, _pi]
            return self._run(f, (_ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), m, n, k), m, n, k, w0, h0,
                             max_iters, interval, eta, eps)
        a = np.ascontiguousarray(a, np.float64)
        m, n = a.shape
        f = self.lib.mo_nmf_serial_dense
        f.argtypes = [_pd, _u64, _u64, _u64, _u64, _u64, _dbl, _dbl, _pd, _pd, _pu, _pd, _u64, _pu,
                      _pu, _pi]
        return self._run(f, (_ptr(a), m, n, k), m, n, k, w0, h0, max_iters, interval, eta, eps)

    def nmf_rnmf(self, a, k, w0, h0, n_workers, n_b=1, max_iters=100, interval=10, eta=0.0, eps=1e-12):
        """Row-partitioned distributed MU simulated over ``n_workers`` ranks (threads-backend
        semantics: ascending-rank all-reduce)."""
        f = self.lib.mo_nmf_rnmf
        f.argtypes = [_pd, _pu, _pu, _pd, _u64, _u64, _u64, _u64, _u64, _u64, _u64, _dbl, _dbl, _pd,
                      _pd, _pu, _pd, _u64, _pu, _pu, _pi]
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp = np.ascontiguousarray(rp, np.uint64)
            ci = np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            pre = (None, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), m, n, k, n_workers, n_b)
        else:
            a = np.ascontiguousarray(a, np.float64)
            m, n = a.shape
            pre = (_ptr(a), None, None, None, m, n, k, n_workers, n_b)
        return self._run(f, pre, m, n, k, w0, h0, max_iters, interval, eta, eps)

    def mu_iteration(self, a, w, h, eps=1e-12):
        a = np.ascontiguousarray(a, np.float64)
        m, n = a.shape
        k = w.shape[1]
        f = self.lib.mo_mu_iteration
        f.argtypes = [_pd, _u64, _u64, _u64, _pd, _pd, _dbl]
        f(_ptr(a), m, n, k, _ptr(w), _ptr(h), eps)

    def relative_error(self, a, w, h):
        w = np.ascontiguousarray(w, np.float64)
        h = np.ascontiguousarray(h, np.float64)
        k = w.shape[1]
        f = self.lib.mo_relative_error
        f.restype = _dbl
        f.argtypes = [_pd, _pu, _pu, _pd, _u64, _u64, _u64, _pd, _pd]
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp = np.ascontiguousarray(rp, np.uint64)
            ci = np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            return f(None, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), m, n, k, _ptr(w), _ptr(h))
        a = np.ascontiguousarray(a, np.float64)
        m, n = a.shape
        return f(_ptr(a), None, None, None, m, n, k, _ptr(w), _ptr(h))

    def gen_sparse(self, m, n, density, seed):
        f = self.lib.mo_gen_sparse
        f.argtypes = [_u64, _u64, _dbl, _u64, _pu, _pu, _pd, _pu]
        rp = np.zeros(m + 1, np.uint64)
        nnz = _u64()
        f(m, n, density, seed, _ptr(rp, _pu), None, None, C.byref(nnz))
        ci = np.zeros(nnz.value, np.uint64)
        v = np.zeros(nnz.value, np.float64)
        f(m, n, density, seed, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), C.byref(nnz))
        return rp, ci, v, (m, n)

    def split_even(self, extent, parts):
        f = self.lib.mo_split_even
        f.argtypes = [_u64, _u64, _pu]
        out = np.zeros(parts + 1, np.uint64)
        f(extent, parts, _ptr(out, _pu))
        return out.astype(np.int64)


class Ref(_Lib):
    """ctypes front-end of the compiled reference (oracle/_ref)."""

    def __init__(self):
        super().__init__(REF_PATH, "ref_")

    def _err(self):
        f = self.lib.ref_last_error
        f.restype = C.c_char_p
        return f().decode()

    def _check(self, st):
        if st == 0:
            return
        msg = self._err()
        raise {1: ValueError, 2: ArithmeticError, 3: OSError, 4: RuntimeError, 5: RuntimeError}.get(
            st, RuntimeError)(f"reference: {msg}")

    def _res(self, m, n, k, cap):
        return (np.zeros((m, k)), np.zeros((k, n)), np.zeros(cap, np.uint64), np.zeros(cap), _u64(), _u64(),
                C.c_int(), np.zeros(7))

    def _pack(self, w, h, ti, te, nt, run, conv, cnt, cap):
        ntr = min(nt.value, cap)
        keys = ["w_update_s", "h_update_s", "allreduce_s", "error_check_s", "io_s", "total_s", "flops"]
        return Result(w, h, ti[:ntr].astype(np.int64), te[:ntr], run.value, bool(conv.value),
                      dict(zip(keys, cnt.tolist())))

    def nmf_serial(self, a, k, w0=None, h0=None, max_iters=100, interval=10, eta=0.0, eps=1e-12, seed=0):
        cap = max_iters // interval + 2
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
        else:
            a = np.ascontiguousarray(a, np.float64)
            m, n = a.shape
        w, h, ti, te, nt, run, conv, cnt = self._res(m, n, k, cap)
        w0p = _ptr(np.ascontiguousarray(w0, np.float64)) if w0 is not None else None
        h0p = _ptr(np.ascontiguousarray(h0, np.float64)) if h0 is not None else None
        keep = (w0, h0)
        if w0 is not None:
            keep = (np.ascontiguousarray(w0, np.float64), np.ascontiguousarray(h0, np.float64))
            w0p, h0p = _ptr(keep[0]), _ptr(keep[1])
        tail = (max_iters, interval, eta, eps, seed, w0p, h0p, _ptr(w), _ptr(h), _ptr(ti, _pu), _ptr(te), cap,
                C.byref(nt), C.byref(run), C.byref(conv), _ptr(cnt))
        tail_t = [_u64, _u64, _dbl, _dbl, _u64, _pd, _pd, _pd, _pd, _pu, _pd, _u64, _pu, _pu, _pi, _pd]
        if isinstance(a, tuple):
            rp = np.ascontiguousarray(rp, np.uint64)
            ci = np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            f = self.lib.ref_nmf_serial_csr
            f.argtypes = [_pu, _pu, _pd, _u64, _u64, _u64] + tail_t
            st = f(_ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), m, n, k, *tail)
        else:
            f = self.lib.ref_nmf_serial_dense
            f.argtypes = [_pd, _u64, _u64, _u64] + tail_t
            st = f(_ptr(a), m, n, k, *tail)
        self._check(st)
        del keep
        return self._pack(w, h, ti, te, nt, run, conv, cnt, cap)

    def nmf_distributed(self, a, k, n_workers, n_b=1, strategy=2, w0=None, h0=None, max_iters=100,
                        interval=10, eta=0.0, eps=1e-12, seed=0):
        cap = max_iters // interval + 2
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp = np.ascontiguousarray(rp, np.uint64)
            ci = np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            ad, rpp, cip, vp = None, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v)
        else:
            a = np.ascontiguousarray(a, np.float64)
            m, n = a.shape
            ad, rpp, cip, vp = _ptr(a), None, None, None
        w, h, ti, te, nt, run, conv, cnt = self._res(m, n, k, cap)
        keep = None
        w0p = h0p = None
        if w0 is not None:
            keep = (np.ascontiguousarray(w0, np.float64), np.ascontiguousarray(h0, np.float64))
            w0p, h0p = _ptr(keep[0]), _ptr(keep[1])
        f = self.lib.ref_nmf_distributed
        f.argtypes = [_pd, _pu, _pu, _pd, _u64, _u64, _u64, C.c_int, _u64, C.c_int, _u64, _u64, _dbl, _dbl,
                      _u64, _pd, _pd, _pd, _pd, _pu, _pd, _u64, _pu, _pu, _pi, _pd]
        st = f(ad, rpp, cip, vp, m, n, k, n_workers, n_b, strategy, max_iters, interval, eta, eps, seed, w0p,
               h0p, _ptr(w), _ptr(h), _ptr(ti, _pu), _ptr(te), cap, C.byref(nt), C.byref(run), C.byref(conv),
               _ptr(cnt))
        self._check(st)
        del keep
        return self._pack(w, h, ti, te, nt, run, conv, cnt, cap)

    def init_factors(self, m, n, k, seed):
        w = np.empty((m, k))
        h = np.empty((k, n))
        f = self.lib.ref_init_factors
        f.argtypes = [_u64, _u64, _u64, _u64, _pd, _pd]
        self._check(f(m, n, k, seed, _ptr(w), _ptr(h)))
        return w, h

    def gen_lowrank(self, m, n, k_true, noise, seed):
        a = np.empty((m, n))
        w0 = np.empty((m, k_true))
        h0 = np.empty((k_true, n))
        f = self.lib.ref_gen_lowrank
        f.argtypes = [_u64, _u64, _u64, _dbl, _u64, _pd, _pd, _pd]
        self._check(f(m, n, k_true, noise, seed, _ptr(a), _ptr(w0), _ptr(h0)))
        return a, w0, h0

    def gen_sparse(self, m, n, density, seed):
        f = self.lib.ref_gen_sparse
        f.argtypes = [_u64, _u64, _dbl, _u64, _pu, _pu, _pd, _pu]
        rp = np.zeros(m + 1, np.uint64)
        nnz = _u64()
        self._check(f(m, n, density, seed, _ptr(rp, _pu), None, None, C.byref(nnz)))
        ci = np.zeros(nnz.value, np.uint64)
        v = np.zeros(nnz.value)
        self._check(f(m, n, density, seed, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v), C.byref(nnz)))
        return rp, ci, v, (m, n)

    def uniform_dense(self, rows, n, seed, stream, row0=0):
        out = np.empty((rows, n))
        f = self.lib.ref_uniform_dense
        f.argtypes = [_u64, _u64, _u64, _u64, _u64, _pd]
        self._check(f(row0, rows, n, seed, stream, _ptr(out)))
        return out

    def make_plan(self, m, n, k, n_workers, n_b, strategy=0):
        slabs = np.zeros((n_workers, 4), np.uint64)
        bat = np.zeros((n_b, 2), np.uint64)
        so = C.c_int()
        f = self.lib.ref_make_plan
        f.argtypes = [_u64, _u64, _u64, C.c_int, _u64, C.c_int, _pu, _pu, _pi]
        self._check(f(m, n, k, n_workers, n_b, strategy, _ptr(slabs, _pu), _ptr(bat, _pu), C.byref(so)))
        return {"strategy": "cnmf" if so.value == 1 else "rnmf", "slabs": slabs.astype(np.int64),
                "batches": bat.astype(np.int64)}

    # Bench reference arm: keep A resident in the library across timed iterations.
    def dense_handle(self, a):
        a = np.ascontiguousarray(a, np.float64)
        f = self.lib.ref_dense_create
        f.restype = C.c_void_p
        f.argtypes = [_pd, _u64, _u64]
        return f(_ptr(a), a.shape[0], a.shape[1])

    def dense_free(self, hnd):
        f = self.lib.ref_dense_destroy
        f.argtypes = [C.c_void_p]
        f(hnd)

    def mu_iteration_handle(self, hnd, w, h, eps=1e-12):
        f = self.lib.ref_mu_iteration_handle
        f.argtypes = [C.c_void_p, _u64, _pd, _pd, _dbl]
        self._check(f(hnd, w.shape[1], _ptr(w), _ptr(h), eps))

    def plan_to_json(self, m, n, k, n_workers, n_b, strategy):
        f = self.lib.ref_plan_to_json
        f.restype = C.c_long
        f.argtypes = [_u64, _u64, _u64, C.c_int, _u64, C.c_int, C.c_char_p, _u64]
        buf = C.create_string_buffer(1 << 20)
        ln = f(m, n, k, n_workers, n_b, strategy, buf, len(buf))
        return buf.raw[:ln].decode()

    def memreport_to_json(self, values7, feasible):
        f = self.lib.ref_memreport_to_json
        f.restype = C.c_long
        f.argtypes = [_pu, C.c_int, C.c_char_p, _u64]
        v = np.ascontiguousarray(values7, np.uint64)
        buf = C.create_string_buffer(4096)
        ln = f(_ptr(v, _pu), int(feasible), buf, len(buf))
        return buf.raw[:ln].decode()

    def json_reformat(self, text, indent=2):
        """nlohmann::json::parse(text).dump(indent) with the reference's JSON library."""
        f = self.lib.ref_json_reformat
        f.restype = C.c_long
        f.argtypes = [C.c_char_p, C.c_int, C.c_char_p, _u64]
        buf = C.create_string_buffer(1 << 22)
        ln = f(text.encode(), indent, buf, len(buf))
        if ln < 0:
            raise ValueError(f"json_reformat failed ({ln}): {self._err()}")
        return buf.raw[:ln].decode()

    def selection_json_csv(self, records, chosen, rationale):
        """The reference's SelectionReport::to_json / to_csv for the given records."""
        rec = np.array([[r["k"], float(r["valid"]), r["runs_used"], r["min_silhouette"], r["mean_silhouette"],
                         r["mean_relative_error"]] for r in records], np.float64).reshape(-1, 6)
        f = self.lib.ref_selection_json_csv
        f.restype = C.c_long
        f.argtypes = [_pd, _u64, C.c_int64, C.c_char_p, C.c_char_p, _u64, C.c_char_p, _u64]
        jb, cb = C.create_string_buffer(1 << 20), C.create_string_buffer(1 << 20)
        rec = np.ascontiguousarray(rec)
        assert f(_ptr(rec), len(rec), -1 if chosen is None else chosen, rationale.encode(), jb, len(jb), cb,
                 len(cb)) == 0
        return jb.value.decode(), cb.value.decode()

    def dense_uniform_handle(self, m, n, seed=42, stream=99, round_f32=True):
        """The uniform synthetic A built in place inside the library (no numpy copy)."""
        f = self.lib.ref_dense_create_uniform
        f.restype = C.c_void_p
        f.argtypes = [_u64, _u64, _u64, _u64, C.c_int]
        return f(m, n, seed, stream, 1 if round_f32 else 0)

    def nmf_serial_handle(self, hnd, m, n, k, w0=None, h0=None, max_iters=100, interval=10, eta=0.0, eps=1e-12,
                          seed=0):
        cap = max_iters // interval + 2
        w, h, ti, te, nt, run, conv, cnt = self._res(m, n, k, cap)
        keep = None
        w0p = h0p = None
        if w0 is not None:
            keep = (np.ascontiguousarray(w0, np.float64), np.ascontiguousarray(h0, np.float64))
            w0p, h0p = _ptr(keep[0]), _ptr(keep[1])
        f = self.lib.ref_nmf_serial_dense_handle
        f.argtypes = [C.c_void_p, _u64, _u64, _u64, _dbl, _dbl, _u64, _pd, _pd, _pd, _pd, _pu, _pd, _u64, _pu, _pu,
                      _pi, _pd]
        st = f(hnd, k, max_iters, interval, eta, eps, seed, w0p, h0p, _ptr(w), _ptr(h), _ptr(ti, _pu), _ptr(te),
               cap, C.byref(nt), C.byref(run), C.byref(conv), _ptr(cnt))
        self._check(st)
        del keep
        return self._pack(w, h, ti, te, nt, run, conv, cnt, cap)

    def csr_handle(self, rp, ci, v, m, n):
        self._csr_keep = (np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint64),
                          np.ascontiguousarray(v, np.float64))
        f = self.lib.ref_csr_create
        f.restype = C.c_void_p
        f.argtypes = [_pu, _pu, _pd, _u64, _u64]
        return f(_ptr(self._csr_keep[0], _pu), _ptr(self._csr_keep[1], _pu), _ptr(self._csr_keep[2]), m, n)

    def csr_free(self, hnd):
        f = self.lib.ref_csr_destroy
        f.argtypes = [C.c_void_p]
        f(hnd)

    def mu_iteration_csr_handle(self, hnd, w, h, eps=1e-12):
        f = self.lib.ref_mu_iteration_csr_handle
        f.argtypes = [C.c_void_p, _u64, _pd, _pd, _dbl]
        self._check(f(hnd, w.shape[1], _ptr(w), _ptr(h), eps))

    # ---- model selection (include/oocnmf/model_selection.hpp) ----
    def select_k(self, a, k_min, k_max, n_perturbations=16, delta=0.03, sil_threshold=0.75, max_iters=500,
                 interval=10, eta=1e-6, eps=1e-12, seed=0):
        """Reference select_k on a dense A: (records list of dicts, chosen_k or None, medians list, rationale)."""
        a = np.ascontiguousarray(a, np.float64)
        m, n = a.shape
        nk = k_max - k_min + 1
        rec = np.zeros((nk, 6))
        med = np.zeros(sum(m * k for k in range(k_min, k_max + 1)))
        chosen = C.c_int64()
        why = C.create_string_buffer(512)
        f = self.lib.ref_select_k_dense
        f.argtypes = [_pd, _u64, _u64, _u64, _u64, _u64, _dbl, _dbl, _u64, _u64, _dbl, _dbl, _u64, _pd,
                      C.POINTER(C.c_int64), _pd, C.c_char_p, _u64]
        self._check(f(_ptr(a), m, n, k_min, k_max, n_perturbations, delta, sil_threshold, max_iters, interval,
                      eta, eps, seed, _ptr(rec), C.byref(chosen), _ptr(med), why, 512))
        records, meds, off = [], [], 0
        for i, k in enumerate(range(k_min, k_max + 1)):
            records.append(dict(k=int(rec[i, 0]), valid=bool(rec[i, 1]), runs_used=int(rec[i, 2]),
                                min_silhouette=rec[i, 3], mean_silhouette=rec[i, 4], mean_relative_error=rec[i, 5]))
            meds.append(med[off:off + m * k].reshape(m, k))
            off += m * k
        return records, (None if chosen.value < 0 else chosen.value), meds, why.value.decode()

    def cluster_silhouette(self, runs):
        """Reference cluster_columns + silhouette over runs (R x m x k)."""
        runs = np.ascontiguousarray(runs, np.float64)
        r, m, k = runs.shape
        med, per = np.zeros((m, k)), np.zeros(k)
        mn, mean, dropped = _dbl(), _dbl(), _u64()
        member = np.zeros(r * k, np.int64)
        f = self.lib.ref_cluster_silhouette
        f.argtypes = [_pd, _u64, _u64, _u64, _pd, _pd, _pd, _pd, _pu, C.POINTER(C.c_int64)]
        self._check(f(_ptr(runs), r, m, k, _ptr(med), _ptr(per), C.byref(mn), C.byref(mean), C.byref(dropped),
                      member.ctypes.data_as(C.POINTER(C.c_int64))))
        return dict(medians=med, per_cluster=per, min_sil=mn.value, mean_sil=mean.value, dropped=dropped.value,
                    member_cluster=member.reshape(r, k))

    def pearson(self, w_true, w_est):
        w_true = np.ascontiguousarray(w_true, np.float64)
        w_est = np.ascontiguousarray(w_est, np.float64)
        corr = np.zeros((w_true.shape[1], w_est.shape[1]))
        f = self.lib.ref_pearson
        f.argtypes = [_pd, _u64, _u64, _pd, _u64, _pd]
        self._check(f(_ptr(w_true), w_true.shape[0], w_true.shape[1], _ptr(w_est), w_est.shape[1], _ptr(corr)))
        return corr

    def perturb_dense(self, a, delta, seed):
        a = np.ascontiguousarray(a, np.float64)
        out = np.zeros_like(a)
        f = self.lib.ref_perturb_dense
        f.argtypes = [_pd, _u64, _u64, _dbl, _u64, _pd]
        self._check(f(_ptr(a), a.shape[0], a.shape[1], delta, seed, _ptr(out)))
        return out

    # ---- matrix files (include/oocnmf/io.hpp) ----
    def write_pdn1(self, path, a):
        b = str(path).encode()
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp, ci = np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            f = self.lib.ref_write_pdn1_csr
            f.argtypes = [C.c_char_p, _u64, _u64, _pu, _pu, _pd]
            self._check(f(b, m, n, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v)))
        else:
            a = np.ascontiguousarray(a, np.float64)
            f = self.lib.ref_write_pdn1_dense
            f.argtypes = [C.c_char_p, _pd, _u64, _u64]
            self._check(f(b, _ptr(a), a.shape[0], a.shape[1]))

    def write_mtx(self, path, a):
        b = str(path).encode()
        if isinstance(a, tuple):
            rp, ci, v, (m, n) = a
            rp, ci = np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint64)
            v = np.ascontiguousarray(v, np.float64)
            f = self.lib.ref_write_mtx_csr
            f.argtypes = [C.c_char_p, _u64, _u64, _pu, _pu, _pd]
            self._check(f(b, m, n, _ptr(rp, _pu), _ptr(ci, _pu), _ptr(v)))
        else:
            a = np.ascontiguousarray(a, np.float64)
            f = self.lib.ref_write_mtx_dense
            f.argtypes = [C.c_char_p, _pd, _u64, _u64]
            self._check(f(b, _ptr(a), a.shape[0], a.shape[1]))

    def read_matrix(self, path):
        """dense ndarray or (row_ptr, col_idx, values, (m, n))"""
        b = str(path).encode()
        f = self.lib.ref_read_matrix
        f.argtypes = [C.c_char_p, _pi, _pu, _pu, _pu, _pd, _pu, _pu, _pd]
        kind, m, n, nnz = C.c_int(), _u64(), _u64(), _u64()
        self._check(f(b, C.byref(kind), C.byref(m), C.byref(n), C.byref(nnz), None, None, None, None))
        if kind.value == 0:
            d = np.zeros((m.value, n.value))
            self._check(f(b, C.byref(kind), C.byref(m), C.byref(n), C.byref(nnz), _ptr(d), None, None, None))
            return d
        rp, ci, v = np.zeros(m.value + 1, np.uint64), np.zeros(nnz.value, np.uint64), np.zeros(nnz.value)
        self._check(f(b, C.byref(kind), C.byref(m), C.byref(n), C.byref(nnz), None, _ptr(rp, _pu), _ptr(ci, _pu),
                      _ptr(v)))
        return rp, ci, v, (m.value, n.value)


port = Port()
ref = Ref()
