"""Python mirror of the reference's MU-NMF API (``oocnmf::`` in /root/reference/proj/include),
driving the B200 C-ABI backend. Names, argument meaning and error behaviour follow the
reference so parity tests read like its own:

* :class:`NmfConfig` / :class:`NmfResult` / :class:`PhaseCounters` — include/oocnmf/nmf.hpp:15-48
* :func:`init_factors` — include/oocnmf/nmf.hpp:53-58 (same counter RNG, bit-identical f64)
* :func:`nmf_serial` — include/oocnmf/nmf.hpp:64, src/nmf_serial.cpp:56-121
* :func:`make_plan` / :func:`choose_strategy` — include/oocnmf/partition.hpp:10-46
* :func:`nmf_distributed` — include/oocnmf/nmf_distributed.hpp:34-36 (row partition)
* exceptions — include/oocnmf/error.hpp:9-36 (+ :class:`DeviceError`)

All arithmetic happens on the GPU; this layer validates, converts and maps status codes.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi


# ----------------------------------------------------------------------------- errors
class ShapeError(ValueError):
    """Contract violation: shapes, windows, configs (reference ShapeError: std::invalid_argument)."""


class DataError(RuntimeError):
    """||A||_F == 0 or non-finite factors."""


class IoError(OSError):
    pass


class CommError(RuntimeError):
    pass


class StoreError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    """CUDA failure or no B200 device (the backend has no CPU fallback)."""


_STATUS = {1: ShapeError, 2: DataError, 3: IoError, 4: CommError, 5: StoreError, 6: DeviceError}


def check(status: int) -> None:
    if status != 0:
        msg = _capi.lib().oocnmf_last_error().decode()
        raise _STATUS.get(status, DeviceError)(msg)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


# ----------------------------------------------------------------------------- types
class FactorInit(enum.Enum):
    uniform01 = 0
    from_files = 1
    resident = 2  # B200 extension: continue from the factors left on the device by a previous solve


@dataclass
class NmfConfig:
    k: int = 1
    eta: float = 1e-4
    max_iters: int = 1000
    error_check_interval: int = 10
    epsilon: float = 1e-12
    seed: int = 0
    init: FactorInit = FactorInit.uniform01
    init_w: Optional[np.ndarray] = None
    init_h: Optional[np.ndarray] = None
    # B200 extensions
    device: int = 0
    error_mode: str = "auto"  # "auto" | "direct" | "trace"

    def validate(self) -> None:
        if self.k < 1:
            raise ShapeError("NmfConfig: k must be >= 1")
        if not self.eta >= 0:
            raise ShapeError("NmfConfig: eta must be >= 0")
        if self.max_iters < 1:
            raise ShapeError("NmfConfig: max_iters must be >= 1")
        if self.error_check_interval < 1:
            raise ShapeError("NmfConfig: error_check_interval must be >= 1")
        if not self.epsilon > 0:
            raise ShapeError("NmfConfig: epsilon must be > 0")
        if self.init == FactorInit.from_files and (self.init_w is None or self.init_h is None):
            raise ShapeError("NmfConfig: init=from_files requires both factors")
        if self.error_mode not in ("auto", "direct", "trace"):
            raise ShapeError("NmfConfig: error_mode must be 'auto', 'direct' or 'trace'")

    def to_c(self) -> _capi.Config:
        return _capi.Config(self.k, self.eta, self.max_iters, self.error_check_interval, self.epsilon,
                            self.seed, self.init.value,
                            {"auto": 0, "direct": 1, "trace": 2}[self.error_mode])


@dataclass
class PhaseCounters:
    h_update_s: float = 0.0
    w_update_s: float = 0.0
    allreduce_s: float = 0.0
    error_check_s: float = 0.0
    io_s: float = 0.0
    total_s: float = 0.0
    flops: float = 0.0
    peak_resident_bytes: int = 0


@dataclass
class NmfResult:
    w: np.ndarray
    h: np.ndarray
    error_trace: List[Tuple[int, float]]
    iterations_run: int
    converged: bool
    counters: PhaseCounters = field(default_factory=PhaseCounters)
    info: dict = field(default_factory=dict)  # device-side timing / launch counts


class CsrMatrix:
    """CSR with u64 indices and f64 values (reference CsrMatrix, matrix.hpp:63-102)."""

    def __init__(self, rows, cols, row_ptr, col_idx, values, _validated=False):
        self.rows, self.cols = int(rows), int(cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
        self.col_idx = np.ascontiguousarray(col_idx, np.uint64)
        self.values = np.ascontiguousarray(values, np.float64)
        if not _validated:  # (downloads of a resident CSR were checked when it was loaded)
            self.validate_structure()

    @property
    def nnz(self):
        return int(self.values.size)

    @property
    def shape(self):
        return (self.rows, self.cols)

    def validate_structure(self):
        rp, ci = self.row_ptr, self.col_idx
        if rp.size != self.rows + 1:
            raise ShapeError("CsrMatrix: row_ptr must have rows+1 entries")
        if rp[0] != 0:
            raise ShapeError("CsrMatrix: row_ptr[0] != 0")
        if rp[-1] != self.values.size or ci.size != self.values.size:
            raise ShapeError("CsrMatrix: row_ptr[rows] disagrees with nnz")
        if np.any(np.diff(rp.astype(np.int64)) < 0):
            raise ShapeError("CsrMatrix: row_ptr decreases")
        if ci.size and np.any(ci >= self.cols):
            raise ShapeError("CsrMatrix: column index out of range")
        if ci.size > 1:
            d = np.diff(ci.astype(np.int64))
            starts = np.zeros(ci.size, bool)
            starts[rp[:-1][rp[:-1] < ci.size].astype(np.int64)] = True
            if np.any((d <= 0) & ~starts[1:]):
                raise ShapeError("CsrMatrix: column indices not strictly increasing within a row")

    def to_dense(self):
        d = np.zeros((self.rows, self.cols))
        rows = np.repeat(np.arange(self.rows), np.diff(self.row_ptr.astype(np.int64)))
        d[rows, self.col_idx.astype(np.int64)] = self.values
        return d

    @staticmethod
    def from_dense(d, zero_tol=0.0):
        d = np.asarray(d, np.float64)
        mask = np.abs(d) > zero_tol
        rp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.uint64)
        r, c = np.nonzero(mask)
        return CsrMatrix(d.shape[0], d.shape[1], rp, c, d[r, c])

    def row_window(self, r0, r1):
        rp = self.row_ptr[r0:r1 + 1].astype(np.int64)
        b, e = int(rp[0]), int(rp[-1])
        return CsrMatrix(r1 - r0, self.cols, (rp - b).astype(np.uint64), self.col_idx[b:e], self.values[b:e])

    def col_window(self, c0, c1):
        """All rows, columns [c0, c1), column indices rebased to the window."""
        ci = self.col_idx.astype(np.int64)
        keep = (ci >= c0) & (ci < c1)
        rows = np.repeat(np.arange(self.rows), np.diff(self.row_ptr.astype(np.int64)))
        rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=self.rows))]).astype(np.uint64)
        return CsrMatrix(self.rows, c1 - c0, rp, (ci[keep] - c0).astype(np.uint64), self.values[keep])


# ----------------------------------------------------------------------------- helpers
def device_count() -> int:
    n = C.c_int()
    check(_capi.lib().oocnmf_device_count(C.byref(n)))
    return n.value


def init_factors(m: int, n: int, k: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """W (m x k) ~ U(seed, 1, i*k+j), H (k x n) ~ U(seed, 2, r*n+j) — reference counter RNG."""
    if m < 1 or n < 1 or k < 1:
        raise ShapeError("init_factors: dimensions must be >= 1")
    w = np.empty((m, k))
    h = np.empty((k, n))
    check(_capi.lib().oocnmf_init_factors_host(m, n, k, seed, _p(w, C.c_double), _p(h, C.c_double)))
    return w, h


def counter_uniform(seed: int, stream: int, index0: int, count: int) -> np.ndarray:
    out = np.empty(count)
    check(_capi.lib().oocnmf_counter_uniform(seed, stream, index0, count, _p(out, C.c_double)))
    return out


def split_even(extent: int, parts: int) -> np.ndarray:
    out = np.zeros(parts + 1, np.uint64)
    check(_capi.lib().oocnmf_split_even(extent, parts, _p(out, C.c_uint64)))
    return out.astype(np.int64)


# ----------------------------------------------------------------------------- context
class Context:
    """One GPU's solver context (C-ABI ``oocnmf_ctx``)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, unique_id: Optional[bytes] = None):
        self._h = C.c_void_p()
        L = _capi.lib()
        if nranks > 1:
            if unique_id is None or len(unique_id) != 128:
                raise ShapeError("Context: a 128-byte NCCL unique id is required for nranks > 1")
            check(L.oocnmf_ctx_create_comm(device, rank, nranks, unique_id, C.byref(self._h)))
        else:
            check(L.oocnmf_ctx_create(device, C.byref(self._h)))
        self.device, self.rank, self.nranks = device, rank, nranks
        self.m = self.n = self.k = self.row0 = self.rows = 0
        self._keep = None

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_capi.lib().oocnmf_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if self._h:
            _capi.lib().oocnmf_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_problem(self, m, n, k, row0=0, rows=None):
        rows = m - row0 if rows is None else rows
        check(_capi.lib().oocnmf_set_problem(self._h, m, n, k, row0, rows))
        self.m, self.n, self.k, self.row0, self.rows = m, n, k, row0, rows
        self.n_global, self.col0 = n, 0

    def load_dense(self, a: np.ndarray):
        a = np.asarray(a)
        if a.shape != (self.rows, self.n):
            raise ShapeError(f"load_dense: expected {self.rows}x{self.n}, got {a.shape}")
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        # a row window of a larger array (the reference's MatrixRef window) goes in place, with
        # its row stride as lda; anything else is made contiguous first
        it = a.itemsize
        if not (a.strides[1] == it and a.strides[0] % it == 0 and a.strides[0] >= a.shape[1] * it):
            a = np.ascontiguousarray(a)
        lda = a.strides[0] // it if a.shape[0] > 1 else self.n
        if a.dtype == np.float32:
            check(_capi.lib().oocnmf_load_dense_f32(self._h, C.cast(a.ctypes.data, C.POINTER(C.c_float)), lda))
        else:
            check(_capi.lib().oocnmf_load_dense_f64(self._h, C.cast(a.ctypes.data, C.POINTER(C.c_double)), lda))

    def load_dense_device(self, ptr: int, lda: int):
        check(_capi.lib().oocnmf_load_dense_device_f32(self._h, C.c_void_p(ptr), lda))

    def download_dense(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = np.empty((self.rows, self.n), np.float32) if out is None else out
        if out.dtype != np.float32 or out.shape != (self.rows, self.n) or not out.flags.c_contiguous:
            raise ShapeError("download_dense: expected a C-contiguous float32 rows x n array")
        check(_capi.lib().oocnmf_download_dense_f32(self._h, out.ctypes.data))
        return out

    def generate_dense_uniform(self, seed=42, stream=99):
        check(_capi.lib().oocnmf_generate_dense_uniform(self._h, seed, stream))

    def load_csr(self, a: CsrMatrix):
        if a.shape != (self.rows, self.n):
            raise ShapeError(f"load_csr: expected {self.rows}x{self.n}, got {a.shape}")
        check(_capi.lib().oocnmf_load_csr_f64(self._h, _p(a.row_ptr, C.c_uint64), _p(a.col_idx, C.c_uint64),
                                              _p(a.values, C.c_double)))

    def generate_csr_uniform(self, density, seed):
        check(_capi.lib().oocnmf_generate_csr_uniform(self._h, density, seed))

    def download_csr(self) -> CsrMatrix:
        nnz = C.c_uint64()
        check(_capi.lib().oocnmf_csr_nnz(self._h, C.byref(nnz)))
        rp = np.empty(self.rows + 1, np.uint64)
        ci = np.empty(max(nnz.value, 1), np.uint64)
        v = np.empty(max(nnz.value, 1))
        check(_capi.lib().oocnmf_download_csr(self._h, _p(rp, C.c_uint64), _p(ci, C.c_uint64), _p(v, C.c_double)))
        return CsrMatrix(self.rows, self.n, rp, ci[:nnz.value], v[:nnz.value], _validated=True)

    def attach_host(self, a: np.ndarray, batch_rows: int = 0):
        """Out-of-core: ``a`` (rows x n float32, ideally pinned) stays in host memory."""
        if a.dtype != np.float32 or a.shape != (self.rows, self.n) or not a.flags.c_contiguous:
            raise ShapeError("attach_host: expected a C-contiguous float32 rows x n array")
        self._keep = a
        check(_capi.lib().oocnmf_attach_host_dense_f32(self._h, a.ctypes.data, self.n, batch_rows))

    def set_factors(self, w: np.ndarray, h: np.ndarray):
        w = np.ascontiguousarray(w, np.float64)
        h = np.ascontiguousarray(h, np.float64)
        if w.shape != (self.rows, self.k) or h.shape != (self.k, self.n):
            raise ShapeError("set_factors: factor shapes do not match the problem")
        check(_capi.lib().oocnmf_set_factors_f64(self._h, _p(w, C.c_double), _p(h, C.c_double)))

    def get_factors(self):
        w = np.empty((self.rows, self.k))
        h = np.empty((self.k, self.n))
        check(_capi.lib().oocnmf_get_factors_f64(self._h, _p(w, C.c_double), _p(h, C.c_double)))
        return w, h

    def set_problem_cols(self, m, n, k, col0, cols):
        """Column partition (CNMF): all m rows, columns [col0, col0 + cols) of the m x n A."""
        check(_capi.lib().oocnmf_set_problem_cols(self._h, m, n, k, col0, cols))
        self.m, self.n, self.k, self.row0, self.rows = m, cols, k, 0, m
        self.n_global, self.col0 = n, col0

    def gather_w(self):
        w = np.empty((self.m, self.k))
        check(_capi.lib().oocnmf_gather_w_f64(self._h, _p(w, C.c_double)))
        return w

    def gather_h(self):
        """CNMF: the full H (k x n_global) on every rank."""
        h = np.empty((self.k, self.n_global))
        check(_capi.lib().oocnmf_gather_h_f64(self._h, _p(h, C.c_double)))
        return h

    def solve(self, cfg: NmfConfig):
        cfg.validate()
        cap = cfg.max_iters // cfg.error_check_interval + 2
        ti = np.zeros(cap, np.uint64)
        te = np.zeros(cap)
        info = _capi.Info()
        c = cfg.to_c()
        check(_capi.lib().oocnmf_solve(self._h, C.byref(c), _p(ti, C.c_uint64), _p(te, C.c_double), cap,
                                       C.byref(info)))
        nt = min(int(info.n_trace), cap)
        return list(zip(ti[:nt].astype(int).tolist(), te[:nt].tolist())), info.as_dict()

    def paths(self) -> Dict[str, bool]:
        """Which B200 paths the current problem runs (reporting only)."""
        f = C.c_int()
        check(_capi.lib().oocnmf_ctx_paths(self._h, C.byref(f)))
        names = ("one_pass", "two_pass_tc", "nvls_h_update", "sharded_h", "csr", "out_of_core")
        return {n: bool(f.value >> i & 1) for i, n in enumerate(names)}

    def set_rank(self, k: int):
        """Change k keeping the resident A (model selection sweeps k over one matrix)."""
        check(_capi.lib().oocnmf_set_rank(self._h, k))
        self.k = k

    def perturb(self, delta: float, seed: int):
        """A <- A0 o U[1-delta, 1+delta] on the device (perturb_dense / perturb_sparse semantics,
        model_selection.cpp:35-60); delta = 0 restores the loaded values."""
        check(_capi.lib().oocnmf_perturb(self._h, float(delta), int(seed)))

    def products(self):
        k, n, rows = self.k, self.n, self.rows
        aht, wta = np.empty((rows, k)), np.empty((k, n))
        hht, wtw = np.empty((k, k)), np.empty((k, k))
        check(_capi.lib().oocnmf_products_f64(self._h, *(_p(x, C.c_double) for x in (aht, wta, hht, wtw))))
        return aht, wta, hht, wtw

    def sq_norm(self):
        out = C.c_double()
        check(_capi.lib().oocnmf_sq_norm(self._h, C.byref(out)))
        return out.value


def _counters(info: dict) -> PhaseCounters:
    return PhaseCounters(**{f: info[f] for f in PhaseCounters.__dataclass_fields__})


# ----------------------------------------------------------------------------- solvers
def nmf_serial(a, cfg: NmfConfig) -> NmfResult:
    """Single-GPU MU-NMF, W update before H update (src/nmf_serial.cpp:56-121).

    ``a``: 2-D ndarray (float64 or float32, nonnegative) or :class:`CsrMatrix`.
    """
    cfg.validate()
    m, n = (a.rows, a.cols) if isinstance(a, CsrMatrix) else np.asarray(a).shape
    if m < 1 or n < 1:
        raise ShapeError(f"nmf_serial: empty input {m}x{n}")
    if cfg.init == FactorInit.from_files:
        if cfg.init_w.shape != (m, cfg.k) or cfg.init_h.shape != (cfg.k, n):
            raise ShapeError("nmf_serial: provided factors do not match A and k")
    with Context(cfg.device) as ctx:
        ctx.set_problem(m, n, cfg.k)
        if isinstance(a, CsrMatrix):
            ctx.load_csr(a)
        else:
            ctx.load_dense(a)
        if cfg.init == FactorInit.from_files:
            ctx.set_factors(cfg.init_w, cfg.init_h)
        trace, info = ctx.solve(cfg)
        w, h = ctx.get_factors()
    return NmfResult(w, h, trace, int(info["iterations_run"]), bool(info["converged"]), _counters(info), info)


class Strategy(enum.Enum):
    cnmf = "cnmf"
    rnmf = "rnmf"


def choose_strategy(m: int, n: int) -> Strategy:
    """CNMF iff n > m (src/partition.cpp:12-14)."""
    return Strategy.cnmf if n > m else Strategy.rnmf


def _ref_json(d) -> str:
    """The reference's nlohmann dump(2) layout: sorted keys, 2-space indent, arrays of numbers on
    one line without spaces."""
    import json
    import re
    s = json.dumps(d, indent=2, sort_keys=True)
    return re.sub(r"\[\s*((?:-?\d+,\s*)*-?\d+)\s*\]", lambda mt: "[" + re.sub(r"\s+", "", mt.group(1)) + "]", s)


@dataclass
class PartitionPlan:
    strategy: Strategy
    n_workers: int
    m: int
    n: int
    k: int
    n_b: int
    slabs: List[Tuple[Tuple[int, int], Tuple[int, int]]]  # per rank: ((row0,row1),(col0,col1))
    batches: List[Tuple[int, int]]

    def to_json(self) -> str:
        """The reference's plan JSON (src/partition.cpp:89-104, nlohmann dump(2))."""
        col = self.strategy == Strategy.cnmf
        d = {"strategy": self.strategy.value, "n_workers": self.n_workers, "m": self.m, "n": self.n, "k": self.k,
             "n_b": self.n_b, "w_role": "replicated" if col else "slab", "h_role": "slab" if col else "replicated"}
        if self.slabs:
            d["workers"] = [{"rank": r, "a_rows": list(rows), "a_cols": list(cols)}
                            for r, (rows, cols) in enumerate(self.slabs)]
        if self.batches:
            d["batches"] = [list(b) for b in self.batches]
        return _ref_json(d)


def make_plan(m, n, k, n_workers, n_b, strategy: Strategy) -> PartitionPlan:
    """Even split with the remainder on the first ranks (src/partition.cpp:49-87)."""
    if m < 1 or n < 1 or k < 1:
        raise ShapeError("make_plan: dimensions must be >= 1")
    if n_workers < 1:
        raise ShapeError("make_plan: need at least one worker")
    if n_b < 1:
        raise ShapeError("make_plan: need at least one batch")
    col = strategy == Strategy.cnmf
    part, bat = (n, m) if col else (m, n)
    if n_workers > part:
        raise ShapeError(f"make_plan: {n_workers} workers exceed the {part} slabs available under {strategy.value}")
    if n_b > bat:
        raise ShapeError(f"make_plan: {n_b} batches exceed the {bat}-extent batched axis")
    s = split_even(part, n_workers)
    b = split_even(bat, n_b)
    slabs = [(((0, m), (int(s[r]), int(s[r + 1]))) if col else ((int(s[r]), int(s[r + 1])), (0, n)))
             for r in range(n_workers)]
    return PartitionPlan(strategy, n_workers, m, n, k, n_b, slabs,
                         [(int(b[i]), int(b[i + 1])) for i in range(n_b)])


@dataclass
class MemoryReport:
    """Per-rank device bytes of the B200 layout (reference MemoryReport, partition.hpp:51-61)."""
    a_slab_bytes: int
    store_peak_bytes: int
    factor_bytes: int
    intermediate_bytes: int
    peak_bytes: int
    min_n_b: int  # 1: in-core fits; > 1: out-of-core row batches; 0: infeasible
    feasible: bool
    in_core: bool

    def to_json(self) -> str:
        """The reference's report JSON (src/partition.cpp:199-209; in_core is not serialised)."""
        return _ref_json({k: getattr(self, k) for k in ("a_slab_bytes", "store_peak_bytes", "factor_bytes",
                                                        "intermediate_bytes", "peak_bytes", "min_n_b", "feasible")})


def memory_estimate(plan: "PartitionPlan", density: float, budget_bytes: int, n_cb: int = 1,
                    num_sms: int = 0) -> MemoryReport:
    """memory_estimate (src/partition.cpp:147-197) for this backend's device layout."""
    if n_cb < 1:
        raise ShapeError("memory_estimate: n_cb must be >= 1")
    r = _capi.MemoryReport()
    check(_capi.lib().oocnmf_memory_estimate(plan.m, plan.n, plan.k, plan.n_workers,
                                             1 if plan.strategy == Strategy.cnmf else 2, float(density),
                                             int(budget_bytes), num_sms, C.byref(r)))
    return MemoryReport(int(r.a_slab_bytes), int(r.store_peak_bytes), int(r.factor_bytes),
                        int(r.intermediate_bytes), int(r.peak_bytes), int(r.min_n_b), bool(r.feasible),
                        bool(r.in_core))


def exchange_unique_id(rank: int, make_id, device: Optional[int] = None, group=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL unique id to every rank with torch.distributed
    (gloo or nccl process group; plumbing only)."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid = make_id()
        if len(uid) != 128:
            raise ShapeError("exchange_unique_id: the id must be 128 bytes")
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
    if dist.get_backend(group) == "nccl":
        t = t.cuda(device)
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


class PhaseTag(enum.IntEnum):
    """Collective tags (include/oocnmf/comm.hpp:13-20)."""
    generic = 0
    w_update = 1
    h_update = 2
    error_check = 3
    gather = 4
    barrier = 5


@dataclass
class CollectiveStats:
    """Per-tag collective statistics (include/oocnmf/comm.hpp:28-43): bytes, calls, seconds
    (device time of the collectives, the solve's own included)."""
    bytes: Dict[PhaseTag, int] = field(default_factory=dict)
    calls: Dict[PhaseTag, int] = field(default_factory=dict)
    seconds: Dict[PhaseTag, float] = field(default_factory=dict)

    def total_bytes(self) -> int:
        return sum(self.bytes.values())

    def total_calls(self) -> int:
        return sum(self.calls.values())

    def total_seconds(self) -> float:
        return sum(self.seconds.values())


class DistComm:
    """One rank of an NCCL group over NVLink (the B200 CommHandle, include/oocnmf/comm.hpp:48-67).
    Built per process from a torch.distributed unique-id exchange, or per thread by
    :func:`spawn_group`; all traffic of the solve goes through NCCL inside the C-ABI library.
    Collectives time out (default 60 s, src/comm.cpp:89-111): a rank whose peer stops
    responding gets :class:`CommError` and the group is poisoned."""

    def __init__(self, rank: int, size: int, device: int, group=None, timeout_s: float = 60.0):
        uid = exchange_unique_id(rank, Context.unique_id, device, group) if size > 1 else b"\0" * 128
        self.rank, self.size, self.device = rank, size, device
        self.ctx = Context(device, rank, size, uid)
        self.set_timeout(timeout_s)

    @classmethod
    def _wrap(cls, ctx: "Context", rank: int, size: int, device: int) -> "DistComm":
        self = cls.__new__(cls)
        self.rank, self.size, self.device, self.ctx = rank, size, device, ctx
        return self

    def all_reduce_sum(self, buf: np.ndarray, tag: PhaseTag = PhaseTag.generic) -> None:
        """In-place elementwise sum of a float64 array across the group (collective)."""
        if buf.dtype != np.float64 or not buf.flags.c_contiguous:
            raise ShapeError("all_reduce_sum: expected a C-contiguous float64 array")
        check(_capi.lib().oocnmf_allreduce_f64(self.ctx._h, _p(buf, C.c_double), buf.size, int(tag)))

    def barrier(self) -> None:
        check(_capi.lib().oocnmf_barrier(self.ctx._h))

    def stats(self) -> CollectiveStats:
        b, c, s = np.zeros(6, np.uint64), np.zeros(6, np.uint64), np.zeros(6)
        check(_capi.lib().oocnmf_comm_stats(self.ctx._h, _p(b, C.c_uint64), _p(c, C.c_uint64), _p(s, C.c_double)))
        return CollectiveStats({t: int(b[t]) for t in PhaseTag}, {t: int(c[t]) for t in PhaseTag},
                               {t: float(s[t]) for t in PhaseTag})

    def reset_stats(self) -> None:
        check(_capi.lib().oocnmf_comm_reset_stats(self.ctx._h))

    def set_timeout(self, seconds: float) -> None:
        check(_capi.lib().oocnmf_set_comm_timeout(self.ctx._h, float(seconds)))

    def close(self):
        self.ctx.close()


def spawn_group(n: int, devices: Optional[Sequence[int]] = None, timeout_s: float = 60.0) -> List[DistComm]:
    """``spawn_group(n, Backend::threads)`` (include/oocnmf/comm.hpp:80-82): n ranks of this
    process, one GPU each (devices, default 0..n-1), sharing one NCCL clique; hand one handle
    to each worker thread."""
    devs = list(range(n)) if devices is None else list(devices)
    if len(devs) != n:
        raise ShapeError("spawn_group: need one device per rank")
    if n > device_count():
        raise ShapeError(f"spawn_group: {n} ranks need {n} GPUs, {device_count()} visible")
    ctxs = (C.c_void_p * n)()
    check(_capi.lib().oocnmf_ctx_create_group(n, (C.c_int * n)(*devs), ctxs))
    out = []
    for r in range(n):
        ctx = Context.__new__(Context)
        ctx._h = C.c_void_p(ctxs[r])
        ctx.device, ctx.rank, ctx.nranks = devs[r], r, n
        ctx.m = ctx.n = ctx.k = ctx.row0 = ctx.rows = 0
        ctx._keep = None
        comm = DistComm._wrap(ctx, r, n, devs[r])
        comm.set_timeout(timeout_s)
        out.append(comm)
    return out


def run_distributed_threads(a, cfg: "NmfConfig", plan: "PartitionPlan", stats_out: Optional[list] = None,
                            devices: Optional[Sequence[int]] = None) -> List["NmfResult"]:
    """All ranks of a one-process group on worker threads, one GPU each
    (src/nmf_distributed.cpp:291-319); returns the per-rank results (index = rank) and, in
    ``stats_out``, each rank's CollectiveStats. The first rank exception is re-raised."""
    import threading

    group = spawn_group(plan.n_workers, devices)
    results: List[Optional[NmfResult]] = [None] * plan.n_workers
    errors: List[Optional[BaseException]] = [None] * plan.n_workers

    def work(r):
        try:
            results[r] = nmf_distributed(a, dataclasses.replace(cfg, device=group[r].device), plan, group[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below, like std::exception_ptr
            errors[r] = e

    threads = [threading.Thread(target=work, args=(r,)) for r in range(plan.n_workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if stats_out is not None:
        stats_out.clear()
        stats_out.extend(g.stats() for g in group)
    for g in group:
        g.close()
    for e in errors:
        if e is not None:
            raise e
    return results  # type: ignore[return-value]


@dataclass
class StoreConfig:
    """include/oocnmf/nmf_distributed.hpp StoreConfig: budget_bytes = HBM staging budget of the
    out-of-core row batches (0 = unlimited: A resident in HBM)."""
    budget_bytes: int = 0
    n_cb: int = 1
    prefetch: bool = False


@dataclass
class StoreCounters:
    """include/oocnmf/chunk_store.hpp:21-28, filled by nmf_distributed."""
    loads: int = 0
    evictions: int = 0
    bytes_read: int = 0
    resident_bytes: int = 0
    peak_resident_bytes: int = 0
    io_seconds: float = 0.0


class _Window:
    """This rank's window of a file-backed A, placed so nmf_distributed's slicing selects it."""

    def __init__(self, part, plan, rank):
        self.part, self.plan, self.rank = part, plan, rank


def _file_window(path, plan: PartitionPlan, rank: int):
    """Read only this rank's slab of a PDN1 file (Pdn1File windows, like the reference's
    ChunkStore over a file); Matrix Market files are parsed whole. Returns an object that the
    RNMF / CNMF branches below slice exactly as they slice an in-memory A."""
    from .io import Pdn1File, read_mtx

    (r0, r1), (c0, c1) = plan.slabs[rank]
    if str(path).endswith(".mtx"):
        full = read_mtx(path)
        shape = full.shape
    else:
        f = Pdn1File(path)
        shape = (f.rows, f.cols)
        if f.is_dense():
            full = None
            win = f.read_dense_window(r0, r1, c0, c1, np.float32)
        else:
            full = None
            win = f.read_csr_rows(r0, r1)
            if plan.strategy == Strategy.cnmf:
                win = win.col_window(c0, c1)
    if shape != (plan.m, plan.n):
        raise ShapeError(f"nmf_distributed: file A is {shape[0]}x{shape[1]}, plan is {plan.m}x{plan.n}")
    if full is not None:
        if isinstance(full, CsrMatrix):
            win = full.row_window(r0, r1) if plan.strategy == Strategy.rnmf else full.col_window(c0, c1)
        else:
            win = np.ascontiguousarray(full[r0:r1, c0:c1], np.float32)
    return _Window(win, plan, rank)


def _batch_rows(n: int, store_cfg: Optional[StoreConfig]) -> int:
    per_row = (n + 127) // 128 * 128 * 4
    return max(128, store_cfg.budget_bytes // 2 // per_row) if store_cfg and store_cfg.budget_bytes else 0


def nmf_distributed(a, cfg: NmfConfig, plan: PartitionPlan, comm: DistComm, host_slab: Optional[np.ndarray] = None,
                    batch_rows: int = 0, store_cfg: Optional[StoreConfig] = None,
                    store_counters: Optional[StoreCounters] = None) -> NmfResult:
    """Row- (RNMF) or column-partitioned (CNMF) MU (src/nmf_distributed.cpp:112-289) —
    collective over ``comm``.

    ``a`` is the full A (ndarray / CsrMatrix; only this rank's window is uploaded), a path to a
    PDN1 / Matrix Market file (ASource::file: this rank reads only its window of a PDN1 file),
    or None with ``host_slab`` (this rank's rows, float32) for the out-of-core mode.
    """
    cfg.validate()
    if cfg.k != plan.k:
        raise ShapeError(f"nmf_distributed: cfg.k={cfg.k} disagrees with plan.k={plan.k}")
    if comm.size != plan.n_workers:
        raise ShapeError(f"nmf_distributed: group size {comm.size} != plan workers {plan.n_workers}")
    import time

    sc = StoreCounters()
    if isinstance(a, (str, os.PathLike)):
        (r0_, r1_), _ = plan.slabs[comm.rank]
        per_row = (plan.n + 127) // 128 * 128 * 4
        dense_pdn1 = False
        if not str(a).endswith(".mtx"):
            from .io import Pdn1File

            f = Pdn1File(a)
            dense_pdn1 = f.is_dense()
        t_io = time.perf_counter()
        if (plan.strategy == Strategy.rnmf and dense_pdn1 and store_cfg and store_cfg.budget_bytes
                and host_slab is None and (r1_ - r0_) * per_row > store_cfg.budget_bytes):
            # ASource::file over budget (src/chunk_store.cpp:106-168): read the window once into
            # page-locked host memory, stream it in budget-sized row batches every iteration
            w = _file_window(a, plan, comm.rank)
            host_slab = np.ascontiguousarray(w.part, np.float32)
            batch_rows = _batch_rows(plan.n, store_cfg)
            sc.bytes_read = (r1_ - r0_) * plan.n * (4 if f.dtype == 1 else 8)
            a = None
        else:
            a = _file_window(a, plan, comm.rank)
            sc.loads, sc.resident_bytes = 1, (r1_ - r0_) * per_row
            sc.peak_resident_bytes = sc.resident_bytes
        sc.io_seconds = time.perf_counter() - t_io
    elif host_slab is None:
        (r0_, r1_), _ = plan.slabs[comm.rank]
        sc.loads = 1
        sc.resident_bytes = sc.peak_resident_bytes = (r1_ - r0_) * ((plan.n + 127) // 128 * 128 * 4)
    if host_slab is not None and not batch_rows:
        batch_rows = _batch_rows(plan.n, store_cfg)
    ctx = comm.ctx
    if plan.strategy == Strategy.cnmf:
        # column partition (src/nmf_distributed.cpp:112-149): W replicated, H column slabs
        if host_slab is not None:
            raise ShapeError("nmf_distributed: out-of-core streaming is row-partitioned (RNMF) only")
        _, (c0, c1) = plan.slabs[comm.rank]
        ctx.set_problem_cols(plan.m, plan.n, plan.k, c0, c1 - c0)
        if isinstance(a, _Window):
            ctx.load_csr(a.part) if isinstance(a.part, CsrMatrix) else ctx.load_dense(a.part)
        elif isinstance(a, CsrMatrix):
            ctx.load_csr(a.col_window(c0, c1))
        else:
            ctx.load_dense(np.ascontiguousarray(np.asarray(a)[:, c0:c1]))
        if cfg.init == FactorInit.from_files:
            ctx.set_factors(cfg.init_w, np.ascontiguousarray(np.asarray(cfg.init_h)[:, c0:c1]))
        trace, info = ctx.solve(cfg)
        w, _ = ctx.get_factors()
        h = ctx.gather_h()
        return NmfResult(w, h, trace, int(info["iterations_run"]), bool(info["converged"]), _counters(info), info)
    (r0, r1), _ = plan.slabs[comm.rank]
    ctx.set_problem(plan.m, plan.n, plan.k, r0, r1 - r0)
    registered = False
    if host_slab is not None:
        if store_cfg is not None and sc.bytes_read:  # our own window buffer: page-lock it
            check(_capi.lib().oocnmf_host_register(host_slab.ctypes.data, host_slab.nbytes))
            registered = True
        ctx.attach_host(host_slab, batch_rows)
    elif isinstance(a, _Window):
        ctx.load_csr(a.part) if isinstance(a.part, CsrMatrix) else ctx.load_dense(a.part)
    elif isinstance(a, CsrMatrix):
        ctx.load_csr(a.row_window(r0, r1))
    else:
        ctx.load_dense(np.asarray(a)[r0:r1])
    if cfg.init == FactorInit.from_files:
        ctx.set_factors(np.asarray(cfg.init_w)[r0:r1], cfg.init_h)
    try:
        trace, info = ctx.solve(cfg)
        _, h = ctx.get_factors()
        w = ctx.gather_w()
    finally:
        if registered:
            ctx.set_problem(plan.m, plan.n, plan.k, r0, r1 - r0)  # detach before unpinning
            _capi.lib().oocnmf_host_unregister(host_slab.ctypes.data)
    if host_slab is not None:
        nb = int(info["h2d_batches"])
        sc.loads, sc.evictions = nb, max(0, nb - 2)
        sc.resident_bytes = sc.peak_resident_bytes = int(info["peak_resident_bytes"])
    if store_counters is not None:
        store_counters.__dict__.update(sc.__dict__)
    return NmfResult(w, h, trace, int(info["iterations_run"]), bool(info["converged"]), _counters(info), info)


# ----------------------------------------------------------------------------- model selection
# Mirrors include/oocnmf/model_selection.hpp (src/model_selection.cpp): P perturbed MU runs per
# candidate k on the GPU, W-column clustering / cosine silhouette / selection rule in the
# library's C++ host core.
@dataclass
class SelectionConfig:
    k_min: int = 1
    k_max: int = 1
    n_perturbations: int = 16
    delta: float = 0.03
    sil_threshold: float = 0.75
    nmf: NmfConfig = field(default_factory=NmfConfig)
    seed: int = 0

    def validate(self, m: int, n: int) -> None:
        if self.k_min < 1 or self.k_max < self.k_min:
            raise ShapeError("SelectionConfig: need 1 <= k_min <= k_max")
        if self.k_max >= min(m, n):
            raise ShapeError("SelectionConfig: k_max must be below min(m, n)")
        if self.n_perturbations < 2:
            raise ShapeError("SelectionConfig: need at least 2 perturbations")
        if not 0.0 < self.delta < 1.0:
            raise ShapeError("SelectionConfig: delta must lie in (0, 1)")
        if not -1.0 <= self.sil_threshold <= 1.0:
            raise ShapeError("SelectionConfig: sil_threshold must lie in [-1, 1]")

    def to_c(self) -> _capi.SelectionConfig:
        return _capi.SelectionConfig(self.k_min, self.k_max, self.n_perturbations, self.delta, self.sil_threshold,
                                     self.nmf.to_c(), self.seed)


@dataclass
class KRecord:
    k: int = 0
    valid: bool = False
    runs_used: int = 0
    min_silhouette: float = 0.0
    mean_silhouette: float = 0.0
    mean_relative_error: float = 0.0
    medians: Optional[np.ndarray] = None  # m x k
    iterations: int = 0  # B200 extension: MU iterations run for this k (all ranks)


@dataclass
class SelectionReport:
    records: List[KRecord]
    chosen_k: Optional[int]
    rationale: str

    def to_json(self) -> str:
        import json
        return json.dumps({"chosen_k": self.chosen_k if self.chosen_k is not None else "none",
                           "rationale": self.rationale,
                           "records": [{"k": r.k, "valid": r.valid, "runs_used": r.runs_used,
                                        "min_silhouette": r.min_silhouette, "mean_silhouette": r.mean_silhouette,
                                        "mean_relative_error": r.mean_relative_error} for r in self.records]},
                          indent=2)

    def to_csv(self) -> str:
        rows = ["k,valid,runs_used,min_silhouette,mean_silhouette,mean_relative_error"]
        rows += [f"{r.k},{int(r.valid)},{r.runs_used},{r.min_silhouette:g},{r.mean_silhouette:g},"
                 f"{r.mean_relative_error:g}" for r in self.records]
        return "\n".join(rows) + "\n"


def _select_on(ctx: "Context", m: int, cfg: SelectionConfig) -> SelectionReport:
    nk = cfg.k_max - cfg.k_min + 1
    recs = (_capi.KRecord * nk)()
    med = np.zeros(sum(m * k for k in range(cfg.k_min, cfg.k_max + 1)))
    chosen = C.c_int64()
    why = C.create_string_buffer(512)
    c = cfg.to_c()
    check(_capi.lib().oocnmf_select_k(ctx._h, C.byref(c), recs, nk, _p(med, C.c_double), C.byref(chosen), why,
                                      512))
    out, off = [], 0
    for i, k in enumerate(range(cfg.k_min, cfg.k_max + 1)):
        r = recs[i]
        out.append(KRecord(int(r.k), bool(r.valid), int(r.runs_used), r.min_silhouette, r.mean_silhouette,
                           r.mean_relative_error, med[off:off + m * k].reshape(m, k).copy(), int(r.iterations)))
        off += m * k
    return SelectionReport(out, None if chosen.value < 0 else int(chosen.value), why.value.decode())


def select_k(a, cfg: SelectionConfig) -> SelectionReport:
    """select_k (src/model_selection.cpp:316-406) on one GPU (cfg.nmf.device): A stays resident
    in HBM, every perturbation is generated there, every run is a GPU MU solve."""
    m, n = (a.rows, a.cols) if isinstance(a, CsrMatrix) else np.asarray(a).shape
    cfg.validate(m, n)
    with Context(cfg.nmf.device) as ctx:
        ctx.set_problem(m, n, cfg.k_min)
        if isinstance(a, CsrMatrix):
            ctx.load_csr(a)
        else:
            ctx.load_dense(a)
        return _select_on(ctx, m, cfg)


def select_k_distributed(a, cfg: SelectionConfig, comm: "DistComm") -> SelectionReport:
    """select_k over an NCCL group: every rank holds the full A, the P runs of each k are spread
    over the ranks as independent replicas, the W factors meet in one all-reduce per k, and every
    rank returns the same report. Collective over ``comm``."""
    m, n = (a.rows, a.cols) if isinstance(a, CsrMatrix) else np.asarray(a).shape
    cfg.validate(m, n)
    ctx = comm.ctx
    ctx.set_problem(m, n, cfg.k_min)
    if isinstance(a, CsrMatrix):
        ctx.load_csr(a)
    else:
        ctx.load_dense(a)
    return _select_on(ctx, m, cfg)


def perturb_dense(a: np.ndarray, delta: float, seed: int, device: int = 0) -> np.ndarray:
    """perturb_dense (model_selection.cpp:35-47), evaluated on the GPU; returns float32."""
    if not 0.0 <= delta < 1.0:
        raise ShapeError("perturb: delta must lie in [0, 1)")
    a = np.asarray(a)
    with Context(device) as ctx:
        ctx.set_problem(a.shape[0], a.shape[1], 1)
        ctx.load_dense(a)
        ctx.perturb(delta, seed)
        return ctx.download_dense()


def perturb_sparse(a: CsrMatrix, delta: float, seed: int, device: int = 0) -> CsrMatrix:
    """perturb_sparse (model_selection.cpp:49-60), evaluated on the GPU (sparsity preserved)."""
    if not 0.0 <= delta < 1.0:
        raise ShapeError("perturb: delta must lie in [0, 1)")
    with Context(device) as ctx:
        ctx.set_problem(a.rows, a.cols, 1)
        ctx.load_csr(a)
        ctx.perturb(delta, seed)
        return ctx.download_csr()


@dataclass
class ColumnClusters:
    member_cluster: np.ndarray  # runs x k: cluster of (run, column), -1 if dropped / unmatched
    medians: np.ndarray         # m x k
    dropped_zero_columns: int
    per_cluster: np.ndarray     # silhouette per cluster
    min_sil: float
    mean_sil: float


def cluster_columns(runs, k: Optional[int] = None) -> ColumnClusters:
    """cluster_columns + silhouette (model_selection.cpp:163-281) over W factors (list of m x k
    arrays or an R x m x k array), in the library's host core."""
    runs = np.ascontiguousarray(np.asarray(runs, dtype=np.float64))
    if runs.ndim != 3 or runs.shape[0] < 2:
        raise ShapeError("cluster_columns: need at least 2 runs of m x k")
    r, m, kk = runs.shape
    if k is not None and k != kk:
        raise ShapeError("cluster_columns: all runs must be m x k")
    med, per = np.zeros((m, kk)), np.zeros(kk)
    mn, mean, dropped = C.c_double(), C.c_double(), C.c_uint64()
    member = np.zeros((r, kk), np.int64)
    check(_capi.lib().oocnmf_cluster_silhouette(_p(runs, C.c_double), r, m, kk, _p(med, C.c_double),
                                                _p(per, C.c_double), C.byref(mn), C.byref(mean), C.byref(dropped),
                                                _p(member, C.c_int64)))
    return ColumnClusters(member, med, int(dropped.value), per, mn.value, mean.value)


def pearson_correlation_matrix(w_true: np.ndarray, w_est: np.ndarray) -> np.ndarray:
    """Entry (i, j): Pearson correlation of column i of w_true and column j of w_est
    (model_selection.cpp:283-314)."""
    wt = np.ascontiguousarray(w_true, np.float64)
    we = np.ascontiguousarray(w_est, np.float64)
    if wt.shape[0] != we.shape[0]:
        raise ShapeError("pearson_correlation_matrix: row counts differ")
    corr = np.zeros((wt.shape[1], we.shape[1]))
    check(_capi.lib().oocnmf_pearson_correlation(_p(wt, C.c_double), wt.shape[0], wt.shape[1], _p(we, C.c_double),
                                                 we.shape[1], _p(corr, C.c_double)))
    return corr
