"""CPU-only tests of the product's host side: the C-ABI library loads and exports every
symbol include/oocnmf_b200.h declares, host helpers match the reference bit-for-bit, config /
shape validation mirrors the reference, there is no silent CPU fallback, and the stream-K
work split the kernels use tiles every pass exactly once."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf
from paper_2202_09518_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "oocnmf_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oocnmf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.EXPORTS)
    assert lib.oocnmf_abi_version() == 1


def test_cpp_headers_forward_to_host_core():
    for h in ("matrix", "nmf", "error", "rng", "partition", "nmf_distributed"):
        txt = open(os.path.join(ROOT, "include", "oocnmf", h + ".hpp")).read()
        assert '#include "oocnmf_b200/oocnmf.hpp"' in txt


def test_host_rng_and_init_bitexact():
    w, h = nmf.init_factors(37, 29, 5, 13)
    w2, h2 = oracle.port.init_factors(37, 29, 5, 13)
    assert np.array_equal(w, w2) and np.array_equal(h, h2)
    u = nmf.counter_uniform(42, 99, 0, 2048 * 3)
    assert np.array_equal(u.reshape(3, 2048), oracle.port.uniform_dense(3, 2048, 42, 99))
    if oracle.ref.available:
        a, b = oracle.ref.init_factors(37, 29, 5, 13)
        assert np.array_equal(w, a) and np.array_equal(h, b)


def test_make_plan_matches_reference():
    for (m, n, k, N, nb) in [(10, 7, 2, 3, 2), (65536, 65536, 32, 8, 1), (100, 80, 4, 7, 3), (9, 9, 1, 9, 9)]:
        p = nmf.make_plan(m, n, k, N, nb, nmf.choose_strategy(m, n))
        if oracle.ref.available:
            r = oracle.ref.make_plan(m, n, k, N, nb, strategy=0)
            assert r["strategy"] == p.strategy.value
            got = np.array([[a[0], a[1], b[0], b[1]] for a, b in p.slabs])
            assert np.array_equal(got, r["slabs"])
            assert np.array_equal(np.array(p.batches), r["batches"])
    assert nmf.choose_strategy(100, 200) == nmf.Strategy.cnmf
    assert nmf.choose_strategy(100, 100) == nmf.Strategy.rnmf
    with pytest.raises(nmf.ShapeError):
        nmf.make_plan(3, 3, 1, 4, 1, nmf.Strategy.rnmf)
    with pytest.raises(nmf.ShapeError):
        nmf.make_plan(3, 3, 1, 1, 4, nmf.Strategy.rnmf)


def test_config_validation_mirrors_reference():
    for bad in (dict(k=0), dict(eta=-1), dict(max_iters=0), dict(error_check_interval=0), dict(epsilon=0),
                dict(init=nmf.FactorInit.from_files), dict(error_mode="x")):
        with pytest.raises(nmf.ShapeError):
            nmf.NmfConfig(**{"k": 2, **bad}).validate()
    with pytest.raises(ValueError):  # ShapeError is-a ValueError (std::invalid_argument)
        nmf.NmfConfig(k=0).validate()


def test_csr_validation():
    with pytest.raises(nmf.ShapeError):
        nmf.CsrMatrix(2, 3, [0, 2, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(nmf.ShapeError):
        nmf.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(nmf.ShapeError):
        nmf.CsrMatrix(1, 3, [0, 1], [3], [1.0])
    d = np.array([[0, 2.0], [0, 0]])
    c = nmf.CsrMatrix.from_dense(d)
    assert np.array_equal(c.to_dense(), d)
    assert c.row_window(0, 1).nnz == 1


@pytest.mark.skipif(nmf.device_count() > 0, reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    with pytest.raises(nmf.DeviceError, match="no CPU fallback"):
        nmf.nmf_serial(np.ones((8, 8)), nmf.NmfConfig(k=2, max_iters=2))


# -------------------------------------------------------------------------- stream-K split
class StreamK:
    """Python restatement of ooc::StreamK (paper_2202_09518_b200/csrc/common.cuh)."""

    def __init__(self, tiles, ipt, g_max):
        self.tiles, self.ipt = tiles, ipt
        self.G = max(1, min(g_max, tiles * ipt))
        self.smax = max((self.begin(c + 1) - 1) // ipt - self.begin(c) // ipt + 1 for c in range(self.G))

    def total(self):
        return self.tiles * self.ipt

    def begin(self, c):
        return c * self.total() // self.G

    def cta_of(self, u):
        return ((u + 1) * self.G + self.total() - 1) // self.total() - 1

    def first_tile(self, c):
        return self.begin(c) // self.ipt

    def slot(self, c, t):
        return c * self.smax + (t - self.first_tile(c))


@pytest.mark.parametrize("tiles,ipt,G", [(512, 2048, 148), (32, 64, 148), (1, 4, 148), (3, 1, 148), (64, 2048, 148),
                                         (5, 7, 3), (17, 13, 148)])
def test_streamk_split_tiles_each_unit_once(tiles, ipt, G):
    sk = StreamK(tiles, ipt, G)
    seen = np.zeros(tiles * ipt, int)
    used_slots = set()
    for c in range(sk.G):
        b, e = sk.begin(c), sk.begin(c + 1)
        assert e > b  # no empty CTA
        seen[b:e] += 1
        for u in (b, e - 1):
            assert sk.cta_of(u) == c
        for t in range(b // ipt, (e - 1) // ipt + 1):
            s = sk.slot(c, t)
            assert 0 <= s < sk.G * sk.smax and s not in used_slots
            used_slots.add(s)
    assert np.all(seen == 1)
    # the consumer's contributor range for each tile covers exactly the CTAs that wrote it
    for t in range(tiles):
        c0, c1 = sk.cta_of(t * ipt), sk.cta_of((t + 1) * ipt - 1)
        writers = [c for c in range(sk.G) if sk.begin(c) < (t + 1) * ipt and sk.begin(c + 1) > t * ipt]
        assert writers == list(range(c0, c1 + 1))
    # balance: every CTA streams the same number of A bytes to within one step
    sizes = [sk.begin(c + 1) - sk.begin(c) for c in range(sk.G)]
    assert max(sizes) - min(sizes) <= 1


def test_memory_estimate_layout_and_batches():
    # config 2 on one 180 GB B200: in core; on an 8 GB budget: out-of-core row batches
    p = nmf.make_plan(65536, 65536, 32, 1, 1, nmf.Strategy.rnmf)
    big = nmf.memory_estimate(p, 1.0, 180 << 30)
    assert big.in_core and big.min_n_b == 1 and big.a_slab_bytes == 65536 * 65536 * 4
    small = nmf.memory_estimate(p, 1.0, 8 << 30)
    assert small.feasible and not small.in_core and small.min_n_b > 1 and small.peak_bytes <= 8 << 30
    tighter = nmf.memory_estimate(p, 1.0, 4 << 30)
    assert tighter.min_n_b >= small.min_n_b                      # fewer bytes -> more batches
    # per-rank slabs shrink with the worker count
    p8 = nmf.make_plan(65536, 65536, 32, 8, 1, nmf.Strategy.rnmf)
    assert nmf.memory_estimate(p8, 1.0, 180 << 30).a_slab_bytes == 8192 * 65536 * 4
    # CSR: 8 B per stored entry in CSR(A) and CSR(A^T), plus both row pointers
    ps = nmf.make_plan(1 << 16, 1 << 16, 16, 1, 1, nmf.Strategy.rnmf)
    rep = nmf.memory_estimate(ps, 1e-3, 180 << 30)
    nnz = int(np.ceil(1e-3 * (1 << 16) * (1 << 16)))
    assert rep.a_slab_bytes == nnz * 16 + 2 * ((1 << 16) + 1) * 8
    with pytest.raises(nmf.ShapeError, match="exceed the budget"):
        nmf.memory_estimate(p, 1.0, 1 << 20)
    with pytest.raises(nmf.ShapeError, match="density"):
        nmf.memory_estimate(p, 0.0, 1 << 30)


def test_plan_and_report_json_match_reference():
    """PartitionPlan.to_json / MemoryReport.to_json byte-identical to the reference's
    (src/partition.cpp:89-104, 199-209: nlohmann dump(2))."""
    import oracle
    from paper_2202_09518_b200.nmf import MemoryReport

    if not oracle.ref.available:
        pytest.skip("needs oracle/_ref")
    for m, n, k, w, nb, st in [(1000, 900, 8, 4, 3, 0), (700, 1300, 16, 3, 2, 1), (10, 10, 2, 1, 1, 0)]:
        plan = nmf.make_plan(m, n, k, w, nb, nmf.Strategy.cnmf if st == 1 else nmf.Strategy.rnmf)
        assert plan.to_json() == oracle.ref.plan_to_json(m, n, k, w, nb, st)
    mr = MemoryReport(1, 2, 3, 4, 5, 6, True, False)
    assert mr.to_json() == oracle.ref.memreport_to_json([1, 2, 3, 4, 5, 6, 0], 1)
