// C-ABI backend: per-GPU context, HBM layout, and the MU iteration loop.
//
// The loop mirrors nmf_serial (src/nmf_serial.cpp:83-117) / the RNMF worker
// (src/nmf_distributed.cpp:151-262): W update, then H update, error every
// error_check_interval iterations and on the last, early exit at eta. Differences that are
// pure B200 engineering:
//  * A lives in HBM as f32 (or streams from host memory out-of-core); factors are f32 with
//    f64 accumulation for every scalar (norms, trace-form error).
//  * The H update's two all-reduces per batch (W^T W, then W^T A_p) are one NCCL
//    all-reduce of a packed [W^T A | W^T W] buffer per iteration.
//  * The error is the trace form ||A||^2 - 2<W^T A, H> + <W^T W, H H^T>, whose terms all
//    exist after the H update, so error checks cost no pass over A; when it reports a small
//    error (where its cancellation hurts) the check is redone with a direct f64 residual.
//  * Nothing syncs the host except error checks (one 16-byte D2H every interval).
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <deque>
#include <mutex>
#include <vector>

#include "kernels.h"
#include "oocnmf_b200.h"

using namespace ooc;

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(OOCNMF_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}
void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(OOCNMF_ERR_COMM, std::string(what) + ": " + ncclGetErrorString(r));
}
template <class F>
int guarded(F&& f) {
    try {
        f();
        return OOCNMF_OK;
    } catch (const Fail& x) {
        g_err = x.msg;
        return x.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return OOCNMF_ERR_DEVICE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OOCNMF_ERR_DEVICE;
    }
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

int pad_k(uint64_t k) {
    if (k < 1) fail(OOCNMF_ERR_SHAPE, "k must be >= 1");
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 32) return 32;
    if (k <= 64) return 64;
    // wide factors (kernels_wide.cu): 64-column groups on the kp = 64 passes
    if (k <= uint64_t(kMaxWideKp)) return int((k + 63) / 64 * 64);
    fail(OOCNMF_ERR_SHAPE, "k=" + std::to_string(k) + " exceeds the supported maximum of " + std::to_string(kMaxWideKp));
}
// tensor-core passes at this kp (wide factors run them per 64-column group)
bool tc_for(int kp) { return tc_supported(kp > 64 ? 64 : std::max(kp, 16)); }

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    bool external = false;  // storage owned elsewhere (the NVLS symmetric Ht): never cudaFree'd
    void release() {
        if (p && !external) cudaFree(p);
        p = nullptr;
        bytes = 0;
        external = false;
    }
    void alloc(size_t b, const char* what) {
        if (b == bytes && p) return;
        release();
        if (b == 0) return;
        const cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(OOCNMF_ERR_DEVICE, std::string("cudaMalloc(") + std::to_string(b) + " B) for " + what +
                                        ": " + cudaGetErrorString(e));
        }
        bytes = b;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

enum class Kind { none, dense, csr, host };

// indices into the f64 scalar scratch
enum Scal { kNormA2 = 0, kErr = 1, kRes = 2, kCross = 3, kNumScal = 8 };

// events recorded per iteration (see solve())
enum Ev { eStart, eAht, eWdone, eWta, eReduced, eComm, eHdone, kEvPerIter };

}  // namespace

struct oocnmf_ctx {
    int device = 0, rank = 0, nranks = 1, num_sms = 148;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    // sharded CSR H update: the reduce-scatter of W^T A runs chunk by chunk on comm_stream
    // (high priority) while the SpMM computes the next chunk (see spmm_wta_reduce_scatter)
    cudaStream_t comm_stream = nullptr;
    static constexpr int kMaxRsChunks = 16;
    cudaEvent_t ev_rs[kMaxRsChunks + 1] = {};
    DevBuf wtp;                  // W^T A in chunk-major order [chunk][rank][rows][kp] (send side)
    bool rs_done = false;        // this iteration's reduce-scatter was issued with the SpMM
    // sharded CSR H: the new H rows reach the other ranks as N broadcasts on comm_stream, and the
    // next A·Ht SpMM consumes Ht slice by slice as they land (own slice first): ev_bc[root]
    bool ag_pending = false;
    std::vector<cudaEvent_t> ev_bc;
    cudaEvent_t ev_hdone = nullptr;
    DevBuf segR;                 // CSR row segments at the rank-slice column boundaries
    int segR_n = 0;
    bool no_check_next = false;  // the iteration being enqueued is not followed by an error check
    bool h_fused = false;        // ... and its H update ran inside the A^T W SpMM
    // sharded CSR H update over NVLS multicast (kernels_nvls.cu, OOCNMF_NVLS=1): the A^T W SpMM
    // writes this rank's partial W^T A into symmetric memory and one kernel reduces, updates and
    // multicasts the rows; Ht itself lives in the symmetric buffer nv.ht while nvls_ready
    NvlsState nv;
    bool nvls_ready = false, nvls_failed = false, nvls_pending = false;

    uint64_t m = 0, n = 0, k = 0, row0 = 0, rows = 0;
    // Column partition (CNMF, src/nmf_distributed.cpp:112-149): this rank owns all m rows and
    // the columns [col0, col0 + n) of n_global; W is replicated, H (Ht) is the local slab.
    bool cnmf = false;
    uint64_t col0 = 0, n_global = 0;
    int kp = 0;
    int64_t mp = 0, np = 0;
    bool problem_set = false;

    Kind kind = Kind::none;
    DevBuf A;                       // dense: mp x np f32
    DevBuf rp, ci, v, rpT, ciT, vT; // csr: slab rows x n and its transpose n x rows
    // column chunks of the two SpMMs (csr_chunks): A over its n columns (gathers Ht), A^T over
    // its rows columns (gathers W); C = 1 is the single-pass SpMM
    struct Chunks {
        DevBuf seg;
        int C = 1, kp = 0;
        int64_t cols = 0;
    } chA, chT;
    int64_t nnz = 0;
    const float* hA = nullptr;      // out-of-core host slab
    uint64_t hlda = 0;
    int64_t batch_rows = 0;
    DevBuf stage[2];
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};

    DevBuf W, Ht, HHt, packed, N1, slots1, slots2, gram_w, gram_h, err_slots, red_slots, scal, flag;
    DevBuf HHt64, WtW64;         // f64 Grams for the trace-form error (f32 copies drive the updates)
    DevBuf W_cat, Ht_cat;        // [F | F - tf32(F)] (rows x 2kp): tensor-core operands only
    DevBuf fix_flags;            // in-kernel stream-K fix-up of pass 2 (tensor-core path)
    bool use_tc = false;         // kp in {32, 64}: tcgen05 passes; else CUDA-core FFMA passes
    StreamK sk1, sk2;            // in-core dense passes
    // one-pass W half (kernels_fused.cu): dense in-core RNMF / serial, kp <= 32
    bool use_fused = false;
    FusedPlan fplan;
    DevBuf fz_idx, fz_slots, fz_count;  // [q0 | t0 | act] ints, P1 partial ring, [count | wdone]
    StreamK sk1b[2], sk2b[2];    // out-of-core: full batch / last batch
    bool norm_valid = false, factors_set = false, factors_valid = false;
    double norm_a2 = 0.0;
    double* hpin = nullptr;      // pinned readback: [err, flag]
    // copy-in / copy-out staging of the C-ABI's pageable-array calls (see Stage), lazily made
    void* stage_pin = nullptr;
    DevBuf stage_dev;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> evs;
    uint64_t launches = 0;
    // CUDA graph of one block of iterations (the launches between two error checks),
    // replayed while its key (buffers, shapes, eps, block length) is unchanged.
    struct Graph {
        std::vector<uint64_t> key;
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;
    };
    std::vector<Graph> graphs;  // small cache: the two event sets of the solve loop alternate
    DevBuf errs, flags, pred;   // device-side error checks: per-check value / NaN flag, predicate
    DevBuf snapW[2], snapH[2];  // eta > 0: the factors at the last two checks (lagged early exit)
    bool graph_broken = false;   // capture failed once: iterate eagerly (same kernels)
    bool capturing = false;

    // model selection: pristine copy of the resident A while it is perturbed; replica mode
    // (every rank holds the full A and solves independently: no collective in the solve)
    DevBuf A0, v0, vT0;
    bool pristine = false, local = false;
    bool collective() const { return nranks > 1 && !local; }
    // Collective bookkeeping (reference CommHandle stats, include/oocnmf/comm.hpp:28-43) and the
    // progress watchdog (src/comm.cpp:89-111): every collective is bracketed by two events; a
    // host wait that sees no collective complete for comm_timeout seconds aborts the
    // communicator (ncclCommAbort) and poisons the context (every later collective fails).
    struct CollMark {
        cudaEvent_t beg, end;
        int tag;
    };
    std::deque<CollMark> marks;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t mark_beg = nullptr;
    uint64_t tag_bytes[6] = {}, tag_calls[6] = {};
    double tag_secs[6] = {};
    double comm_timeout = 60.0;
    bool poisoned = false;
    // RNMF on CSR: W^T A is n x k (537 MB at config 3), so instead of all-reducing it and
    // repeating the n-row H update on every rank, the ranks reduce-scatter it, update their
    // own n/N rows of H, and all-gather H (the same bytes as the all-reduce, 1/N of the update).
    // Needs whole 128-row tiles per rank (n a multiple of 128 N, as at config 3); else all-reduce.
    // Dense RNMF can do the same (OOCNMF_SHARD_H=1); W^T A is only 8.4 MB at config 2, and the
    // all-reduce + replicated H update measured faster (649 vs 607 it/s at N = 4), so it is off.
    // OOCNMF_SHARD_H=1 / 0 forces the sharded / replicated H update for both kinds.
    // Dense: only with the NVLS H update on the one-pass path (OOCNMF_NVLS=1), which needs it.
    bool shard_h() const {
        static const int force = [] {  // dense measured slower at N = 4 (607 vs 649 it/s): off by default
            const char* e = std::getenv("OOCNMF_SHARD_H");
            return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
        }();
        const bool want = force >= 0 ? force == 1 : (kind == Kind::csr || dense_nvls());
        return collective() && !cnmf && want && (kind == Kind::csr || kind == Kind::dense) &&
               np % (int64_t(kTile) * nranks) == 0;
    }
    bool dense_nvls() const {
        static const bool on = [] {
            const char* e = std::getenv("OOCNMF_NVLS");
            return e && e[0] == '1';
        }();
        return on && kind == Kind::dense && use_fused && nvls_compiled();
    }
    int64_t h_rows() const { return shard_h() ? np / nranks : np; }
    int64_t h_row0() const { return shard_h() ? h_rows() * rank : 0; }

    float* wta() const { return packed.as<float>(); }
    float* wtw() const { return packed.as<float>() + np * kp; }
    int64_t packed_count() const { return np * kp + int64_t(kp) * kp; }
};

namespace {

void set_dev(oocnmf_ctx* c) { ck(cudaSetDevice(c->device), "cudaSetDevice"); }

void need_problem(oocnmf_ctx* c) {
    if (!c->problem_set) fail(OOCNMF_ERR_SHAPE, "oocnmf_set_problem has not been called");
}

void count(oocnmf_ctx* c, cudaError_t e, const char* what) {
    ck(e, what);
    ++c->launches;
}

// ------------------------------------------------------------------ collectives
// PhaseTag values (include/oocnmf/comm.hpp:13-20)
enum Tag { kTagGeneric = 0, kTagW = 1, kTagH = 2, kTagErr = 3, kTagGather = 4, kTagBarrier = 5 };

cudaEvent_t pool_event(oocnmf_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}
// Open / close the bracket of one collective (or one NCCL group) on stream s.
void coll_begin(oocnmf_ctx* c, cudaStream_t s) {
    if (!c->comm) return;
    c->mark_beg = pool_event(c);
    ck(cudaEventRecord(c->mark_beg, s), "event");
}
void coll_end(oocnmf_ctx* c, cudaStream_t s, int tag, size_t bytes) {
    if (!c->comm || !c->mark_beg) return;
    cudaEvent_t e = pool_event(c);
    ck(cudaEventRecord(e, s), "event");
    c->marks.push_back({c->mark_beg, e, tag});
    c->mark_beg = nullptr;
    c->tag_bytes[tag] += bytes;
    c->tag_calls[tag] += 1;
}
// Retire completed collectives (their device time goes to the tag); returns how many.
size_t reap_marks(oocnmf_ctx* c) {
    size_t n = 0;
    while (!c->marks.empty()) {
        const auto& m = c->marks.front();
        const cudaError_t q = cudaEventQuery(m.end);
        if (q != cudaSuccess) break;  // not ready (or a fault, reported by the caller's wait)
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m.beg, m.end) == cudaSuccess) c->tag_secs[m.tag] += ms * 1e-3;
        cudaGetLastError();
        c->ev_pool.push_back(m.beg);
        c->ev_pool.push_back(m.end);
        c->marks.pop_front();
        ++n;
    }
    return n;
}
// Abort the group after a collective failure. A live context (timeout, NCCL async error) gets
// ncclCommAbort — on a helper thread, bounded, since an abort that itself blocks must not turn
// the failure into a hang — and its streams are drained (bounded). After a device fault the
// context is lost: nothing is waited for. Either way the context is poisoned.
[[noreturn]] void abort_comm(oocnmf_ctx* c, const std::string& why, bool device_fault = false) {
    ncclComm_t comm = c->comm;
    c->comm = nullptr;
    c->poisoned = true;
    auto bounded = [](auto&& done, int max_ms) {
        for (int ms = 0; ms < max_ms && !done(); ms += 10) std::this_thread::sleep_for(std::chrono::milliseconds(10));
    };
    if (comm && !device_fault) {
        auto flag = std::make_shared<std::atomic<bool>>(false);
        std::thread t([comm, flag] {
            ncclCommAbort(comm);
            flag->store(true);
        });
        bounded([&] { return flag->load(); }, 10000);
        if (flag->load())
            t.join();
        else
            t.detach();
        bounded([&] {
            return cudaStreamQuery(c->stream) != cudaErrorNotReady && cudaStreamQuery(c->comm_stream) != cudaErrorNotReady;
        }, 10000);
    }
    cudaGetLastError();
    for (auto& m : c->marks) c->ev_pool.push_back(m.beg), c->ev_pool.push_back(m.end);
    c->marks.clear();
    fail(OOCNMF_ERR_COMM, "rank " + std::to_string(c->rank) + " of " + std::to_string(c->nranks) + ": " + why +
                              "; communicator aborted (the group is poisoned)");
}
void need_comm(const oocnmf_ctx* c) {
    if (c->poisoned) fail(OOCNMF_ERR_COMM, "communicator was aborted after an earlier collective failure");
}
// A failing NCCL call on the group (a dead peer detected at enqueue, an async error surfacing
// at group end): abort and poison like a timeout.
void ncc(oocnmf_ctx* c, ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress) abort_comm(c, std::string(what) + ": " + ncclGetErrorString(r));
}
// Host wait for an event (or the whole stream when e is null). With a communicator it polls:
// no collective completing for comm_timeout seconds, or an NCCL async error, aborts the group
// instead of hanging on a dead peer.
void wait_for(oocnmf_ctx* c, cudaStream_t s, cudaEvent_t e, const char* what) {
    if (!c->comm) {
        ck(e ? cudaEventSynchronize(e) : cudaStreamSynchronize(s), what);
        return;
    }
    auto last = std::chrono::steady_clock::now();
    for (int spins = 0;; ++spins) {
        const cudaError_t q = e ? cudaEventQuery(e) : cudaStreamQuery(s);
        if (reap_marks(c)) last = std::chrono::steady_clock::now();
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) {
            // a device fault while collectives are in flight: typically a peer process died and
            // its NVLink-mapped buffers vanished under the NCCL kernels (the context is lost)
            if (!c->marks.empty())
                abort_comm(c, std::string("device error (") + cudaGetErrorString(q) + ") while waiting for " + what +
                                  " with collectives in flight (a peer rank failed?)",
                           true);
            ck(q, what);
        }
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
            abort_comm(c, std::string("NCCL async error (") + ncclGetErrorString(ar) + ") while waiting for " + what);
        const double idle = std::chrono::duration<double>(std::chrono::steady_clock::now() - last).count();
        if (!c->marks.empty() && idle > c->comm_timeout)
            abort_comm(c, "no collective completed for " + std::to_string(c->comm_timeout) +
                              " s while waiting for " + what + " (unresponsive peer)");
        if (spins < 4096)
            std::this_thread::yield();
        else
            std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

// Column-chunked SpMM plan (kernels_sparse.cu, launch_spmm_seg): chunk the gathered operand
// so each pass's slice stays in L2, when the traffic model says the chunk passes move fewer
// bytes than one gathering pass. Per row: one pass gathers nnz_row x kp x 4 bytes from DRAM;
// C passes read 16 bytes of segment bounds and read + write the kp x 4 accumulator row per
// pass, plus the gathered operand once. OOCNMF_SPMM_CHUNK_MB sets the slice size (default
// 40 MB: a third of the 126 MB L2); 0 disables chunking.
void plan_chunks(oocnmf_ctx* c, oocnmf_ctx::Chunks& ch, const int64_t* rp, const int32_t* ci, int64_t rows,
                 int64_t cols) {
    const char* e = std::getenv("OOCNMF_SPMM_CHUNK_MB");  // (fractions allowed: tests force chunks)
    const int64_t target = int64_t((e ? std::atof(e) : 40.0) * 1048576.0);
    const char* f = std::getenv("OOCNMF_SPMM_CHUNK_FORCE");
    const bool force = f && *f && *f != '0';
    const int kp = c->kp;
    ch.kp = kp;
    ch.C = 1;
    ch.seg.release();
    const int64_t b_bytes = cols * kp * 4;
    if (target <= 0 || rows <= 0 || b_bytes <= target || kp > 64) return;  // (no wide chunk kernel)
    const int C = int((b_bytes + target - 1) / target);
    const double nnz_row = double(c->nnz) / double(rows);
    const double one_pass = nnz_row * kp * 4;
    const double chunked = C * 16.0 + (2.0 * C - 1.0) * kp * 4 + double(b_bytes) / double(rows);
    // (measured at config 3, 42 entries per row: 8-13 chunk passes of ~4 entries per row are
    // latency-bound on the per-row bounds and accumulator round trips — 5.5-6.8 ms against
    // 3.8 ms for the one gathering pass — so chunks also need >= 16 entries per row each)
    if (C > 64 || (!force && (chunked * 1.25 > one_pass || nnz_row < 16.0 * C))) return;
    ch.C = C;
    ch.cols = (cols + C - 1) / C;
    ch.seg.alloc(size_t(C + 1) * rows * 8, "spmm chunks");
    ck(launch_csr_segments(rp, ci, rows, ch.cols, C, ch.seg.as<int64_t>(), c->stream), "csr chunks");
}

void ensure_chunks(oocnmf_ctx* c) {
    if (c->kind != Kind::csr) return;
    if (c->chA.kp != c->kp)
        plan_chunks(c, c->chA, c->rp.as<int64_t>(), c->ci.as<int32_t>(), int64_t(c->rows), int64_t(c->n));
    if (c->chT.kp != c->kp)
        plan_chunks(c, c->chT, c->rpT.as<int64_t>(), c->ciT.as<int32_t>(), int64_t(c->n), int64_t(c->rows));
}

// out = A · Ht (transpose = false: rows x kp) or A^T · W (n x kp), chunked per the plan.
void spmm(oocnmf_ctx* c, bool transpose, const float* B, float* out, cudaStream_t s) {
    const auto& ch = transpose ? c->chT : c->chA;
    const int64_t* rp = (transpose ? c->rpT : c->rp).as<int64_t>();
    const int32_t* ci = (transpose ? c->ciT : c->ci).as<int32_t>();
    const float* v = (transpose ? c->vT : c->v).as<float>();
    const int64_t rows = transpose ? int64_t(c->n) : int64_t(c->rows);
    if (ch.C <= 1) {
        count(c, launch_spmm(c->kp, rp, ci, v, rows, B, out, s), transpose ? "spmm At W" : "spmm A Ht");
        return;
    }
    const int64_t* seg = ch.seg.as<int64_t>();
    for (int k = 0; k < ch.C; ++k)
        count(c, launch_spmm_seg(c->kp, seg + k * rows, seg + (k + 1) * rows, ci, v, rows, B, out, k > 0, s),
              transpose ? "spmm At W (chunk)" : "spmm A Ht (chunk)");
}

void nvls_release(oocnmf_ctx* c);

void alloc_factors(oocnmf_ctx* c) {
    const int kp = c->kp;
    if (c->nvls_ready && c->nv.ht_bytes != size_t(c->np) * kp * 4) nvls_release(c);  // (collective: set_rank)
    c->W.alloc(size_t(c->mp) * kp * 4, "W");
    c->Ht.alloc(size_t(c->np) * kp * 4, "Ht");
    if (c->use_tc) {
        c->W_cat.alloc(size_t(c->mp) * 2 * kp * 4, "W_cat");
        c->Ht_cat.alloc(size_t(c->np) * 2 * kp * 4, "Ht_cat");
        ck(cudaMemsetAsync(c->W_cat.p, 0, c->W_cat.bytes, c->stream), "memset");
        ck(cudaMemsetAsync(c->Ht_cat.p, 0, c->Ht_cat.bytes, c->stream), "memset");
    } else {
        c->W_cat.release();
        c->Ht_cat.release();
    }
    c->HHt.alloc(size_t(kp) * kp * 4, "HHt");
    c->HHt64.alloc(size_t(kp) * kp * 8, "HHt64");
    c->WtW64.alloc(size_t(kp) * kp * 8, "WtW64");
    c->packed.alloc(size_t(c->packed_count()) * 4, "packed");
    const int gw = factor_grid(c->mp / kTile), gh = factor_grid(c->np / kTile);
    // (also the one-pass kernel's per-CTA Gram slots: one per SM)
    c->gram_w.alloc(size_t(std::max(gw, c->num_sms)) * kp * kp * 8, "gram_w");
    c->gram_h.alloc(size_t(gh) * kp * kp * 8, "gram_h");
    c->err_slots.alloc(size_t(std::max(gh, sqnorm_grid())) * 8, "err_slots");
    c->red_slots.alloc(size_t(sqnorm_grid()) * 8, "red_slots");
    c->scal.alloc(kNumScal * 8, "scalars");
    c->flag.alloc(4, "flag");
    ck(cudaMemsetAsync(c->W.p, 0, c->W.bytes, c->stream), "memset W");
    ck(cudaMemsetAsync(c->Ht.p, 0, c->Ht.bytes, c->stream), "memset Ht");
    ck(cudaMemsetAsync(c->flag.p, 0, 4, c->stream), "memset flag");
}

// OOCNMF_FUSED=0 keeps the two-pass W half; OOCNMF_FUSED_D sets the P2 lag in row blocks
// (default 1: two 32 MB blocks of A in L2 at n = 65536 — at 2 the third block pushes the A
// re-reads out of L2, 32 GB instead of 19 GB of DRAM reads per launch); OOCNMF_FUSED_P2FIRST=1
// orders each step P2(s - D) before P1(s); OOCNMF_FUSED_POL picks the L2 policies of the two A
// loads (0: normal / first, 1: last / first, 2: normal / normal).
// The one-pass kernel pays a fixed W-update latency per 128-row block (~4 us: every CTA's
// partial published, gathered and summed); it beats the two streaming passes once a row block
// is large enough to hide it. Measured on B200 (tools/fused_crossover.py,
// profiles/r2_fused_crossover.jsonl): np = 65536 +8-13 %; np = 32768 (lag 2) +3-7 % at
// kp = 16, -3..-8 % at kp = 32; np = 16384 -20-35 %; np = 8192 -55 %.
// OOCNMF_FUSED=0 / 1 turns it off / on regardless of the shape.
bool fused_wanted(const oocnmf_ctx* c) {
    const char* e = std::getenv("OOCNMF_FUSED");
    if (e && e[0] == '0') return false;
    const bool forced = e && e[0] == '1';
    const int64_t min_cols = c->kp == 16 ? 32768 : 65536;
    return c->use_tc && !c->cnmf && (forced || c->np >= min_cols) &&
           fused_supported(c->kp, c->mp, c->np, c->num_sms);
}
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}
// P2 lags P1 by D row blocks; the D + 2 blocks in flight (128 np 4 bytes each) must stay in
// L2 for P2's re-read, so D is what 64 MiB holds beyond the two in use, clamped to [1, 4]
// (np = 65536: 1, 32768: 2, <= 16384: 4).
int fused_lag(int64_t np) {
    const int64_t blk = int64_t(kTile) * np * 4;
    return int(std::max<int64_t>(1, std::min<int64_t>(4, (int64_t(64) << 20) / blk - 2)));
}

void plan_fused_buffers(oocnmf_ctx* c) {
    FusedPlan& fp = c->fplan;
    plan_fused(fp, c->mp, c->np, c->num_sms, env_int("OOCNMF_FUSED_D", fused_lag(c->np)));
    std::vector<int> idx;
    idx.insert(idx.end(), fp.q0.begin(), fp.q0.end());
    idx.insert(idx.end(), fp.t0.begin(), fp.t0.end());
    idx.insert(idx.end(), fp.act.begin(), fp.act.end());
    c->fz_idx.alloc(idx.size() * 4, "fused plan");
    ck(cudaMemcpy(c->fz_idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice), "H2D fused plan");
    c->fz_slots.alloc(fused_slot_bytes(c->kp, fp), "fused P1 slots");
    // CTAs without P1 work never publish: their slots must read as zeros in the updaters' gather
    ck(cudaMemsetAsync(c->fz_slots.p, 0, c->fz_slots.bytes, c->stream), "memset fused slots");
    c->fz_count.alloc(size_t(3) * fp.NB * 4, "fused counters");  // count[NB] | wdone[2 NB]
}

void plan_dense(oocnmf_ctx* c) {
    c->use_fused = fused_wanted(c);
    if (c->use_fused) plan_fused_buffers(c);
    const int step = c->use_tc ? kTcStep : kFfmaStep;
    plan_aht(c->sk1, c->mp, c->np, c->num_sms, step);
    plan_wta(c->sk2, c->mp, c->np, c->num_sms, step);
    c->slots1.alloc(size_t(c->sk1.G * c->sk1.smax) * kTile * c->kp * 4, "slots1");
    c->slots2.alloc(size_t(c->sk2.G * c->sk2.smax) * kTile * c->kp * 4, "slots2");
    c->fix_flags.alloc(size_t(c->sk2.G * c->sk2.smax) * 4 * 4, "fix flags");
    ck(cudaMemsetAsync(c->fix_flags.p, 0, c->fix_flags.bytes, c->stream), "memset");
    if (c->cnmf || c->kp > 64) {
        c->N1.alloc(size_t(c->mp) * c->kp * 4, "AHt");
        ck(cudaMemsetAsync(c->N1.p, 0, c->N1.bytes, c->stream), "memset");
    }
}

void reset_source(oocnmf_ctx* c) {
    c->A.release();
    c->rp.release(), c->ci.release(), c->v.release();
    c->rpT.release(), c->ciT.release(), c->vT.release();
    c->chA.seg.release(), c->chT.seg.release();
    c->segR.release(), c->segR_n = 0, c->ag_pending = false;
    c->chA.C = c->chT.C = 1, c->chA.kp = c->chT.kp = 0;
    c->stage[0].release(), c->stage[1].release();
    c->hA = nullptr;
    c->kind = Kind::none;
    c->norm_valid = false;
    c->A0.release(), c->v0.release(), c->vT0.release();
    c->pristine = false;
}

void compute_norm(oocnmf_ctx* c) {
    double* slots = c->red_slots.as<double>();
    double* out = c->scal.as<double>() + kNormA2;
    if (c->kind == Kind::dense) {
        count(c, launch_sq_norm_dense(c->A.as<float>(), c->np, c->mp, c->np, slots, c->stream), "sq_norm");
    } else if (c->kind == Kind::csr) {
        count(c, launch_sq_norm_vals(c->v.as<float>(), c->nnz, slots, c->stream), "sq_norm");
    } else {
        // out-of-core: stream the slab once through the staging buffers.
        double acc = 0.0;
        std::vector<double> part(sqnorm_grid());
        for (int64_t b0 = 0; b0 < int64_t(c->rows); b0 += c->batch_rows) {
            const int64_t br = std::min<int64_t>(c->batch_rows, int64_t(c->rows) - b0);
            ck(cudaMemcpy2DAsync(c->stage[0].p, c->np * 4, c->hA + b0 * c->hlda, c->hlda * 4, c->n * 4, br,
                                 cudaMemcpyHostToDevice, c->stream),
               "H2D batch");
            count(c, launch_sq_norm_dense(c->stage[0].as<float>(), c->np, br, c->np, slots, c->stream), "sq_norm");
            count(c, launch_reduce_f64(slots, sqnorm_grid(), out, c->stream), "reduce");
            double v = 0;
            ck(cudaMemcpyAsync(&v, out, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
            ck(cudaStreamSynchronize(c->stream), "sync");
            acc += v;
        }
        ck(cudaMemcpyAsync(out, &acc, 8, cudaMemcpyHostToDevice, c->stream), "H2D");
        ck(cudaStreamSynchronize(c->stream), "sync");
        goto reduced;
    }
    count(c, launch_reduce_f64(slots, sqnorm_grid(), out, c->stream), "reduce_f64");
reduced:
    if (c->collective()) {
        coll_begin(c, c->stream);
        ncc(c, ncclAllReduce(out, out, 1, ncclDouble, ncclSum, c->comm, c->stream), "allreduce norm");
        coll_end(c, c->stream, kTagErr, 8);  // ||A||^2 (src/nmf_distributed.cpp:232, error_check)
    }
    // (into the pinned scratch: a pageable D2H would block the host behind a hung collective,
    // out of the watchdog's reach)
    ck(cudaMemcpyAsync(c->hpin + 4, out, 8, cudaMemcpyDeviceToHost, c->stream), "D2H norm");
    wait_for(c, c->stream, nullptr, "||A||^2 all-reduce");
    std::memcpy(&c->norm_a2, c->hpin + 4, 8);
    c->norm_valid = true;
}

// [F | F_lo] operand copies: only the dense tensor-core passes read them (the CSR SpMMs read
// W / Ht), so CSR solves skip writing them (2 GB per iteration at config 3)
float* wlo(oocnmf_ctx* c) { return c->use_tc && c->kind != Kind::csr ? c->W_cat.as<float>() : nullptr; }
float* htlo(oocnmf_ctx* c) { return c->use_tc && c->kind != Kind::csr ? c->Ht_cat.as<float>() : nullptr; }

// Pass 1 over an A slab (rows_p x np, rows_p a multiple of 128): slots <- A·Ht partials.
// Wide factors (kp > 64): each pass runs once per 64-column group of the [F_g | F_lo_g]
// group-interleaved operand (kp = 64 tensor-core passes), and its stream-K partials are
// reduced into the group's columns of a plain rows x kp output right away.
bool wide(const oocnmf_ctx* c) { return c->kp > 64; }
cudaError_t pass1(oocnmf_ctx* c, const float* A, int64_t rows_p, float* slots, const StreamK& sk, cudaStream_t s,
                  float* out = nullptr) {
    if (wide(c)) {
        if (!out) return cudaErrorInvalidValue;
        for (int g = 0; g < c->kp / 64; ++g) {
            cudaError_t e = launch_aht_tc(64, A, c->np, rows_p, c->np, c->Ht_cat.as<float>() + 128 * g, slots, sk, s,
                                          2 * c->kp);
            if (e == cudaSuccess) e = launch_streamk_reduce_ld(slots, sk, out + 64 * g, c->kp, false, s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    if (c->use_tc) return launch_aht_tc(c->kp, A, c->np, rows_p, c->np, c->Ht_cat.as<float>(), slots, sk, s);
    return launch_aht(c->kp, A, c->np, c->Ht.as<float>(), slots, sk, s);
}
// Pass 2 over an A slab with its W rows (W rows x kp, Wcat rows x 2kp): slots <- A^T·W partials
// (out_final set: reduced into it; wide factors always reduce into out_final, adding to it when
// accumulate is set).
cudaError_t pass2(oocnmf_ctx* c, const float* A, int64_t rows_p, const float* W, const float* Wcat, float* slots,
                  const StreamK& sk, cudaStream_t s, float* out_final = nullptr, bool accumulate = false) {
    if (wide(c)) {
        if (!out_final) return cudaErrorInvalidValue;
        for (int g = 0; g < c->kp / 64; ++g) {
            cudaError_t e = launch_wta_tc(64, A, c->np, rows_p, c->np, Wcat + 128 * g, slots, sk, s, nullptr, nullptr,
                                          0u, 2 * c->kp);
            if (e == cudaSuccess) e = launch_streamk_reduce_ld(slots, sk, out_final + 64 * g, c->kp, accumulate, s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    if (c->use_tc)
        return launch_wta_tc(c->kp, A, c->np, rows_p, c->np, Wcat, slots, sk, s, out_final,
                             out_final ? c->fix_flags.as<unsigned>() : nullptr, 1u);
    return launch_wta(c->kp, A, c->np, W, slots, sk, s);
}

// HH^T from the per-CTA Gram slots of the last H pass; under CNMF each rank holds a column
// slab of H, so the f32 and f64 Grams are summed over the ranks (the reference's HH^T
// all-reduce, src/nmf_distributed.cpp:115).
void finish_hht(oocnmf_ctx* c, int64_t rows, bool partial) {
    const int kp = c->kp;
    count(c, launch_reduce_slots(c->gram_h.as<double>(), factor_grid(rows / kTile), int64_t(kp) * kp,
                                 c->HHt.as<float>(), c->HHt64.as<double>(), c->stream),
          "reduce HHt");
    if (partial) {
        coll_begin(c, c->stream);
        nck(ncclGroupStart(), "ncclGroupStart");
        ncc(c, ncclAllReduce(c->HHt.p, c->HHt.p, size_t(kp) * kp, ncclFloat, ncclSum, c->comm, c->stream),
            "allreduce HHt");
        ncc(c, ncclAllReduce(c->HHt64.p, c->HHt64.p, size_t(kp) * kp, ncclDouble, ncclSum, c->comm, c->stream),
            "allreduce HHt64");
        ncc(c, ncclGroupEnd(), "ncclGroupEnd");
        coll_end(c, c->stream, kTagW, size_t(kp) * kp * 12);  // CNMF HH^T (nmf_distributed.cpp:116)
    }
}

// HH^T of the current Ht (gram only; also refreshes Ht_cat for the tensor-core pass).
void gram_h(oocnmf_ctx* c) {
    const int kp = c->kp;
    count(c, launch_factor_update(kp, c->Ht.as<float>(), c->np, nullptr, nullptr, nullptr, nullptr, 0.f, false,
                                  c->gram_h.as<double>(), nullptr, c->flag.as<int>(), htlo(c), c->stream),
          "gram H");
    finish_hht(c, c->np, c->cnmf && c->collective());  // a CNMF rank holds a column slab of H
}

// CNMF: A·H^T of this rank's column slab (in N1) summed over the ranks before the
// (replicated) W update (src/nmf_distributed.cpp:124).
void allreduce_aht(oocnmf_ctx* c) {
    if (c->cnmf && c->collective()) {
        coll_begin(c, c->stream);
        ncc(c, ncclAllReduce(c->N1.p, c->N1.p, size_t(c->mp) * c->kp, ncclFloat, ncclSum, c->comm, c->stream),
            "allreduce AHt");
        coll_end(c, c->stream, kTagW, size_t(c->mp) * c->kp * 4);  // nmf_distributed.cpp:124
    }
}

// A timing event: inside a graph capture it must be an external event-record node.
void record(oocnmf_ctx* c, cudaEvent_t e, cudaStream_t s) {
    ck(c->capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s), "event");
}

// CSR W update fused into the A·Ht SpMM (launch_spmm_mu) whenever the numerator is local and
// one-pass: not under CNMF (A·Ht is all-reduced first) nor with column-chunked SpMM passes.
// OOCNMF_FUSE_W=0 selects the separate SpMM + factor-update kernels (bit-identical results).
bool fuse_w_update(const oocnmf_ctx* c) {
    if (c->kind != Kind::csr || c->cnmf || c->chA.C > 1 || c->kp > 64) return false;
    const char* e = std::getenv("OOCNMF_FUSE_W");
    return !(e && *e == '0');
}
// The H update fused into the A^T W SpMM likewise, when W^T A needs no collective (one rank,
// or the replicas of model selection) — on iterations not followed by an error check, whose
// trace-form cross term <W^T A, H> needs the numerator the fused kernel never stores.
// OOCNMF_FUSE_H=0 keeps the separate kernels.
// ---- the NVLS sharded H update (kernels_nvls.cu) -------------------------------------------
// CSR row partitions with a sharded H (shard_h) and a single-pass A^T W SpMM, from 4 ranks
// (config 3 at N = 4: 292 vs 268 it/s; at N = 2, where multicast moves more bytes than a ring,
// 183 vs 185.5). OOCNMF_NVLS=1 / 0 forces it on (from 2 ranks) / off.
bool nvls_wanted(const oocnmf_ctx* c) {
    static const int force = [] {
        const char* e = std::getenv("OOCNMF_NVLS");
        return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
    }();
    const bool want = force >= 0 ? force == 1 : c->nranks >= 4;
    const bool path = c->kind == Kind::csr ? c->chT.C <= 1 : (c->kind == Kind::dense && c->use_fused);
    return want && !c->nvls_failed && nvls_compiled() && path && c->shard_h() &&
           (c->kp == 16 || c->kp == 32 || c->kp == 64);
}
// Collective: every rank of the group reaches it in the same iteration. Moves Ht into the
// symmetric buffer (the NCCL paths keep using it as plain device memory).
void nvls_setup_ctx(oocnmf_ctx* c) {
    std::string why;
    const size_t bytes = size_t(c->np) * c->kp * 4;
    if (!nvls_setup(c->nv, c->comm, bytes, bytes, c->num_sms * 8, c->stream, &why)) {
        c->nvls_failed = true;
        if (c->rank == 0) std::fprintf(stderr, "[oocnmf] NVLS H update unavailable (%s): NCCL collectives\n", why.c_str());
        return;
    }
    ck(cudaMemcpyAsync(c->nv.ht, c->Ht.p, bytes, cudaMemcpyDeviceToDevice, c->stream), "copy Ht");
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->Ht.release();
    c->Ht.p = c->nv.ht, c->Ht.bytes = bytes, c->Ht.external = true;
    c->nvls_ready = true;
}
// Collective: the symmetric buffers released (called when Ht is reallocated for a new rank, or
// at context destruction; Ht's contents are not needed either way).
void nvls_release(oocnmf_ctx* c) {
    if (!c->nvls_ready) return;
    cudaStreamSynchronize(c->stream);
    c->Ht.release();  // external: not freed here, the next alloc_factors makes a private Ht
    nvls_teardown(c->nv, c->comm);
    c->nvls_ready = c->nvls_pending = false;
}
bool nvls_use(const oocnmf_ctx* c) { return c->nvls_ready && c->no_check_next && nvls_wanted(c); }

bool fuse_h_update(const oocnmf_ctx* c) {
    if (c->kind != Kind::csr || c->cnmf || c->collective() || c->chT.C > 1 || c->kp > 64) return false;
    const char* e = std::getenv("OOCNMF_FUSE_H");
    return !(e && *e == '0');
}

// Sharded CSR H update, compute/communication overlap: rank r's rows of W^T A are
// [r hr, (r+1) hr). The SpMM A^T W runs in S row chunks; chunk c covers sub-range c of every
// rank's segment and is written in chunk-major order ([rank][rows][kp] contiguous), so it is
// exactly one ncclReduceScatter's send buffer. Each chunk's reduce-scatter is issued on the
// high-priority comm stream as soon as its SpMM launches retire, landing in this rank's rows of
// W^T A while the SpMM computes the next chunk; only the last chunk's transfer is exposed.
// OOCNMF_RS_CHUNKS sets S (default 4; 1 = the unoverlapped reduce-scatter in h_update).
int rs_chunks(oocnmf_ctx* c) {
    static const int S = [] {
        const char* e = std::getenv("OOCNMF_RS_CHUNKS");
        const int v = e ? std::atoi(e) : 4;
        return std::clamp(v, 1, int(oocnmf_ctx::kMaxRsChunks));
    }();
    return c->shard_h() && c->chT.C <= 1 ? int(std::min<int64_t>(S, c->h_rows())) : 1;
}

// Sharded CSR H update: overlap the H all-gather with the next iteration's A·Ht SpMM
// (OOCNMF_AG_OVERLAP=0 keeps the single all-gather).
bool ag_overlap(const oocnmf_ctx* c) {
    static const bool on = [] {  // measured slower at N = 4 (221 vs 269 it/s): off by default
        const char* e = std::getenv("OOCNMF_AG_OVERLAP");
        return e && e[0] == '1';
    }();
    return on && c->kind == Kind::csr && c->shard_h() && c->chA.C <= 1;
}
// The main stream waits for every pending Ht slice (anything but the sliced SpMM reads all of Ht).
void ht_ready(oocnmf_ctx* c) {
    if (!c->ag_pending) return;
    ck(cudaStreamWaitEvent(c->stream, c->ev_bc[c->nranks - 1], 0), "wait H broadcasts");
    c->ag_pending = false;
}
// A·Ht into N1 over the rank slices of Ht: this rank's slice first, then the others as their
// broadcasts land (k_spmm_seg over the column ranges, accumulating).
void spmm_aht_sliced(oocnmf_ctx* c, cudaStream_t s) {
    const int N = c->nranks;
    const int64_t rows = int64_t(c->rows), hr = c->h_rows();
    if (c->segR_n != N) {
        c->segR.alloc(size_t(N + 1) * rows * 8, "rank-slice segments");
        ck(launch_csr_segments(c->rp.as<int64_t>(), c->ci.as<int32_t>(), rows, hr, N, c->segR.as<int64_t>(), s),
           "rank-slice segments");
        c->segR_n = N;
    }
    const int64_t* seg = c->segR.as<int64_t>();
    bool first = true;
    for (int i = -1; i < N; ++i) {
        const int r = i < 0 ? c->rank : i;
        if (i >= 0 && r == c->rank) continue;
        if (i >= 0) ck(cudaStreamWaitEvent(s, c->ev_bc[r], 0), "wait H slice");
        count(c, launch_spmm_seg(c->kp, seg + int64_t(r) * rows, seg + int64_t(r + 1) * rows, c->ci.as<int32_t>(),
                                 c->v.as<float>(), rows, c->Ht.as<float>(), c->N1.as<float>(), !first, s),
              "spmm A Ht (slice)");
        first = false;
    }
    c->ag_pending = false;
}

void spmm_wta_reduce_scatter(oocnmf_ctx* c, cudaStream_t s) {
    const int kp = c->kp, N = c->nranks, S = rs_chunks(c);
    const int64_t hr = c->h_rows(), h0 = c->h_row0(), n = int64_t(c->n);
    if (c->wtp.bytes != size_t(c->np) * kp * 4) {
        c->wtp.alloc(size_t(c->np) * kp * 4, "W^T A (chunk-major)");
        ck(cudaMemsetAsync(c->wtp.p, 0, c->wtp.bytes, s), "memset");  // padding rows stay 0
    }
    float* wtp = c->wtp.as<float>();
    const int64_t* rpT = c->rpT.as<int64_t>();
    for (int ch = 0; ch < S; ++ch) {
        const int64_t r0 = hr * ch / S, r1 = hr * (ch + 1) / S, len = r1 - r0;
        float* base = wtp + size_t(N) * r0 * kp;
        for (int r = 0; r < N; ++r) {
            const int64_t g0 = int64_t(r) * hr + r0, g1 = std::min(int64_t(r) * hr + r1, n);
            if (g1 > g0)
                count(c, launch_spmm(kp, rpT + g0, c->ciT.as<int32_t>(), c->vT.as<float>(), g1 - g0,
                                     c->W.as<float>(), base + size_t(r) * len * kp, s),
                      "spmm At W (chunk)");
        }
        ck(cudaEventRecord(c->ev_rs[ch], s), "event");
        ck(cudaStreamWaitEvent(c->comm_stream, c->ev_rs[ch], 0), "wait");
        coll_begin(c, c->comm_stream);
        ncc(c, ncclReduceScatter(base, c->wta() + size_t(h0 + r0) * kp, size_t(len) * kp, ncclFloat, ncclSum, c->comm,
                              c->comm_stream),
            "reduce-scatter WtA (chunk)");
        coll_end(c, c->comm_stream, kTagH, size_t(N) * len * kp * 4);
    }
    ck(cudaEventRecord(c->ev_rs[oocnmf_ctx::kMaxRsChunks], c->comm_stream), "event");
    c->rs_done = true;
}

// W update + accumulation of the rank-local [W^T A | W^T W] into c->packed.
void w_update_and_wta(oocnmf_ctx* c, float eps, bool timed, cudaEvent_t* ev) {
    const int kp = c->kp;
    const int gw = factor_grid(c->mp / kTile);
    cudaStream_t s = c->stream;
    auto rec = [&](int i) {
        if (timed) record(c, ev[i], s);
    };
    rec(eStart);
    if (c->kind == Kind::dense && c->use_fused) {
        // one pass over A: P1, the W update and P2 (W^T A of the new W) in one kernel; then the
        // Gram of the new W
        if (!c->nvls_ready && nvls_wanted(c)) nvls_setup_ctx(c);
        const bool nvls = nvls_use(c);  // W^T A into symmetric memory for the NVLS H update
        const FusedPlan& fp = c->fplan;
        ck(cudaMemsetAsync(c->fz_count.p, 0, c->fz_count.bytes, s), "memset fused counters");
        const int* idx = c->fz_idx.as<int>();
        FusedArgs a{};
        static const int p2f = env_int("OOCNMF_FUSED_P2FIRST", 0);
        a.NB = fp.NB, a.D = fp.D, a.NS = fp.NS, a.G1 = fp.G1, a.drain_units = tc::tc_drain_units();
        a.p2_first = p2f;
        a.q0 = idx, a.t0 = idx + fp.G + 1, a.act = idx + 2 * (fp.G + 1);
        a.p1slots = c->fz_slots.as<float>();
        a.count = c->fz_count.as<unsigned>(), a.wdone = a.count + fp.NB;
        a.W = c->W.as<float>(), a.Wcat = c->W_cat.as<float>(), a.HHt = c->HHt.as<float>();
        a.eps = eps, a.flag = c->flag.as<int>(), a.wta = nvls ? static_cast<float*>(c->nv.wp) : c->wta();
        c->nvls_pending = nvls;
        fused_policies(a);
        // the Gram of the new W is accumulated by the updater warps (one f64 slot per CTA);
        // OOCNMF_FUSED_WGRAM=0: the separate Gram pass over W instead
        static const bool wgram_in_kernel = env_int("OOCNMF_FUSED_WGRAM", 1) != 0;
        a.wgram = wgram_in_kernel ? c->gram_w.as<double>() : nullptr;
        count(c, launch_mu_fused(kp, fp, c->A.as<float>(), c->mp, c->np, c->Ht_cat.as<float>(), a, s), "mu fused");
        rec(eAht);
        if (!wgram_in_kernel)
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, nullptr, nullptr, nullptr, nullptr, eps, false,
                                          c->gram_w.as<double>(), nullptr, c->flag.as<int>(), nullptr, s),
                  "W Gram");
        count(c, launch_reduce_slots(c->gram_w.as<double>(), wgram_in_kernel ? fp.G : gw, int64_t(kp) * kp, c->wtw(),
                                     c->WtW64.as<double>(), s),
              "reduce WtW");
        rec(eWdone);
        rec(eWta);
        rec(eReduced);
    } else if (c->kind == Kind::dense) {
        count(c, pass1(c, c->A.as<float>(), c->mp, c->slots1.as<float>(), c->sk1, s, c->N1.as<float>()), "aht");
        rec(eAht);
        if (c->cnmf || wide(c)) {
            // the column slab's A·H^T partials -> one m x kp buffer, summed over the ranks (wide
            // factors: already reduced there by the group passes)
            if (!wide(c))
                count(c, launch_streamk_reduce(kp, c->slots1.as<float>(), c->sk1, c->N1.as<float>(), false, s),
                      "reduce AHt");
            allreduce_aht(c);
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, c->N1.as<float>(), nullptr, nullptr,
                                          c->HHt.as<float>(), eps, true, c->gram_w.as<double>(), nullptr,
                                          c->flag.as<int>(), wlo(c), s),
                  "W update");
        } else {
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, nullptr, c->slots1.as<float>(), &c->sk1,
                                          c->HHt.as<float>(), eps, true, c->gram_w.as<double>(), nullptr,
                                          c->flag.as<int>(), wlo(c), s),
                  "W update");
        }
        count(c, launch_reduce_slots(c->gram_w.as<double>(), gw, int64_t(kp) * kp, c->wtw(), c->WtW64.as<double>(), s), "reduce WtW");
        rec(eWdone);
        if (c->use_tc) {
            // the tensor-core pass reduces its own stream-K partials into W^T A
            count(c, pass2(c, c->A.as<float>(), c->mp, c->W.as<float>(), wlo(c), c->slots2.as<float>(), c->sk2, s,
                           c->wta()),
                  "wta");
            rec(eWta);
        } else {
            count(c, pass2(c, c->A.as<float>(), c->mp, c->W.as<float>(), wlo(c), c->slots2.as<float>(), c->sk2, s),
                  "wta");
            rec(eWta);
            count(c, launch_streamk_reduce(kp, c->slots2.as<float>(), c->sk2, c->wta(), false, s), "reduce WtA");
        }
        rec(eReduced);
    } else if (c->kind == Kind::csr) {
        if (!c->nvls_ready && nvls_wanted(c)) nvls_setup_ctx(c);
        if (c->ag_pending) {
            // H slices still arriving: the SpMM consumes them as they land, then the W update
            spmm_aht_sliced(c, s);
            rec(eAht);
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, c->N1.as<float>(), nullptr, nullptr,
                                          c->HHt.as<float>(), eps, true, c->gram_w.as<double>(), nullptr,
                                          c->flag.as<int>(), nullptr, s),
                  "W update");
        } else if (fuse_w_update(c)) {
            // A·Ht and the W update in one pass over the rows, then the Gram of the new W
            count(c, launch_spmm_mu(kp, c->rp.as<int64_t>(), c->ci.as<int32_t>(), c->v.as<float>(), c->rows,
                                    c->Ht.as<float>(), c->W.as<float>(), c->HHt.as<float>(), eps, c->flag.as<int>(), s),
                  "spmm A Ht + W update");
            rec(eAht);
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, nullptr, nullptr, nullptr, nullptr, eps, false,
                                          c->gram_w.as<double>(), nullptr, c->flag.as<int>(), nullptr, s),
                  "W Gram");
        } else {
            spmm(c, false, c->Ht.as<float>(), c->N1.as<float>(), s);
            rec(eAht);
            allreduce_aht(c);
            count(c, launch_factor_update(kp, c->W.as<float>(), c->mp, c->N1.as<float>(), nullptr, nullptr,
                                          c->HHt.as<float>(), eps, true, c->gram_w.as<double>(), nullptr,
                                          c->flag.as<int>(), nullptr, s),
                  "W update");
        }
        count(c, launch_reduce_slots(c->gram_w.as<double>(), gw, int64_t(kp) * kp, c->wtw(), c->WtW64.as<double>(), s), "reduce WtW");
        rec(eWdone);
        if (c->no_check_next && fuse_h_update(c)) {
            count(c, launch_spmm_mu(kp, c->rpT.as<int64_t>(), c->ciT.as<int32_t>(), c->vT.as<float>(), c->n,
                                    c->W.as<float>(), c->Ht.as<float>(), c->wtw(), eps, c->flag.as<int>(), s),
                  "spmm At W + H update");
            c->h_fused = true;
        } else if (nvls_use(c)) {
            // this rank's partial W^T A into symmetric memory; h_update reduces it over NVLS
            spmm(c, true, c->W.as<float>(), static_cast<float*>(c->nv.wp), s);
            c->nvls_pending = true;
        } else if (rs_chunks(c) > 1) {
            spmm_wta_reduce_scatter(c, s);
        } else {
            spmm(c, true, c->W.as<float>(), c->wta(), s);
        }
        rec(eWta);
        rec(eReduced);
    } else {
        // Out-of-core fused row-batch schedule: each batch crosses the host link once and
        // serves both its W rows' update and its W^T A contribution.
        const int64_t nb = (int64_t(c->rows) + c->batch_rows - 1) / c->batch_rows;
        const int gwb = factor_grid(c->batch_rows / kTile);
        for (int64_t b = 0; b < nb; ++b) {
            const int si = int(b & 1);
            const int64_t b0 = b * c->batch_rows;
            const int64_t br = std::min<int64_t>(c->batch_rows, int64_t(c->rows) - b0);
            const int64_t brp = round_up(br, kTile);
            const StreamK& s1 = (br == c->batch_rows) ? c->sk1b[0] : c->sk1b[1];
            const StreamK& s2 = (br == c->batch_rows) ? c->sk2b[0] : c->sk2b[1];
            float* st = c->stage[si].as<float>();
            ck(cudaStreamWaitEvent(c->copy_stream, c->ev_free[si], 0), "wait free");
            if (brp != br)
                ck(cudaMemsetAsync(st + br * c->np, 0, size_t(brp - br) * c->np * 4, c->copy_stream), "memset tail");
            ck(cudaMemcpy2DAsync(st, c->np * 4, c->hA + b0 * c->hlda, c->hlda * 4, c->n * 4, br,
                                 cudaMemcpyHostToDevice, c->copy_stream),
               "H2D batch");
            ck(cudaEventRecord(c->ev_copied[si], c->copy_stream), "event");
            ck(cudaStreamWaitEvent(s, c->ev_copied[si], 0), "wait copied");
            float* Wb = c->W.as<float>() + b0 * kp;
            float* Wlob = c->use_tc ? c->W_cat.as<float>() + b0 * 2 * kp : nullptr;
            count(c, pass1(c, st, brp, c->slots1.as<float>(), s1, s, c->N1.as<float>()), "aht");
            count(c, launch_factor_update(kp, Wb, brp, wide(c) ? c->N1.as<float>() : nullptr,
                                          wide(c) ? nullptr : c->slots1.as<float>(), &s1, c->HHt.as<float>(), eps,
                                          true, c->gram_w.as<double>() + b * gwb * kp * kp, nullptr,
                                          c->flag.as<int>(), Wlob, s),
                  "W update");
            if (wide(c)) {
                count(c, pass2(c, st, brp, Wb, Wlob, c->slots2.as<float>(), s2, s, c->wta(), b > 0), "wta");
            } else {
                count(c, pass2(c, st, brp, Wb, Wlob, c->slots2.as<float>(), s2, s), "wta");
                count(c, launch_streamk_reduce(kp, c->slots2.as<float>(), s2, c->wta(), b > 0, s), "reduce WtA");
            }
            ck(cudaEventRecord(c->ev_free[si], s), "event");
        }
        count(c, launch_reduce_slots(c->gram_w.as<double>(), nb * gwb, int64_t(kp) * kp, c->wtw(), c->WtW64.as<double>(), s), "reduce WtW");
        rec(eAht);
        rec(eWdone);
        rec(eWta);
        rec(eReduced);
    }
}

void h_update(oocnmf_ctx* c, float eps, bool timed, cudaEvent_t* ev) {
    const int kp = c->kp;
    cudaStream_t s = c->stream;
    const int64_t hr = c->h_rows(), h0 = c->h_row0();
    if (c->nvls_pending) {
        // W^T W (f32 for the update, f64 for the trace-form error) over NCCL, then one kernel:
        // reduce this rank's rows of W^T A over NVLS, update them, multicast the new rows
        coll_begin(c, s);
        nck(ncclGroupStart(), "ncclGroupStart");
        ncc(c, ncclAllReduce(c->wtw(), c->wtw(), size_t(kp) * kp, ncclFloat, ncclSum, c->comm, s), "allreduce WtW");
        ncc(c, ncclAllReduce(c->WtW64.p, c->WtW64.p, size_t(kp) * kp, ncclDouble, ncclSum, c->comm, s),
            "allreduce WtW64");
        ncc(c, ncclGroupEnd(), "ncclGroupEnd");
        coll_end(c, s, kTagH, size_t(kp) * kp * 12);
        if (timed) record(c, ev[eComm], s);
        NvlsArgs a{};
        a.mc_wp = static_cast<const float*>(c->nv.mc[0]);
        a.mc_ht = static_cast<float*>(c->nv.mc[1]);
        a.mc_bar = static_cast<unsigned*>(c->nv.mc[2]);
        a.bar = static_cast<const unsigned*>(c->nv.bar);
        a.ht = c->Ht.as<float>(), a.wtw = c->wtw(), a.flag = c->flag.as<int>();
        a.row0 = h0, a.rows = hr, a.epoch = c->nv.epoch++, a.nranks = c->nranks, a.eps = eps;
        // a peer that never arrives: the kernel traps after twice the group timeout (>= 30 s),
        // after the watchdog has already raised CommError on the host
        a.timeout_ns = uint64_t(std::max(30.0, 2.0 * c->comm_timeout) * 1e9);
        coll_begin(c, s);
        static const int ctas_per_sm = std::clamp(env_int("OOCNMF_NVLS_CTAS", 1), 1, 8);  // developer knob
        count(c, launch_h_update_nvls(kp, a, c->num_sms * ctas_per_sm, s), "NVLS H update");
        coll_end(c, s, kTagH, size_t(c->nranks) * hr * kp * 4 * 2);  // the reduce-scatter + all-gather it replaces
        if (float* hc = htlo(c)) count(c, launch_split_cat(c->Ht.as<float>(), hc, c->np, kp, s), "split H");
        count(c, launch_factor_update(kp, c->Ht.as<float>() + h0 * kp, hr, nullptr, nullptr, nullptr, nullptr, eps,
                                      false, c->gram_h.as<double>(), nullptr, c->flag.as<int>(), nullptr, s),
              "H Gram");
        finish_hht(c, hr, true);
        c->nvls_pending = false;
        if (timed) record(c, ev[eHdone], s);
        return;
    }
    if (c->shard_h()) {
        // reduce-scatter W^T A (each rank keeps its n/N rows, in place) + the small Grams; with
        // the overlapped SpMM the scatter is already on the comm stream
        const size_t slice = size_t(hr) * kp;
        float* wta = c->wta();
        if (c->rs_done) ck(cudaStreamWaitEvent(s, c->ev_rs[oocnmf_ctx::kMaxRsChunks], 0), "wait reduce-scatter");
        coll_begin(c, s);
        nck(ncclGroupStart(), "ncclGroupStart");
        if (!c->rs_done)
            ncc(c, ncclReduceScatter(wta, wta + size_t(c->rank) * slice, slice, ncclFloat, ncclSum, c->comm, s),
                "reduce-scatter WtA");
        ncc(c, ncclAllReduce(c->wtw(), c->wtw(), size_t(kp) * kp, ncclFloat, ncclSum, c->comm, s), "allreduce WtW");
        ncc(c, ncclAllReduce(c->WtW64.p, c->WtW64.p, size_t(kp) * kp, ncclDouble, ncclSum, c->comm, s),
            "allreduce WtW64");
        ncc(c, ncclGroupEnd(), "ncclGroupEnd");
        coll_end(c, s, kTagH, (c->rs_done ? 0 : size_t(c->nranks) * slice * 4) + size_t(kp) * kp * 12);
        c->rs_done = false;
    } else if (c->collective() && !c->cnmf) {
        // One fused NCCL launch: the packed f32 [W^T A | W^T W] the update consumes and the f64
        // W^T W the trace-form error consumes. (CNMF: W^T A of the column slab and W^T W of the
        // replicated W are already complete on every rank.)
        // (the f64 copy only ahead of an error check: nothing else reads it)
        const bool with64 = !c->no_check_next;
        coll_begin(c, s);
        nck(ncclGroupStart(), "ncclGroupStart");
        ncc(c, ncclAllReduce(c->packed.p, c->packed.p, size_t(c->packed_count()), ncclFloat, ncclSum, c->comm, s),
            "allreduce [WtA|WtW]");
        if (with64)
            ncc(c, ncclAllReduce(c->WtW64.p, c->WtW64.p, size_t(kp) * kp, ncclDouble, ncclSum, c->comm, s),
                "allreduce WtW64");
        ncc(c, ncclGroupEnd(), "ncclGroupEnd");
        coll_end(c, s, kTagH, size_t(c->packed_count()) * 4 + (with64 ? size_t(kp) * kp * 8 : 0));  // nmf_distributed.cpp:171,178
    }
    if (timed) record(c, ev[eComm], s);
    // sharded H: the [H | H_lo] operand of the next pass is rebuilt from the gathered H below
    float* hcat = c->shard_h() ? nullptr : htlo(c);
    if (c->h_fused) {  // updated inside the SpMM: the Gram of the new rows only
        count(c, launch_factor_update(kp, c->Ht.as<float>(), hr, nullptr, nullptr, nullptr, nullptr, eps, false,
                                      c->gram_h.as<double>(), nullptr, c->flag.as<int>(), nullptr, s),
              "H Gram");
        c->h_fused = false;
    } else {
        count(c, launch_factor_update(kp, c->Ht.as<float>() + h0 * kp, hr, c->wta() + h0 * kp, nullptr, nullptr,
                                      c->wtw(), eps, true, c->gram_h.as<double>(), c->err_slots.as<double>(),
                                      c->flag.as<int>(), hcat ? hcat + h0 * 2 * kp : nullptr, s),
              "H update");
    }
    if (c->shard_h() && ag_overlap(c)) {
        // the all-gather as N broadcasts on the comm stream; the next SpMM starts on this rank's
        // slice and picks up the others as their events fire (spmm_aht_sliced)
        if (int(c->ev_bc.size()) < c->nranks) {
            c->ev_bc.resize(c->nranks, nullptr);
            for (auto& e : c->ev_bc)
                if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            if (!c->ev_hdone) ck(cudaEventCreateWithFlags(&c->ev_hdone, cudaEventDisableTiming), "event");
        }
        ck(cudaEventRecord(c->ev_hdone, s), "event");
        ck(cudaStreamWaitEvent(c->comm_stream, c->ev_hdone, 0), "wait H update");
        coll_begin(c, c->comm_stream);
        for (int r = 0; r < c->nranks; ++r) {
            float* sl = c->Ht.as<float>() + size_t(r) * hr * kp;
            ncc(c, ncclBroadcast(sl, sl, size_t(hr) * kp, ncclFloat, r, c->comm, c->comm_stream), "broadcast H slice");
            ck(cudaEventRecord(c->ev_bc[r], c->comm_stream), "event");
        }
        coll_end(c, c->comm_stream, kTagH, size_t(c->nranks) * hr * kp * 4);
        c->ag_pending = true;
    } else if (c->shard_h()) {
        coll_begin(c, s);
        ncc(c, ncclAllGather(c->Ht.as<float>() + h0 * kp, c->Ht.p, size_t(hr) * kp, ncclFloat, c->comm, s),
            "all-gather H");
        coll_end(c, s, kTagH, size_t(c->nranks) * hr * kp * 4);
        if (htlo(c)) count(c, launch_split_cat(c->Ht.as<float>(), htlo(c), c->np, kp, s), "split H");
    }
    finish_hht(c, hr, c->collective() && (c->cnmf || c->shard_h()));
    if (timed) record(c, ev[eHdone], s);
}


// Below this trace-form estimate of the relative error, error_mode auto re-evaluates the
// error with the direct residual: the trace form subtracts O(||A||^2) terms, so an f32-level
// relative error of ~1e-7 in them grows by 1/err^2 (SURVEY.md §7 hard part 2).
constexpr double kAutoDirectBelow = 0.1;

// Enqueue the error evaluation of one check with no host round trip: errs[slot] <- the
// relative error, flags[slot] <- the sticky non-finite flag. error_mode 0 (auto) computes the
// trace form and then the direct residual predicated on the device-side estimate being below
// kAutoDirectBelow (the residual kernels and the second finalize read the predicate and exit
// when it is 0); 1 (direct) always takes the residual; 2 (trace) never. Out-of-core runs use
// the trace form only.
void enqueue_check(oocnmf_ctx* c, int error_mode, uint64_t slot) {
    ht_ready(c);  // the direct residual reads all of Ht
    const int kp = c->kp;
    cudaStream_t s = c->stream;
    double* scal = c->scal.as<double>();
    double* out = c->errs.as<double>() + slot;
    int* pred = c->pred.as<int>();
    const bool direct = error_mode != 2 && c->kind != Kind::host;
    const double threshold = error_mode == 1 ? INFINITY : kAutoDirectBelow;
    const double* eslots = c->err_slots.as<double>();
    int64_t n_err = factor_grid(c->h_rows() / kTile);
    if (c->collective() && (c->cnmf || c->shard_h())) {
        // CNMF / sharded H: <W^T A, H> is a sum over the ranks' slabs
        count(c, launch_reduce_f64(eslots, n_err, scal + kCross, s), "reduce cross");
        coll_begin(c, s);
        ncc(c, ncclAllReduce(scal + kCross, scal + kCross, 1, ncclDouble, ncclSum, c->comm, s), "allreduce cross");
        coll_end(c, s, kTagErr, 8);
        eslots = scal + kCross;
        n_err = 1;
    }
    count(c, launch_finalize_error(kp, eslots, n_err, c->WtW64.as<double>(), c->HHt64.as<double>(), scal + kNormA2,
                                   nullptr, out, s, nullptr, direct ? pred : nullptr, threshold),
          "finalize");
    if (direct) {
        if (c->kind == Kind::dense) {
            count(c, launch_residual_dense(kp, c->A.as<float>(), c->np, c->rows, c->n, c->W.as<float>(),
                                           c->Ht.as<float>(), c->red_slots.as<double>(), s, pred),
                  "residual");
            count(c, launch_reduce_f64(c->red_slots.as<double>(), sqnorm_grid(), scal + kRes, s), "reduce");
            if (c->collective()) {
                coll_begin(c, s);
                ncc(c, ncclAllReduce(scal + kRes, scal + kRes, 1, ncclDouble, ncclSum, c->comm, s), "allreduce res");
                coll_end(c, s, kTagErr, 8);  // nmf_distributed.cpp:254
            }
            count(c, launch_finalize_error(kp, nullptr, 0, c->WtW64.as<double>(), c->HHt64.as<double>(),
                                           scal + kNormA2, scal + kRes, out, s, pred),
                  "finalize direct");
        } else {
            count(c, launch_residual_csr(kp, c->rp.as<int64_t>(), c->ci.as<int32_t>(), c->v.as<float>(), c->rows,
                                         c->n, c->W.as<float>(), c->Ht.as<float>(), c->red_slots.as<double>(), s,
                                         pred),
                  "cross");
            count(c, launch_reduce_f64(c->red_slots.as<double>(), sqnorm_grid(), scal + kCross, s), "reduce");
            if (c->collective()) {
                coll_begin(c, s);
                ncc(c, ncclAllReduce(scal + kCross, scal + kCross, 1, ncclDouble, ncclSum, c->comm, s),
                    "allreduce cross");
                coll_end(c, s, kTagErr, 8);
            }
            count(c, launch_finalize_error(kp, scal + kCross, 1, c->WtW64.as<double>(), c->HHt64.as<double>(),
                                           scal + kNormA2, nullptr, out, s, pred),
                  "finalize direct");
        }
    }
    ck(cudaMemcpyAsync(c->flags.as<int>() + slot, c->flag.p, 4, cudaMemcpyDeviceToDevice, s), "flag");
}

void ensure_events(oocnmf_ctx* c, size_t n) {
    while (c->evs.size() < n) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        c->evs.push_back(e);
    }
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
    return ms;
}

void prepare_factors(oocnmf_ctx* c, const oocnmf_config* cfg) {
    if (cfg->init == 1) {
        if (!c->factors_set)
            fail(OOCNMF_ERR_SHAPE, "init=from_files requires factors (oocnmf_set_factors_f64)");
    } else if (cfg->init == 2) {
        if (!c->factors_valid) fail(OOCNMF_ERR_SHAPE, "init=continue requires resident factors");
    } else {
        ck(cudaMemsetAsync(c->W.p, 0, c->W.bytes, c->stream), "memset W");
        ck(cudaMemsetAsync(c->Ht.p, 0, c->Ht.bytes, c->stream), "memset Ht");
        count(c, launch_init_factors(c->W.as<float>(), c->Ht.as<float>(), c->kp, c->k, c->rows, c->row0, c->n,
                                     c->n_global, c->col0, cfg->seed, c->stream),
              "init");
    }
    c->factors_valid = true;
}

// `count` MU iterations; iteration i records its events into ev + kEvPerIter * i. In-core
// single-rank problems replay a captured CUDA graph of the whole block (one launch instead of
// ~10 per iteration); OOCNMF_NO_GRAPH=1 iterates eagerly.
void run_iterations(oocnmf_ctx* c, float eps, uint64_t count, cudaEvent_t* ev) {
    static const bool no_graph = [] {
        const char* e = std::getenv("OOCNMF_NO_GRAPH");
        return e && e[0] == '1';
    }();
    auto eager = [&] {
        for (uint64_t i = 0; i < count; ++i) {
            c->no_check_next = i + 1 < count;  // a block's last iteration precedes its error check
            w_update_and_wta(c, eps, true, ev + kEvPerIter * i);
            h_update(c, eps, true, ev + kEvPerIter * i);
        }
        c->no_check_next = false;
    };
    // Graphs for single-rank solves only: replaying NCCL work from graphs made every launch
    // pay NCCL's graph/non-graph mixing synchronisation (4 x B200: 555 it/s with graphs, 634
    // eager, 627 with NCCL_GRAPH_MIXING_SUPPORT=0), while the eager loop keeps the queue full
    // now that the error checks no longer sync the host.
    if (no_graph || c->graph_broken || c->kind == Kind::host || c->collective()) return eager();
    uint32_t eps_bits;
    std::memcpy(&eps_bits, &eps, 4);
    const std::vector<uint64_t> key = {
        uint64_t(c->kind), uint64_t(c->kp), uint64_t(c->mp), uint64_t(c->np), c->rows, count, eps_bits,
        uint64_t(c->use_tc), uint64_t(c->collective()), uint64_t(c->cnmf), uint64_t(reinterpret_cast<uintptr_t>(c->comm)),
        uint64_t(reinterpret_cast<uintptr_t>(ev)), uint64_t(reinterpret_cast<uintptr_t>(c->A.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->rp.p)), uint64_t(reinterpret_cast<uintptr_t>(c->rpT.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->W.p)), uint64_t(reinterpret_cast<uintptr_t>(c->Ht.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->W_cat.p)), uint64_t(reinterpret_cast<uintptr_t>(c->Ht_cat.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->packed.p)), uint64_t(reinterpret_cast<uintptr_t>(c->slots1.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->slots2.p)), uint64_t(reinterpret_cast<uintptr_t>(c->N1.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->gram_w.p)), uint64_t(reinterpret_cast<uintptr_t>(c->gram_h.p)),
        uint64_t(c->sk1.G), uint64_t(c->sk1.tiles), uint64_t(c->sk2.G), uint64_t(c->sk2.tiles),
        uint64_t(reinterpret_cast<uintptr_t>(c->chA.seg.p)), uint64_t(reinterpret_cast<uintptr_t>(c->chT.seg.p)),
        uint64_t(c->chA.C), uint64_t(c->chT.C), uint64_t(fuse_w_update(c)), uint64_t(fuse_h_update(c)),
        uint64_t(c->use_fused), uint64_t(reinterpret_cast<uintptr_t>(c->fz_idx.p)),
        uint64_t(reinterpret_cast<uintptr_t>(c->fz_slots.p)), uint64_t(reinterpret_cast<uintptr_t>(c->fz_count.p)),
        uint64_t(c->fplan.D), uint64_t(c->HHt.p ? reinterpret_cast<uintptr_t>(c->HHt.p) : 0)};
    oocnmf_ctx::Graph* hit = nullptr;
    for (auto& g : c->graphs)
        if (g.key == key) hit = &g;
    if (!hit) {
        if (c->graphs.size() >= 4) {
            cudaGraphExecDestroy(c->graphs.front().exec);
            c->graphs.erase(c->graphs.begin());
        }
        cudaGraphExec_t exec = nullptr;
        const uint64_t l0 = c->launches;
        cudaGraph_t g = nullptr;
        bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            c->capturing = true;
            try {
                eager();
            } catch (...) {
                c->capturing = false;
                cudaStreamEndCapture(c->stream, &g);
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                c->launches = l0;
                c->graph_broken = true;  // replay eagerly from now on
                return eager();
            }
            c->capturing = false;
            ok = cudaStreamEndCapture(c->stream, &g) == cudaSuccess && g;
        }
        ok = ok && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        const uint64_t nl = c->launches - l0;
        c->launches = l0;
        if (!ok) {
            cudaGetLastError();
            c->graph_broken = true;
            return eager();
        }
        c->graphs.push_back({key, exec, nl});
        hit = &c->graphs.back();
    }
    ck(cudaGraphLaunch(hit->exec, c->stream), "cudaGraphLaunch");
    c->launches += hit->launches;
}

void solve_impl(oocnmf_ctx* c, const oocnmf_config* cfg, uint64_t* trace_iter, double* trace_err,
                uint64_t trace_cap, oocnmf_info* info) {
    need_problem(c);
    if (!cfg) fail(OOCNMF_ERR_SHAPE, "null config");
    if (cfg->k != c->k)
        fail(OOCNMF_ERR_SHAPE, "config k=" + std::to_string(cfg->k) + " disagrees with problem k=" + std::to_string(c->k));
    if (!(cfg->eta >= 0)) fail(OOCNMF_ERR_SHAPE, "NmfConfig: eta must be >= 0");
    if (cfg->max_iters < 1) fail(OOCNMF_ERR_SHAPE, "NmfConfig: max_iters must be >= 1");
    if (cfg->error_check_interval < 1) fail(OOCNMF_ERR_SHAPE, "NmfConfig: error_check_interval must be >= 1");
    if (!(cfg->epsilon > 0)) fail(OOCNMF_ERR_SHAPE, "NmfConfig: epsilon must be > 0");
    if (cfg->error_mode < 0 || cfg->error_mode > 2) fail(OOCNMF_ERR_SHAPE, "error_mode must be 0, 1 or 2");
    if (cfg->error_mode == 1 && c->kind == Kind::host)
        fail(OOCNMF_ERR_SHAPE, "error_mode=direct is not supported out-of-core");
    if (c->kind == Kind::none) fail(OOCNMF_ERR_SHAPE, "no A loaded");
    if (c->collective()) need_comm(c);

    const auto t0 = std::chrono::steady_clock::now();
    c->launches = 0;
    oocnmf_info inf{};
    prepare_factors(c, cfg);
    ensure_chunks(c);
    if (!c->norm_valid) compute_norm(c);
    if (c->norm_a2 == 0.0) fail(OOCNMF_ERR_DATA, "nmf: ||A||_F is zero");
    ck(cudaMemsetAsync(c->flag.p, 0, 4, c->stream), "memset flag");
    gram_h(c);

    const float eps = float(cfg->epsilon);
    const uint64_t interval = cfg->error_check_interval;
    const double flops_per_iter = 4.0 * double(c->rows) * double(c->n) * double(c->k) +
                                  2.0 * double(c->rows + c->n) * double(c->k) * double(c->k);
    // Two event sets alternate between consecutive blocks (a block = the iterations up to and
    // including one error check), so the host reads a block's timings while the next one runs;
    // the checks themselves are evaluated on the device into errs / flags. Only eta > 0 needs
    // each value on the host before the next block (early exit), and then the loop syncs.
    const size_t set_size = size_t(kEvPerIter) * interval + 2;
    ensure_events(c, 2 * set_size);
    const uint64_t max_checks = cfg->max_iters / interval + 2;
    c->errs.alloc(std::max<size_t>(c->errs.bytes, max_checks * 8), "errs");
    c->flags.alloc(std::max<size_t>(c->flags.bytes, max_checks * 4), "flags");
    c->pred.alloc(std::max<size_t>(c->pred.bytes, 4), "pred");
    struct Pending {
        uint64_t iters;
        cudaEvent_t* ev;
    };
    std::vector<Pending> pend;
    const bool fused_run = c->kind == Kind::dense && c->use_fused;
    auto drain = [&](const Pending& p) {
        cudaEvent_t* ce = p.ev + kEvPerIter * p.iters;
        wait_for(c, c->stream, ce[1], "an iteration block");
        for (uint64_t i = 0; i < p.iters; ++i) {
            cudaEvent_t* e = p.ev + kEvPerIter * i;
            if (fused_run) {
                inf.fused_pass_ms += elapsed(e[eStart], e[eAht]);
                inf.fused_pass_launches += 1;
            } else {
                inf.aht_pass_ms += elapsed(e[eStart], e[eAht]);
                inf.wta_pass_ms += elapsed(e[eWdone], e[eWta]);
                inf.aht_pass_launches += 1;
                inf.wta_pass_launches += 1;
            }
            inf.w_update_s += elapsed(e[eStart], e[eWdone]) * 1e-3;
            inf.allreduce_s += elapsed(e[eReduced], e[eComm]) * 1e-3;
            inf.h_update_s += (elapsed(e[eWdone], e[eReduced]) + elapsed(e[eComm], e[eHdone])) * 1e-3;
        }
        inf.error_check_s += elapsed(ce[0], ce[1]) * 1e-3;
    };
    static const bool force_sync = [] {
        const char* e = std::getenv("OOCNMF_SYNC_CHECKS");
        return e && e[0] == '1';
    }();
    // eta > 0: the early exit (nmf_serial.cpp:111 `if (err <= cfg.eta) break`) is taken one
    // block late so the device never idles on the host: block b is enqueued before check b-1's
    // value is read. Each check therefore snapshots W and Ht (two alternating device copies,
    // ~5 us at config 2), and an exit at check b-1 restores its snapshot, discarding block b.
    const bool sync_each = cfg->eta > 0.0 || force_sync;
    if (sync_each)
        for (int p = 0; p < 2; ++p) {
            c->snapW[p].alloc(c->W.bytes, "W snapshot");
            c->snapH[p].alloc(c->Ht.bytes, "Ht snapshot");
        }
    std::vector<uint64_t> check_iter;
    uint64_t iter = 0, nt = 0;
    bool converged = false, stopped = false;
    // decide on the check enqueued as block bb (its values were copied to hpin[2 (bb & 1)]);
    // returns true when the solve stops there
    auto decide = [&](uint64_t bb, cudaEvent_t done) -> bool {
        wait_for(c, c->stream, done, "an error check");
        double e = 0.0;
        int f = 0;
        std::memcpy(&e, c->hpin + 2 * (bb & 1), 8);
        std::memcpy(&f, c->hpin + 2 * (bb & 1) + 1, 4);
        if (f) return true;  // reported below, with the iteration of the first bad check
        if (e <= cfg->eta) {
            converged = true;
            return true;
        }
        return false;
    };
    cudaEvent_t prev_done = nullptr;
    for (uint64_t next = 1, b = 0; next <= cfg->max_iters; ++b) {
        const uint64_t block = std::min<uint64_t>(interval - (next - 1) % interval, cfg->max_iters - next + 1);
        cudaEvent_t* ev = c->evs.data() + set_size * (b & 1);
        if (pend.size() == 2) {  // the set this block reuses belongs to block b - 2
            drain(pend.front());
            pend.erase(pend.begin());
        }
        run_iterations(c, eps, block, ev);
        cudaEvent_t* ce = ev + kEvPerIter * block;
        ck(cudaEventRecord(ce[0], c->stream), "event");
        enqueue_check(c, cfg->error_mode, nt);
        if (sync_each) {
            double* hp = c->hpin + 2 * (b & 1);
            ck(cudaMemcpyAsync(hp, c->errs.as<double>() + nt, 8, cudaMemcpyDeviceToHost, c->stream), "D2H err");
            ck(cudaMemcpyAsync(hp + 1, c->flags.as<int>() + nt, 4, cudaMemcpyDeviceToHost, c->stream), "D2H flag");
            ck(cudaMemcpyAsync(c->snapW[b & 1].p, c->W.p, c->W.bytes, cudaMemcpyDeviceToDevice, c->stream), "snapshot W");
            ck(cudaMemcpyAsync(c->snapH[b & 1].p, c->Ht.p, c->Ht.bytes, cudaMemcpyDeviceToDevice, c->stream),
               "snapshot Ht");
        }
        ck(cudaEventRecord(ce[1], c->stream), "event");
        pend.push_back({block, ev});
        inf.flops += flops_per_iter * double(block);
        iter = next + block - 1;
        next += block;
        check_iter.push_back(iter);
        ++nt;
        if (sync_each) {
            if (b > 0 && decide(b - 1, prev_done)) {
                // stop at check b - 1: drop block b and restore the factors as they were there
                wait_for(c, c->stream, nullptr, "the discarded block");
                ck(cudaMemcpyAsync(c->W.p, c->snapW[(b - 1) & 1].p, c->W.bytes, cudaMemcpyDeviceToDevice, c->stream),
                   "restore W");
                ck(cudaMemcpyAsync(c->Ht.p, c->snapH[(b - 1) & 1].p, c->Ht.bytes, cudaMemcpyDeviceToDevice,
                                   c->stream),
                   "restore Ht");
                inf.flops -= flops_per_iter * double(block);
                --nt;
                check_iter.pop_back();
                iter = check_iter.back();
                stopped = true;
                break;
            }
            prev_done = ce[1];
        }
    }
    if (sync_each && !stopped && nt > 0) decide(nt - 1, prev_done);
    wait_for(c, c->stream, nullptr, "the solve");
    for (const auto& p : pend) drain(p);
    std::vector<double> errs(nt);
    std::vector<int> flags(nt);
    ck(cudaMemcpy(errs.data(), c->errs.p, nt * 8, cudaMemcpyDeviceToHost), "D2H errs");
    ck(cudaMemcpy(flags.data(), c->flags.p, nt * 4, cudaMemcpyDeviceToHost), "D2H flags");
    if (!sync_each) {
        // eta = 0 runs without host round trips; the reference still stops at a check whose
        // error is <= 0 (an exact fit), so the trace ends at the first such check. (The factors
        // are then those of the last iteration: at an exact fit the MU ratios are 1.)
        for (uint64_t i = 0; i < nt; ++i)
            if (!flags[i] && errs[i] <= cfg->eta) {
                nt = i + 1;
                iter = check_iter[i];
                converged = true;
                break;
            } else if (flags[i]) {
                break;
            }
    }
    for (uint64_t i = 0; i < nt; ++i) {
        if (flags[i])
            fail(OOCNMF_ERR_DATA, "nmf: non-finite factor entries at iteration " + std::to_string(check_iter[i]));
        if (trace_iter && i < trace_cap) {
            trace_iter[i] = check_iter[i];
            trace_err[i] = errs[i];
        }
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    inf.iterations_run = iter;
    inf.converged = converged ? 1 : 0;
    inf.n_trace = nt;
    inf.gpu_launches = c->launches;
    if (c->kind == Kind::host) {
        inf.io_s = 0;  // overlapped with compute; reported through h2d_bytes
        inf.h2d_bytes = double(inf.iterations_run) * double(c->rows) * double(c->n) * 4.0;
        inf.h2d_batches = inf.iterations_run * uint64_t((int64_t(c->rows) + c->batch_rows - 1) / c->batch_rows);
        inf.peak_resident_bytes = uint64_t(c->stage[0].bytes + c->stage[1].bytes);
    }
    inf.total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (info) *info = inf;
}

void set_problem_impl(oocnmf_ctx* c, uint64_t m, uint64_t n, uint64_t k, uint64_t row0, uint64_t rows) {
    if (m < 1 || n < 1 || k < 1) fail(OOCNMF_ERR_SHAPE, "nmf: dimensions must be >= 1");
    if (rows < 1 || row0 + rows > m) fail(OOCNMF_ERR_SHAPE, "row slab out of bounds");
    if (n > uint64_t(INT32_MAX) || rows > uint64_t(INT32_MAX))
        fail(OOCNMF_ERR_SHAPE, "dimension exceeds the 2^31 index range of the device layout");
    reset_source(c);
    c->m = m, c->n = n, c->k = k, c->row0 = row0, c->rows = rows;
    c->cnmf = false, c->col0 = 0, c->n_global = n;
    // Tensor-core passes for every k (measured on B200: the FFMA passes reach only 64% / 48% /
    // 32% of the HBM roofline at kp = 8 / 16 / 32); k <= 8 rides in the kp = 16 layout. The
    // FFMA passes remain selectable (OOCNMF_FORCE_FFMA=1) as an independent cross-check.
    const char* force = std::getenv("OOCNMF_FORCE_FFMA");
    int kp = pad_k(k);
    c->use_tc = (kp > 64 || !(force && force[0] == '1')) && tc_for(kp);
    if (kp > 64 && !c->use_tc) fail(OOCNMF_ERR_DEVICE, "k > 64 needs the tensor-core passes");
    if (c->use_tc) kp = std::max(kp, 16);
    c->kp = kp;
    c->mp = round_up(int64_t(rows), kTile);
    c->np = round_up(int64_t(n), kTile);
    c->problem_set = true;
    c->factors_set = c->factors_valid = false;
    alloc_factors(c);
}

// Change k keeping the resident A (model selection sweeps k over one matrix).
void set_rank_impl(oocnmf_ctx* c, uint64_t k) {
    need_problem(c);
    if (k < 1) fail(OOCNMF_ERR_SHAPE, "k must be >= 1");
    const char* force = std::getenv("OOCNMF_FORCE_FFMA");
    int kp = pad_k(k);
    c->use_tc = (kp > 64 || !(force && force[0] == '1')) && tc_for(kp);
    if (kp > 64 && !c->use_tc) fail(OOCNMF_ERR_DEVICE, "k > 64 needs the tensor-core passes");
    if (c->use_tc) kp = std::max(kp, 16);
    c->k = k;
    c->kp = kp;
    c->factors_set = c->factors_valid = false;
    alloc_factors(c);
    if (c->kind == Kind::dense) plan_dense(c);
    if (c->kind == Kind::csr) {
        c->N1.alloc(size_t(c->mp) * c->kp * 4, "AHt");
        ck(cudaMemsetAsync(c->N1.p, 0, c->N1.bytes, c->stream), "memset");
        ck(cudaMemsetAsync(c->packed.p, 0, c->packed.bytes, c->stream), "memset");
    }
    if (c->kind == Kind::host) fail(OOCNMF_ERR_SHAPE, "set_rank: re-attach the out-of-core source after a rank change");
    ck(cudaStreamSynchronize(c->stream), "sync");
}

// A <- A0 o (1 - delta + 2 delta U(seed, 21, .)) from the pristine copy (kept on first use).
void perturb_impl(oocnmf_ctx* c, double delta, uint64_t seed) {
    need_problem(c);
    if (c->cnmf) fail(OOCNMF_ERR_SHAPE, "perturb: needs a row-window context (model selection holds the full A)");
    if (!(delta >= 0.0 && delta < 1.0)) fail(OOCNMF_ERR_SHAPE, "perturb: delta must lie in [0, 1)");
    cudaStream_t s = c->stream;
    if (c->kind == Kind::dense) {
        if (!c->pristine) {
            c->A0.alloc(c->A.bytes, "A0");
            ck(cudaMemcpyAsync(c->A0.p, c->A.p, c->A.bytes, cudaMemcpyDeviceToDevice, s), "copy A0");
            c->pristine = true;
        }
        count(c, launch_perturb_dense(c->A0.as<float>(), c->A.as<float>(), c->np, c->rows, c->n, c->row0, c->n, seed,
                                      delta, s),
              "perturb");
    } else if (c->kind == Kind::csr) {
        const size_t vb = size_t(std::max<int64_t>(c->nnz, 1)) * 4;
        if (!c->pristine) {
            c->v0.alloc(vb, "v0");
            c->vT0.alloc(vb, "vT0");
            ck(cudaMemcpyAsync(c->v0.p, c->v.p, vb, cudaMemcpyDeviceToDevice, s), "copy v0");
            ck(cudaMemcpyAsync(c->vT0.p, c->vT.p, vb, cudaMemcpyDeviceToDevice, s), "copy vT0");
            c->pristine = true;
        }
        count(c, launch_perturb_csr(c->v0.as<float>(), c->v.as<float>(), c->rp.as<int64_t>(), c->ci.as<int32_t>(),
                                    c->rows, c->row0, c->n, seed, delta, false, s),
              "perturb");
        count(c, launch_perturb_csr(c->vT0.as<float>(), c->vT.as<float>(), c->rpT.as<int64_t>(),
                                    c->ciT.as<int32_t>(), c->n, c->row0, c->n, seed, delta, true, s),
              "perturb T");
    } else {
        fail(OOCNMF_ERR_SHAPE, "perturb: needs a resident (dense or CSR) A");
    }
    ck(cudaStreamSynchronize(s), "sync");
    c->norm_valid = false;
}

void load_dense_common(oocnmf_ctx* c) {
    need_problem(c);
    reset_source(c);
    c->A.alloc(size_t(c->mp) * c->np * 4, "A");
    ck(cudaMemsetAsync(c->A.p, 0, c->A.bytes, c->stream), "memset A");
    c->kind = Kind::dense;
    plan_dense(c);
}

// ----------------------------------------------------------------- pageable copy-in / copy-out
// The reference API hands arrays over in pageable host memory (f64 values, u64 indices,
// reference layouts). The calls that take or return them stream through two pinned slots:
// host threads pack the caller's array into one slot while the other slot's DMA and the
// on-device layout work (narrowing, padding, transposition) run, so the host copy, the PCIe
// transfer and the conversion overlap and no layout loop runs on one host core.
//
// A transfer moves `count` elements of one or more parts; part p's element e is elem bytes
// at host + e * stride. A chunk of len elements occupies the slot as the parts back to back
// (part p at len * sum of the earlier parts' elem).
struct Part {
    const void* host;  // copy-in source / copy-out destination (cast away const for the latter)
    size_t elem, stride;
};

constexpr size_t kStageSlot = size_t(64) << 20;

// OOCNMF_STAGE_SLOT_KB: smaller slots (tests drive the multi-chunk pipeline at small sizes)
size_t stage_slot_target() {
    const char* e = std::getenv("OOCNMF_STAGE_SLOT_KB");
    const long long kb = e ? std::atoll(e) : 0;
    return kb > 0 ? size_t(kb) << 10 : kStageSlot;
}

// Page-locked staging buffers outlive their contexts: pinning 128 MB costs ~0.1-0.3 s, which
// a one-shot call (context create, upload, solve, download, destroy) would otherwise pay every
// time. A context takes a buffer of its size from this process-wide free list (or pins a new
// one) and returns it on destruction; buffers are never unpinned (UVA: usable by any device).
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<size_t, void*>> free;
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // intentionally leaked: process lifetime
    return *p;
}
void* pinned_take(size_t bytes) {
    {
        std::lock_guard<std::mutex> g(pinned_pool().mu);
        auto& f = pinned_pool().free;
        for (size_t i = 0; i < f.size(); ++i)
            if (f[i].first == bytes) {
                void* p = f[i].second;
                f.erase(f.begin() + i);
                return p;
            }
    }
    void* p = nullptr;
    ck(cudaMallocHost(&p, bytes), "cudaMallocHost (staging)");
    return p;
}
void pinned_give(void* p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> g(pinned_pool().mu);
    pinned_pool().free.emplace_back(bytes, p);
}

size_t stage_slot_bytes(oocnmf_ctx* c, size_t unit) {
    const size_t want = std::max(stage_slot_target(), unit);
    if (!c->stage_pin || c->stage_dev.bytes != 2 * want) {
        if (c->stage_pin) pinned_give(c->stage_pin, c->stage_dev.bytes), c->stage_pin = nullptr;
        c->stage_pin = pinned_take(2 * want);
        c->stage_dev.alloc(2 * want, "staging");
        for (auto& e : c->stage_ev)
            if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    return c->stage_dev.bytes / 2;
}

// OOCNMF_PROFILE_IO=1: per-phase wall times of the copy-in calls on stderr
bool io_profile() {
    static const bool on = [] {
        const char* e = std::getenv("OOCNMF_PROFILE_IO");
        return e && *e && *e != '0';
    }();
    return on;
}
double io_clock() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// host threads for packing the staging slots (OOCNMF_IO_THREADS overrides; default: all cores
// up to 16 — a pageable memcpy runs at ~4-5 GB/s per core, the link at ~55 GB/s)
int host_threads() {
    static const int n = [] {
        const char* e = std::getenv("OOCNMF_IO_THREADS");
        if (e && std::atoi(e) > 0) return std::atoi(e);
        return int(std::clamp<unsigned>(std::thread::hardware_concurrency(), 1u, 16u));
    }();
    return n;
}

// Pack (in = true: host parts -> slot) or unpack (slot -> host parts) elements [off, off + len).
void pack_chunk(const std::vector<Part>& parts, char* slot, int64_t off, int64_t len, bool in) {
    struct Job {
        char* slot;
        char* host;
        size_t elem, stride;
    };
    std::vector<Job> jobs;
    size_t at = 0;
    for (const Part& p : parts) {
        jobs.push_back({slot + at, const_cast<char*>(static_cast<const char*>(p.host)) + off * p.stride, p.elem,
                        p.stride});
        at += size_t(len) * p.elem;
    }
    const int nt = host_threads();
    auto work = [&](int t) {
        for (const Job& j : jobs) {
            if (j.stride == j.elem) {  // contiguous: split the bytes
                const size_t bytes = size_t(len) * j.elem, per = (bytes + nt - 1) / nt;
                const size_t b = std::min(bytes, t * per), e = std::min(bytes, b + per);
                if (in)
                    std::memcpy(j.slot + b, j.host + b, e - b);
                else
                    std::memcpy(j.host + b, j.slot + b, e - b);
            } else {  // strided: split the elements
                const int64_t per = (len + nt - 1) / nt, b = std::min(len, t * per), e = std::min(len, b + per);
                for (int64_t q = b; q < e; ++q) {
                    if (in)
                        std::memcpy(j.slot + q * j.elem, j.host + q * j.stride, j.elem);
                    else
                        std::memcpy(j.host + q * j.stride, j.slot + q * j.elem, j.elem);
                }
            }
        }
    };
    const size_t total = size_t(len) * (at / std::max<int64_t>(len, 1));
    if (nt == 1 || total < (size_t(1) << 20)) {
        for (int t = 0; t < nt; ++t) work(t);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& t : pool) t.join();
}

// Copy-in: consume(dev_slot, off, len) enqueues on c->stream the device work that reads the
// staged chunk (parts back to back in dev_slot).
// Small transfers skip the slots (their first use allocates 128 MB of pinned memory, ~50 ms):
// one device buffer, the driver's pageable copy per part (2-D when strided).
bool direct_transfer(oocnmf_ctx* c, size_t bytes) {
    const char* f = std::getenv("OOCNMF_STAGE_FORCE");  // tests: always take the slots
    if (f && *f && *f != '0') return false;
    return bytes <= (size_t(4) << 20) || (!c->stage_pin && bytes <= (size_t(64) << 20));
}

template <class Consume>
void copy_in(oocnmf_ctx* c, const std::vector<Part>& parts, int64_t count, Consume&& consume) {
    if (count <= 0) return;
    size_t unit = 0;
    for (const Part& p : parts) unit += p.elem;
    if (direct_transfer(c, size_t(count) * unit)) {
        DevBuf tmp;
        tmp.alloc(size_t(count) * unit, "copy-in");
        size_t at = 0;
        for (const Part& p : parts) {
            if (p.stride == p.elem)
                ck(cudaMemcpyAsync(tmp.as<char>() + at, p.host, size_t(count) * p.elem, cudaMemcpyHostToDevice,
                                   c->stream),
                   "H2D");
            else
                ck(cudaMemcpy2DAsync(tmp.as<char>() + at, p.elem, p.host, p.stride, p.elem, size_t(count),
                                     cudaMemcpyHostToDevice, c->stream),
                   "H2D");
            at += size_t(count) * p.elem;
        }
        consume(tmp.as<char>(), int64_t(0), count);
        ck(cudaStreamSynchronize(c->stream), "sync");
        return;
    }
    const size_t slot = stage_slot_bytes(c, unit);
    const int64_t chunk = std::max<int64_t>(1, int64_t(slot / unit));
    double t_wait = 0, t_pack = 0;
    const double t0 = io_clock();
    for (int64_t off = 0, i = 0; off < count; off += chunk, ++i) {
        const int si = int(i & 1);
        const int64_t len = std::min(chunk, count - off);
        char* hs = static_cast<char*>(c->stage_pin) + si * slot;
        char* ds = c->stage_dev.as<char>() + si * slot;
        const double ta = io_clock();
        if (i >= 2) ck(cudaEventSynchronize(c->stage_ev[si]), "sync");
        const double tb = io_clock();
        pack_chunk(parts, hs, off, len, true);
        t_wait += tb - ta, t_pack += io_clock() - tb;
        ck(cudaMemcpyAsync(ds, hs, size_t(len) * unit, cudaMemcpyHostToDevice, c->stream), "H2D");
        consume(ds, off, len);
        ck(cudaEventRecord(c->stage_ev[si], c->stream), "event");
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (io_profile())
        std::fprintf(stderr, "[oocnmf io] copy_in %.1f MB: %.1f ms (host pack %.1f ms, slot waits %.1f ms, %d threads)\n",
                     double(count) * unit / 1e6, (io_clock() - t0) * 1e3, t_pack * 1e3, t_wait * 1e3, host_threads());
}

// Copy-out: produce(dev_slot, off, len) enqueues on c->stream the device work that writes the
// chunk (parts back to back) into dev_slot.
template <class Produce>
void copy_out(oocnmf_ctx* c, const std::vector<Part>& parts, int64_t count, Produce&& produce) {
    if (count <= 0) return;
    size_t unit = 0;
    for (const Part& p : parts) unit += p.elem;
    if (direct_transfer(c, size_t(count) * unit)) {
        const double t0 = io_clock();
        DevBuf tmp;
        tmp.alloc(size_t(count) * unit, "copy-out");
        const double t1 = io_clock();
        produce(tmp.as<char>(), int64_t(0), count);
        size_t at = 0;
        for (const Part& p : parts) {
            if (p.stride == p.elem)
                ck(cudaMemcpyAsync(const_cast<void*>(p.host), tmp.as<char>() + at, size_t(count) * p.elem,
                                   cudaMemcpyDeviceToHost, c->stream),
                   "D2H");
            else
                ck(cudaMemcpy2DAsync(const_cast<void*>(p.host), p.stride, tmp.as<char>() + at, p.elem, p.elem,
                                     size_t(count), cudaMemcpyDeviceToHost, c->stream),
                   "D2H");
            at += size_t(count) * p.elem;
        }
        ck(cudaStreamSynchronize(c->stream), "sync");
        const double t2 = io_clock();
        tmp.release();
        if (io_profile())
            std::fprintf(stderr, "[oocnmf io] copy_out %.1f MB direct: alloc %.1f ms, produce+D2H %.1f ms, free %.1f ms\n",
                         double(count) * unit / 1e6, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (io_clock() - t2) * 1e3);
        return;
    }
    const size_t slot = stage_slot_bytes(c, unit);
    const int64_t chunk = std::max<int64_t>(1, int64_t(slot / unit));
    const int64_t nchunks = (count + chunk - 1) / chunk;
    auto issue = [&](int64_t i) {
        const int si = int(i & 1);
        const int64_t off = i * chunk, len = std::min(chunk, count - off);
        char* ds = c->stage_dev.as<char>() + si * slot;
        produce(ds, off, len);
        ck(cudaMemcpyAsync(static_cast<char*>(c->stage_pin) + si * slot, ds, size_t(len) * unit,
                           cudaMemcpyDeviceToHost, c->stream),
           "D2H");
        ck(cudaEventRecord(c->stage_ev[si], c->stream), "event");
    };
    issue(0);
    for (int64_t i = 0; i < nchunks; ++i) {
        if (i + 1 < nchunks) issue(i + 1);  // its slot was unpacked in the previous round
        const int si = int(i & 1);
        ck(cudaEventSynchronize(c->stage_ev[si]), "sync");
        const int64_t off = i * chunk, len = std::min(chunk, count - off);
        pack_chunk(parts, static_cast<char*>(c->stage_pin) + si * slot, off, len, false);
    }
}

// Device layout of the factors: W rows x kp (row i at W + i kp), Ht n x kp. The reference's:
// W m x k row-major, H k x n row-major (f64).
void import_w(oocnmf_ctx* c, const double* w) {
    ck(cudaMemsetAsync(c->W.p, 0, c->W.bytes, c->stream), "memset");
    const int64_t k = int64_t(c->k), kp = c->kp;
    copy_in(c, {Part{w, size_t(k) * 8, size_t(k) * 8}}, int64_t(c->rows), [&](char* ds, int64_t off, int64_t len) {
        ck(launch_strided_cast(CastKind::f64_f32, ds, k, 1, c->W.as<float>() + off * kp, kp, 1, len, k, c->stream),
           "import W");
    });
}
void import_h(oocnmf_ctx* c, const double* h) {
    ck(cudaMemsetAsync(c->Ht.p, 0, c->Ht.bytes, c->stream), "memset");
    const int64_t n = int64_t(c->n), kp = c->kp;
    // element = one row r of H (n values) -> column r of Ht
    copy_in(c, {Part{h, size_t(n) * 8, size_t(n) * 8}}, int64_t(c->k), [&](char* ds, int64_t off, int64_t len) {
        ck(launch_strided_cast(CastKind::f64_f32, ds, n, 1, c->Ht.as<float>() + off, 1, kp, len, n, c->stream),
           "import H");
    });
}
void export_w(oocnmf_ctx* c, const float* W, int64_t rows, double* w) {
    const int64_t k = int64_t(c->k), kp = c->kp;
    copy_out(c, {Part{w, size_t(k) * 8, size_t(k) * 8}}, rows, [&](char* ds, int64_t off, int64_t len) {
        ck(launch_strided_cast(CastKind::f32_f64, W + off * kp, kp, 1, ds, k, 1, len, k, c->stream), "export W");
    });
}
// H rows [0, k) of the local n columns into h (row stride ldh doubles)
void export_h(oocnmf_ctx* c, double* h, int64_t ldh) {
    const int64_t n = int64_t(c->n), kp = c->kp;
    copy_out(c, {Part{h, size_t(n) * 8, size_t(ldh) * 8}}, int64_t(c->k), [&](char* ds, int64_t off, int64_t len) {
        ck(launch_strided_cast(CastKind::f32_f64, c->Ht.as<float>() + off, 1, kp, ds, n, 1, len, n, c->stream),
           "export H");
    });
}

void csr_finish(oocnmf_ctx* c) {
    // CSR(A^T) once: A is iteration-invariant.
    c->rpT.alloc(size_t(c->n + 1) * 8, "rpT");
    c->ciT.alloc(size_t(std::max<int64_t>(c->nnz, 1)) * 4, "ciT");
    c->vT.alloc(size_t(std::max<int64_t>(c->nnz, 1)) * 4, "vT");
    ck(csr_transpose(c->rp.as<int64_t>(), c->ci.as<int32_t>(), c->v.as<float>(), c->rows, c->n, c->nnz,
                     c->rpT.as<int64_t>(), c->ciT.as<int32_t>(), c->vT.as<float>(), c->stream),
       "csr transpose");
    c->N1.alloc(size_t(c->mp) * c->kp * 4, "AHt");
    ck(cudaMemsetAsync(c->N1.p, 0, c->N1.bytes, c->stream), "memset");
    ck(cudaMemsetAsync(c->packed.p, 0, c->packed.bytes, c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->kind = Kind::csr;
}

}  // namespace

namespace ooc {
// Shared with the host-side translation units (selection.cpp): the thread-local message
// oocnmf_last_error() returns.
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace ooc

// =============================================================================== C-ABI
extern "C" {

const char* oocnmf_last_error(void) { return g_err.c_str(); }

int oocnmf_problem_dims(const oocnmf_ctx* c, uint64_t* m, uint64_t* n, uint64_t* k, uint64_t* row0, uint64_t* rows) {
    return guarded([&] {
        if (!c->problem_set) fail(OOCNMF_ERR_SHAPE, "oocnmf_set_problem has not been called");
        *m = c->m, *n = c->n, *k = c->k, *row0 = c->row0, *rows = c->rows;
    });
}
int oocnmf_abi_version(void) { return OOCNMF_ABI_VERSION; }

int oocnmf_device_count(int* count_out) {
    return guarded([&] {
        int nd = 0;
        const cudaError_t e = cudaGetDeviceCount(&nd);
        if (e != cudaSuccess) {
            cudaGetLastError();
            nd = 0;
        }
        *count_out = nd;
    });
}

int oocnmf_counter_uniform(uint64_t seed, uint64_t stream, uint64_t index0, uint64_t cnt, double* out) {
    return guarded([&] {
        const uint64_t key = rng_key(seed, stream);
        for (uint64_t i = 0; i < cnt; ++i) out[i] = rng_u01(key, index0 + i);
    });
}

int oocnmf_init_factors_host(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, double* w, double* h) {
    return guarded([&] {
        if (m < 1 || n < 1 || k < 1) fail(OOCNMF_ERR_SHAPE, "init_factors: dimensions must be >= 1");
        const uint64_t kw = rng_key(seed, kStreamW), kh = rng_key(seed, kStreamH);
        for (uint64_t i = 0; i < m * k; ++i) w[i] = rng_u01(kw, i);
        for (uint64_t i = 0; i < k * n; ++i) h[i] = rng_u01(kh, i);
    });
}

int oocnmf_split_even(uint64_t extent, uint64_t parts, uint64_t* begins) {
    return guarded([&] {
        if (parts < 1) fail(OOCNMF_ERR_SHAPE, "split_even: parts must be >= 1");
        const uint64_t base = extent / parts, rem = extent % parts;
        uint64_t pos = 0;
        for (uint64_t p = 0; p < parts; ++p) {
            begins[p] = pos;
            pos += base + (p < rem ? 1 : 0);
        }
        begins[parts] = pos;
    });
}

// Establish the group's NVLink / network connections during communicator creation, while every
// rank is alive (NCCL otherwise connects lazily inside the first collective, where a peer that
// died meanwhile blocks the host in the NCCL call for its own ~60 s socket timeout, out of reach
// of the progress watchdog). Respects a caller's own NCCL_RUNTIME_CONNECT.
static void eager_connect() { setenv("NCCL_RUNTIME_CONNECT", "0", 0); }

static void ctx_init_common(oocnmf_ctx* c, int device) {
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
        cudaGetLastError();
        fail(OOCNMF_ERR_DEVICE, "no CUDA device available (the B200 backend has no CPU fallback)");
    }
    if (device < 0 || device >= nd) fail(OOCNMF_ERR_DEVICE, "device index out of range");
    c->device = device;
    set_dev(c);
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) fail(OOCNMF_ERR_DEVICE, "requires an sm_100 (Blackwell B200) device");
    c->num_sms = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
    int prio_lo = 0, prio_hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "stream priorities");
    ck(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio_hi), "stream");
    for (auto& e : c->ev_rs) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (int i = 0; i < 2; ++i) {
        ck(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming), "event");
    }
    ck(cudaMallocHost(&c->hpin, 64), "cudaMallocHost");
}

int oocnmf_ctx_create(int device, oocnmf_ctx** out) {
    return guarded([&] {
        *out = nullptr;
        auto* c = new oocnmf_ctx();
        try {
            ctx_init_common(c, device);
        } catch (...) {
            oocnmf_ctx_destroy(c);
            throw;
        }
        *out = c;
    });
}

int oocnmf_comm_unique_id(unsigned char id[128]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId uid;
        nck(ncclGetUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(id, &uid, 128);
    });
}

int oocnmf_ctx_create_comm(int device, int rank, int nranks, const unsigned char id[128], oocnmf_ctx** out) {
    return guarded([&] {
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(OOCNMF_ERR_SHAPE, "bad rank/nranks");
        auto* c = new oocnmf_ctx();
        try {
            ctx_init_common(c, device);
            c->rank = rank;
            c->nranks = nranks;
            if (nranks > 1) {
                ncclUniqueId uid;
                std::memcpy(&uid, id, 128);
                eager_connect();
                nck(ncclCommInitRank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
            }
        } catch (...) {
            oocnmf_ctx_destroy(c);
            throw;
        }
        *out = c;
    });
}

int oocnmf_ctx_destroy(oocnmf_ctx* c) {
    if (!c) return OOCNMF_OK;
    return guarded([&] {
        cudaSetDevice(c->device);
        if (c->stream) cudaStreamSynchronize(c->stream);
        if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
        if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
        // the graphs hold NCCL work on c->comm: release them before the communicator
        for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
        c->graphs.clear();
        if (c->nvls_ready && !c->poisoned) nvls_release(c);  // collective (all ranks destroy together)
        if (c->comm) ncclCommDestroy(c->comm);
        for (auto e : c->evs) cudaEventDestroy(e);
        for (auto& m : c->marks) c->ev_pool.push_back(m.beg), c->ev_pool.push_back(m.end);
        if (c->mark_beg) c->ev_pool.push_back(c->mark_beg);
        for (auto e : c->ev_pool) cudaEventDestroy(e);
        for (int i = 0; i < 2; ++i) {
            if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
            if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
        }
        if (c->hpin) cudaFreeHost(c->hpin);
        if (c->stage_pin) pinned_give(c->stage_pin, c->stage_dev.bytes);
        for (auto e : c->stage_ev)
            if (e) cudaEventDestroy(e);
        if (c->stream) cudaStreamDestroy(c->stream);
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
        if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
        for (auto e : c->ev_rs)
            if (e) cudaEventDestroy(e);
        for (auto e : c->ev_bc)
            if (e) cudaEventDestroy(e);
        if (c->ev_hdone) cudaEventDestroy(c->ev_hdone);
        delete c;
    });
}

int oocnmf_ctx_rank(const oocnmf_ctx* c, int* rank, int* nranks) {
    return guarded([&] {
        *rank = c->rank;
        *nranks = c->nranks;
    });
}

int oocnmf_ctx_paths(const oocnmf_ctx* c, int* flags) {
    return guarded([&] {
        int f = 0;
        if (c->kind == Kind::dense && c->use_fused) f |= 1;
        if ((c->kind == Kind::dense || c->kind == Kind::host) && c->use_tc && !c->use_fused) f |= 2;
        if (c->nvls_ready) f |= 4;
        if (c->shard_h()) f |= 8;
        if (c->kind == Kind::csr) f |= 16;
        if (c->kind == Kind::host) f |= 32;
        *flags = f;
    });
}

int oocnmf_set_problem(oocnmf_ctx* c, uint64_t m, uint64_t n, uint64_t k, uint64_t row0, uint64_t rows) {
    return guarded([&] {
        set_dev(c);
        set_problem_impl(c, m, n, k, row0, rows);
    });
}

int oocnmf_load_dense_f64(oocnmf_ctx* c, const double* a, uint64_t lda) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (lda < c->n) fail(OOCNMF_ERR_SHAPE, "lda < n");
        load_dense_common(c);
        // rows through the staging slots, narrowed and padded in HBM
        copy_in(c, {Part{a, size_t(c->n) * 8, size_t(lda) * 8}}, int64_t(c->rows),
                [&](char* ds, int64_t off, int64_t len) {
                    ck(launch_cast_pad_f64(reinterpret_cast<const double*>(ds), c->n, len, c->n,
                                           c->A.as<float>() + off * c->np, c->np, c->stream),
                       "cast");
                });
    });
}

int oocnmf_load_dense_f32(oocnmf_ctx* c, const float* a, uint64_t lda) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (lda < c->n) fail(OOCNMF_ERR_SHAPE, "lda < n");
        load_dense_common(c);
        cudaPointerAttributes at{};
        const bool pinned = cudaPointerGetAttributes(&at, a) == cudaSuccess && at.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pinned) {  // page-locked (oocnmf_host_register / cudaMallocHost): one DMA
            ck(cudaMemcpy2DAsync(c->A.p, c->np * 4, a, lda * 4, c->n * 4, c->rows, cudaMemcpyHostToDevice,
                                 c->stream),
               "H2D A");
            ck(cudaStreamSynchronize(c->stream), "sync");
            return;
        }
        copy_in(c, {Part{a, size_t(c->n) * 4, size_t(lda) * 4}}, int64_t(c->rows),
                [&](char* ds, int64_t off, int64_t len) {
                    ck(cudaMemcpy2DAsync(c->A.as<float>() + off * c->np, c->np * 4, ds, c->n * 4, c->n * 4, len,
                                         cudaMemcpyDeviceToDevice, c->stream),
                       "copy A");
                });
    });
}

int oocnmf_load_dense_device_f32(oocnmf_ctx* c, const float* d_a, uint64_t lda) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (lda < c->n) fail(OOCNMF_ERR_SHAPE, "lda < n");
        load_dense_common(c);
        ck(cudaMemcpy2DAsync(c->A.p, c->np * 4, d_a, lda * 4, c->n * 4, c->rows, cudaMemcpyDeviceToDevice,
                             c->stream),
           "D2D A");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int oocnmf_generate_dense_uniform(oocnmf_ctx* c, uint64_t seed, uint64_t stream) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (c->cnmf) fail(OOCNMF_ERR_SHAPE, "generators produce row windows; load a column slab instead");
        load_dense_common(c);
        ck(launch_gen_dense_uniform(c->A.as<float>(), c->np, c->rows, c->n, c->row0, c->n, seed, stream, c->stream),
           "generate");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int oocnmf_load_csr_f64(oocnmf_ctx* c, const uint64_t* row_ptr, const uint64_t* col_idx, const double* vals) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (row_ptr[0] != 0) fail(OOCNMF_ERR_SHAPE, "CsrMatrix: row_ptr[0] must be 0");
        const double t_start = io_clock();
        const int64_t nnz = int64_t(row_ptr[c->rows]);
        if (nnz < 0 || uint64_t(nnz) > c->rows * c->n)
            fail(OOCNMF_ERR_SHAPE, "CsrMatrix: row_ptr must be nondecreasing");
        reset_source(c);
        c->nnz = nnz;
        c->rp.alloc(size_t(c->rows + 1) * 8, "rp");
        c->ci.alloc(size_t(std::max<int64_t>(nnz, 1)) * 4, "ci");
        c->v.alloc(size_t(std::max<int64_t>(nnz, 1)) * 4, "v");
        DevBuf bad;
        bad.alloc(4, "flags");
        ck(cudaMemsetAsync(bad.p, 0, 4, c->stream), "memset");
        // row_ptr: u64 -> i64 is the same bits
        copy_in(c, {Part{row_ptr, 8, 8}}, int64_t(c->rows + 1), [&](char* ds, int64_t off, int64_t len) {
            ck(cudaMemcpyAsync(c->rp.as<int64_t>() + off, ds, size_t(len) * 8, cudaMemcpyDeviceToDevice, c->stream),
               "copy rp");
        });
        // entries: narrowed to (i32, f32) with the column-range check on device
        copy_in(c, {Part{col_idx, 8, 8}, Part{vals, 8, 8}}, nnz, [&](char* ds, int64_t off, int64_t len) {
            ck(launch_csr_ingest(reinterpret_cast<const uint64_t*>(ds), reinterpret_cast<const double*>(ds + len * 8),
                                 len, c->n, c->ci.as<int32_t>() + off, c->v.as<float>() + off, bad.as<unsigned>(),
                                 c->stream),
               "csr ingest");
        });
        const double t_entries = io_clock();
        ck(launch_csr_check_rows(c->rp.as<int64_t>(), c->ci.as<int32_t>(), c->rows, nnz, bad.as<unsigned>(),
                                 c->stream),
           "csr check");
        unsigned flags = 0;
        ck(cudaMemcpyAsync(&flags, bad.p, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        // the reference constructor's messages, in its order of checks
        const char* msg = flags & kCsrBadRowPtr   ? "CsrMatrix: row_ptr must be nondecreasing"
                          : flags & kCsrBadColumn ? "CsrMatrix: column index out of range"
                          : flags & kCsrBadOrder  ? "CsrMatrix: column indices must strictly increase within a row"
                                                  : nullptr;
        if (msg) {
            reset_source(c);
            fail(OOCNMF_ERR_SHAPE, msg);
        }
        const double t_check = io_clock();
        csr_finish(c);
        if (io_profile())
            std::fprintf(stderr, "[oocnmf io] load_csr: %.1f ms upload+ingest, %.1f ms check, %.1f ms transpose\n",
                         (t_entries - t_start) * 1e3, (t_check - t_entries) * 1e3, (io_clock() - t_check) * 1e3);
    });
}

int oocnmf_generate_csr_uniform(oocnmf_ctx* c, double density, uint64_t seed) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (!(density >= 0.0) || density > 1.0) fail(OOCNMF_ERR_SHAPE, "density must lie in [0, 1]");
        if (c->cnmf) fail(OOCNMF_ERR_SHAPE, "generators produce row windows; load a column slab instead");
        reset_source(c);
        // U < density  <=>  bits53 < ceil(density * 2^53)  (exact: power-of-two scaling)
        const uint64_t thresh = uint64_t(std::ceil(density * 0x1.0p53));
        c->rp.alloc(size_t(c->rows + 1) * 8, "rp");
        DevBuf counts;
        counts.alloc(size_t(c->rows + 1) * 8, "counts");
        ck(cudaMemsetAsync(counts.p, 0, counts.bytes, c->stream), "memset");
        ck(launch_gen_csr_count(c->rows, c->row0, c->n, thresh, seed, counts.as<int64_t>(), c->stream), "gen count");
        ck(exclusive_scan_i64(counts.as<int64_t>(), c->rp.as<int64_t>(), c->rows + 1, c->stream), "scan");
        int64_t nnz = 0;
        ck(cudaMemcpyAsync(&nnz, c->rp.as<int64_t>() + c->rows, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->nnz = nnz;
        c->ci.alloc(size_t(std::max<int64_t>(nnz, 1)) * 4, "ci");
        c->v.alloc(size_t(std::max<int64_t>(nnz, 1)) * 4, "v");
        ck(launch_gen_csr_fill(c->rows, c->row0, c->n, thresh, seed, c->rp.as<int64_t>(), c->ci.as<int32_t>(),
                               c->v.as<float>(), c->stream),
           "gen fill");
        csr_finish(c);
    });
}

int oocnmf_attach_host_dense_f32(oocnmf_ctx* c, const float* a, uint64_t lda, uint64_t batch_rows) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (c->cnmf) fail(OOCNMF_ERR_SHAPE, "out-of-core streaming is row-partitioned (RNMF) only");
        if (lda < c->n) fail(OOCNMF_ERR_SHAPE, "lda < n");
        reset_source(c);
        int64_t br = int64_t(batch_rows);
        if (br == 0) br = std::max<int64_t>(kTile, ((int64_t(512) << 20) / (c->np * 4)) / kTile * kTile);
        br = round_up(br, kTile);
        br = std::min<int64_t>(br, c->mp);
        c->batch_rows = br;
        c->hA = a;
        c->hlda = lda;
        for (int i = 0; i < 2; ++i) {
            c->stage[i].alloc(size_t(br) * c->np * 4, "stage");
            ck(cudaMemsetAsync(c->stage[i].p, 0, c->stage[i].bytes, c->stream), "memset stage");
            ck(cudaEventRecord(c->ev_free[i], c->stream), "event");
        }
        const int64_t nb = (int64_t(c->rows) + br - 1) / br;
        const int64_t last = round_up(int64_t(c->rows) - (nb - 1) * br, kTile);
        const int step = c->use_tc ? kTcStep : kFfmaStep;
        plan_aht(c->sk1b[0], br, c->np, c->num_sms, step);
        plan_aht(c->sk1b[1], last, c->np, c->num_sms, step);
        plan_wta(c->sk2b[0], br, c->np, c->num_sms, step);
        plan_wta(c->sk2b[1], last, c->np, c->num_sms, step);
        const int64_t s1 = std::max(c->sk1b[0].G * c->sk1b[0].smax, c->sk1b[1].G * c->sk1b[1].smax);
        const int64_t s2 = std::max(c->sk2b[0].G * c->sk2b[0].smax, c->sk2b[1].G * c->sk2b[1].smax);
        c->slots1.alloc(size_t(s1) * kTile * c->kp * 4, "slots1");
        c->slots2.alloc(size_t(s2) * kTile * c->kp * 4, "slots2");
        if (c->kp > 64) c->N1.alloc(size_t(br) * c->kp * 4, "AHt (batch)");  // wide: plain numerators
        c->gram_w.alloc(size_t(nb) * factor_grid(br / kTile) * c->kp * c->kp * 8, "gram_w");
        ck(cudaMemsetAsync(c->gram_w.p, 0, c->gram_w.bytes, c->stream), "memset");
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->kind = Kind::host;
    });
}

int oocnmf_host_register(void* p, uint64_t bytes) {
    return guarded([&] { ck(cudaHostRegister(p, bytes, cudaHostRegisterDefault), "cudaHostRegister"); });
}
int oocnmf_host_unregister(void* p) {
    return guarded([&] { ck(cudaHostUnregister(p), "cudaHostUnregister"); });
}

int oocnmf_download_dense_f32(oocnmf_ctx* c, float* a) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (c->kind != Kind::dense) fail(OOCNMF_ERR_SHAPE, "no dense A resident in HBM");
        ck(cudaMemcpy2DAsync(a, c->n * 4, c->A.p, c->np * 4, c->n * 4, c->rows, cudaMemcpyDeviceToHost, c->stream),
           "D2H A");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int oocnmf_csr_nnz(oocnmf_ctx* c, uint64_t* nnz) {
    return guarded([&] {
        if (c->kind != Kind::csr) fail(OOCNMF_ERR_SHAPE, "no CSR A resident in HBM");
        *nnz = uint64_t(c->nnz);
    });
}

int oocnmf_download_csr(oocnmf_ctx* c, uint64_t* row_ptr, uint64_t* col_idx, double* vals) {
    return guarded([&] {
        set_dev(c);
        if (c->kind != Kind::csr) fail(OOCNMF_ERR_SHAPE, "no CSR A resident in HBM");
        copy_out(c, {Part{row_ptr, 8, 8}}, int64_t(c->rows + 1), [&](char* ds, int64_t off, int64_t len) {
            ck(cudaMemcpyAsync(ds, c->rp.as<int64_t>() + off, size_t(len) * 8, cudaMemcpyDeviceToDevice, c->stream),
               "copy rp");
        });
        copy_out(c, {Part{col_idx, 8, 8}, Part{vals, 8, 8}}, c->nnz, [&](char* ds, int64_t off, int64_t len) {
            ck(launch_strided_cast(CastKind::i32_u64, c->ci.as<int32_t>() + off, 1, 1, ds, 1, 1, len, 1, c->stream),
               "widen ci");
            ck(launch_strided_cast(CastKind::f32_f64, c->v.as<float>() + off, 1, 1, ds + len * 8, 1, 1, len, 1,
                                   c->stream),
               "widen v");
        });
    });
}

int oocnmf_set_factors_f64(oocnmf_ctx* c, const double* w, const double* h) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        import_w(c, w);
        import_h(c, h);
        c->factors_set = c->factors_valid = true;
    });
}

int oocnmf_get_factors_f64(oocnmf_ctx* c, double* w, double* h) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (!c->factors_valid) fail(OOCNMF_ERR_SHAPE, "factors are not initialised");
        if (w) export_w(c, c->W.as<float>(), int64_t(c->rows), w);
        if (h) export_h(c, h, int64_t(c->n));
    });
}

int oocnmf_gather_w_f64(oocnmf_ctx* c, double* w_full) {
    if (c && c->cnmf) return oocnmf_get_factors_f64(c, w_full, nullptr);  // W is replicated under CNMF
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        const int N = c->nranks, kp = c->kp;
        std::vector<uint64_t> beg(N + 1);
        {
            const uint64_t base = c->m / N, rem = c->m % N;
            uint64_t pos = 0;
            for (int p = 0; p < N; ++p) beg[p] = pos, pos += base + (uint64_t(p) < rem ? 1 : 0);
            beg[N] = pos;
        }
        if (beg[c->rank] != c->row0 || beg[c->rank + 1] != c->row0 + c->rows)
            fail(OOCNMF_ERR_SHAPE, "gather_w requires split_even row slabs");
        const int64_t maxr = int64_t(beg[1] - beg[0]);
        // A rank's W holds round_up(rows, 128) rows, which can be fewer than maxr (a rank with
        // maxr - 1 rows, a multiple of 128): the send side is this rank's slot of `all`, filled
        // with its rows and zero-padded to maxr, so NCCL never reads past the W allocation.
        DevBuf all;
        all.alloc(size_t(N) * maxr * kp * 4, "gather");
        float* mine = all.as<float>() + size_t(c->rank) * maxr * kp;
        const size_t own = size_t(c->rows) * kp * 4;
        ck(cudaMemcpyAsync(mine, c->W.p, own, cudaMemcpyDeviceToDevice, c->stream), "copy W");
        if (size_t(maxr) * kp * 4 > own)
            ck(cudaMemsetAsync(reinterpret_cast<char*>(mine) + own, 0, size_t(maxr) * kp * 4 - own, c->stream),
               "memset W tail");
        if (N > 1) {
            need_comm(c);
            coll_begin(c, c->stream);
            ncc(c, ncclAllGather(mine, all.p, size_t(maxr) * kp, ncclFloat, c->comm, c->stream), "allgather W");
            coll_end(c, c->stream, kTagGather, size_t(N) * maxr * kp * 4);  // nmf_distributed.cpp:280
            wait_for(c, c->stream, nullptr, "W all-gather");
        }
        for (int p = 0; p < N; ++p)
            export_w(c, all.as<float>() + size_t(p) * maxr * kp, int64_t(beg[p + 1] - beg[p]), w_full + beg[p] * c->k);
    });
}

int oocnmf_solve(oocnmf_ctx* c, const oocnmf_config* cfg, uint64_t* trace_iter, double* trace_err,
                 uint64_t trace_cap, oocnmf_info* info) {
    return guarded([&] {
        set_dev(c);
        solve_impl(c, cfg, trace_iter, trace_err, trace_cap, info);
    });
}

int oocnmf_sq_norm(oocnmf_ctx* c, double* out) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (c->kind == Kind::none) fail(OOCNMF_ERR_SHAPE, "no A loaded");
        if (!c->norm_valid) compute_norm(c);
        *out = c->norm_a2;
    });
}

int oocnmf_products_f64(oocnmf_ctx* c, double* aht, double* wta, double* hht, double* wtw) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (c->kind != Kind::dense && c->kind != Kind::csr) fail(OOCNMF_ERR_SHAPE, "products need in-core A");
        if (!c->factors_valid) fail(OOCNMF_ERR_SHAPE, "factors are not initialised");
        const int kp = c->kp;
        cudaStream_t s = c->stream;
        DevBuf t1;
        t1.alloc(size_t(c->mp) * kp * 4, "aht");
        if (c->kind == Kind::dense) {
            if (c->use_tc) {
                ck(launch_split_cat(c->Ht.as<float>(), c->Ht_cat.as<float>(), c->np, kp, s), "split");
                ck(launch_split_cat(c->W.as<float>(), c->W_cat.as<float>(), c->mp, kp, s), "split");
            }
            ck(pass1(c, c->A.as<float>(), c->mp, c->slots1.as<float>(), c->sk1, s, t1.as<float>()), "aht");
            if (!wide(c))
                ck(launch_streamk_reduce(kp, c->slots1.as<float>(), c->sk1, t1.as<float>(), false, s), "reduce");
            if (wide(c)) {
                ck(pass2(c, c->A.as<float>(), c->mp, c->W.as<float>(), wlo(c), c->slots2.as<float>(), c->sk2, s,
                         c->wta()),
                   "wta");
            } else {
                ck(pass2(c, c->A.as<float>(), c->mp, c->W.as<float>(), wlo(c), c->slots2.as<float>(), c->sk2, s),
                   "wta");
                ck(launch_streamk_reduce(kp, c->slots2.as<float>(), c->sk2, c->wta(), false, s), "reduce");
            }
        } else {
            ensure_chunks(c);
            spmm(c, false, c->Ht.as<float>(), t1.as<float>(), s);
            spmm(c, true, c->W.as<float>(), c->wta(), s);
        }
        gram_h(c);
        ck(launch_factor_update(kp, c->W.as<float>(), c->mp, nullptr, nullptr, nullptr, nullptr, 0.f, false,
                                c->gram_w.as<double>(), nullptr, c->flag.as<int>(), nullptr, s),
           "gram W");
        ck(launch_reduce_slots(c->gram_w.as<double>(), factor_grid(c->mp / kTile), int64_t(kp) * kp, c->wtw(), c->WtW64.as<double>(), s),
           "reduce");
        std::vector<float> a1(size_t(c->mp) * kp), a2(size_t(c->np) * kp), g1(size_t(kp) * kp), g2(size_t(kp) * kp);
        ck(cudaMemcpyAsync(a1.data(), t1.p, a1.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(a2.data(), c->wta(), a2.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(g1.data(), c->HHt.p, g1.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(g2.data(), c->wtw(), g2.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        const uint64_t k = c->k;
        for (uint64_t i = 0; i < c->rows; ++i)
            for (uint64_t j = 0; j < k; ++j) aht[i * k + j] = a1[i * kp + j];
        for (uint64_t r = 0; r < k; ++r)
            for (uint64_t j = 0; j < c->n; ++j) wta[r * c->n + j] = a2[j * kp + r];
        for (uint64_t r = 0; r < k; ++r)
            for (uint64_t j = 0; j < k; ++j) {
                hht[r * k + j] = g1[r * kp + j];
                wtw[r * k + j] = g2[r * kp + j];
            }
    });
}

int oocnmf_set_problem_cols(oocnmf_ctx* c, uint64_t m, uint64_t n, uint64_t k, uint64_t col0, uint64_t cols) {
    return guarded([&] {
        set_dev(c);
        if (cols < 1 || col0 + cols > n) fail(OOCNMF_ERR_SHAPE, "column slab out of bounds");
        set_problem_impl(c, m, cols, k, 0, m);
        c->cnmf = true, c->col0 = col0, c->n_global = n;
    });
}

int oocnmf_gather_h_f64(oocnmf_ctx* c, double* h_full) {
    return guarded([&] {
        set_dev(c);
        need_problem(c);
        if (!c->factors_valid) fail(OOCNMF_ERR_SHAPE, "factors are not initialised");
        // zero-padded sum over the ranks' column slabs (the reference's gather,
        // src/nmf_distributed.cpp:267-273), assembled in HBM
        const int64_t ng = int64_t(c->n_global);
        DevBuf d;
        d.alloc(c->k * c->n_global * 8, "gather H");
        ck(cudaMemsetAsync(d.p, 0, d.bytes, c->stream), "memset");
        ck(launch_strided_cast(CastKind::f32_f64, c->Ht.as<float>(), 1, c->kp, d.as<double>() + c->col0, ng, 1,
                               int64_t(c->k), int64_t(c->n), c->stream),
           "export H");
        if (c->collective()) {
            need_comm(c);
            coll_begin(c, c->stream);
            ncc(c, ncclAllReduce(d.p, d.p, c->k * c->n_global, ncclDouble, ncclSum, c->comm, c->stream), "allreduce H");
            coll_end(c, c->stream, kTagGather, c->k * c->n_global * 8);  // nmf_distributed.cpp:272
            wait_for(c, c->stream, nullptr, "H gather");
        }
        copy_out(c, {Part{h_full, size_t(ng) * 8, size_t(ng) * 8}}, int64_t(c->k),
                 [&](char* ds, int64_t off, int64_t len) {
                     ck(cudaMemcpyAsync(ds, d.as<double>() + off * ng, size_t(len) * ng * 8,
                                        cudaMemcpyDeviceToDevice, c->stream),
                        "copy H");
                 });
    });
}

int oocnmf_memory_estimate(uint64_t m, uint64_t n, uint64_t k, int n_workers, int strategy, double density,
                           uint64_t budget_bytes, int num_sms, oocnmf_memory_report* out) {
    return guarded([&] {
        if (m < 1 || n < 1 || k < 1) fail(OOCNMF_ERR_SHAPE, "memory_estimate: dimensions must be >= 1");
        if (n_workers < 1) fail(OOCNMF_ERR_SHAPE, "memory_estimate: need at least one worker");
        if (!(density > 0.0) || density > 1.0) fail(OOCNMF_ERR_SHAPE, "memory_estimate: density must be in (0, 1]");
        if (budget_bytes == 0) fail(OOCNMF_ERR_SHAPE, "memory_estimate: budget must be > 0");
        const bool cnmf = strategy == 1;
        const int sms = num_sms > 0 ? num_sms : 148;
        const uint64_t N = uint64_t(n_workers);
        const int64_t rows = int64_t(cnmf ? m : (m + N - 1) / N), cols = int64_t(cnmf ? (n + N - 1) / N : n);
        int kp = pad_k(k);
        kp = std::max(kp, 16);  // the tensor-core layout
        const int64_t mp = round_up(rows, kTile), np = round_up(cols, kTile);
        const bool dense = density >= 1.0;
        // resident A
        uint64_t a_bytes;
        if (dense) {
            a_bytes = uint64_t(mp) * np * 4;
        } else {
            const double nnz = std::ceil(density * double(rows) * double(cols));
            a_bytes = uint64_t(nnz) * 8 * 2 + uint64_t(rows + 1) * 8 + uint64_t(cols + 1) * 8;
        }
        const uint64_t factors = uint64_t(mp + np) * kp * 4 * 3;  // W, Ht and [F | F_lo] copies
        auto inter_for = [&](int64_t mrows) {
            StreamK s1, s2;
            plan_aht(s1, mrows, np, sms, kTcStep);
            plan_wta(s2, mrows, np, sms, kTcStep);
            uint64_t b = uint64_t(np * kp + kp * kp) * 4;                                   // packed
            b += uint64_t(s1.G * s1.smax + s2.G * s2.smax) * kTile * kp * 4;              // slots
            b += uint64_t(factor_grid(mp / kTile) + factor_grid(np / kTile)) * kp * kp * 8; // Gram slots
            if (!dense || cnmf) b += uint64_t(mp) * kp * 4;                               // A·H^T
            return b + (1u << 20);                                                         // scalars, flags
        };
        oocnmf_memory_report r{};
        r.a_slab_bytes = a_bytes;
        r.factor_bytes = factors;
        r.intermediate_bytes = inter_for(mp);
        r.peak_bytes = a_bytes + factors + r.intermediate_bytes;
        if (r.peak_bytes <= budget_bytes) {
            r.min_n_b = 1, r.feasible = 1, r.in_core = 1;
        } else if (dense && !cnmf) {
            // out-of-core row batches: two staging buffers of br rows
            const uint64_t fixed = factors + r.intermediate_bytes;
            if (fixed > budget_bytes)
                fail(OOCNMF_ERR_SHAPE, "memory_estimate: factor arrays alone (" + std::to_string(fixed) +
                                           " B) exceed the budget of " + std::to_string(budget_bytes) + " B");
            const int64_t br = int64_t((budget_bytes - fixed) / (2 * uint64_t(np) * 4)) / kTile * kTile;
            if (br >= kTile) {
                r.min_n_b = uint64_t((rows + br - 1) / br);
                r.store_peak_bytes = 2 * uint64_t(br) * np * 4;
                r.peak_bytes = r.store_peak_bytes + fixed;
                r.feasible = 1;
            }
        }
        *out = r;
    });
}

int oocnmf_set_rank(oocnmf_ctx* c, uint64_t k) {
    return guarded([&] {
        set_dev(c);
        set_rank_impl(c, k);
    });
}

int oocnmf_perturb(oocnmf_ctx* c, double delta, uint64_t seed) {
    return guarded([&] {
        set_dev(c);
        perturb_impl(c, delta, seed);
    });
}

int oocnmf_set_local(oocnmf_ctx* c, int local) {
    return guarded([&] {
        c->local = local != 0;
        c->norm_valid = false;
    });
}

int oocnmf_allreduce_sum_f64(oocnmf_ctx* c, double* buf, uint64_t count) {
    return oocnmf_allreduce_f64(c, buf, count, kTagGeneric);
}

int oocnmf_allreduce_f64(oocnmf_ctx* c, double* buf, uint64_t count, int tag) {
    return guarded([&] {
        set_dev(c);
        if (tag < 0 || tag > 5) fail(OOCNMF_ERR_SHAPE, "all_reduce_sum: unknown PhaseTag");
        if (c->nranks <= 1 || count == 0) {
            c->tag_calls[tag] += 1;  // loopback: counted like the reference's single-rank group
            c->tag_bytes[tag] += count * 8;
            return;
        }
        DevBuf d;
        d.alloc(count * 8, "allreduce scratch");
        need_comm(c);
        ck(cudaMemcpyAsync(d.p, buf, count * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
        coll_begin(c, c->stream);
        ncc(c, ncclAllReduce(d.p, d.p, count, ncclDouble, ncclSum, c->comm, c->stream), "allreduce");
        coll_end(c, c->stream, tag, count * 8);
        wait_for(c, c->stream, nullptr, "all_reduce_sum");  // (before the pageable D2H, which would block)
        ck(cudaMemcpy(buf, d.p, count * 8, cudaMemcpyDeviceToHost), "D2H");
    });
}

int oocnmf_barrier(oocnmf_ctx* c) {
    return guarded([&] {
        set_dev(c);
        if (c->nranks <= 1) {
            c->tag_calls[kTagBarrier] += 1;
            return;
        }
        need_comm(c);
        DevBuf d;
        d.alloc(4, "barrier");
        ck(cudaMemsetAsync(d.p, 0, 4, c->stream), "memset");
        coll_begin(c, c->stream);
        ncc(c, ncclAllReduce(d.p, d.p, 1, ncclFloat, ncclSum, c->comm, c->stream), "barrier");
        coll_end(c, c->stream, kTagBarrier, 0);
        wait_for(c, c->stream, nullptr, "barrier");
    });
}

int oocnmf_comm_stats(oocnmf_ctx* c, uint64_t bytes[6], uint64_t calls[6], double seconds[6]) {
    return guarded([&] {
        set_dev(c);
        reap_marks(c);
        for (int t = 0; t < 6; ++t) {
            if (bytes) bytes[t] = c->tag_bytes[t];
            if (calls) calls[t] = c->tag_calls[t];
            if (seconds) seconds[t] = c->tag_secs[t];
        }
    });
}

int oocnmf_comm_reset_stats(oocnmf_ctx* c) {
    return guarded([&] {
        set_dev(c);
        reap_marks(c);
        for (int t = 0; t < 6; ++t) c->tag_bytes[t] = c->tag_calls[t] = 0, c->tag_secs[t] = 0.0;
    });
}

int oocnmf_set_comm_timeout(oocnmf_ctx* c, double seconds) {
    return guarded([&] {
        if (!(seconds > 0)) fail(OOCNMF_ERR_SHAPE, "comm timeout must be > 0");
        c->comm_timeout = seconds;
    });
}

int oocnmf_ctx_create_group(int n, const int* devices, oocnmf_ctx** out) {
    return guarded([&] {
        if (n < 1) fail(OOCNMF_ERR_SHAPE, "spawn_group: need at least one rank");
        for (int r = 0; r < n; ++r) out[r] = nullptr;
        std::vector<int> devs(devices, devices + n);
        for (int r = 0; r < n; ++r)
            for (int q = 0; q < r; ++q)
                if (devs[q] == devs[r])
                    fail(OOCNMF_ERR_SHAPE, "spawn_group: one GPU per rank (device " + std::to_string(devs[r]) +
                                               " repeats; NCCL runs one rank per device)");
        std::vector<oocnmf_ctx*> cs(n, nullptr);
        try {
            for (int r = 0; r < n; ++r) {
                cs[r] = new oocnmf_ctx();
                ctx_init_common(cs[r], devs[r]);
                cs[r]->rank = r;
                cs[r]->nranks = n;
            }
            if (n > 1) {
                std::vector<ncclComm_t> comms(n);
                eager_connect();
                nck(ncclCommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
                for (int r = 0; r < n; ++r) cs[r]->comm = comms[r];
            }
        } catch (...) {
            for (auto* c : cs)
                if (c) oocnmf_ctx_destroy(c);
            throw;
        }
        for (int r = 0; r < n; ++r) out[r] = cs[r];
    });
}

static int one_shot(int device, uint64_t m, uint64_t n, const oocnmf_config* cfg, const double* w0, const double* h0,
                    double* w_out, double* h_out, uint64_t* ti, double* te, uint64_t cap, oocnmf_info* info,
                    int (*load)(oocnmf_ctx*, const void*), const void* src) {
    double tp[6];
    tp[0] = io_clock();
    oocnmf_ctx* c = nullptr;
    int st = oocnmf_ctx_create(device, &c);
    if (st) return st;
    if (!cfg) {
        oocnmf_ctx_destroy(c);
        g_err = "null config";
        return OOCNMF_ERR_SHAPE;
    }
    st = oocnmf_set_problem(c, m, n, cfg->k, 0, m);
    tp[1] = io_clock();
    if (!st) st = load(c, src);
    if (!st && cfg->init == 1) {
        if (!w0 || !h0) {
            g_err = "NmfConfig: init=from_files requires both factors";
            st = OOCNMF_ERR_SHAPE;
        } else {
            st = oocnmf_set_factors_f64(c, w0, h0);
        }
    }
    tp[2] = io_clock();
    if (!st) st = oocnmf_solve(c, cfg, ti, te, cap, info);
    tp[3] = io_clock();
    if (!st) st = oocnmf_get_factors_f64(c, w_out, h_out);
    tp[4] = io_clock();
    const std::string keep = g_err;
    oocnmf_ctx_destroy(c);
    g_err = keep;
    tp[5] = io_clock();
    if (io_profile())
        std::fprintf(stderr, "[oocnmf io] one-shot: create+problem %.1f ms, load %.1f ms, solve %.1f ms, "
                     "factors out %.1f ms, destroy %.1f ms\n", (tp[1] - tp[0]) * 1e3, (tp[2] - tp[1]) * 1e3,
                     (tp[3] - tp[2]) * 1e3, (tp[4] - tp[3]) * 1e3, (tp[5] - tp[4]) * 1e3);
    return st;
}

struct CsrSrc {
    const uint64_t *rp, *ci;
    const double* v;
};

int oocnmf_nmf_serial_dense_f64(int device, const double* a, uint64_t m, uint64_t n, const oocnmf_config* cfg,
                                const double* w0, const double* h0, double* w_out, double* h_out, uint64_t* ti,
                                double* te, uint64_t cap, oocnmf_info* info) {
    auto ld = [](oocnmf_ctx* c, const void* p) {
        return oocnmf_load_dense_f64(c, static_cast<const double*>(p), c->n);
    };
    return one_shot(device, m, n, cfg, w0, h0, w_out, h_out, ti, te, cap, info, ld, a);
}

int oocnmf_nmf_serial_dense_f32(int device, const float* a, uint64_t m, uint64_t n, const oocnmf_config* cfg,
                                const double* w0, const double* h0, double* w_out, double* h_out, uint64_t* ti,
                                double* te, uint64_t cap, oocnmf_info* info) {
    auto ld = [](oocnmf_ctx* c, const void* p) {
        return oocnmf_load_dense_f32(c, static_cast<const float*>(p), c->n);
    };
    return one_shot(device, m, n, cfg, w0, h0, w_out, h_out, ti, te, cap, info, ld, a);
}

int oocnmf_nmf_serial_csr_f64(int device, const uint64_t* row_ptr, const uint64_t* col_idx, const double* vals,
                              uint64_t m, uint64_t n, const oocnmf_config* cfg, const double* w0, const double* h0,
                              double* w_out, double* h_out, uint64_t* ti, double* te, uint64_t cap,
                              oocnmf_info* info) {
    CsrSrc src{row_ptr, col_idx, vals};
    auto ld = [](oocnmf_ctx* c, const void* p) {
        const auto* s = static_cast<const CsrSrc*>(p);
        return oocnmf_load_csr_f64(c, s->rp, s->ci, s->v);
    };
    return one_shot(device, m, n, cfg, w0, h0, w_out, h_out, ti, te, cap, info, ld, &src);
}

}  // extern "C"
