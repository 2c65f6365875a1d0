// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the *unmodified* reference library compiled from
// /root/reference/proj/src (see oracle/Makefile). It lets tests/, bench.py's
// cpu_baseline / --impl reference leg, and __graft_entry__.smoke() drive the
// reference CPU solver through plain pointers. Nothing here re-implements an
// algorithm: every call forwards to the reference's own functions.
//
//   ref_nmf_serial_*        -> oocnmf::nmf_serial          (src/nmf_serial.cpp:56)
//   ref_nmf_distributed_*   -> oocnmf::run_distributed_threads (src/nmf_distributed.cpp:291)
//   ref_gen_lowrank         -> oocnmf::gen_lowrank          (src/synth.cpp:18)
//   ref_gen_sparse_*        -> oocnmf::gen_sparse_random    (src/synth.cpp:60)
//   ref_init_factors        -> oocnmf::init_factors         (src/nmf_serial.cpp:50)
//   ref_mu_iteration        -> the body of nmf_serial's loop (src/nmf_serial.cpp:84-101)
//   ref_make_plan           -> oocnmf::make_plan            (src/partition.cpp:49)
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "oocnmf/io.hpp"
#include "oocnmf/kernels.hpp"
#include "oocnmf/model_selection.hpp"
#include "oocnmf/nmf.hpp"
#include "oocnmf/nmf_distributed.hpp"
#include "oocnmf/partition.hpp"
#include "oocnmf/rng.hpp"
#include "oocnmf/synth.hpp"

#include <nlohmann/json.hpp>

using namespace oocnmf;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        return fail(e, 1);
    } catch (const DataError& e) {
        return fail(e, 2);
    } catch (const IoError& e) {
        return fail(e, 3);
    } catch (const CommError& e) {
        return fail(e, 4);
    } catch (const StoreError& e) {
        return fail(e, 5);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

DenseMatrix copy_dense(const double* p, std::uint64_t r, std::uint64_t c) {
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

struct Out {
    double* w;
    double* h;
    std::uint64_t* trace_it;
    double* trace_err;
    std::uint64_t trace_cap;
    std::uint64_t* n_trace;
    std::uint64_t* iters_run;
    int* converged;
    double* counters;  // [w_update_s, h_update_s, allreduce_s, error_check_s, io_s, total_s, flops]
};

void write_out(const NmfResult& r, const Out& o) {
    std::memcpy(o.w, r.w.data(), r.w.size() * sizeof(double));
    std::memcpy(o.h, r.h.data(), r.h.size() * sizeof(double));
    const std::uint64_t n = r.error_trace.size();
    *o.n_trace = n;
    for (std::uint64_t i = 0; i < n && i < o.trace_cap; ++i) {
        o.trace_it[i] = r.error_trace[i].first;
        o.trace_err[i] = r.error_trace[i].second;
    }
    *o.iters_run = r.iterations_run;
    *o.converged = r.converged ? 1 : 0;
    if (o.counters) {
        const auto& c = r.counters;
        double v[7] = {c.w_update_s, c.h_update_s, c.allreduce_s, c.error_check_s,
                       c.io_s,       c.total_s,    c.flops};
        std::memcpy(o.counters, v, sizeof v);
    }
}

NmfConfig make_cfg(std::uint64_t k, std::uint64_t max_iters, std::uint64_t interval, double eta,
                   double eps, std::uint64_t seed, const double* w0, const double* h0,
                   std::uint64_t m, std::uint64_t n) {
    NmfConfig cfg;
    cfg.k = k;
    cfg.max_iters = max_iters;
    cfg.error_check_interval = interval;
    cfg.eta = eta;
    cfg.epsilon = eps;
    cfg.seed = seed;
    if (w0 && h0) {
        cfg.init = FactorInit::from_files;
        cfg.init_w = copy_dense(w0, m, k);
        cfg.init_h = copy_dense(h0, k, n);
    }
    return cfg;
}

CsrMatrix make_csr(std::uint64_t m, std::uint64_t n, const std::uint64_t* rp, const std::uint64_t* ci,
                   const double* v) {
    const std::uint64_t nnz = rp[m];
    return CsrMatrix(m, n, std::vector<index_t>(rp, rp + m + 1), std::vector<index_t>(ci, ci + nnz),
                     std::vector<double>(v, v + nnz));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_nmf_serial_dense(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t k,
                         std::uint64_t max_iters, std::uint64_t interval, double eta, double eps,
                         std::uint64_t seed, const double* w0, const double* h0, double* w,
                         double* h, std::uint64_t* trace_it, double* trace_err,
                         std::uint64_t trace_cap, std::uint64_t* n_trace, std::uint64_t* iters_run,
                         int* converged, double* counters) {
    return guarded([&] {
        DenseMatrix A = copy_dense(a, m, n);
        NmfConfig cfg = make_cfg(k, max_iters, interval, eta, eps, seed, w0, h0, m, n);
        write_out(nmf_serial(MatrixRef(A), cfg),
                  {w, h, trace_it, trace_err, trace_cap, n_trace, iters_run, converged, counters});
    });
}

int ref_nmf_serial_csr(const std::uint64_t* rp, const std::uint64_t* ci, const double* v,
                       std::uint64_t m, std::uint64_t n, std::uint64_t k, std::uint64_t max_iters,
                       std::uint64_t interval, double eta, double eps, std::uint64_t seed,
                       const double* w0, const double* h0, double* w, double* h,
                       std::uint64_t* trace_it, double* trace_err, std::uint64_t trace_cap,
                       std::uint64_t* n_trace, std::uint64_t* iters_run, int* converged,
                       double* counters) {
    return guarded([&] {
        CsrMatrix A = make_csr(m, n, rp, ci, v);
        NmfConfig cfg = make_cfg(k, max_iters, interval, eta, eps, seed, w0, h0, m, n);
        write_out(nmf_serial(MatrixRef(A), cfg),
                  {w, h, trace_it, trace_err, trace_cap, n_trace, iters_run, converged, counters});
    });
}

// Threads-backend distributed run; returns rank 0's result (identical on all ranks).
// strategy: 0 = choose_strategy(m, n), 1 = CNMF, 2 = RNMF. a_csr_* may be null for dense.
int ref_nmf_distributed(const double* a_dense, const std::uint64_t* rp, const std::uint64_t* ci,
                        const double* v, std::uint64_t m, std::uint64_t n, std::uint64_t k,
                        int n_workers, std::uint64_t n_b, int strategy, std::uint64_t max_iters,
                        std::uint64_t interval, double eta, double eps, std::uint64_t seed,
                        const double* w0, const double* h0, double* w, double* h,
                        std::uint64_t* trace_it, double* trace_err, std::uint64_t trace_cap,
                        std::uint64_t* n_trace, std::uint64_t* iters_run, int* converged,
                        double* counters) {
    return guarded([&] {
        DenseMatrix Ad;
        CsrMatrix As;
        MatrixRef ref;
        if (a_dense) {
            Ad = copy_dense(a_dense, m, n);
            ref = MatrixRef(Ad);
        } else {
            As = make_csr(m, n, rp, ci, v);
            ref = MatrixRef(As);
        }
        const Strategy s = strategy == 0   ? choose_strategy(m, n)
                           : strategy == 1 ? Strategy::cnmf
                                           : Strategy::rnmf;
        PartitionPlan plan = make_plan(m, n, k, n_workers, n_b, s);
        NmfConfig cfg = make_cfg(k, max_iters, interval, eta, eps, seed, w0, h0, m, n);
        auto res = run_distributed_threads(ASource::memory(ref), cfg, plan);
        write_out(res[0],
                  {w, h, trace_it, trace_err, trace_cap, n_trace, iters_run, converged, counters});
    });
}

int ref_init_factors(std::uint64_t m, std::uint64_t n, std::uint64_t k, std::uint64_t seed,
                     double* w, double* h) {
    return guarded([&] {
        auto [W, H] = init_factors(m, n, k, seed);
        std::memcpy(w, W.data(), W.size() * sizeof(double));
        std::memcpy(h, H.data(), H.size() * sizeof(double));
    });
}

int ref_gen_lowrank(std::uint64_t m, std::uint64_t n, std::uint64_t k_true, double noise,
                    std::uint64_t seed, double* a, double* w0, double* h0) {
    return guarded([&] {
        LowrankSpec spec{m, n, k_true, noise, seed};
        LowrankData d = gen_lowrank(spec);
        std::memcpy(a, d.a.data(), d.a.size() * sizeof(double));
        if (w0) std::memcpy(w0, d.w0.data(), d.w0.size() * sizeof(double));
        if (h0) std::memcpy(h0, d.h0.data(), d.h0.size() * sizeof(double));
    });
}

// Two-call protocol: first with col_idx == nullptr to learn nnz (written to *nnz_out and
// rp), then again with buffers sized nnz.
int ref_gen_sparse(std::uint64_t m, std::uint64_t n, double density, std::uint64_t seed,
                   std::uint64_t* rp, std::uint64_t* ci, double* v, std::uint64_t* nnz_out) {
    return guarded([&] {
        CsrMatrix s = gen_sparse_random(SparseSpec{m, n, density, seed});
        *nnz_out = s.nnz();
        std::memcpy(rp, s.row_ptr().data(), (m + 1) * sizeof(std::uint64_t));
        if (ci) {
            std::memcpy(ci, s.col_idx().data(), s.nnz() * sizeof(std::uint64_t));
            std::memcpy(v, s.values().data(), s.nnz() * sizeof(double));
        }
    });
}

// CounterRng(seed, stream).uniform(i * n + j) for a row window [row0, row0 + rows).
int ref_uniform_dense(std::uint64_t row0, std::uint64_t rows, std::uint64_t n, std::uint64_t seed,
                      std::uint64_t stream, double* out) {
    return guarded([&] {
        CounterRng rng(seed, stream);
        for (std::uint64_t i = 0; i < rows; ++i)
            for (std::uint64_t j = 0; j < n; ++j) out[i * n + j] = rng.uniform((row0 + i) * n + j);
    });
}

// One MU iteration (W update then H update) on caller-owned factors, exactly the body of
// nmf_serial's loop (src/nmf_serial.cpp:84-101), without the error check. Used by the
// bench's reference arm on a bounded row sample.
int ref_mu_iteration(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t k, double* w,
                     double* h, double eps) {
    return guarded([&] {
        DenseMatrix A(m, n, std::vector<double>(a, a + m * n));
        DenseMatrix W = copy_dense(w, m, k), H = copy_dense(h, k, n);
        DenseMatrix ht = transpose(H);
        DenseMatrix hht = gram_t(MatrixRef(ht));
        DenseMatrix aht = matmul(MatrixRef(A), ht);
        DenseMatrix whht = matmul(MatrixRef(W), hht);
        hadamard_update(W, aht, whht, eps);
        DenseMatrix wtw = gram_t(MatrixRef(W));
        DenseMatrix wta(k, n);
        matmul_ta_acc(MatrixRef(W), MatrixRef(A), wta);
        DenseMatrix wtwh = matmul(MatrixRef(wtw), H);
        hadamard_update(H, wta, wtwh, eps);
        std::memcpy(w, W.data(), W.size() * sizeof(double));
        std::memcpy(h, H.data(), H.size() * sizeof(double));
    });
}

// Same, but A is already an oocnmf::DenseMatrix held by the caller across calls (avoids the
// per-call copy in timed loops): create/destroy a handle.
void* ref_dense_create(const double* a, std::uint64_t m, std::uint64_t n) {
    return new DenseMatrix(m, n, std::vector<double>(a, a + m * n));
}
void ref_dense_destroy(void* p) { delete static_cast<DenseMatrix*>(p); }
int ref_mu_iteration_handle(void* a_handle, std::uint64_t k, double* w, double* h, double eps) {
    return guarded([&] {
        const DenseMatrix& A = *static_cast<DenseMatrix*>(a_handle);
        const std::uint64_t m = A.rows(), n = A.cols();
        DenseMatrix W = copy_dense(w, m, k), H = copy_dense(h, k, n);
        DenseMatrix ht = transpose(H);
        DenseMatrix hht = gram_t(MatrixRef(ht));
        DenseMatrix aht = matmul(MatrixRef(A), ht);
        DenseMatrix whht = matmul(MatrixRef(W), hht);
        hadamard_update(W, aht, whht, eps);
        DenseMatrix wtw = gram_t(MatrixRef(W));
        DenseMatrix wta(k, n);
        matmul_ta_acc(MatrixRef(W), MatrixRef(A), wta);
        DenseMatrix wtwh = matmul(MatrixRef(wtw), H);
        hadamard_update(H, wta, wtwh, eps);
        std::memcpy(w, W.data(), W.size() * sizeof(double));
        std::memcpy(h, H.data(), H.size() * sizeof(double));
    });
}

// The uniform synthetic A (CounterRng(seed, stream).uniform(i * n + j), as
// bench/kernels_bench.cpp:12-18), optionally rounded to f32, built in place in a
// DenseMatrix held by the caller: a full-size (65536^2, 34 GB) A then exists once, not as a
// numpy array plus the DenseMatrix copy nmf_serial would otherwise need.
void* ref_dense_create_uniform(std::uint64_t m, std::uint64_t n, std::uint64_t seed, std::uint64_t stream,
                               int round_f32) {
    auto* A = new DenseMatrix(m, n);
    double* a = A->data();
    const CounterRng rng(seed, stream);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(m); ++i)
        for (std::uint64_t j = 0; j < n; ++j) {
            const double v = rng.uniform(std::uint64_t(i) * n + j);
            a[std::uint64_t(i) * n + j] = round_f32 ? double(float(v)) : v;
        }
    return A;
}

// nmf_serial (src/nmf_serial.cpp:56) on a held DenseMatrix.
int ref_nmf_serial_dense_handle(void* a_handle, std::uint64_t k, std::uint64_t max_iters, std::uint64_t interval,
                                double eta, double eps, std::uint64_t seed, const double* w0, const double* h0,
                                double* w, double* h, std::uint64_t* trace_it, double* trace_err,
                                std::uint64_t trace_cap, std::uint64_t* n_trace, std::uint64_t* iters_run,
                                int* converged, double* counters) {
    return guarded([&] {
        const DenseMatrix& A = *static_cast<DenseMatrix*>(a_handle);
        NmfConfig cfg = make_cfg(k, max_iters, interval, eta, eps, seed, w0, h0, A.rows(), A.cols());
        write_out(nmf_serial(MatrixRef(A), cfg),
                  {w, h, trace_it, trace_err, trace_cap, n_trace, iters_run, converged, counters});
    });
}

// PartitionPlan::to_json / MemoryReport::to_json of the reference (src/partition.cpp:89,199) into
// buf (NUL-terminated); returns the length or -1 if cap is too small.
long ref_plan_to_json(std::uint64_t m, std::uint64_t n, std::uint64_t k, int n_workers, std::uint64_t n_b,
                      int strategy, char* buf, std::uint64_t cap) {
    const PartitionPlan p = make_plan(m, n, k, n_workers, n_b, strategy == 1 ? Strategy::cnmf : Strategy::rnmf);
    const std::string j = p.to_json();
    if (j.size() + 1 > cap) return -1;
    std::memcpy(buf, j.c_str(), j.size() + 1);
    return long(j.size());
}
long ref_memreport_to_json(const std::uint64_t* v7, int feasible, char* buf, std::uint64_t cap) {
    MemoryReport r;
    r.a_slab_bytes = v7[0], r.store_peak_bytes = v7[1], r.factor_bytes = v7[2], r.intermediate_bytes = v7[3];
    r.peak_bytes = v7[4], r.min_n_b = v7[5], r.feasible = feasible != 0;
    const std::string j = r.to_json();
    if (j.size() + 1 > cap) return -1;
    std::memcpy(buf, j.c_str(), j.size() + 1);
    return long(j.size());
}

// nlohmann::json::parse(text).dump(indent) with the JSON library the reference is compiled
// against: the fixed-point check of the B200 CLI's JSON writer (csrc/json_out.hpp).
long ref_json_reformat(const char* text, int indent, char* buf, std::uint64_t cap) {
    std::string j;
    try {
        j = nlohmann::json::parse(text).dump(indent);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
    if (j.size() + 1 > cap) return -1;
    std::memcpy(buf, j.c_str(), j.size() + 1);
    return long(j.size());
}

// SelectionReport::to_json / to_csv (src/model_selection.cpp:408-434) of a report holding the
// given records (rec6 as ref_select_k_dense writes them), chosen k (-1 = none) and rationale.
long ref_selection_json_csv(const double* rec6, std::uint64_t nrec, std::int64_t chosen, const char* why,
                            char* json_buf, std::uint64_t json_cap, char* csv_buf, std::uint64_t csv_cap) {
    SelectionReport rep;
    for (std::uint64_t i = 0; i < nrec; ++i) {
        KRecord r;
        const double* o = rec6 + 6 * i;
        r.k = index_t(o[0]), r.valid = o[1] != 0, r.runs_used = index_t(o[2]);
        r.min_silhouette = o[3], r.mean_silhouette = o[4], r.mean_relative_error = o[5];
        rep.records.push_back(std::move(r));
    }
    if (chosen >= 0) rep.chosen_k = index_t(chosen);
    rep.rationale = why;
    const std::string j = rep.to_json(), c = rep.to_csv();
    if (j.size() + 1 > json_cap || c.size() + 1 > csv_cap) return -1;
    std::memcpy(json_buf, j.c_str(), j.size() + 1);
    std::memcpy(csv_buf, c.c_str(), c.size() + 1);
    return 0;
}

// CSR variant for the sparse bench sample (A held by the library across timed iterations).
void* ref_csr_create(const std::uint64_t* rp, const std::uint64_t* ci, const double* v, std::uint64_t m,
                     std::uint64_t n) {
    return new CsrMatrix(make_csr(m, n, rp, ci, v));
}
void ref_csr_destroy(void* p) { delete static_cast<CsrMatrix*>(p); }
int ref_mu_iteration_csr_handle(void* a_handle, std::uint64_t k, double* w, double* h, double eps) {
    return guarded([&] {
        const CsrMatrix& A = *static_cast<CsrMatrix*>(a_handle);
        const std::uint64_t m = A.rows(), n = A.cols();
        DenseMatrix W = copy_dense(w, m, k), H = copy_dense(h, k, n);
        DenseMatrix ht = transpose(H);
        DenseMatrix hht = gram_t(MatrixRef(ht));
        DenseMatrix aht = matmul(MatrixRef(A), ht);
        DenseMatrix whht = matmul(MatrixRef(W), hht);
        hadamard_update(W, aht, whht, eps);
        DenseMatrix wtw = gram_t(MatrixRef(W));
        DenseMatrix wta(k, n);
        matmul_ta_acc(MatrixRef(W), MatrixRef(A), wta);
        DenseMatrix wtwh = matmul(MatrixRef(wtw), H);
        hadamard_update(H, wta, wtwh, eps);
        std::memcpy(w, W.data(), W.size() * sizeof(double));
        std::memcpy(h, H.data(), H.size() * sizeof(double));
    });
}

// Partition plan: writes per-rank [row_begin,row_end,col_begin,col_end] and batch ranges.
int ref_make_plan(std::uint64_t m, std::uint64_t n, std::uint64_t k, int n_workers,
                  std::uint64_t n_b, int strategy, std::uint64_t* slabs4, std::uint64_t* batches2,
                  int* strategy_out) {
    return guarded([&] {
        const Strategy s = strategy == 0   ? choose_strategy(m, n)
                           : strategy == 1 ? Strategy::cnmf
                                           : Strategy::rnmf;
        PartitionPlan p = make_plan(m, n, k, n_workers, n_b, s);
        for (int r = 0; r < n_workers; ++r) {
            slabs4[4 * r + 0] = p.slabs[r].a_rows.begin;
            slabs4[4 * r + 1] = p.slabs[r].a_rows.end;
            slabs4[4 * r + 2] = p.slabs[r].a_cols.begin;
            slabs4[4 * r + 3] = p.slabs[r].a_cols.end;
        }
        for (std::uint64_t b = 0; b < n_b; ++b) {
            batches2[2 * b] = p.batches[b].begin;
            batches2[2 * b + 1] = p.batches[b].end;
        }
        *strategy_out = p.strategy == Strategy::cnmf ? 1 : 2;
    });
}

// ---- model selection (include/oocnmf/model_selection.hpp) ----
// select_k on a dense A. rec6: per k [k, valid, runs_used, min_sil, mean_sil, mean_err];
// chosen: -1 if none; medians (optional): sum over k of m*k doubles, k ascending.
int ref_select_k_dense(const double* a, std::uint64_t m, std::uint64_t n, std::uint64_t k_min,
                       std::uint64_t k_max, std::uint64_t n_pert, double delta, double sil_threshold,
                       std::uint64_t max_iters, std::uint64_t interval, double eta, double eps,
                       std::uint64_t seed, double* rec6, std::int64_t* chosen, double* medians,
                       char* why, std::uint64_t why_cap) {
    return guarded([&] {
        DenseMatrix A = copy_dense(a, m, n);
        SelectionConfig cfg;
        cfg.k_min = k_min, cfg.k_max = k_max, cfg.n_perturbations = n_pert;
        cfg.delta = delta, cfg.sil_threshold = sil_threshold, cfg.seed = seed;
        cfg.nmf.max_iters = max_iters, cfg.nmf.error_check_interval = interval;
        cfg.nmf.eta = eta, cfg.nmf.epsilon = eps;
        SelectionReport rep = select_k(MatrixRef(A), cfg);
        double* med = medians;
        for (std::size_t i = 0; i < rep.records.size(); ++i) {
            const KRecord& r = rep.records[i];
            double* o = rec6 + 6 * i;
            o[0] = double(r.k), o[1] = r.valid ? 1.0 : 0.0, o[2] = double(r.runs_used);
            o[3] = r.min_silhouette, o[4] = r.mean_silhouette, o[5] = r.mean_relative_error;
            if (med) {
                for (index_t e = 0; e < m * r.k; ++e) med[e] = r.valid ? r.medians.data()[e] : 0.0;
                med += m * r.k;
            }
        }
        *chosen = rep.chosen_k ? std::int64_t(*rep.chosen_k) : -1;
        if (why && why_cap) {
            const std::size_t len = std::min<std::size_t>(rep.rationale.size(), why_cap - 1);
            std::memcpy(why, rep.rationale.data(), len);
            why[len] = 0;
        }
    });
}

int ref_cluster_silhouette(const double* runs, std::uint64_t nruns, std::uint64_t m, std::uint64_t k,
                           double* medians, double* per_cluster, double* min_sil, double* mean_sil,
                           std::uint64_t* dropped, std::int64_t* member_cluster) {
    return guarded([&] {
        std::vector<DenseMatrix> ws;
        for (std::uint64_t r = 0; r < nruns; ++r) ws.push_back(copy_dense(runs + r * m * k, m, k));
        ColumnClusters cl = cluster_columns(ws, k);
        for (std::uint64_t e = 0; e < nruns * k; ++e) member_cluster[e] = -1;
        for (std::uint64_t c = 0; c < k; ++c)
            for (const auto& [r, col] : cl.member_ids[c]) member_cluster[r * k + col] = std::int64_t(c);
        std::memcpy(medians, cl.medians.data(), m * k * sizeof(double));
        *dropped = cl.dropped_zero_columns;
        SilhouetteScore s = silhouette(cl);
        std::memcpy(per_cluster, s.per_cluster.data(), k * sizeof(double));
        *min_sil = s.min_sil;
        *mean_sil = s.mean_sil;
    });
}

int ref_pearson(const double* wt, std::uint64_t m, std::uint64_t k1, const double* we, std::uint64_t k2,
                double* corr) {
    return guarded([&] {
        DenseMatrix c = pearson_correlation_matrix(copy_dense(wt, m, k1), copy_dense(we, m, k2));
        std::memcpy(corr, c.data(), k1 * k2 * sizeof(double));
    });
}

int ref_perturb_dense(const double* a, std::uint64_t m, std::uint64_t n, double delta, std::uint64_t seed,
                      double* out) {
    return guarded([&] {
        DenseMatrix A = copy_dense(a, m, n);
        DenseMatrix P = perturb_dense(MatrixRef(A), delta, seed);
        std::memcpy(out, P.data(), m * n * sizeof(double));
    });
}

// ---- matrix files (include/oocnmf/io.hpp) ----
int ref_write_pdn1_dense(const char* path, const double* a, std::uint64_t m, std::uint64_t n) {
    return guarded([&] { write_pdn1(path, copy_dense(a, m, n)); });
}
int ref_write_mtx_dense(const char* path, const double* a, std::uint64_t m, std::uint64_t n) {
    return guarded([&] { write_mtx(path, copy_dense(a, m, n)); });
}
static CsrMatrix io_csr(std::uint64_t m, std::uint64_t n, const std::uint64_t* rp, const std::uint64_t* ci,
                          const double* v) {
    return CsrMatrix(m, n, std::vector<index_t>(rp, rp + m + 1), std::vector<index_t>(ci, ci + rp[m]),
                     std::vector<double>(v, v + rp[m]));
}
int ref_write_pdn1_csr(const char* path, std::uint64_t m, std::uint64_t n, const std::uint64_t* rp,
                       const std::uint64_t* ci, const double* v) {
    return guarded([&] { write_pdn1(path, io_csr(m, n, rp, ci, v)); });
}
int ref_write_mtx_csr(const char* path, std::uint64_t m, std::uint64_t n, const std::uint64_t* rp,
                      const std::uint64_t* ci, const double* v) {
    return guarded([&] { write_mtx(path, io_csr(m, n, rp, ci, v)); });
}
// read_matrix: dims first (outputs null), then fill
int ref_read_matrix(const char* path, int* kind, std::uint64_t* m, std::uint64_t* n, std::uint64_t* nnz,
                    double* dense, std::uint64_t* rp, std::uint64_t* ci, double* v) {
    return guarded([&] {
        AnyMatrix a = read_matrix(path);
        *kind = a.is_dense() ? 0 : 1;
        *m = a.rows(), *n = a.cols();
        *nnz = a.is_dense() ? 0 : a.sparse().nnz();
        if (a.is_dense() && dense) std::memcpy(dense, a.dense().data(), a.dense().size() * sizeof(double));
        if (!a.is_dense() && rp) {
            const CsrMatrix& s = a.sparse();
            for (index_t i = 0; i <= s.rows(); ++i) rp[i] = s.row_ptr()[i];
            for (index_t p = 0; p < s.nnz(); ++p) ci[p] = s.col_idx()[p], v[p] = s.values()[p];
        }
    });
}

}  // extern "C"
