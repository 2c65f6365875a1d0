/*
 * TEST INFRASTRUCTURE ONLY — the CPU parity oracle. Not part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.
 *
 * A plain-C restatement of the reference's serial and row-partitioned MU-NMF
 * (arxiv 2202.09518 "pyDNMF-GPU", as restated by /root/reference/proj). Every
 * loop keeps the reference's f64 summation order so this file reproduces the
 * reference bit-for-bit when both are compiled with -ffp-contract=off
 * (tests/test_oracle.py pins that against oracle/_ref and against the golden
 * values in tests/golden/).
 *
 *   counter RNG          include/oocnmf/rng.hpp:11-45
 *   init_factors         src/nmf_serial.cpp:31-54
 *   nmf_serial loop      src/nmf_serial.cpp:56-121
 *   matmul_acc           src/kernels.cpp:28-68     (dense + CSR)
 *   matmul_ta_acc        src/kernels.cpp:78-125    (dense + CSR scatter)
 *   gram_acc (upper+mirror) src/kernels.cpp:127-173
 *   hadamard_update      src/kernels.cpp:207-244
 *   sq_frobenius         src/kernels.cpp:246-268
 *   residual_sq (256-row blocks) src/kernels.cpp:272-327
 *   RNMF worker          src/nmf_distributed.cpp:151-289 (threads backend:
 *                        ascending-rank all-reduce, src/comm.cpp:77-87)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MO_GOLDEN 0x9E3779B97F4A7C15ULL

uint64_t mo_mix(uint64_t z) {
    z += MO_GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t mo_key(uint64_t seed, uint64_t stream) {
    return mo_mix(seed ^ mo_mix(stream + 0x632BE59BD9B4E019ULL));
}

static double mo_u01(uint64_t key, uint64_t idx) {
    return (double)(mo_mix(key + (idx + 1) * MO_GOLDEN) >> 11) * 0x1.0p-53;
}

double mo_uniform(uint64_t seed, uint64_t stream, uint64_t idx) {
    return mo_u01(mo_key(seed, stream), idx);
}

/* out[i*n + j] = U(seed, stream, (row0+i)*n + j) */
void mo_uniform_dense(uint64_t row0, uint64_t rows, uint64_t n, uint64_t seed, uint64_t stream,
                      double* out) {
    const uint64_t key = mo_key(seed, stream);
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < n; ++j) out[i * n + j] = mo_u01(key, (row0 + i) * n + j);
}

/* W (m x k) from stream 1, H (k x n) from stream 2 (nmf_serial.cpp:17-18). */
void mo_init_factors(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, double* w, double* h) {
    const uint64_t kw = mo_key(seed, 1), kh = mo_key(seed, 2);
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < k; ++j) w[i * k + j] = mo_u01(kw, i * k + j);
    for (uint64_t r = 0; r < k; ++r)
        for (uint64_t j = 0; j < n; ++j) h[r * n + j] = mo_u01(kh, r * n + j);
}

/* ------------------------------------------------------------------ A */
/* A is either dense row-major (ld = n) or CSR with u64 indices. A "view" is a
 * row window [r0, r1) and column window [c0, c1) of the stored matrix. */
typedef struct {
    const double* dense;
    const uint64_t* rp;
    const uint64_t* ci;
    const double* v;
    uint64_t m, n;
} mo_mat;

typedef struct {
    const mo_mat* a;
    uint64_t r0, r1, c0, c1;
} mo_view;

static mo_view full_view(const mo_mat* a) {
    mo_view v = {a, 0, a->m, 0, a->n};
    return v;
}

/* acc (rows x kc) += A_view @ B, B rows indexed by view-local column (ld = kc). */
static void matmul_acc(mo_view a, const double* b, uint64_t kc, double* acc) {
    const uint64_t rows = a.r1 - a.r0, cols = a.c1 - a.c0;
    for (uint64_t r = 0; r < rows; ++r) {
        double* out = acc + r * kc;
        const uint64_t gi = a.r0 + r;
        if (a.a->dense) {
            const double* arow = a.a->dense + gi * a.a->n + a.c0;
            for (uint64_t q = 0; q < cols; ++q) {
                const double av = arow[q];
                const double* brow = b + q * kc;
                for (uint64_t c = 0; c < kc; ++c) out[c] += av * brow[c];
            }
        } else {
            for (uint64_t p = a.a->rp[gi]; p < a.a->rp[gi + 1]; ++p) {
                const uint64_t j = a.a->ci[p];
                if (j < a.c0 || j >= a.c1) continue;
                const double av = a.a->v[p];
                const double* brow = b + (j - a.c0) * kc;
                for (uint64_t c = 0; c < kc; ++c) out[c] += av * brow[c];
            }
        }
    }
}

/* plain dense acc (r x c) += x (r x q) @ y (q x c); ldx/ldy/ldacc given. */
static void dmm(const double* x, uint64_t ldx, const double* y, uint64_t ldy, double* acc,
                uint64_t ldacc, uint64_t r_, uint64_t q_, uint64_t c_) {
    for (uint64_t r = 0; r < r_; ++r) {
        double* out = acc + r * ldacc;
        for (uint64_t q = 0; q < q_; ++q) {
            const double xv = x[r * ldx + q];
            const double* yrow = y + q * ldy;
            for (uint64_t c = 0; c < c_; ++c) out[c] += xv * yrow[c];
        }
    }
}

/* acc (k x cols) += W^T @ A_view; W rows aligned with the view's rows (ld k). */
static void matmul_ta_acc(const double* w, uint64_t k, mo_view a, double* acc) {
    const uint64_t rows = a.r1 - a.r0, cols = a.c1 - a.c0;
    if (a.a->dense) {
        /* i-outer for cache reuse; each acc[r][c] still sums over ascending i. */
        for (uint64_t i = 0; i < rows; ++i) {
            const double* arow = a.a->dense + (a.r0 + i) * a.a->n + a.c0;
            for (uint64_t r = 0; r < k; ++r) {
                const double wv = w[i * k + r];
                double* out = acc + r * cols;
                for (uint64_t c = 0; c < cols; ++c) out[c] += wv * arow[c];
            }
        }
    } else {
        for (uint64_t i = 0; i < rows; ++i) {
            const double* wrow = w + i * k;
            const uint64_t gi = a.r0 + i;
            for (uint64_t p = a.a->rp[gi]; p < a.a->rp[gi + 1]; ++p) {
                const uint64_t j = a.a->ci[p];
                if (j < a.c0 || j >= a.c1) continue;
                const double av = a.a->v[p];
                const uint64_t lc = j - a.c0;
                for (uint64_t r = 0; r < k; ++r) acc[r * cols + lc] += av * wrow[r];
            }
        }
    }
}

/* g (k x k) = x^T x for x (rows x k, ld k): upper triangle, ascending rows, mirrored. */
static void gram(const double* x, uint64_t rows, uint64_t k, double* g) {
    memset(g, 0, k * k * sizeof(double));
    /* i-outer; each g[r][c] (c >= r) still accumulates over ascending i from 0. */
    for (uint64_t i = 0; i < rows; ++i) {
        const double* xi = x + i * k;
        for (uint64_t r = 0; r < k; ++r)
            for (uint64_t c = r; c < k; ++c) g[r * k + c] += xi[r] * xi[c];
    }
    for (uint64_t r = 0; r < k; ++r)
        for (uint64_t c = r + 1; c < k; ++c) g[c * k + r] = g[r * k + c];
}

static void transpose(const double* x, uint64_t r, uint64_t c, double* y) {
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t j = 0; j < c; ++j) y[j * r + i] = x[i * c + j];
}

/* t[i, col0+j] = t*nu/(de+eps) over a (rows x cols) window of t (ld ldt). */
static void hadamard(double* t, uint64_t ldt, const double* nu, const double* de, uint64_t rows,
                     uint64_t cols, double eps) {
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j)
            t[i * ldt + j] = t[i * ldt + j] * nu[i * cols + j] / (de[i * cols + j] + eps);
}

static double sq_frobenius(mo_view a) {
    double sum = 0.0;
    if (a.a->dense) {
        for (uint64_t i = a.r0; i < a.r1; ++i) {
            const double* row = a.a->dense + i * a.a->n + a.c0;
            for (uint64_t j = 0; j < a.c1 - a.c0; ++j) sum += row[j] * row[j];
        }
    } else {
        for (uint64_t i = a.r0; i < a.r1; ++i)
            for (uint64_t p = a.a->rp[i]; p < a.a->rp[i + 1]; ++p)
                if (a.a->ci[p] >= a.c0 && a.a->ci[p] < a.c1) sum += a.a->v[p] * a.a->v[p];
    }
    return sum;
}

/* sum (A_view - W[w_row0..] H[:, h_col0..])^2 in 256-row blocks. h is k x ldh. */
static double residual_sq(mo_view a, const double* w, uint64_t w_row0, const double* h,
                          uint64_t ldh, uint64_t h_col0, uint64_t k) {
    const uint64_t rows = a.r1 - a.r0, ncols = a.c1 - a.c0, block = 256;
    double* wh = (double*)malloc(block * ncols * sizeof(double));
    double total = 0.0;
    for (uint64_t b0 = 0; b0 < rows; b0 += block) {
        const uint64_t b1 = rows < b0 + block ? rows : b0 + block;
        memset(wh, 0, (b1 - b0) * ncols * sizeof(double));
        dmm(w + (w_row0 + b0) * k, k, h + h_col0, ldh, wh, ncols, b1 - b0, k, ncols);
        double block_sum = 0.0;
        for (uint64_t i = b0; i < b1; ++i) {
            const uint64_t gi = a.r0 + i;
            const double* whrow = wh + (i - b0) * ncols;
            if (a.a->dense) {
                const double* arow = a.a->dense + gi * a.a->n + a.c0;
                for (uint64_t j = 0; j < ncols; ++j) {
                    const double d = arow[j] - whrow[j];
                    block_sum += d * d;
                }
            } else {
                uint64_t p = a.a->rp[gi];
                const uint64_t pe = a.a->rp[gi + 1];
                while (p < pe && a.a->ci[p] < a.c0) ++p;
                for (uint64_t j = 0; j < ncols; ++j) {
                    double av = 0.0;
                    if (p < pe && a.a->ci[p] == a.c0 + j) av = a.a->v[p++];
                    const double d = av - whrow[j];
                    block_sum += d * d;
                }
            }
        }
        total += block_sum;
    }
    free(wh);
    return total;
}

static int all_finite(const double* x, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* status: 0 ok, 1 shape, 2 data (zero norm / non-finite) */
typedef struct {
    uint64_t* trace_it;
    double* trace_err;
    uint64_t trace_cap;
    uint64_t n_trace;
    uint64_t iters_run;
    int converged;
} mo_trace;

static void push_trace(mo_trace* t, uint64_t it, double err) {
    if (t->n_trace < t->trace_cap) {
        t->trace_it[t->n_trace] = it;
        t->trace_err[t->n_trace] = err;
    }
    t->n_trace++;
}

/* nmf_serial (src/nmf_serial.cpp:56-121). w (m x k) and h (k x n) hold the initial
 * factors on entry (caller draws them with mo_init_factors or supplies files) and the
 * result on exit. */
static int nmf_serial_impl(const mo_mat* A, uint64_t k, uint64_t max_iters, uint64_t interval,
                           double eta, double eps, double* w, double* h, mo_trace* tr) {
    const uint64_t m = A->m, n = A->n;
    if (k < 1 || max_iters < 1 || interval < 1 || !(eps > 0) || !(eta >= 0) || m < 1 || n < 1)
        return 1;
    mo_view av = full_view(A);
    const double norm_a_sq = sq_frobenius(av);
    if (norm_a_sq == 0.0) return 2;
    const double norm_a = sqrt(norm_a_sq);

    double* ht = malloc(n * k * sizeof(double));
    double* hht = malloc(k * k * sizeof(double));
    double* aht = malloc(m * k * sizeof(double));
    double* whht = malloc(m * k * sizeof(double));
    double* wtw = malloc(k * k * sizeof(double));
    double* wta = malloc(k * n * sizeof(double));
    double* wtwh = malloc(k * n * sizeof(double));
    int status = 0;
    uint64_t iter;
    tr->n_trace = 0;
    tr->converged = 0;
    for (iter = 1; iter <= max_iters; ++iter) {
        transpose(h, k, n, ht);
        gram(ht, n, k, hht);
        memset(aht, 0, m * k * sizeof(double));
        matmul_acc(av, ht, k, aht);
        memset(whht, 0, m * k * sizeof(double));
        dmm(w, k, hht, k, whht, k, m, k, k);
        hadamard(w, k, aht, whht, m, k, eps);

        gram(w, m, k, wtw);
        memset(wta, 0, k * n * sizeof(double));
        matmul_ta_acc(w, k, av, wta);
        memset(wtwh, 0, k * n * sizeof(double));
        dmm(wtw, k, h, n, wtwh, n, k, k, n);
        hadamard(h, n, wta, wtwh, k, n, eps);

        if (iter % interval == 0 || iter == max_iters) {
            if (!all_finite(w, m * k) || !all_finite(h, k * n)) {
                status = 2;
                break;
            }
            const double err = sqrt(residual_sq(av, w, 0, h, n, 0, k)) / norm_a;
            push_trace(tr, iter, err);
            if (err <= eta) {
                tr->converged = 1;
                break;
            }
        }
    }
    tr->iters_run = iter < max_iters ? iter : max_iters;
    free(ht), free(hht), free(aht), free(whht), free(wtw), free(wta), free(wtwh);
    return status;
}

int mo_nmf_serial_dense(const double* a, uint64_t m, uint64_t n, uint64_t k, uint64_t max_iters,
                        uint64_t interval, double eta, double eps, double* w, double* h,
                        uint64_t* trace_it, double* trace_err, uint64_t trace_cap,
                        uint64_t* n_trace, uint64_t* iters_run, int* converged) {
    mo_mat A = {a, 0, 0, 0, m, n};
    mo_trace t = {trace_it, trace_err, trace_cap, 0, 0, 0};
    int s = nmf_serial_impl(&A, k, max_iters, interval, eta, eps, w, h, &t);
    *n_trace = t.n_trace, *iters_run = t.iters_run, *converged = t.converged;
    return s;
}

int mo_nmf_serial_csr(const uint64_t* rp, const uint64_t* ci, const double* v, uint64_t m,
                      uint64_t n, uint64_t k, uint64_t max_iters, uint64_t interval, double eta,
                      double eps, double* w, double* h, uint64_t* trace_it, double* trace_err,
                      uint64_t trace_cap, uint64_t* n_trace, uint64_t* iters_run, int* converged) {
    mo_mat A = {0, rp, ci, v, m, n};
    mo_trace t = {trace_it, trace_err, trace_cap, 0, 0, 0};
    int s = nmf_serial_impl(&A, k, max_iters, interval, eta, eps, w, h, &t);
    *n_trace = t.n_trace, *iters_run = t.iters_run, *converged = t.converged;
    return s;
}

/* ---------------------------------------------------------------- RNMF */
/* Split [0, extent) into parts ranges, the first (extent mod parts) one longer
 * (src/partition.cpp:20-32). */
void mo_split_even(uint64_t extent, uint64_t parts, uint64_t* begins /* parts+1 */) {
    const uint64_t base = extent / parts, rem = extent % parts;
    uint64_t pos = 0;
    for (uint64_t p = 0; p < parts; ++p) {
        begins[p] = pos;
        pos += base + (p < rem ? 1 : 0);
    }
    begins[parts] = pos;
}

/* Row-partitioned distributed MU over n_workers simulated ranks with n_b column
 * batches, reproducing the threads backend (ascending-rank all-reduce). W on exit is
 * the gathered m x k factor, H the replicated k x n factor. */
int mo_nmf_rnmf(const double* a_dense, const uint64_t* rp, const uint64_t* ci, const double* v,
                uint64_t m, uint64_t n, uint64_t k, uint64_t n_workers, uint64_t n_b,
                uint64_t max_iters, uint64_t interval, double eta, double eps, double* w,
                double* h, uint64_t* trace_it, double* trace_err, uint64_t trace_cap,
                uint64_t* n_trace, uint64_t* iters_run, int* converged) {
    if (n_workers < 1 || n_workers > m || n_b < 1 || n_b > n || k < 1 || max_iters < 1 ||
        interval < 1 || !(eps > 0))
        return 1;
    mo_mat A = {a_dense, rp, ci, v, m, n};
    uint64_t* slab = malloc((n_workers + 1) * sizeof(uint64_t));
    uint64_t* bat = malloc((n_b + 1) * sizeof(uint64_t));
    mo_split_even(m, n_workers, slab);
    mo_split_even(n, n_b, bat);
    const uint64_t N = n_workers;
    /* per-rank buffers; h is replicated (each rank holds the same values) */
    double* hs = malloc(N * k * n * sizeof(double));
    for (uint64_t r = 0; r < N; ++r) memcpy(hs + r * k * n, h, k * n * sizeof(double));
    double* ht = malloc(n * k * sizeof(double));
    double* hht = malloc(k * k * sizeof(double));
    double* aht = malloc(m * k * sizeof(double));
    double* whht = malloc(m * k * sizeof(double));
    double* wtw_r = malloc(N * k * k * sizeof(double));
    double* wtw = malloc(k * k * sizeof(double));
    const uint64_t maxb = bat[1] - bat[0];
    double* wta_r = malloc(N * k * maxb * sizeof(double));
    double* wta = malloc(k * maxb * sizeof(double));
    double* wtwh = malloc(k * maxb * sizeof(double));
    double* hcols = malloc(k * maxb * sizeof(double));
    int status = 0;

    /* ||A||^2: per-rank batch sums, then ascending-rank reduce */
    double norm_sq = 0.0;
    for (uint64_t r = 0; r < N; ++r) {
        double local = 0.0;
        for (uint64_t p = 0; p < n_b; ++p) {
            mo_view bv = {&A, slab[r], slab[r + 1], bat[p], bat[p + 1]};
            local += sq_frobenius(bv);
        }
        norm_sq = r == 0 ? local : norm_sq + local;
    }
    if (norm_sq == 0.0) status = 2;
    const double norm_a = sqrt(norm_sq);

    uint64_t iter = 0, nt = 0;
    int conv = 0;
    for (iter = 1; status == 0 && iter <= max_iters; ++iter) {
        /* W update: local per rank (H replicated) */
        for (uint64_t r = 0; r < N; ++r) {
            const uint64_t rows = slab[r + 1] - slab[r];
            double* wr = w + slab[r] * k;
            const double* hr = hs + r * k * n;
            transpose(hr, k, n, ht);
            gram(ht, n, k, hht);
            memset(aht, 0, rows * k * sizeof(double));
            for (uint64_t p = 0; p < n_b; ++p) {
                mo_view bv = {&A, slab[r], slab[r + 1], bat[p], bat[p + 1]};
                matmul_acc(bv, ht + bat[p] * k, k, aht);
            }
            memset(whht, 0, rows * k * sizeof(double));
            dmm(wr, k, hht, k, whht, k, rows, k, k);
            hadamard(wr, k, aht, whht, rows, k, eps);
        }
        /* H update: all-reduce W^T W, then per batch all-reduce W^T A_p */
        for (uint64_t r = 0; r < N; ++r)
            gram(w + slab[r] * k, slab[r + 1] - slab[r], k, wtw_r + r * k * k);
        memcpy(wtw, wtw_r, k * k * sizeof(double));
        for (uint64_t r = 1; r < N; ++r)
            for (uint64_t i = 0; i < k * k; ++i) wtw[i] += wtw_r[r * k * k + i];
        for (uint64_t p = 0; p < n_b; ++p) {
            const uint64_t cols = bat[p + 1] - bat[p];
            for (uint64_t r = 0; r < N; ++r) {
                memset(wta_r + r * k * cols, 0, k * cols * sizeof(double));
                mo_view bv = {&A, slab[r], slab[r + 1], bat[p], bat[p + 1]};
                matmul_ta_acc(w + slab[r] * k, k, bv, wta_r + r * k * cols);
            }
            memcpy(wta, wta_r, k * cols * sizeof(double));
            for (uint64_t r = 1; r < N; ++r)
                for (uint64_t i = 0; i < k * cols; ++i) wta[i] += wta_r[r * k * cols + i];
            for (uint64_t r = 0; r < N; ++r) {
                double* hr = hs + r * k * n;
                for (uint64_t i = 0; i < k; ++i)
                    memcpy(hcols + i * cols, hr + i * n + bat[p], cols * sizeof(double));
                memset(wtwh, 0, k * cols * sizeof(double));
                dmm(wtw, k, hcols, cols, wtwh, cols, k, k, cols);
                hadamard(hr + bat[p], n, wta, wtwh, k, cols, eps);
            }
        }
        if (iter % interval == 0 || iter == max_iters) {
            if (!all_finite(w, m * k) || !all_finite(hs, k * n)) {
                status = 2;
                break;
            }
            double tot = 0.0;
            for (uint64_t r = 0; r < N; ++r) {
                double local = 0.0;
                for (uint64_t p = 0; p < n_b; ++p) {
                    mo_view bv = {&A, slab[r], slab[r + 1], bat[p], bat[p + 1]};
                    local += residual_sq(bv, w + slab[r] * k, 0, hs + r * k * n, n, bat[p], k);
                }
                tot = r == 0 ? local : tot + local;
            }
            const double err = sqrt(tot) / norm_a;
            if (nt < trace_cap) trace_it[nt] = iter, trace_err[nt] = err;
            ++nt;
            if (err <= eta) {
                conv = 1;
                break;
            }
        }
    }
    memcpy(h, hs, k * n * sizeof(double));
    *n_trace = nt;
    *iters_run = iter < max_iters ? iter : max_iters;
    *converged = conv;
    free(slab), free(bat), free(hs), free(ht), free(hht), free(aht), free(whht);
    free(wtw_r), free(wtw), free(wta_r), free(wta), free(wtwh), free(hcols);
    return status;
}

/* One MU iteration (W then H) without the error check — bench cpu_baseline "port" leg. */
int mo_mu_iteration(const double* a, uint64_t m, uint64_t n, uint64_t k, double* w, double* h,
                    double eps) {
    mo_mat A = {a, 0, 0, 0, m, n};
    mo_view av = full_view(&A);
    double* ht = malloc(n * k * sizeof(double));
    double* hht = malloc(k * k * sizeof(double));
    double* aht = calloc(m * k, sizeof(double));
    double* whht = calloc(m * k, sizeof(double));
    double* wtw = malloc(k * k * sizeof(double));
    double* wta = calloc(k * n, sizeof(double));
    double* wtwh = calloc(k * n, sizeof(double));
    transpose(h, k, n, ht);
    gram(ht, n, k, hht);
    matmul_acc(av, ht, k, aht);
    dmm(w, k, hht, k, whht, k, m, k, k);
    hadamard(w, k, aht, whht, m, k, eps);
    gram(w, m, k, wtw);
    matmul_ta_acc(w, k, av, wta);
    dmm(wtw, k, h, n, wtwh, n, k, k, n);
    hadamard(h, n, wta, wtwh, k, n, eps);
    free(ht), free(hht), free(aht), free(whht), free(wtw), free(wta), free(wtwh);
    return 0;
}

/* Relative error ||A - WH|| / ||A|| (kernels.cpp:329-338), used by tests on GPU output. */
double mo_relative_error(const double* a_dense, const uint64_t* rp, const uint64_t* ci,
                         const double* v, uint64_t m, uint64_t n, uint64_t k, const double* w,
                         const double* h) {
    mo_mat A = {a_dense, rp, ci, v, m, n};
    mo_view av = full_view(&A);
    return sqrt(residual_sq(av, w, 0, h, n, 0, k)) / sqrt(sq_frobenius(av));
}

/* Reference-semantics sparse generator (src/synth.cpp:60-86): cell (i, j) is present iff
 * U(seed,14,i*n+j) < density, value U(seed,15,i*n+j). Two-call protocol like the shim. */
int mo_gen_sparse(uint64_t m, uint64_t n, double density, uint64_t seed, uint64_t* rp,
                  uint64_t* ci, double* v, uint64_t* nnz_out) {
    const uint64_t km = mo_key(seed, 14), kv = mo_key(seed, 15);
    uint64_t nnz = 0;
    rp[0] = 0;
    for (uint64_t i = 0; i < m; ++i) {
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t flat = i * n + j;
            if (mo_u01(km, flat) < density) {
                if (ci) ci[nnz] = j, v[nnz] = mo_u01(kv, flat);
                ++nnz;
            }
        }
        rp[i + 1] = nnz;
    }
    *nnz_out = nnz;
    return 0;
}
