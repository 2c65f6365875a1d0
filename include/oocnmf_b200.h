/*
 * oocnmf_b200.h — C-ABI of the B200-native Frobenius multiplicative-update (MU) NMF
 * backend (liboocnmf_b200.so). Plain pointers and sizes only; no torch or C++ types.
 *
 * This is the drop-in boundary for the reference's MU-NMF path. The reference
 * (/root/reference/proj, a C++20 restatement of pyDNMF-GPU, arXiv 2202.09518) has no
 * FFI of its own; its callers bind the C++ API below, which our C++ host core
 * (include/oocnmf/<name>.hpp -> include/oocnmf_b200/oocnmf.hpp) re-exports on top of these
 * entry points. Each entry point names the reference interface it replaces:
 *
 *   oocnmf_nmf_serial_dense_f64 / _csr_f64
 *        replaces NmfResult nmf_serial(MatrixRef, const NmfConfig&)
 *        (include/oocnmf/nmf.hpp:64, src/nmf_serial.cpp:56-121)
 *   oocnmf_ctx_create_comm + oocnmf_set_problem(row0, rows) + oocnmf_solve
 *        replaces nmf_distributed(ASource, NmfConfig, PartitionPlan, CommHandle&, ...)
 *        for the row partition (include/oocnmf/nmf_distributed.hpp:34-36,
 *        src/nmf_distributed.cpp:151-289); the CommHandle all-reduce
 *        (include/oocnmf/comm.hpp:61, src/comm.cpp:139-147) becomes NCCL over NVLink.
 *   oocnmf_attach_host_dense_f32(batch_rows)
 *        replaces the ChunkStore batch server for file/host-backed A
 *        (include/oocnmf/chunk_store.hpp:53-58): A stays in (pinned) host memory and is
 *        streamed to HBM in row batches on a copy stream.
 *   oocnmf_init_factors_host
 *        replaces init_factors(m, n, k, seed) (include/oocnmf/nmf.hpp:53-58): the same
 *        SplitMix64 counter RNG (include/oocnmf/rng.hpp:11-40), bit-identical f64.
 *   oocnmf_split_even
 *        the partition rule of make_plan (src/partition.cpp:20-32).
 *
 * Errors: every function returns an oocnmf_status; oocnmf_last_error() (thread-local)
 * carries the message. The C++ host core maps the codes onto the reference's exception
 * types (include/oocnmf/error.hpp:9-36): SHAPE->ShapeError, DATA->DataError,
 * IO->IoError, COMM->CommError, STORE->StoreError, DEVICE->DeviceError (new,
 * std::runtime_error). There is no CPU fallback: without a CUDA device every compute
 * entry point returns OOCNMF_ERR_DEVICE.
 */
#ifndef OOCNMF_B200_H
#define OOCNMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOCNMF_ABI_VERSION 1

typedef enum {
    OOCNMF_OK = 0,
    OOCNMF_ERR_SHAPE = 1,  /* ShapeError  — bad dims/config/window */
    OOCNMF_ERR_DATA = 2,   /* DataError   — ||A|| == 0, non-finite factors */
    OOCNMF_ERR_IO = 3,     /* IoError */
    OOCNMF_ERR_COMM = 4,   /* CommError   — NCCL failure */
    OOCNMF_ERR_STORE = 5,  /* StoreError  — host batch buffer misuse */
    OOCNMF_ERR_DEVICE = 6  /* DeviceError — CUDA failure / no device */
} oocnmf_status;

/* Mirrors NmfConfig (include/oocnmf/nmf.hpp:15-27) plus two backend knobs. */
typedef struct {
    uint64_t k;
    double eta;                    /* default 1e-4 */
    uint64_t max_iters;            /* default 1000 */
    uint64_t error_check_interval; /* default 10 */
    double epsilon;                /* default 1e-12 */
    uint64_t seed;                 /* default 0 */
    int32_t init;                  /* 0 = uniform01 (counter RNG), 1 = from factors set by
                                      oocnmf_set_factors_f64 (FactorInit::from_files),
                                      2 = continue from the factors resident on the device
                                      (warm restart after a previous oocnmf_solve) */
    int32_t error_mode;            /* 0 = auto: trace form ||A||^2 - 2<W^T A,H> + <W^T W,H H^T>
                                      (free: every term exists after the H update), re-done
                                      with the direct residual when it reports < 0.1 (where
                                      the trace form's cancellation costs accuracy);
                                      1 = direct residual (f64) at every check;
                                      2 = trace form only */
} oocnmf_config;

/* Mirrors PhaseCounters (include/oocnmf/nmf.hpp:30-39) + NmfResult scalars + kernel
 * timing measured with CUDA events on the launching stream. */
typedef struct {
    double h_update_s, w_update_s, allreduce_s, error_check_s, io_s, total_s, flops;
    uint64_t peak_resident_bytes;
    uint64_t iterations_run;
    int32_t converged;
    int32_t reserved;
    uint64_t n_trace;
    /* device-side timing (ms, summed over all launches of that kernel) */
    double aht_pass_ms;  /* A·H^T streaming pass (dense) or SpMM (CSR) */
    double wta_pass_ms;  /* A^T·W streaming pass (dense) or SpMM on CSR(A^T) */
    uint64_t aht_pass_launches;
    uint64_t wta_pass_launches;
    uint64_t gpu_launches; /* all kernels this library launched inside oocnmf_solve */
    double h2d_bytes;      /* host->device bytes moved inside oocnmf_solve (out-of-core) */
    double fused_pass_ms;  /* one-pass dense W half (A read once: A·H^T, W update, W^T·A) */
    uint64_t fused_pass_launches;
    uint64_t h2d_batches;  /* out-of-core: row batches copied host -> device inside the solve */
} oocnmf_info;

typedef struct oocnmf_ctx oocnmf_ctx;

const char* oocnmf_last_error(void);
int oocnmf_abi_version(void);
int oocnmf_device_count(int* count);

/* Host-side helpers (no device needed). */
int oocnmf_init_factors_host(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, double* w,
                             double* h);
int oocnmf_counter_uniform(uint64_t seed, uint64_t stream, uint64_t index0, uint64_t count,
                           double* out);
int oocnmf_split_even(uint64_t extent, uint64_t parts, uint64_t* begins /* parts + 1 */);

/* ----- context: one per GPU (one host thread / process per GPU) ----- */
int oocnmf_ctx_create(int device, oocnmf_ctx** out);
/* NCCL communicator: rank 0 calls oocnmf_comm_unique_id, ships the 128 bytes to the other
 * ranks (any transport; torch.distributed in the Python layer), every rank then calls
 * oocnmf_ctx_create_comm collectively. */
int oocnmf_comm_unique_id(unsigned char id[128]);
int oocnmf_ctx_create_comm(int device, int rank, int nranks, const unsigned char id[128],
                           oocnmf_ctx** out);
int oocnmf_ctx_destroy(oocnmf_ctx* ctx);
int oocnmf_ctx_rank(const oocnmf_ctx* ctx, int* rank, int* nranks);
/* Which B200 paths the context's current problem uses (reporting only; no reference
 * counterpart): bit 0 the one-pass dense kernel, bit 1 the two streaming tensor-core passes,
 * bit 2 the NVLS multicast H update, bit 3 the sharded H update, bit 4 CSR, bit 5 out-of-core. */
int oocnmf_ctx_paths(const oocnmf_ctx* ctx, int* flags);

/* Global A is m x n with k latent features; this rank owns rows [row0, row0 + rows)
 * (the RNMF slab of PartitionPlan, src/partition.cpp:72-85). */
int oocnmf_set_problem(oocnmf_ctx* ctx, uint64_t m, uint64_t n, uint64_t k, uint64_t row0,
                       uint64_t rows);

/* The problem set on this context (for layered callers). */
int oocnmf_problem_dims(const oocnmf_ctx* ctx, uint64_t* m, uint64_t* n, uint64_t* k, uint64_t* row0,
                        uint64_t* rows);

/* Column partition (CNMF, src/nmf_distributed.cpp:112-149, partition.cpp:12-14): this rank
 * owns all m rows and the columns [col0, col0 + cols) of the m x n A. W (m x k) is replicated,
 * H is the local k x cols slab; per iteration the ranks sum A·H^T (m x k) and H H^T (k x k)
 * with NCCL. Load the column slab (m x cols) with oocnmf_load_dense_* / oocnmf_load_csr_f64
 * (column indices local to the slab); oocnmf_set_factors_f64 takes the full W and the H slab;
 * oocnmf_gather_h_f64 returns the full H (k x n) on every rank. */
int oocnmf_set_problem_cols(oocnmf_ctx* ctx, uint64_t m, uint64_t n, uint64_t k, uint64_t col0,
                            uint64_t cols);
int oocnmf_gather_h_f64(oocnmf_ctx* ctx, double* h_full);

/* A sources (pick one). Dense values are stored in HBM as f32 row-major. */
int oocnmf_load_dense_f64(oocnmf_ctx* ctx, const double* a_slab, uint64_t lda);
int oocnmf_load_dense_f32(oocnmf_ctx* ctx, const float* a_slab, uint64_t lda);
int oocnmf_load_dense_device_f32(oocnmf_ctx* ctx, const float* d_a_slab, uint64_t lda);
/* A[i][j] = (float) CounterRng(seed, stream).uniform(i * n + j), generated in HBM
 * (the bench/kernels_bench.cpp:12-18 input at any size). */
int oocnmf_generate_dense_uniform(oocnmf_ctx* ctx, uint64_t seed, uint64_t stream);
/* CSR slab: row_ptr has rows+1 entries starting at 0, col_idx global in [0, n). */
int oocnmf_load_csr_f64(oocnmf_ctx* ctx, const uint64_t* row_ptr, const uint64_t* col_idx,
                        const double* vals);
/* Reference-semantics sparse generator (src/synth.cpp:60-86), evaluated in HBM for this
 * rank's rows: cell present iff U(seed,14,i*n+j) < density, value U(seed,15,i*n+j). */
int oocnmf_generate_csr_uniform(oocnmf_ctx* ctx, double density, uint64_t seed);
/* Out-of-core: A stays in host memory (pinned if the caller registered/allocated it so)
 * and streams to HBM in row batches of batch_rows (0 = auto from free HBM). */
int oocnmf_attach_host_dense_f32(oocnmf_ctx* ctx, const float* a_slab, uint64_t lda,
                                 uint64_t batch_rows);
int oocnmf_host_register(void* p, uint64_t bytes);   /* cudaHostRegister (pin) */
int oocnmf_host_unregister(void* p);
/* Copy the resident dense A slab (rows x n, f32) back to host memory (ld = n). */
int oocnmf_download_dense_f32(oocnmf_ctx* ctx, float* a_slab);
/* Resident CSR slab: nnz, then row_ptr (rows+1), col_idx, vals (f32 widened to f64). */
int oocnmf_csr_nnz(oocnmf_ctx* ctx, uint64_t* nnz);
int oocnmf_download_csr(oocnmf_ctx* ctx, uint64_t* row_ptr, uint64_t* col_idx, double* vals);

/* ----- factors ----- */
int oocnmf_set_factors_f64(oocnmf_ctx* ctx, const double* w_slab /* rows x k */,
                           const double* h /* k x n */);
int oocnmf_get_factors_f64(oocnmf_ctx* ctx, double* w_slab, double* h);
/* Gather every rank's W slab into w_full (m x k) on every rank (ncclAllGather). */
int oocnmf_gather_w_f64(oocnmf_ctx* ctx, double* w_full);

/* ----- solve: the MU loop (src/nmf_serial.cpp:83-117 / src/nmf_distributed.cpp:239-262).
 * Collective across ranks of a communicator context. Writes up to trace_cap
 * (iteration, relative error) pairs. */
int oocnmf_solve(oocnmf_ctx* ctx, const oocnmf_config* cfg, uint64_t* trace_iter,
                 double* trace_err, uint64_t trace_cap, oocnmf_info* info);

/* Diagnostics for parity tests: with the current factors, compute A·H^T (rows x k) and
 * the rank-local A^T·W (k x n), H H^T and W^T W (k x k) without updating anything. */
int oocnmf_products_f64(oocnmf_ctx* ctx, double* aht, double* wta, double* hht, double* wtw);
/* Squared Frobenius norm of the resident A slab (f64 accumulation). */
int oocnmf_sq_norm(oocnmf_ctx* ctx, double* out);

/* ----- model selection (NMFk), the consumer of the MU path -----
 * replaces select_k / cluster_columns / silhouette / pearson_correlation_matrix /
 * perturb_dense / perturb_sparse (include/oocnmf/model_selection.hpp:14-84,
 * src/model_selection.cpp:35-406). */

/* Mirrors SelectionConfig (model_selection.hpp:15-24). nmf.k and nmf.seed are overridden per
 * run (k swept, seed = derive_seed(seed, k, 2p + 1 + attempt * 1000003)). */
typedef struct {
    uint64_t k_min, k_max;
    uint64_t n_perturbations; /* P, default 16 */
    double delta;             /* default 0.03, in (0, 1) */
    double sil_threshold;     /* default 0.75, in [-1, 1] */
    oocnmf_config nmf;        /* per-run template */
    uint64_t seed;
} oocnmf_selection_config;

/* Mirrors KRecord (model_selection.hpp:27-35); the medians matrix is returned separately. */
typedef struct {
    uint64_t k;
    int32_t valid;            /* at least two runs survived */
    int32_t reserved;
    uint64_t runs_used;
    double min_silhouette, mean_silhouette, mean_relative_error;
    uint64_t iterations;      /* B200 extension: MU iterations run for this k, all ranks */
} oocnmf_k_record;

/* Change k keeping the resident A (re-allocates the factors). */
int oocnmf_set_rank(oocnmf_ctx* ctx, uint64_t k);
/* perturb_dense / perturb_sparse on the resident A: A <- A0 o (1 - delta + 2 delta U) with
 * U = CounterRng(seed, 21).uniform(i * n + j) over stored entries (model_selection.cpp:35-60),
 * A0 the values loaded last (kept on the device on first use; delta = 0 restores them). */
int oocnmf_perturb(oocnmf_ctx* ctx, double delta, uint64_t seed);
/* Replica mode on a communicator context: solves run rank-locally (every rank holds its own
 * full A), no collective inside oocnmf_solve. */
int oocnmf_set_local(oocnmf_ctx* ctx, int local);
/* Sum a host f64 buffer over the ranks of a communicator context (NCCL, in place). */
int oocnmf_allreduce_sum_f64(oocnmf_ctx* ctx, double* buf, uint64_t count);

/* ---- collectives of the group (reference CommHandle, include/oocnmf/comm.hpp:48-67) ----
 * tag: PhaseTag (comm.hpp:13-20): 0 generic, 1 w_update, 2 h_update, 3 error_check, 4 gather,
 * 5 barrier. All are collective (every rank calls them) and blocking. */
int oocnmf_allreduce_f64(oocnmf_ctx* ctx, double* buf, uint64_t count, int tag);  /* all_reduce_sum */
int oocnmf_barrier(oocnmf_ctx* ctx);                                              /* barrier */
/* CollectiveStats (comm.hpp:28-43): per tag bytes, calls, seconds (device time of the
 * collectives, the solve's own included); any pointer may be null. */
int oocnmf_comm_stats(oocnmf_ctx* ctx, uint64_t bytes[6], uint64_t calls[6], double seconds[6]);
int oocnmf_comm_reset_stats(oocnmf_ctx* ctx);
/* Failure semantics (src/comm.cpp:89-111: 60 s timeout, then the group is poisoned): a host
 * wait that sees no collective complete for `seconds` (or an NCCL async error) aborts the
 * communicator (ncclCommAbort) and returns OOCNMF_ERR_COMM; every later collective on the
 * context fails with OOCNMF_ERR_COMM. Default 60 s. */
int oocnmf_set_comm_timeout(oocnmf_ctx* ctx, double seconds);
/* spawn_group(n, Backend::threads) (comm.hpp:80-82): n contexts of one process on
 * devices[0..n) (distinct), one NCCL communicator clique (ncclCommInitAll); each context is
 * then driven by its own host thread (run_distributed_threads, nmf_distributed.hpp:40). */
int oocnmf_ctx_create_group(int n, const int* devices, oocnmf_ctx** out);
/* select_k (model_selection.cpp:316-406) on the full A resident in ctx (row0 = 0, rows = m):
 * P perturbed MU runs per k on the GPU, then cluster_columns / silhouette / selection rule on
 * the host. On a communicator context the runs of each k are spread over the ranks as
 * replicas (each rank must hold the full A) and the W factors are summed into every rank with
 * one NCCL all-reduce per k, so every rank returns the same report.
 * records: cap >= k_max - k_min + 1 entries. medians (optional): sum over k of m * k doubles,
 * k ascending, each m x k row-major. chosen_k: -1 if no k qualified. rationale: truncated to
 * rationale_cap bytes including the NUL. */
int oocnmf_select_k(oocnmf_ctx* ctx, const oocnmf_selection_config* cfg, oocnmf_k_record* records,
                    uint64_t cap, double* medians, int64_t* chosen_k, char* rationale,
                    uint64_t rationale_cap);
/* Host-side (no device): cluster_columns + silhouette (model_selection.cpp:163-281) over W
 * factors runs[r] (m x k row-major, r < nruns, nruns >= 2). Outputs medians (m x k),
 * per_cluster (k), the min / mean silhouette, the dropped zero-norm columns and, optionally,
 * member_cluster[r * k + c] = cluster of column c of run r (-1: dropped or unmatched). */
int oocnmf_cluster_silhouette(const double* runs, uint64_t nruns, uint64_t m, uint64_t k, double* medians,
                              double* per_cluster, double* min_sil, double* mean_sil, uint64_t* dropped,
                              int64_t* member_cluster);
/* pearson_correlation_matrix (model_selection.cpp:283-314): corr (k1 x k2), host-side. */
int oocnmf_pearson_correlation(const double* w_true, uint64_t m, uint64_t k1, const double* w_est,
                               uint64_t k2, double* corr);

/* ----- memory_estimate (include/oocnmf/partition.hpp:51-64, src/partition.cpp:147-197) -----
 * Per-rank device bytes of THIS backend's layout (f32, padded to 128, tensor-core [F | F_lo]
 * copies, stream-K slots) for the largest slab of a plan, and the row-batch count the
 * out-of-core mode needs to fit budget_bytes. min_n_b = 1: the in-core path fits; > 1:
 * out-of-core with that many row batches (dense RNMF); 0: infeasible. Host-side. */
typedef struct {
    uint64_t a_slab_bytes;       /* A slab resident in HBM (CSR: values + indices, both CSR(A) and CSR(A^T)) */
    uint64_t store_peak_bytes;   /* out-of-core: the two row-batch staging buffers at min_n_b */
    uint64_t factor_bytes;       /* W, H and their tensor-core [F | F_lo] copies */
    uint64_t intermediate_bytes; /* packed W^T A, stream-K slots, Gram / error slots, A·H^T (CSR / CNMF) */
    uint64_t peak_bytes;         /* (a_slab or store_peak) + factors + intermediates */
    uint64_t min_n_b;
    int32_t feasible;
    int32_t in_core;
} oocnmf_memory_report;
/* strategy: 1 = CNMF, 2 = RNMF; density 1 = dense; num_sms 0 = 148 */
int oocnmf_memory_estimate(uint64_t m, uint64_t n, uint64_t k, int n_workers, int strategy, double density,
                           uint64_t budget_bytes, int num_sms, oocnmf_memory_report* out);

/* ----- matrix files (include/oocnmf/io.hpp:28-66, src/io.cpp), host-side -----
 * PDN1: "PDNMF\0v1", u8 kind (0 dense, 1 CSR), u8 dtype, u64 rows, u64 cols, little-endian;
 * dense payload row-major; CSR payload u64 nnz, u64 row_ptr[rows+1], u64 col_idx[nnz], values.
 * dtype 0 = f64 (the reference's only type), 1 = f32 (B200 extension in the reserved byte).
 * Matrix Market: array (column-major) / coordinate, real or integer, general. */
int oocnmf_pdn1_info(const char* path, int32_t* kind, int32_t* dtype, uint64_t* rows, uint64_t* cols,
                     uint64_t* nnz);
/* dense window [r0, r1) x [c0, c1), row-major (Pdn1File::read_dense_window) */
int oocnmf_pdn1_read_dense(const char* path, uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1, double* out);
int oocnmf_pdn1_read_dense_f32(const char* path, uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1,
                               float* out);
/* CSR rows [r0, r1), row_ptr rebased, global column indices (Pdn1File::read_csr_rows) */
int oocnmf_pdn1_csr_rows_nnz(const char* path, uint64_t r0, uint64_t r1, uint64_t* nnz);
int oocnmf_pdn1_read_csr_rows(const char* path, uint64_t r0, uint64_t r1, uint64_t* row_ptr, uint64_t* col_idx,
                              double* vals);
int oocnmf_pdn1_write_dense(const char* path, const double* a, uint64_t rows, uint64_t cols, int32_t dtype);
int oocnmf_pdn1_write_dense_f32(const char* path, const float* a, uint64_t rows, uint64_t cols);
int oocnmf_pdn1_write_csr(const char* path, uint64_t rows, uint64_t cols, const uint64_t* row_ptr,
                          const uint64_t* col_idx, const double* vals, int32_t dtype);
/* kind 0 = array (dense), 1 = coordinate (CSR; repeated cells keep their last value) */
int oocnmf_mtx_info(const char* path, int32_t* kind, uint64_t* rows, uint64_t* cols, uint64_t* nnz);
int oocnmf_mtx_read(const char* path, double* dense_out, uint64_t* row_ptr, uint64_t* col_idx, double* vals);
int oocnmf_mtx_write_dense(const char* path, const double* a, uint64_t rows, uint64_t cols);
int oocnmf_mtx_write_csr(const char* path, uint64_t rows, uint64_t cols, const uint64_t* row_ptr,
                         const uint64_t* col_idx, const double* vals);

/* ----- one-shot drop-ins for nmf_serial(MatrixRef a, const NmfConfig& cfg) on host
 * buffers: upload, solve, download. w0/h0 are used iff cfg->init == 1. */
int oocnmf_nmf_serial_dense_f64(int device, const double* a, uint64_t m, uint64_t n,
                                const oocnmf_config* cfg, const double* w0, const double* h0,
                                double* w_out, double* h_out, uint64_t* trace_iter,
                                double* trace_err, uint64_t trace_cap, oocnmf_info* info);
int oocnmf_nmf_serial_dense_f32(int device, const float* a, uint64_t m, uint64_t n,
                                const oocnmf_config* cfg, const double* w0, const double* h0,
                                double* w_out, double* h_out, uint64_t* trace_iter,
                                double* trace_err, uint64_t trace_cap, oocnmf_info* info);
int oocnmf_nmf_serial_csr_f64(int device, const uint64_t* row_ptr, const uint64_t* col_idx,
                              const double* vals, uint64_t m, uint64_t n,
                              const oocnmf_config* cfg, const double* w0, const double* h0,
                              double* w_out, double* h_out, uint64_t* trace_iter,
                              double* trace_err, uint64_t trace_cap, oocnmf_info* info);

#ifdef __cplusplus
}
#endif
#endif /* OOCNMF_B200_H */
