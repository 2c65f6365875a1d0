// Host-callable launchers for the MU-NMF device kernels (one TU per kernel family).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"

namespace ooc {

// Device layout (per rank): A slab mp x np f32 row-major (zero-padded to multiples of
// 128), W mp x kp, Ht np x kp (H stored transposed so both factors are "tall"), kp in
// {8, 16, 32, 64} (k zero-padded; padding is exact for MU: padded entries stay 0).
// The tensor-core path also keeps W_cat / Ht_cat (rows x 2kp) = [F | F - tf32(F)].
constexpr int kTile = 128;  // rows (pass 1, W update) / columns (pass 2, H update) per tile

// ---- dense streaming passes ----
// Stream-K plans: tiles of 128 rows (pass 1) / 128 columns (pass 2), reduction steps of
// `step` columns / rows (32 for the FFMA kernels, kTcStep for the tensor-core kernels).
constexpr int kFfmaStep = 32, kTcStep = 64;
void plan_aht(StreamK& sk, int64_t mp, int64_t np, int num_sms, int step);
void plan_wta(StreamK& sk, int64_t mp, int64_t np, int num_sms, int step);
// CUDA-core (FFMA) passes, kernels_dense.cu: any kp.
cudaError_t launch_aht(int kp, const float* A, int64_t lda, const float* Ht, float* slots,
                       const StreamK& sk, cudaStream_t s);
cudaError_t launch_wta(int kp, const float* A, int64_t lda, const float* W, float* slots,
                       const StreamK& sk, cudaStream_t s);
// Tensor-core passes, kernels_tc.cu: kp in {32, 64}, 3xTF32 split precision; the factor
// operand is its [F | F_lo] concatenation (rows x 2kp).
bool tc_supported(int kp);
// ldb: row stride of the [F | F_lo] operand in floats (0 = 2 kp; wide factors pass the full
// 2 kp_total with the group's column offset folded into the pointer)
cudaError_t launch_aht_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np,
                          const float* Ht_cat, float* slots, const StreamK& sk, cudaStream_t s, int64_t ldb = 0);
// out_final (optional): the pass reduces its stream-K partials itself (ascending CTA order)
// and writes the np x kp result there; flags: 4 u32 per slot, zero before the launch (the
// kernel leaves them zero again), epoch: the nonzero "published" value.
cudaError_t launch_wta_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np,
                          const float* W_cat, float* slots, const StreamK& sk, cudaStream_t s,
                          float* out_final = nullptr, unsigned* flags = nullptr, unsigned epoch = 0,
                          int64_t ldb = 0);

// ---- one-pass dense MU W-half (kernels_fused.cu): P1 (A·Ht partials), the W update, and
// P2 (W^T A with the new W) in one persistent tcgen05 kernel, A read from HBM once ----
struct FusedArgs {
    int NB, D, NS, G1;     // row blocks, P2 lookahead (blocks), P1 slot ring depth, P1 publishers
    int drain_units;       // P1 chain length (kernels_tc.cu numerics)
    int p2_first;          // unit order of step s: P2(s - D) before P1(s) (else after)
    const int* q0;         // [G + 1] P1 chunk (64 cols) range per CTA
    const int* t0;         // [G + 1] owned W^T A tile (128 cols) range per CTA
    const int* act;        // [G1] CTAs with P1 work, ascending
    float* p1slots;        // [NS][G][128][kp] published P1 partials
    unsigned* count;       // [NB] P1 partials published per block (zero before the launch)
    unsigned* wdone;       // [2 NB] rows of each 64-row half block updated (zero before the launch)
    float* W;              // mp x kp, updated in place
    float* Wcat;           // mp x 2kp [W | W_lo] of the new W
    const float* HHt;      // kp x kp
    float eps;
    int* flag;             // non-finite W entries
    float* wta;            // np x kp: W^T A (transposed) of the new W
    uint64_t pol_p1, pol_p2;  // L2 policies of the A loads of P1 / P2
    uint64_t pol_p1s;         // P1 loads of the streamed (not kept) column tiles
    double* wgram;            // [G][kp * kp] per-CTA W^T W of the new rows (nullptr: not computed)
    int keep_num, keep_den;   // column tile j kept in L2 for P2 iff j % keep_den < keep_num
};
struct FusedPlan {
    int G = 0, NB = 0, NT = 0, NQ = 0, D = 1, NS = 3, G1 = 0;
    std::vector<int> q0, t0, act;
};
bool fused_supported(int kp, int64_t mp, int64_t np, int num_sms);
size_t fused_slot_bytes(int kp, const FusedPlan& fp);  // the P1 slot ring (rows padded to 128 B)
namespace tc {
int tc_drain_units();  // kernels_tc.cu: K steps per TMEM accumulation chain
}
void plan_fused(FusedPlan& fp, int64_t mp, int64_t np, int num_sms, int lookahead);
// L2 policies of the one-pass kernel's A loads (OOCNMF_FUSED_POL / _KEEP, defaults measured best)
void fused_policies(FusedArgs& a);

// kernels_nvls.cu: the sharded H update fused with its reduce-scatter and all-gather over NVLS
// multicast (NCCL >= 2.28 symmetric memory). mc_* are multicast addresses of the symmetric
// buffers, bar / ht this rank's local views.
struct NvlsArgs {
    const float* mc_wp;   // partial W^T A (np x kp), multicast
    float* mc_ht;         // Ht (np x kp), multicast
    unsigned* mc_bar;     // per-CTA barrier counters, multicast
    const unsigned* bar;  // the same counters, local
    const float* ht;      // Ht, local (the old rows)
    const float* wtw;     // kp x kp W^T W (already all-reduced)
    int* flag;
    int64_t row0, rows;   // this rank's rows of H
    unsigned epoch;       // launches so far on this group (the barrier phase)
    int nranks;
    float eps;
    uint64_t timeout_ns;  // barrier spin limit (trap) for a peer that never arrives
};
bool nvls_compiled();
// Symmetric buffers of one group (all ncclMemAlloc'd and registered as NCCL_WIN_COLL_SYMMETRIC
// windows on every rank) and the device communicator with the lsa multicast mapping.
struct NvlsState {
    void* wp = nullptr;   // partial W^T A
    void* ht = nullptr;   // Ht
    void* bar = nullptr;  // barrier counters
    size_t wp_bytes = 0, ht_bytes = 0, bar_bytes = 0;
    void* win[3] = {};       // ncclWindow_t of wp, ht, bar
    void* devcomm = nullptr; // ncclDevComm (heap)
    void* mc[3] = {};        // multicast base addresses of wp, ht, bar
    unsigned epoch = 0;
};
// Collective over comm (every rank, same sizes): allocate, zero, register, create the device
// communicator, resolve the multicast addresses. On failure returns false with *why set and
// leaves nothing allocated.
bool nvls_setup(NvlsState& st, ncclComm_t comm, size_t wp_bytes, size_t ht_bytes, int nbar, cudaStream_t s,
                std::string* why);
void nvls_teardown(NvlsState& st, ncclComm_t comm);  // collective
cudaError_t launch_h_update_nvls(int kp, const NvlsArgs& a, int grid, cudaStream_t s);
cudaError_t launch_mu_fused(int kp, const FusedPlan& fp, const float* A, int64_t mp, int64_t np, const float* Ht_cat,
                            const FusedArgs& args, cudaStream_t s);

// ---- factor kernels (kernels_factor.cu) ----
// F (rows x kp, rows a multiple of 128) <- F * N / (F G + eps) rowwise, where N is either
// a plain rows x kp matrix (n_plain) or stream-K partials (n_slots, sk). Emits per-CTA
// partial Gram F_new^T F_new in f64 (gram_slots[gridDim][kp*kp]), per-CTA f64 partial
// sum(N .* F_new) (err_slots, may be null) and sets *flag on non-finite output.
// update == false: only emit the Gram of F (no update). cat_out (may be null) receives the
// rows of [F | F - tf32(F)] (rows x 2kp) for the tensor-core passes.
int factor_grid(int64_t tiles);
cudaError_t launch_factor_update(int kp, float* F, int64_t rows, const float* n_plain,
                                 const float* n_slots, const StreamK* sk, const float* G,
                                 float eps, bool update, double* gram_slots, double* err_slots,
                                 int* flag, float* cat_out, cudaStream_t s);
// out[e] = sum_s slots[s*E + e] in f64 (fixed order), E = count; written as f32 (out32) and,
// if out64 != null, f64.
cudaError_t launch_reduce_slots(const double* slots, int64_t nslots, int64_t count, float* out32,
                                double* out64, cudaStream_t s);
// out (tiles*128 x kp) <- [out +] sum of each tile's stream-K partials (ascending CTA order).
cudaError_t launch_streamk_reduce(int kp, const float* slots, const StreamK& sk, float* out,
                                  bool accumulate, cudaStream_t s);
// trace slot <- sqrt(max(0, nA2 - 2 sum(err_slots) + <WtW, HHt>)) / sqrt(nA2)   (f64)
// Predication (no host round trip): if pred_in is set and *pred_in == 0 the kernel does
// nothing; if pred_out is set it receives (err < threshold).
cudaError_t launch_finalize_error(int kp, const double* err_slots, int64_t n_err,
                                  const double* wtw, const double* hht, const double* norm_a2,
                                  const double* direct_res /* null = trace form */,
                                  double* out_err, cudaStream_t s, const int* pred_in = nullptr,
                                  int* pred_out = nullptr, double threshold = 0.0);

// ---- setup kernels (kernels_setup.cu) ----
cudaError_t launch_gen_dense_uniform(float* A, int64_t lda, int64_t rows, int64_t cols,
                                     int64_t row0, int64_t n_global, uint64_t seed,
                                     uint64_t stream, cudaStream_t s);
// W rows [row0, row0 + rows) and H columns [col0, col0 + n) of n_global (Ht, n x kp)
cudaError_t launch_init_factors(float* W, float* Ht, int kp, int64_t k, int64_t rows,
                                int64_t row0, int64_t n, int64_t n_global, int64_t col0, uint64_t seed,
                                cudaStream_t s);
// out(r, c) = in(r, c) over an R x C block with element strides (is_*, os_*), casting the type.
enum class CastKind { f32_f64, f64_f32, i32_u64 };
cudaError_t launch_strided_cast(CastKind kind, const void* in, int64_t is_r, int64_t is_c, void* out, int64_t os_r,
                                int64_t os_c, int64_t R, int64_t C, cudaStream_t s);
cudaError_t launch_cast_pad_f64(const double* src, int64_t ld_src, int64_t rows, int64_t cols,
                                float* dst, int64_t ld_dst, cudaStream_t s);
// Partial f64 sums of squares of A (dense, padded) -> out_slots[sqnorm_grid()].
int sqnorm_grid();
cudaError_t launch_sq_norm_dense(const float* A, int64_t lda, int64_t rows, int64_t cols,
                                 double* out_slots, cudaStream_t s);
cudaError_t launch_sq_norm_vals(const float* v, int64_t nnz, double* out_slots, cudaStream_t s);
cudaError_t launch_reduce_f64(const double* slots, int64_t n, double* out, cudaStream_t s);
// Direct residual sum((A - W Ht^T)^2) partials for the rows x cols window (f64).
cudaError_t launch_residual_dense(int kp, const float* A, int64_t lda, int64_t rows,
                                  int64_t cols, const float* W, const float* Ht,
                                  double* out_slots, cudaStream_t s, const int* pred = nullptr);
cudaError_t launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t s);
// Model-selection perturbation of the resident A (dense window, or CSR values; transposed:
// the CSR(A^T) copy), out = f32(in * (1 - delta + 2 delta U(seed, 21, i * n + j))).
cudaError_t launch_perturb_dense(const float* in, float* out, int64_t lda, int64_t rows, int64_t cols,
                                 int64_t row0, int64_t n, uint64_t seed, double delta, cudaStream_t s);
cudaError_t launch_perturb_csr(const float* in, float* out, const int64_t* rp, const int32_t* ci, int64_t rows,
                               int64_t row0, int64_t n, uint64_t seed, double delta, bool transposed,
                               cudaStream_t s);
// cat (rows x 2kp) <- [F | F - tf32_trunc(F)] for F (rows x kp)
cudaError_t launch_split_cat(const float* F, float* cat, int64_t rows, int kp, cudaStream_t s);

// ---- k > 64 (kernels_wide.cu): kp a multiple of 64 up to kMaxWideKp; the contractions run
// per 64-column group on the kp = 64 passes, factor operands group-interleaved [F_g | F_lo_g] ----
constexpr int kMaxWideKp = 512;
// gram / err slots: nslots (= factor_grid(rows / kTile), the count the caller reduces)
cudaError_t launch_factor_update_wide(int kp, float* F, int64_t rows, const float* n_plain, const float* G, float eps,
                                      bool update, double* gram_slots, int nslots, double* err_slots, int* flag,
                                      float* cat_out, cudaStream_t s);
cudaError_t launch_spmm_wide(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows, const float* B,
                             float* out, cudaStream_t s);
cudaError_t launch_residual_dense_wide(int kp, const float* A, int64_t lda, int64_t rows, int64_t cols, const float* W,
                                       const float* Ht, double* out_slots, int nslots, cudaStream_t s, const int* pred);
cudaError_t launch_cross_csr_wide(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                                  const float* W, const float* Ht, double* out_slots, int nslots, cudaStream_t s,
                                  const int* pred);
// a kp = 64 pass's stream-K partials -> a 64-column group of a wider output (row stride ldo)
cudaError_t launch_streamk_reduce_ld(const float* slots, const StreamK& sk, float* out, int64_t ldo, bool accumulate,
                                     cudaStream_t s);

// ---- CSR kernels (kernels_sparse.cu) ----
// out (rows x kp) = CSR(rp, ci, v) · B (B rows indexed by column, kp wide).
cudaError_t launch_spmm(int kp, const int64_t* rp, const int32_t* ci, const float* v,
                        int64_t rows, const float* B, float* out, cudaStream_t s);
// Column chunks of a CSR with column-sorted rows: seg[c * rows + i] = first entry of row i
// with column >= c * chunk_cols (c = 0..C); chunk c of row i is [seg[c][i], seg[c+1][i]).
cudaError_t launch_csr_segments(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t chunk_cols, int C,
                                int64_t* seg, cudaStream_t s);
// out (rows x kp) = (or +=, accumulate) the chunk [lo[i], hi[i]) of each row of a CSR · B.
cudaError_t launch_spmm_seg(int kp, const int64_t* lo, const int64_t* hi, const int32_t* ci, const float* v,
                            int64_t rows, const float* B, float* out, bool accumulate, cudaStream_t s);
// F[row] <- F * (CSR · B)[row] * rcp_rn(F[row] · G + eps) for rows [0, rows): the SpMM fused with
// the MU update of the same rows (non-finite results set *flag). The Gram of the new F is left
// to launch_factor_update(update = false).
cudaError_t launch_spmm_mu(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                           const float* B, float* F, const float* G, float eps, int* flag, cudaStream_t s);
cudaError_t launch_residual_csr(int kp, const int64_t* rp, const int32_t* ci, const float* v,
                                int64_t rows, int64_t cols, const float* W, const float* Ht,
                                double* out_slots, cudaStream_t s,
                                const int* pred = nullptr);
// Transpose a CSR (rows x cols) into CSR^T (cols x rows), entries of each output row in
// ascending source-row order (deterministic). Scratch allocated internally.
cudaError_t csr_transpose(const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                          int64_t cols, int64_t nnz, int64_t* rpT, int32_t* ciT, float* vT,
                          cudaStream_t s);
// Reference-semantics generator: counts per row, then fill (row_ptr must be scanned between).
cudaError_t launch_gen_csr_count(int64_t rows, int64_t row0, int64_t n, uint64_t thresh,
                                 uint64_t seed, int64_t* counts, cudaStream_t s);
cudaError_t launch_gen_csr_fill(int64_t rows, int64_t row0, int64_t n, uint64_t thresh,
                                uint64_t seed, const int64_t* rp, int32_t* ci, float* v,
                                cudaStream_t s);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
// CSR upload: narrow a chunk of reference-format entries (u64 column, f64 value) to the device
// layout, flagging columns >= n; then check the row structure of the whole upload.
constexpr unsigned kCsrBadRowPtr = 1u, kCsrBadColumn = 2u, kCsrBadOrder = 4u;
cudaError_t launch_csr_ingest(const uint64_t* ci_in, const double* v_in, int64_t count, uint64_t n,
                              int32_t* ci, float* v, unsigned* bad, cudaStream_t s);
cudaError_t launch_csr_check_rows(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t nnz,
                                  unsigned* bad, cudaStream_t s);

}  // namespace ooc
