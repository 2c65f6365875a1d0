// Kernels for k > 64 ("wide" factors, kp a multiple of 64 up to kMaxWideKp): the reference
// accepts any k (include/oocnmf/nmf.hpp:15-27) and the paper's scaling study runs k = 128 and
// 256. The streaming contractions run on the kp = 64 tensor-core passes, once
// per 64-column group of the factor (solver.cu pass1 / pass2, [F_g | F_lo_g] group-interleaved
// operand layout); these kernels are the pieces whose width the kp <= 64 kernels hard-wire:
//   k_factor_update_wide   F <- F * N / (F G + eps) (plain numerator), the trace-form partial
//                          sum(N .* F_new), the NaN flag and the [F | F_lo] group-interleaved copy
//   k_gram_wide            per-slot partial F^T F (f64, upper 64 x 64 tiles, mirrored on read)
//   k_spmm_wide            CSR · B, one warp per row
//   k_residual_dense_wide  f64 sum((A - W Ht^T)^2) of the dense window
//   k_cross_csr_wide       f64 sum_nz a_ij (W_i · Ht_j)
//   k_streamk_reduce_ld    a kp = 64 pass's stream-K partials into a 64-column group of a wider
//                          output (row stride ldo)
// They are CUDA-core kernels: at k >= 128 the contractions dominate (4 m n k flop per
// iteration) and run on the tensor cores; these touch only the factors (rows x kp).
#include "kernels.h"

namespace ooc {
namespace {

constexpr int kWideRows = 8;  // factor rows per CTA in the update kernel

// One CTA of 256 threads per kWideRows rows; thread t owns columns t, t + 256, ... of every row.
__global__ void __launch_bounds__(256) k_factor_update_wide(float* __restrict__ F, int64_t rows, int kp,
                                                             const float* __restrict__ N,
                                                             const float* __restrict__ G, float eps,
                                                             double* __restrict__ err_slots,
                                                             int* __restrict__ flag, float* __restrict__ cat) {
    extern __shared__ float fs[];  // kWideRows x kp rows of F
    __shared__ double red[256];
    double eacc = 0.0;
    bool bad = false;
    const int ngroups_total = int((rows + kWideRows - 1) / kWideRows);
    for (int64_t blk = blockIdx.x; blk < ngroups_total; blk += gridDim.x) {
        const int64_t r0 = blk * kWideRows;
        const int nr = int(rows - r0 < kWideRows ? rows - r0 : kWideRows);
        for (int e = threadIdx.x; e < nr * kp; e += blockDim.x) fs[e] = F[r0 * kp + e];
        __syncthreads();
        float e32 = 0.f;
        for (int j = threadIdx.x; j < kp; j += blockDim.x) {
            float de[kWideRows];
#pragma unroll
            for (int r = 0; r < kWideRows; ++r) de[r] = 0.f;
            for (int q = 0; q < kp; ++q) {
                const float g = __ldg(G + int64_t(q) * kp + j);
#pragma unroll
                for (int r = 0; r < kWideRows; ++r) de[r] = fmaf(fs[r * kp + q], g, de[r]);
            }
#pragma unroll
            for (int r = 0; r < kWideRows; ++r) {
                if (r >= nr) break;
                const int64_t at = (r0 + r) * kp + j;
                const float nu = N[at];
                // t * nu / (de + eps) as (t * nu) * rcp_rn(de + eps), as kernels_factor.cu
                const float fn = (fs[r * kp + j] * nu) * __frcp_rn(de[r] + eps);
                bad |= !isfinite(fn);
                e32 = fmaf(nu, fn, e32);
                F[at] = fn;
                if (cat) {
                    float* cw = cat + (r0 + r) * 2 * kp + 128 * (j >> 6) + (j & 63);
                    cw[0] = fn;
                    cw[64] = tf32_lo(fn);
                }
            }
        }
        eacc += double(e32);
        __syncthreads();
    }
    if (err_slots) {
        red[threadIdx.x] = eacc;
        __syncthreads();
        for (int st = 128; st > 0; st >>= 1) {
            if (int(threadIdx.x) < st) red[threadIdx.x] += red[threadIdx.x + st];
            __syncthreads();
        }
        if (threadIdx.x == 0) err_slots[blockIdx.x] = red[0];  // (grid == nslots)
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Partial Gram of a row range into slot blockIdx.x (kp x kp f64): the CTA walks its rows in
// chunks of 32 staged in shared memory; thread (ti, tj) of a 16 x 16 grid accumulates the 4 x 4
// micro-tile (4 ti + a, 4 tj + b) of every upper 64 x 64 tile (I <= J) in f32 per chunk, then
// in f64; lower tiles are mirrored from the upper ones (bitwise symmetric, as the reference's
// gram_t, src/kernels.cpp:127-147).
__global__ void __launch_bounds__(256) k_gram_wide(const float* __restrict__ F, int64_t rows, int kp,
                                                    double* __restrict__ slots, int nslots) {
    extern __shared__ float fs[];  // 32 x kp
    const int nt = kp / 64;
    const int ti = threadIdx.x / 16, tj = threadIdx.x % 16;
    const int64_t per = (rows + nslots - 1) / nslots;
    const int64_t ra = int64_t(blockIdx.x) * per, rb = ra + per < rows ? ra + per : rows;
    double* out = slots + int64_t(blockIdx.x) * kp * kp;
    for (int I = 0; I < nt; ++I)
        for (int J = I; J < nt; ++J) {
            double acc[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = 0.0;
            for (int64_t c0 = ra; c0 < rb; c0 += 32) {
                const int nr = int(rb - c0 < 32 ? rb - c0 : 32);
                __syncthreads();
                for (int e = threadIdx.x; e < nr * kp; e += blockDim.x) fs[e] = F[c0 * kp + e];
                __syncthreads();
                float a32[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) a32[e] = 0.f;
                for (int r = 0; r < nr; ++r) {
                    float x[4], y[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) x[a] = fs[r * kp + 64 * I + 4 * ti + a], y[a] = fs[r * kp + 64 * J + 4 * tj + a];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) a32[a * 4 + b] = fmaf(x[a], y[b], a32[a * 4 + b]);
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[e] += double(a32[e]);
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int i = 64 * I + 4 * ti + a, j = 64 * J + 4 * tj + b;
                    out[int64_t(i) * kp + j] = acc[a * 4 + b];
                    if (I != J) out[int64_t(j) * kp + i] = acc[a * 4 + b];
                }
        }
    // diagonal tiles: make the tile itself bitwise symmetric (upper triangle wins)
    __syncthreads();
    for (int I = 0; I < nt; ++I)
        for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
            const int i = 64 * I + e / 64, j = 64 * I + e % 64;
            if (j < i) out[int64_t(i) * kp + j] = out[int64_t(j) * kp + i];
        }
}

// out (rows x kp) = CSR · B (B rows of width kp); one warp per row, lane owns kp / 32 columns
__global__ void __launch_bounds__(256) k_spmm_wide(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                    const float* __restrict__ v, int64_t rows,
                                                    const float* __restrict__ B, int kp, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int per = kp / 32;  // 2 .. 16
    for (int64_t r = warp0; r < rows; r += nw) {
        float acc[16];
        for (int q = 0; q < per; ++q) acc[q] = 0.f;
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
            const float a = v[p];
            const float* b = B + int64_t(ci[p]) * kp + lane;
            for (int q = 0; q < per; ++q) acc[q] = fmaf(a, __ldg(b + 32 * q), acc[q]);
        }
        for (int q = 0; q < per; ++q) out[r * kp + lane + 32 * q] = acc[q];
    }
}

// f64 partial sums of (A_ij - W_i · Ht_j)^2; one warp per (row, 32-column strip)
__global__ void __launch_bounds__(256) k_residual_dense_wide(const float* __restrict__ A, int64_t lda, int64_t rows,
                                                              int64_t cols, const float* __restrict__ W,
                                                              const float* __restrict__ Ht, int kp,
                                                              double* __restrict__ out_slots, const int* pred) {
    __shared__ double red[256];
    if (pred && *pred == 0) return;
    double acc = 0.0;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = tid; e < rows * cols; e += nth) {
        const int64_t i = e / cols, j = e % cols;
        const float* w = W + i * kp;
        const float* h = Ht + j * kp;
        float d = 0.f;
        for (int q = 0; q < kp; ++q) d = fmaf(__ldg(w + q), __ldg(h + q), d);
        const double r = double(A[i * lda + j]) - double(d);
        acc += r * r;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (int(threadIdx.x) < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) out_slots[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k_cross_csr_wide(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                         const float* __restrict__ v, int64_t rows,
                                                         const float* __restrict__ W, const float* __restrict__ Ht,
                                                         int kp, double* __restrict__ out_slots, const int* pred) {
    __shared__ double red[256];
    if (pred && *pred == 0) return;
    double acc = 0.0;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < rows; i += nth)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const float* w = W + i * kp;
            const float* h = Ht + int64_t(ci[p]) * kp;
            float d = 0.f;
            for (int q = 0; q < kp; ++q) d = fmaf(__ldg(w + q), __ldg(h + q), d);
            acc += double(v[p]) * double(d);
        }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (int(threadIdx.x) < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) out_slots[blockIdx.x] = red[0];
}

// stream-K partials of a kp = 64 pass -> columns [0, 64) of out rows (row stride ldo)
__global__ void k_streamk_reduce_ld(const float* __restrict__ slots, StreamK sk, float* __restrict__ out,
                                    int64_t ldo, int accumulate) {
    const int64_t t = blockIdx.x;
    const int64_t c0 = sk.cta_of(t * sk.ipt), c1 = sk.cta_of((t + 1) * sk.ipt - 1);
    for (int q = threadIdx.x; q < kTile * 64; q += blockDim.x) {
        const int r = q / 64, j = q % 64;
        float* o = out + (t * kTile + r) * ldo + j;
        float s = accumulate ? *o : 0.f;
        for (int64_t c = c0; c <= c1; ++c) s += slots[sk.slot(c, t) * int64_t(kTile * 64) + q];
        *o = s;
    }
}

int wide_grid() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms * 4;
}

}  // namespace

cudaError_t launch_factor_update_wide(int kp, float* F, int64_t rows, const float* n_plain, const float* G, float eps,
                                      bool update, double* gram_slots, int nslots, double* err_slots, int* flag,
                                      float* cat_out, cudaStream_t s) {
    if (kp % 64 || kp > kMaxWideKp) return cudaErrorInvalidValue;
    if (update) {
        if (!n_plain) return cudaErrorInvalidValue;
        const int grid = nslots;  // one err slot per CTA, the slot count the caller reduces
        const size_t smem = size_t(kWideRows) * kp * 4;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_factor_update_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_factor_update_wide<<<grid, 256, smem, s>>>(F, rows, kp, n_plain, G, eps, err_slots, flag, cat_out);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    } else if (cat_out) {
        cudaError_t e = launch_split_cat(F, cat_out, rows, kp, s);
        if (e != cudaSuccess) return e;
    }
    if (gram_slots) {
        const size_t smem = size_t(32) * kp * 4;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_gram_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_gram_wide<<<nslots, 256, smem, s>>>(F, rows, kp, gram_slots, nslots);
    }
    return cudaGetLastError();
}

cudaError_t launch_spmm_wide(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows, const float* B,
                             float* out, cudaStream_t s) {
    if (kp % 64 || kp > kMaxWideKp) return cudaErrorInvalidValue;
    const int64_t warps = rows, blocks = (warps * 32 + 255) / 256;
    k_spmm_wide<<<unsigned(blocks < wide_grid() ? blocks : wide_grid()), 256, 0, s>>>(rp, ci, v, rows, B, kp, out);
    return cudaGetLastError();
}

cudaError_t launch_residual_dense_wide(int kp, const float* A, int64_t lda, int64_t rows, int64_t cols, const float* W,
                                       const float* Ht, double* out_slots, int nslots, cudaStream_t s, const int* pred) {
    k_residual_dense_wide<<<nslots, 256, 0, s>>>(A, lda, rows, cols, W, Ht, kp, out_slots, pred);
    return cudaGetLastError();
}

cudaError_t launch_cross_csr_wide(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                                  const float* W, const float* Ht, double* out_slots, int nslots, cudaStream_t s,
                                  const int* pred) {
    k_cross_csr_wide<<<nslots, 256, 0, s>>>(rp, ci, v, rows, W, Ht, kp, out_slots, pred);
    return cudaGetLastError();
}

cudaError_t launch_streamk_reduce_ld(const float* slots, const StreamK& sk, float* out, int64_t ldo, bool accumulate,
                                     cudaStream_t s) {
    k_streamk_reduce_ld<<<unsigned(sk.tiles), 256, 0, s>>>(slots, sk, out, ldo, accumulate ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace ooc
