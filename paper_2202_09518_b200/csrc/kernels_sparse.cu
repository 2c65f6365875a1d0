// CSR path of the MU iteration (config 3: sparse synthetic A).
//
//   A·H^T   CSR SpMM, one row per (sub)warp, lanes span the kp outputs so each nonzero
//           gathers one contiguous kp-wide row of Ht (reference: matmul_acc CSR,
//           src/kernels.cpp:46-67)
//   A^T·W   the reference scatters a_ij·W[i,:] into column j serially
//           (src/kernels.cpp:102-124). A is iteration-invariant, so we build CSR(A^T)
//           once (stable radix sort by column => deterministic order) and run the same
//           gather SpMM on it: no atomics, no scatter.
//   generator  reference semantics of gen_sparse_random (src/synth.cpp:60-86) on device.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace ooc {
namespace {

template <int KP>
__global__ void __launch_bounds__(256) k_spmm(const int64_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci,
                                              const float* __restrict__ v, int64_t rows,
                                              const float* __restrict__ B, float* __restrict__ out) {
    constexpr int LPR = KP < 32 ? KP : 32;  // lanes per row
    constexpr int VEC = KP / LPR;           // outputs per lane
    constexpr int RPW = 32 / LPR;           // rows per warp
    const int lane = threadIdx.x & 31, sub = lane / LPR, l = lane % LPR;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wg = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wg * RPW < rows; wg += warps) {
        const int64_t row = wg * RPW + sub;
        const bool live = row < rows;
        const int64_t beg = live ? rp[row] : 0, end = live ? rp[row + 1] : 0;
        float acc[VEC];
#pragma unroll
        for (int t = 0; t < VEC; ++t) acc[t] = 0.f;
        for (int64_t p0 = beg; __any_sync(0xffffffffu, p0 < end); p0 += LPR) {
            const int64_t p = p0 + l;
            const int col = p < end ? ci[p] : 0;
            const float val = p < end ? v[p] : 0.f;
#pragma unroll
            for (int t = 0; t < LPR; ++t) {
                const int c = __shfl_sync(0xffffffffu, col, sub * LPR + t);
                const float w = __shfl_sync(0xffffffffu, val, sub * LPR + t);
                if (p0 + t < end) {
                    if constexpr (VEC == 1) {
                        acc[0] = fmaf(w, B[int64_t(c) * KP + l], acc[0]);
                    } else {
                        const float2 b = reinterpret_cast<const float2*>(B + int64_t(c) * KP)[l];
                        acc[0] = fmaf(w, b.x, acc[0]);
                        acc[1] = fmaf(w, b.y, acc[1]);
                    }
                }
            }
        }
        if (live) {
            if constexpr (VEC == 1)
                out[row * KP + l] = acc[0];
            else
                reinterpret_cast<float2*>(out + row * KP)[l] = make_float2(acc[0], acc[1]);
        }
    }
}

// Vectorised variant: each lane owns 4 consecutive outputs (one float4 of the factor row), so
// a warp covers 128 / kp rows at once (kp = 32: 8 lanes per row, 4 rows per warp) — four times
// the independent gathers in flight per warp and a quarter of the load instructions of the
// one-float-per-lane kernel.
template <int KP>
__global__ void __launch_bounds__(256) k_spmm_v4(const int64_t* __restrict__ rp,
                                                 const int32_t* __restrict__ ci,
                                                 const float* __restrict__ v, int64_t rows,
                                                 const float* __restrict__ B, float* __restrict__ out) {
    constexpr int LPR = KP / 4;    // lanes per row
    constexpr int RPW = 32 / LPR;  // rows per warp
    const int lane = threadIdx.x & 31, sub = lane / LPR, l = lane % LPR;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wg = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wg * RPW < rows; wg += warps) {
        const int64_t row = wg * RPW + sub;
        const bool live = row < rows;
        const int64_t beg = live ? rp[row] : 0, end = live ? rp[row + 1] : 0;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p0 = beg; __any_sync(0xffffffffu, p0 < end); p0 += LPR) {
            const int64_t p = p0 + l;
            const int col = p < end ? ci[p] : 0;
            const float val = p < end ? v[p] : 0.f;
#pragma unroll
            for (int t = 0; t < LPR; ++t) {
                const int c = __shfl_sync(0xffffffffu, col, sub * LPR + t);
                const float w = __shfl_sync(0xffffffffu, val, sub * LPR + t);
                if (p0 + t < end) {
                    const float4 b = __ldg(reinterpret_cast<const float4*>(B + int64_t(c) * KP) + l);
                    acc.x = fmaf(w, b.x, acc.x);
                    acc.y = fmaf(w, b.y, acc.y);
                    acc.z = fmaf(w, b.z, acc.z);
                    acc.w = fmaf(w, b.w, acc.w);
                }
            }
        }
        if (live) reinterpret_cast<float4*>(out + row * KP)[l] = acc;
    }
}

// ---------------------------------------------------------------------------- column chunks
// A uniformly sparse A gathers a random kp-wide row of B per nonzero: 42 gathers per B row at
// config 3, each a DRAM read because B (512 MB) is four times the L2. Splitting the columns
// into chunks whose B slice fits in L2 and running one pass per chunk turns those gathers
// into L2 hits: B is read from DRAM once, the A entries once, and the price is the f32
// output accumulated across the chunk passes (read + write per chunk). Rows are sorted by
// column, so chunk c of row i is the contiguous range [seg[c][i], seg[c+1][i]).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ld_hint_f4(const float* a, uint64_t pol) {
    float4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_hint_i32(const int32_t* a, uint64_t pol) {
    int r;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ float ld_hint_f32(const float* a, uint64_t pol) {
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ int64_t ld_hint_i64(const int64_t* a, uint64_t pol) {
    int64_t r;
    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(r) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_hint_f4(float* a, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ float4 ld_plain_hint_f4(const float* a, uint64_t pol) {
    float4 r;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(a), "l"(pol));
    return r;
}

__global__ void k_csr_segments(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t rows,
                               int64_t chunk_cols, int C, int64_t* __restrict__ seg) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
         i += int64_t(gridDim.x) * blockDim.x) {
        int64_t p = rp[i];
        const int64_t e = rp[i + 1];
        seg[i] = p;
        for (int c = 1; c < C; ++c) {
            const int64_t lim = int64_t(c) * chunk_cols;
            while (p < e && ci[p] < lim) ++p;
            seg[int64_t(c) * rows + i] = p;
        }
        seg[int64_t(C) * rows + i] = e;
    }
}

// k_spmm_v4 over one column chunk: row i's entries [lo[i], hi[i]); B gathers marked
// evict-last (the chunk's slice is what L2 should keep), the streams evict-first.
template <int KP>
__global__ void __launch_bounds__(256) k_spmm_seg(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                                  const int32_t* __restrict__ ci, const float* __restrict__ v,
                                                  int64_t rows, const float* __restrict__ B,
                                                  float* __restrict__ out, int accumulate) {
    constexpr int LPR = KP / 4;    // lanes per row
    constexpr int RPW = 32 / LPR;  // rows per warp
    const int lane = threadIdx.x & 31, sub = lane / LPR, l = lane % LPR;
    const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wg = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wg * RPW < rows; wg += warps) {
        const int64_t row = wg * RPW + sub;
        const bool live = row < rows;
        const int64_t beg = live ? ld_hint_i64(lo + row, stream) : 0, end = live ? ld_hint_i64(hi + row, stream) : 0;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p0 = beg; __any_sync(0xffffffffu, p0 < end); p0 += LPR) {
            const int64_t p = p0 + l;
            const int col = p < end ? ld_hint_i32(ci + p, stream) : 0;
            const float val = p < end ? ld_hint_f32(v + p, stream) : 0.f;
#pragma unroll
            for (int t = 0; t < LPR; ++t) {
                const int c = __shfl_sync(0xffffffffu, col, sub * LPR + t);
                const float w = __shfl_sync(0xffffffffu, val, sub * LPR + t);
                if (p0 + t < end) {
                    const float4 b = ld_hint_f4(B + int64_t(c) * KP + 4 * l, keep);
                    acc.x = fmaf(w, b.x, acc.x);
                    acc.y = fmaf(w, b.y, acc.y);
                    acc.z = fmaf(w, b.z, acc.z);
                    acc.w = fmaf(w, b.w, acc.w);
                }
            }
        }
        if (live) {
            float* o = out + row * KP + 4 * l;
            if (accumulate) {
                const float4 prev = ld_plain_hint_f4(o, stream);
                acc.x += prev.x, acc.y += prev.y, acc.z += prev.z, acc.w += prev.w;
            }
            st_hint_f4(o, acc, stream);
        }
    }
}

__device__ double block_sum256(double v) {
    __shared__ double sh[256];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    return sh[0];
}

// k_spmm_v4 fused with the MU update of the same rows (the W update of a local-numerator CSR
// solve): the row's A·Ht stays in the lane group's registers and becomes the numerator of
// F[row] <- F * nu * rcp_rn(F·G + eps) (kernels_factor.cu's formula and summation order, so
// the result is bit-identical to SpMM + k_factor_update), instead of a 537 MB round trip
// through HBM and a second pass over F. The Gram of the new rows follows in
// k_factor_update's Gram-only mode. Bounded to 48 registers: 5 resident CTAs per SM like the
// plain SpMM (54 registers / 4 CTAs cost 0.1 ms per pass at config 3).
template <int KP>
__global__ void __launch_bounds__(256, 5) k_spmm_mu(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                 const float* __restrict__ v, int64_t rows,
                                                 const float* __restrict__ B, float* __restrict__ F,
                                                 const float* __restrict__ G, float eps, int* __restrict__ flag) {
    constexpr int LPR = KP / 4;    // lanes per row
    constexpr int RPW = 32 / LPR;  // rows per warp
    __shared__ __align__(16) float Gs[KP * KP];
    for (int e = threadIdx.x; e < KP * KP; e += blockDim.x) Gs[e] = G[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, sub = lane / LPR, l = lane % LPR;
    const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    bool bad = false;
    for (int64_t wg = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wg * RPW < rows; wg += warps) {
        const int64_t row = wg * RPW + sub;
        const bool live = row < rows;
        const int64_t beg = live ? rp[row] : 0, end = live ? rp[row + 1] : 0;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t p0 = beg; __any_sync(0xffffffffu, p0 < end); p0 += LPR) {
            const int64_t p = p0 + l;
            const int col = p < end ? ci[p] : 0;
            const float val = p < end ? v[p] : 0.f;
#pragma unroll
            for (int t = 0; t < LPR; ++t) {
                const int c = __shfl_sync(0xffffffffu, col, sub * LPR + t);
                const float w = __shfl_sync(0xffffffffu, val, sub * LPR + t);
                if (p0 + t < end) {
                    const float4 b = __ldg(reinterpret_cast<const float4*>(B + int64_t(c) * KP) + l);
                    acc.x = fmaf(w, b.x, acc.x);
                    acc.y = fmaf(w, b.y, acc.y);
                    acc.z = fmaf(w, b.z, acc.z);
                    acc.w = fmaf(w, b.w, acc.w);
                }
            }
        }
        // the update: lane l owns columns 4l..4l+3 of the row; F[row][q] comes from lane q/4
        float4* frow = reinterpret_cast<float4*>(F + (live ? row : 0) * KP);
        const float4 f = live ? frow[l] : make_float4(0.f, 0.f, 0.f, 0.f);
        float de0 = 0.f, de1 = 0.f, de2 = 0.f, de3 = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < LPR; ++q4) {
            const float fx = __shfl_sync(0xffffffffu, f.x, sub * LPR + q4);
            const float fy = __shfl_sync(0xffffffffu, f.y, sub * LPR + q4);
            const float fz = __shfl_sync(0xffffffffu, f.z, sub * LPR + q4);
            const float fw = __shfl_sync(0xffffffffu, f.w, sub * LPR + q4);
            const float fq[4] = {fx, fy, fz, fw};
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const float4 g = *reinterpret_cast<const float4*>(Gs + (4 * q4 + qq) * KP + 4 * l);
                de0 = fmaf(fq[qq], g.x, de0);
                de1 = fmaf(fq[qq], g.y, de1);
                de2 = fmaf(fq[qq], g.z, de2);
                de3 = fmaf(fq[qq], g.w, de3);
            }
        }
        if (live) {
            float4 nf;
            nf.x = (f.x * acc.x) * __frcp_rn(de0 + eps);
            nf.y = (f.y * acc.y) * __frcp_rn(de1 + eps);
            nf.z = (f.z * acc.z) * __frcp_rn(de2 + eps);
            nf.w = (f.w * acc.w) * __frcp_rn(de3 + eps);
            bad |= !isfinite(nf.x) || !isfinite(nf.y) || !isfinite(nf.z) || !isfinite(nf.w);
            frow[l] = nf;
        }
    }
    if (bad) atomicOr(flag, 1);
}

// sum over nonzeros of a_ij * (W_i · Ht_j)  (f64) — the cross term of ||A - WH||^2.
template <int KP>
__global__ void __launch_bounds__(256) k_cross_csr(const int64_t* __restrict__ rp,
                                                   const int32_t* __restrict__ ci,
                                                   const float* __restrict__ v, int64_t rows,
                                                   const float* __restrict__ W,
                                                   const float* __restrict__ Ht,
                                                   double* __restrict__ out, const int* __restrict__ pred) {
    if (pred && *pred == 0) return;  // device-side predication (error_mode auto)
    double acc = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
         i += int64_t(gridDim.x) * blockDim.x) {
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int64_t j = ci[p];
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < KP; ++q) s = fma(double(W[i * KP + q]), double(Ht[j * KP + q]), s);
            acc += double(v[p]) * s;
        }
    }
    const double s = block_sum256(acc);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void k_row_ids(const int64_t* __restrict__ rp, int64_t rows, int32_t* __restrict__ rid) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
         i += int64_t(gridDim.x) * blockDim.x)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) rid[p] = int32_t(i);
}

__global__ void k_col_hist(const int32_t* __restrict__ ci, int64_t nnz,
                           unsigned long long* __restrict__ cnt) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nnz;
         p += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(cnt + ci[p], 1ull);
}

// (I: the permutation's index type — int64 once nnz exceeds the int32 range)
template <class I>
__global__ void k_gather_t(const I* __restrict__ perm, const int32_t* __restrict__ rid,
                           const float* __restrict__ v, int64_t nnz, int32_t* __restrict__ ciT,
                           float* __restrict__ vT) {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = perm[q];
        ciT[q] = rid[p];
        vT[q] = v[p];
    }
}

template <class I>
__global__ void k_iota(I* x, int64_t n) {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x)
        x[q] = I(q);
}

// Generator: each thread tests kCpt consecutive cells of a row; rows are strided over blocks.
constexpr int kCpt = 16;

__device__ __forceinline__ uint32_t hit_mask(uint64_t km, uint64_t flat0, int64_t j0, int64_t n,
                                             uint64_t thresh) {
    uint32_t m = 0;
#pragma unroll
    for (int t = 0; t < kCpt; ++t)
        if (j0 + t < n && rng_bits53(km, flat0 + t) < thresh) m |= 1u << t;
    return m;
}

__global__ void __launch_bounds__(256) k_gen_csr_count(int64_t rows, int64_t row0, int64_t n,
                                                       uint64_t thresh, uint64_t km,
                                                       int64_t* __restrict__ counts) {
    __shared__ int64_t sh[256];
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        int64_t c = 0;
        const uint64_t base = uint64_t(row0 + i) * uint64_t(n);
        for (int64_t j0 = int64_t(threadIdx.x) * kCpt; j0 < n; j0 += 256 * kCpt)
            c += __popc(hit_mask(km, base + j0, j0, n, thresh));
        sh[threadIdx.x] = c;
        __syncthreads();
        for (int s = 128; s > 0; s >>= 1) {
            if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) counts[i] = sh[0];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_gen_csr_fill(int64_t rows, int64_t row0, int64_t n,
                                                      uint64_t thresh, uint64_t km, uint64_t kv,
                                                      const int64_t* __restrict__ rp,
                                                      int32_t* __restrict__ ci,
                                                      float* __restrict__ v) {
    using Scan = cub::BlockScan<int, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int total_sh;
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        int64_t pos = rp[i];
        const uint64_t base = uint64_t(row0 + i) * uint64_t(n);
        for (int64_t c0 = 0; c0 < n; c0 += 256 * kCpt) {
            const int64_t j0 = c0 + int64_t(threadIdx.x) * kCpt;
            const uint32_t m = j0 < n ? hit_mask(km, base + j0, j0, n, thresh) : 0u;
            int off, total;
            Scan(tmp).ExclusiveSum(int(__popc(m)), off, total);
            uint32_t mm = m;
            int64_t q = pos + off;
            while (mm) {
                const int t = __ffs(mm) - 1;
                mm &= mm - 1;
                ci[q] = int32_t(j0 + t);
                v[q] = __double2float_rn(double(rng_bits53(kv, base + j0 + t)) * 0x1.0p-53);
                ++q;
            }
            if (threadIdx.x == 0) total_sh = total;
            __syncthreads();
            pos += total_sh;
            __syncthreads();
        }
    }
}

unsigned grid_for(int64_t work) {
    const int64_t b = (work + 255) / 256;
    return unsigned(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

}  // namespace

cudaError_t launch_spmm(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                        const float* B, float* out, cudaStream_t s) {
    if (kp > 64) return launch_spmm_wide(kp, rp, ci, v, rows, B, out, s);
    static const int mode = [] {  // OOCNMF_SPMM=1: the one-float-per-lane kernel (developer knob)
        const char* e = std::getenv("OOCNMF_SPMM");
        return e ? std::atoi(e) : 4;
    }();
    if (mode == 4 && kp >= 8) {
        const int64_t warps = (rows * (kp / 4) + 31) / 32;
        const unsigned grid = grid_for(warps * 32);
        switch (kp) {
            case 8: k_spmm_v4<8><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
            case 16: k_spmm_v4<16><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
            case 32: k_spmm_v4<32><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
            case 64: k_spmm_v4<64><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    const int64_t warps = (rows * (kp < 32 ? kp : 32) + 31) / 32;
    const unsigned grid = grid_for(warps * 32);
    switch (kp) {
        case 8: k_spmm<8><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
        case 16: k_spmm<16><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
        case 32: k_spmm<32><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
        case 64: k_spmm<64><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_csr_segments(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t chunk_cols, int C,
                                int64_t* seg, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    k_csr_segments<<<grid_for(rows), 256, 0, s>>>(rp, ci, rows, chunk_cols, C, seg);
    return cudaGetLastError();
}

cudaError_t launch_spmm_seg(int kp, const int64_t* lo, const int64_t* hi, const int32_t* ci, const float* v,
                            int64_t rows, const float* B, float* out, bool accumulate, cudaStream_t s) {
    const int64_t warps = (rows * (kp / 4) + 31) / 32;
    const unsigned grid = grid_for(warps * 32);
    const int acc = accumulate ? 1 : 0;
    switch (kp) {
        case 8: k_spmm_seg<8><<<grid, 256, 0, s>>>(lo, hi, ci, v, rows, B, out, acc); break;
        case 16: k_spmm_seg<16><<<grid, 256, 0, s>>>(lo, hi, ci, v, rows, B, out, acc); break;
        case 32: k_spmm_seg<32><<<grid, 256, 0, s>>>(lo, hi, ci, v, rows, B, out, acc); break;
        case 64: k_spmm_seg<64><<<grid, 256, 0, s>>>(lo, hi, ci, v, rows, B, out, acc); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_spmm_mu(int kp, const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                           const float* B, float* F, const float* G, float eps, int* flag, cudaStream_t s) {
    const int64_t warps = (rows * (kp / 4) + 31) / 32;
    const unsigned grid = grid_for(warps * 32);
    switch (kp) {
        case 8: k_spmm_mu<8><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, F, G, eps, flag); break;
        case 16: k_spmm_mu<16><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, F, G, eps, flag); break;
        case 32: k_spmm_mu<32><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, F, G, eps, flag); break;
        case 64: k_spmm_mu<64><<<grid, 256, 0, s>>>(rp, ci, v, rows, B, F, G, eps, flag); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_residual_csr(int kp, const int64_t* rp, const int32_t* ci, const float* v,
                                int64_t rows, int64_t cols, const float* W, const float* Ht,
                                double* out_slots, cudaStream_t s, const int* pred) {
    (void)cols;
    const unsigned grid = 4 * 148;
    if (kp > 64) return launch_cross_csr_wide(kp, rp, ci, v, rows, W, Ht, out_slots, int(grid), s, pred);
    switch (kp) {
        case 8: k_cross_csr<8><<<grid, 256, 0, s>>>(rp, ci, v, rows, W, Ht, out_slots, pred); break;
        case 16: k_cross_csr<16><<<grid, 256, 0, s>>>(rp, ci, v, rows, W, Ht, out_slots, pred); break;
        case 32: k_cross_csr<32><<<grid, 256, 0, s>>>(rp, ci, v, rows, W, Ht, out_slots, pred); break;
        case 64: k_cross_csr<64><<<grid, 256, 0, s>>>(rp, ci, v, rows, W, Ht, out_slots, pred); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s);
    if (e != cudaSuccess) return e;
    void* tmp = nullptr;
    if ((e = cudaMallocAsync(&tmp, bytes, s)) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, s);
    cudaFreeAsync(tmp, s);
    return e;
}

// Stable radix sort of the entries by column (cub), carrying the entry index: the transpose
// keeps ascending row order inside each column (deterministic CSR(A^T)). The permutation is
// int32 while nnz fits, int64 beyond (a B200 holds A and A^T past 2^31 entries).
template <class I>
cudaError_t csr_transpose_t(const int64_t* rp, const int32_t* ci, const float* v, int64_t rows, int64_t cols,
                            int64_t nnz, int64_t* rpT, int32_t* ciT, float* vT, cudaStream_t s) {
    cudaError_t e;
    int32_t *rid = nullptr, *keys_out = nullptr;
    I *perm_in = nullptr, *perm = nullptr;
    unsigned long long* cnt = nullptr;
    void* tmp = nullptr;
    size_t bytes = 0;
    const int64_t nz = nnz > 0 ? nnz : 1;
#define OOC_TRY(x)                   \
    if ((e = (x)) != cudaSuccess) {  \
        goto done;                   \
    }
    OOC_TRY(cudaMallocAsync(&rid, nz * sizeof(int32_t), s));
    OOC_TRY(cudaMallocAsync(&keys_out, nz * sizeof(int32_t), s));
    OOC_TRY(cudaMallocAsync(&perm_in, nz * sizeof(I), s));
    OOC_TRY(cudaMallocAsync(&perm, nz * sizeof(I), s));
    OOC_TRY(cudaMallocAsync(&cnt, (cols + 1) * sizeof(unsigned long long), s));
    OOC_TRY(cudaMemsetAsync(cnt, 0, (cols + 1) * sizeof(unsigned long long), s));
    if (nnz > 0) {
        k_row_ids<<<grid_for(rows), 256, 0, s>>>(rp, rows, rid);
        k_iota<I><<<grid_for(nnz), 256, 0, s>>>(perm_in, nnz);
        k_col_hist<<<grid_for(nnz), 256, 0, s>>>(ci, nnz, cnt);
        int bits = 1;
        while ((int64_t(1) << bits) < cols) ++bits;
        OOC_TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ci, keys_out, perm_in, perm, nnz, 0,
                                                bits, s));
        OOC_TRY(cudaMallocAsync(&tmp, bytes, s));
        OOC_TRY(cub::DeviceRadixSort::SortPairs(tmp, bytes, ci, keys_out, perm_in, perm, nnz, 0, bits,
                                                s));
        k_gather_t<I><<<grid_for(nnz), 256, 0, s>>>(perm, rid, v, nnz, ciT, vT);
    }
    static_assert(sizeof(unsigned long long) == sizeof(int64_t), "");
    OOC_TRY(exclusive_scan_i64(reinterpret_cast<const int64_t*>(cnt), rpT, cols + 1, s));
    e = cudaGetLastError();
done:
#undef OOC_TRY
    if (rid) cudaFreeAsync(rid, s);
    if (keys_out) cudaFreeAsync(keys_out, s);
    if (perm_in) cudaFreeAsync(perm_in, s);
    if (perm) cudaFreeAsync(perm, s);
    if (cnt) cudaFreeAsync(cnt, s);
    if (tmp) cudaFreeAsync(tmp, s);
    return e;
}

cudaError_t csr_transpose(const int64_t* rp, const int32_t* ci, const float* v, int64_t rows,
                          int64_t cols, int64_t nnz, int64_t* rpT, int32_t* ciT, float* vT,
                          cudaStream_t s) {
    if (nnz > int64_t(INT32_MAX)) return csr_transpose_t<int64_t>(rp, ci, v, rows, cols, nnz, rpT, ciT, vT, s);
    return csr_transpose_t<int32_t>(rp, ci, v, rows, cols, nnz, rpT, ciT, vT, s);
}

cudaError_t launch_gen_csr_count(int64_t rows, int64_t row0, int64_t n, uint64_t thresh, uint64_t seed,
                                 int64_t* counts, cudaStream_t s) {
    const unsigned grid = unsigned(rows < 148 * 16 ? rows : 148 * 16);
    k_gen_csr_count<<<grid, 256, 0, s>>>(rows, row0, n, thresh, rng_key(seed, kStreamSparseMask), counts);
    return cudaGetLastError();
}

cudaError_t launch_gen_csr_fill(int64_t rows, int64_t row0, int64_t n, uint64_t thresh, uint64_t seed,
                                const int64_t* rp, int32_t* ci, float* v, cudaStream_t s) {
    const unsigned grid = unsigned(rows < 148 * 16 ? rows : 148 * 16);
    k_gen_csr_fill<<<grid, 256, 0, s>>>(rows, row0, n, thresh, rng_key(seed, kStreamSparseMask),
                                        rng_key(seed, kStreamSparseVal), rp, ci, v);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------- ingest
// Upload path of oocnmf_load_csr_f64: the reference's CsrMatrix arrays (u64 columns, f64
// values; include/oocnmf/matrix.hpp) arrive in chunks and are narrowed to the device layout
// (i32 columns, f32 values) here, with the reference constructor's checks
// (src/matrix.cpp CsrMatrix validation) done on device instead of on one host core.
namespace {

__global__ void k_csr_ingest(const uint64_t* __restrict__ ci_in, const double* __restrict__ v_in,
                             int64_t count, uint64_t n, int32_t* __restrict__ ci, float* __restrict__ v,
                             unsigned* __restrict__ bad) {
    bool out_of_range = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = ci_in[i];
        out_of_range |= c >= n;
        ci[i] = int32_t(c);
        v[i] = float(v_in[i]);
    }
    if (__any_sync(0xffffffffu, out_of_range) && (threadIdx.x & 31) == 0) atomicOr(bad, kCsrBadColumn);
}

// One thread per row. A row pointer outside [0, nnz] or below its predecessor is reported as
// "not nondecreasing" (a nondecreasing row_ptr from 0 to nnz stays inside), so the column walk
// never leaves the arrays.
__global__ void k_csr_check_rows(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 int64_t rows, int64_t nnz, unsigned* __restrict__ bad) {
    unsigned flags = 0;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = rp[r], e = rp[r + 1];
        if (b < 0 || e < b || e > nnz) {
            flags |= kCsrBadRowPtr;
            continue;
        }
        for (int64_t p = b + 1; p < e; ++p)
            if (ci[p] <= ci[p - 1]) {
                flags |= kCsrBadOrder;
                break;
            }
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (flags && (threadIdx.x & 31) == 0) atomicOr(bad, flags);
}

int ingest_grid(int64_t work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return int(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, int64_t(sms) * 8)));
}

}  // namespace

cudaError_t launch_csr_ingest(const uint64_t* ci_in, const double* v_in, int64_t count, uint64_t n,
                              int32_t* ci, float* v, unsigned* bad, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    k_csr_ingest<<<ingest_grid(count), 256, 0, s>>>(ci_in, v_in, count, n, ci, v, bad);
    return cudaGetLastError();
}

cudaError_t launch_csr_check_rows(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t nnz,
                                  unsigned* bad, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    k_csr_check_rows<<<ingest_grid(rows), 256, 0, s>>>(rp, ci, rows, nnz, bad);
    return cudaGetLastError();
}

}  // namespace ooc
