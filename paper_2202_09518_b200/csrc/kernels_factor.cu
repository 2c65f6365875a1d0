// Factor-side kernels of one MU iteration: the fused multiplicative update with its
// epsilon guard and Gram / trace-error partials, plus deterministic slot reductions.
//
// Reference semantics kept (src/kernels.cpp):
//   hadamard_update  t <- t * nu / (de + eps)              (:207-244)
//   denominator      de = F · G  (W·HH^T, or (W^T W)·H)     (nmf_serial.cpp:89,98)
//   gram_t           symmetric k x k, mirrored triangle     (:127-179)
// With H stored transposed (Ht, n x kp) both factors are row-major "tall" matrices, so one
// kernel updates W rows (G = HH^T, N = A·H^T) and Ht rows (G = W^T W, N = (W^T A)^T).
#include "kernels.h"

namespace ooc {
namespace {

// A CTA handles 64-row units (half of a 128-row stream-K tile) with four threads per row,
// each owning kp/4 columns. The update is a short dependent chain per thread, so what sets its
// speed is how many units are in flight per SM: small CTAs, few registers (the row is staged
// in shared memory instead of registers), several CTAs resident per SM.
constexpr int kUnitRows = 64;
constexpr int kRowThreads = 4;
constexpr int kFuThreads = kUnitRows * kRowThreads;  // 256
constexpr int kFuMaxGrid = 16 * 148;

// Fixed-shape block reduction of a double (deterministic).
__device__ double block_sum_f64(double v, double* sh) {
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) sh[tid] += sh[tid + s];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// Register-blocked Gram of a 64-row unit over 256 threads: thread t < NBLK owns a TI x TJ
// block (rows i0.., cols j0..) of the kp x kp result.
template <int KP>
struct GramBlock {
    static constexpr int T = KP >= 64 ? 4 : (KP >= 32 ? 2 : 1);
    static constexpr int TI = T, TJ = T;
    static constexpr int NJB = KP / TJ;           // blocks along j
    static constexpr int NBLK = (KP / TI) * NJB;  // <= 256
    static constexpr int FS = KP + 4;             // f32 smem row stride (16-byte aligned rows)
};

template <int KP>
__global__ void __launch_bounds__(kFuThreads, 3)
    k_factor_update(float* __restrict__ F, int64_t units, const float* __restrict__ n_plain,
                    const float* __restrict__ n_slots, StreamK sk, const float* __restrict__ G,
                    float eps, int update, double* __restrict__ gram_slots,
                    double* __restrict__ err_slots, int* __restrict__ flag, float* __restrict__ cat_out) {
    using GB = GramBlock<KP>;
    constexpr int FS = GB::FS;
    constexpr int QW = KP / kRowThreads;  // columns owned by each thread of a row
    extern __shared__ __align__(16) unsigned char fu_smem[];
    double* red = reinterpret_cast<double*>(fu_smem);
    float* Gs = reinterpret_cast<float*>(red + kFuThreads);
    float* Fs = Gs + KP * KP;
    const int tid = threadIdx.x;
    const int lr = tid / kRowThreads, part = tid % kRowThreads;  // local row, column quarter
    const int c0 = part * QW;
    if (update)
        for (int e = tid; e < KP * KP; e += kFuThreads) Gs[e] = G[e];

    const int bi = tid / GB::NJB, bj = tid % GB::NJB;
    const int i0 = bi * GB::TI, j0 = bj * GB::TJ;
    const bool gram_owner = tid < GB::NBLK;
    double gacc[GB::TI * GB::TJ];
#pragma unroll
    for (int q = 0; q < GB::TI * GB::TJ; ++q) gacc[q] = 0.0;
    double eacc = 0.0;
    bool bad = false;

    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t row = u * kUnitRows + lr;
        const int64_t t = u / (kTile / kUnitRows);                  // stream-K tile
        const int trow = int(u % (kTile / kUnitRows)) * kUnitRows + lr;  // row within the tile
        float fo[QW];
        {
            const float* fr = F + row * KP + c0;
#pragma unroll
            for (int j = 0; j < QW; ++j) fo[j] = fr[j];
        }
        if (update) {
#pragma unroll
            for (int j = 0; j < QW; ++j) Fs[lr * FS + c0 + j] = fo[j];
            float nu[QW];
            if (n_plain) {
                const float* nr = n_plain + row * KP + c0;
#pragma unroll
                for (int j = 0; j < QW; ++j) nu[j] = nr[j];
            } else {
#pragma unroll
                for (int j = 0; j < QW; ++j) nu[j] = 0.f;
                const int64_t s0 = sk.cta_of(t * sk.ipt), s1 = sk.cta_of((t + 1) * sk.ipt - 1);
                for (int64_t c = s0; c <= s1; ++c) {
                    const float* nr = n_slots + sk.slot(c, t) * int64_t(kTile * KP) + int64_t(trow) * KP + c0;
#pragma unroll
                    for (int j = 0; j < QW; ++j) nu[j] += nr[j];
                }
            }
            __syncthreads();  // Gs (first unit) and this unit's rows staged
            // de = f · G: f[q] is a broadcast read of the row in smem, G rows are 128-bit loads
            float de[QW];
#pragma unroll
            for (int j = 0; j < QW; ++j) de[j] = 0.f;
            const float* frow = Fs + lr * FS;
#pragma unroll 8
            for (int q = 0; q < KP; ++q) {
                const float fq = frow[q];
#pragma unroll
                for (int j = 0; j < QW; ++j) de[j] = fmaf(fq, Gs[q * KP + c0 + j], de[j]);
            }
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < QW; ++j) {
                const float nf = fo[j] * nu[j] / (de[j] + eps);
                bad |= !isfinite(nf);
                fo[j] = nf;
                e += double(nu[j]) * double(nf);
            }
            eacc += e;
            float* fw = F + row * KP + c0;
#pragma unroll
            for (int j = 0; j < QW; ++j) fw[j] = fo[j];
            __syncthreads();  // everyone has read the old rows from Fs
        }
        if (cat_out) {
            // [F | F - tf32(F)] row of the tensor-core operand (one TMA box carries both halves)
            float* cw = cat_out + row * 2 * KP;
#pragma unroll
            for (int j = 0; j < QW; ++j) {
                cw[c0 + j] = fo[j];
                cw[KP + c0 + j] = tf32_lo(fo[j]);
            }
        }
        // Gram partial of the unit: f32 sums over its 64 rows (FP64 issue rate is far below
        // FP32), accumulated across units and CTAs in f64. Its ~1e-7 relative error only
        // reaches the error estimate through the trace form, which error_mode auto uses only
        // where err > 0.1 (there it moves err by < 1e-5 relative).
#pragma unroll
        for (int j = 0; j < QW; ++j) Fs[lr * FS + c0 + j] = fo[j];
        __syncthreads();
        if (gram_owner) {
            float gt[GB::TI * GB::TJ];
#pragma unroll
            for (int q = 0; q < GB::TI * GB::TJ; ++q) gt[q] = 0.f;
#pragma unroll 8
            for (int r = 0; r < kUnitRows; ++r) {
                const float* fr = Fs + r * FS;
                float fi[GB::TI], fj[GB::TJ];
#pragma unroll
                for (int a = 0; a < GB::TI; ++a) fi[a] = fr[i0 + a];
#pragma unroll
                for (int b = 0; b < GB::TJ; ++b) fj[b] = fr[j0 + b];
#pragma unroll
                for (int a = 0; a < GB::TI; ++a)
#pragma unroll
                    for (int b = 0; b < GB::TJ; ++b) gt[a * GB::TJ + b] = fmaf(fi[a], fj[b], gt[a * GB::TJ + b]);
            }
#pragma unroll
            for (int q = 0; q < GB::TI * GB::TJ; ++q) gacc[q] += double(gt[q]);
        }
        __syncthreads();
    }
    if (gram_owner) {
        double* gout = gram_slots + int64_t(blockIdx.x) * KP * KP;
#pragma unroll
        for (int a = 0; a < GB::TI; ++a)
#pragma unroll
            for (int b = 0; b < GB::TJ; ++b) {
                const int i = i0 + a, j = j0 + b;
                // mirror the upper triangle so the Gram is symmetric to the bit
                const double v = gacc[a * GB::TJ + b];
                if (i <= j) gout[i * KP + j] = v, gout[j * KP + i] = v;
            }
    }
    if (err_slots) {
        const double s = block_sum_f64(eacc, red);
        if (tid == 0) err_slots[blockIdx.x] = s;
    }
    if (bad) atomicOr(flag, 1);
}

// One warp per output element; lanes stride the slots, then a fixed shuffle tree.
__global__ void k_reduce_slots(const double* __restrict__ slots, int64_t nslots, int64_t count,
                               float* __restrict__ out32, double* __restrict__ out64) {
    const int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= count) return;
    double s = 0.0;
    for (int64_t q = lane; q < nslots; q += 32) s += slots[q * count + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        out32[e] = float(s);
        if (out64) out64[e] = s;
    }
}

template <int KP>
__global__ void k_streamk_reduce(const float* __restrict__ slots, StreamK sk, float* __restrict__ out,
                                 int accumulate) {
    const int64_t t = blockIdx.x;
    const int64_t c0 = sk.cta_of(t * sk.ipt), c1 = sk.cta_of((t + 1) * sk.ipt - 1);
    constexpr int N4 = kTile * KP / 4;
    float4* o = reinterpret_cast<float4*>(out + t * int64_t(kTile * KP));
    for (int q = threadIdx.x; q < N4; q += blockDim.x) {
        float4 s = accumulate ? o[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t c = c0; c <= c1; ++c) {
            const float4 v = reinterpret_cast<const float4*>(slots + sk.slot(c, t) * int64_t(kTile * KP))[q];
            s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
        }
        o[q] = s;
    }
}

__global__ void k_finalize_error(int kp, const double* __restrict__ err_slots, int64_t n_err,
                                 const double* __restrict__ wtw, const double* __restrict__ hht,
                                 const double* __restrict__ norm_a2,
                                 const double* __restrict__ direct_res, double* __restrict__ out) {
    __shared__ double sh[256];
    const int tid = threadIdx.x;
    double res;
    if (direct_res) {
        res = *direct_res;
    } else {
        double a = 0.0;
        for (int64_t q = tid; q < n_err; q += blockDim.x) a += err_slots[q];
        const double cross = block_sum_f64(a, sh);
        double b = 0.0;
        for (int e = tid; e < kp * kp; e += blockDim.x) b += wtw[e] * hht[e];
        const double quad = block_sum_f64(b, sh);
        res = *norm_a2 - 2.0 * cross + quad;
    }
    if (tid == 0) *out = sqrt(res > 0.0 ? res : 0.0) / sqrt(*norm_a2);
}

}  // namespace

int factor_grid(int64_t tiles) {
    const int64_t units = tiles * (kTile / kUnitRows);
    return int(units < kFuMaxGrid ? units : kFuMaxGrid);
}

cudaError_t launch_factor_update(int kp, float* F, int64_t rows, const float* n_plain,
                                 const float* n_slots, const StreamK* sk, const float* G,
                                 float eps, bool update, double* gram_slots, double* err_slots,
                                 int* flag, float* cat_out, cudaStream_t s) {
    const int64_t tiles = rows / kTile;
    const int64_t units = tiles * (kTile / kUnitRows);
    const int grid = factor_grid(tiles);
    StreamK skv = sk ? *sk : StreamK{};
#define OOC_FU(K)                                                                              \
    case K: {                                                                                  \
        const int smem = int(kFuThreads * sizeof(double) + K * K * sizeof(float) +            \
                             kUnitRows * GramBlock<K>::FS * sizeof(float));                    \
        cudaError_t e = cudaFuncSetAttribute(                                                  \
            k_factor_update<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
        if (e != cudaSuccess) return e;                                                        \
        k_factor_update<K><<<grid, kFuThreads, smem, s>>>(F, units, n_plain, n_slots, skv, G,  \
                                                         eps, update ? 1 : 0, gram_slots,      \
                                                         err_slots, flag, cat_out);            \
        break;                                                                                 \
    }
    switch (kp) {
        OOC_FU(8)
        OOC_FU(16)
        OOC_FU(32)
        OOC_FU(64)
        default: return cudaErrorInvalidValue;
    }
#undef OOC_FU
    return cudaGetLastError();
}

cudaError_t launch_reduce_slots(const double* slots, int64_t nslots, int64_t count, float* out32,
                                double* out64, cudaStream_t s) {
    const int64_t threads = count * 32;
    k_reduce_slots<<<unsigned((threads + 255) / 256), 256, 0, s>>>(slots, nslots, count, out32, out64);
    return cudaGetLastError();
}

cudaError_t launch_streamk_reduce(int kp, const float* slots, const StreamK& sk, float* out,
                                  bool accumulate, cudaStream_t s) {
    switch (kp) {
        case 8: k_streamk_reduce<8><<<unsigned(sk.tiles), 256, 0, s>>>(slots, sk, out, accumulate); break;
        case 16: k_streamk_reduce<16><<<unsigned(sk.tiles), 256, 0, s>>>(slots, sk, out, accumulate); break;
        case 32: k_streamk_reduce<32><<<unsigned(sk.tiles), 256, 0, s>>>(slots, sk, out, accumulate); break;
        case 64: k_streamk_reduce<64><<<unsigned(sk.tiles), 256, 0, s>>>(slots, sk, out, accumulate); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_finalize_error(int kp, const double* err_slots, int64_t n_err, const double* wtw,
                                  const double* hht, const double* norm_a2, const double* direct_res,
                                  double* out_err, cudaStream_t s) {
    k_finalize_error<<<1, 256, 0, s>>>(kp, err_slots, n_err, wtw, hht, norm_a2, direct_res, out_err);
    return cudaGetLastError();
}

}  // namespace ooc
