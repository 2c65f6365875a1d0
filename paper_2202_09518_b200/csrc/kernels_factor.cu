// Factor-side kernels of one MU iteration: the fused multiplicative update with its
// epsilon guard and Gram / trace-error partials, plus deterministic slot reductions.
//
// Reference semantics kept (src/kernels.cpp):
//   hadamard_update  t <- t * nu / (de + eps)              (:207-244)
//   denominator      de = F · G  (W·HH^T, or (W^T W)·H)     (nmf_serial.cpp:89,98)
//   gram_t           upper triangle accumulated, mirrored   (:127-179)
// With H stored transposed (Ht, n x kp) both factors are row-major "tall" matrices, so one
// kernel updates W rows (G = HH^T, N = A·H^T) and Ht rows (G = W^T W, N = (W^T A)^T).
#include "kernels.h"

namespace ooc {
namespace {

constexpr int kFuThreads = 128;  // one thread per factor row of a 128-row tile

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

template <int KP>
__global__ void __launch_bounds__(kFuThreads)
    k_factor_update(float* __restrict__ F, int64_t tiles, const float* __restrict__ n_plain,
                    const float* __restrict__ n_slots, StreamK sk, const float* __restrict__ G,
                    float eps, int update, double* __restrict__ gram_slots,
                    double* __restrict__ err_slots, int* __restrict__ flag, float* __restrict__ cat_out) {
    constexpr int FS = KP + 1;
    extern __shared__ __align__(16) unsigned char fu_smem[];
    double* red = reinterpret_cast<double*>(fu_smem);
    float* Gs = reinterpret_cast<float*>(red + kFuThreads);
    double* Fs = reinterpret_cast<double*>(Gs + KP * KP);
    const int tid = threadIdx.x;
    if (update)
        for (int e = tid; e < KP * KP; e += kFuThreads) Gs[e] = G[e];

    constexpr int NE = (KP * KP + kFuThreads - 1) / kFuThreads;  // gram entries per thread
    double gacc[NE];  // f64: the Gram feeds <W^T W, H H^T> of the trace-form error
#pragma unroll
    for (int q = 0; q < NE; ++q) gacc[q] = 0.0;
    double eacc = 0.0;
    bool bad = false;
    __syncthreads();

    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t row = t * kTile + tid;
        float f[KP];
        {
            const float4* fr = reinterpret_cast<const float4*>(F + row * KP);
#pragma unroll
            for (int j4 = 0; j4 < KP / 4; ++j4) {
                const float4 v = fr[j4];
                f[4 * j4] = v.x, f[4 * j4 + 1] = v.y, f[4 * j4 + 2] = v.z, f[4 * j4 + 3] = v.w;
            }
        }
        if (update) {
            float nu[KP];
            if (n_plain) {
                const float4* nr = reinterpret_cast<const float4*>(n_plain + row * KP);
#pragma unroll
                for (int j4 = 0; j4 < KP / 4; ++j4) {
                    const float4 v = nr[j4];
                    nu[4 * j4] = v.x, nu[4 * j4 + 1] = v.y, nu[4 * j4 + 2] = v.z, nu[4 * j4 + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < KP; ++j) nu[j] = 0.f;
                const int64_t c0 = sk.cta_of(t * sk.ipt), c1 = sk.cta_of((t + 1) * sk.ipt - 1);
                for (int64_t c = c0; c <= c1; ++c) {
                    const float4* nr = reinterpret_cast<const float4*>(
                        n_slots + sk.slot(c, t) * int64_t(kTile * KP) + int64_t(tid) * KP);
#pragma unroll
                    for (int j4 = 0; j4 < KP / 4; ++j4) {
                        const float4 v = nr[j4];
                        nu[4 * j4] += v.x, nu[4 * j4 + 1] += v.y, nu[4 * j4 + 2] += v.z,
                            nu[4 * j4 + 3] += v.w;
                    }
                }
            }
            float de[KP];
#pragma unroll
            for (int j = 0; j < KP; ++j) de[j] = 0.f;
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const float fq = f[q];
#pragma unroll
                for (int j = 0; j < KP; ++j) de[j] = fmaf(fq, Gs[q * KP + j], de[j]);
            }
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < KP; ++j) {
                const float nf = f[j] * nu[j] / (de[j] + eps);
                bad |= !isfinite(nf);
                f[j] = nf;
                e += double(nu[j]) * double(nf);
            }
            eacc += e;
            float4* fw = reinterpret_cast<float4*>(F + row * KP);
#pragma unroll
            for (int j4 = 0; j4 < KP / 4; ++j4)
                fw[j4] = make_float4(f[4 * j4], f[4 * j4 + 1], f[4 * j4 + 2], f[4 * j4 + 3]);
        }
        if (cat_out) {
            // [F | F - tf32(F)] row of the tensor-core operand (one TMA box carries both halves)
            float4* cw = reinterpret_cast<float4*>(cat_out + row * 2 * KP);
#pragma unroll
            for (int j4 = 0; j4 < KP / 4; ++j4) {
                float l[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float x = f[4 * j4 + q];
                    l[q] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
                }
                cw[j4] = make_float4(f[4 * j4], f[4 * j4 + 1], f[4 * j4 + 2], f[4 * j4 + 3]);
                cw[KP / 4 + j4] = make_float4(l[0], l[1], l[2], l[3]);
            }
        }
        // Gram partial of this tile: entries (i <= j), ascending rows.
        // Rows go to smem already widened to f64 (f32 x f32 products are exact in f64); each
        // thread then runs NE independent accumulation chains over the 128 rows (rows outer),
        // so the f64 FMA latency is hidden by ILP instead of serialising 128-long chains.
#pragma unroll
        for (int j = 0; j < KP; ++j) Fs[tid * FS + j] = double(f[j]);
        __syncthreads();
        {
            // thread t owns entries e = t + 128 q: column j = e % KP, rows i = e / KP
            const int j0 = tid % KP;
            for (int r = 0; r < kTile; ++r) {
                const double fj = Fs[r * FS + j0];
#pragma unroll
                for (int q = 0; q < NE; ++q) {
                    const int e = tid + q * kFuThreads;
                    if (e < KP * KP) gacc[q] = fma(Fs[r * FS + e / KP], fj, gacc[q]);
                }
            }
        }
        __syncthreads();
    }
    double* gout = gram_slots + int64_t(blockIdx.x) * KP * KP;
#pragma unroll
    for (int q = 0; q < NE; ++q) {
        const int e = tid + q * kFuThreads;
        if (e < KP * KP) {
            const int i = e / KP, j = e % KP;
            if (i <= j) {
                gout[i * KP + j] = gacc[q];
                gout[j * KP + i] = gacc[q];
            }
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

int factor_grid(int64_t tiles) { return int(tiles < 1184 ? tiles : 1184); }

cudaError_t launch_factor_update(int kp, float* F, int64_t rows, const float* n_plain,
                                 const float* n_slots, const StreamK* sk, const float* G,
                                 float eps, bool update, double* gram_slots, double* err_slots,
                                 int* flag, float* cat_out, cudaStream_t s) {
    const int64_t tiles = rows / kTile;
    const int grid = factor_grid(tiles);
    StreamK skv = sk ? *sk : StreamK{};
#define OOC_FU(K)                                                                              \
    case K: {                                                                                  \
        const int smem = int(kFuThreads * sizeof(double) + K * K * sizeof(float) +            \
                             kFuThreads * (K + 1) * sizeof(double));                           \
        cudaError_t e = cudaFuncSetAttribute(                                                  \
            k_factor_update<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
        if (e != cudaSuccess) return e;                                                        \
        k_factor_update<K><<<grid, kFuThreads, smem, s>>>(F, tiles, n_plain, n_slots, skv, G,  \
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
