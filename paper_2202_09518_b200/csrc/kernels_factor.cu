// Factor-side kernels of one MU iteration: the fused multiplicative update with its
// epsilon guard and Gram / trace-error partials, plus deterministic slot reductions.
//
// Reference semantics kept (src/kernels.cpp):
//   hadamard_update  t <- t * nu / (de + eps)              (:207-244)
//   denominator      de = F · G  (W·HH^T, or (W^T W)·H)     (nmf_serial.cpp:89,98)
//   gram_t           symmetric k x k, mirrored triangle     (:127-179)
// With H stored transposed (Ht, n x kp) both factors are row-major "tall" matrices, so one
// kernel updates W rows (G = HH^T, N = A·H^T) and Ht rows (G = W^T W, N = (W^T A)^T).
#include <cstdlib>

#include "kernels.h"

namespace ooc {
namespace {

// A CTA of 512 threads owns whole 128-row tiles and loops over them:
//   1. the tile's F rows and numerator rows (plain, or the sum of the tile's stream-K
//      partials in ascending CTA order) are staged in shared memory with coalesced loads,
//      each thread keeping all of its kp/4 loads in flight;
//   2. warp w updates 32 rows x one quarter of the columns: lane = row, so f[q] is a
//      conflict-free read of the lane's own (padded) row and the G row segment is the same
//      for the whole warp (a broadcast) — kp/4 FMAs per f[q], 3 wavefronts per 8 FMAs; the
//      update f * n / (de + eps) and its n·f_new term of the trace-form error follow;
//   3. the new rows go back to global memory (and [F | lo(F)] for the tensor-core operand)
//      with coalesced stores;
//   4. Gram partial: thread (block b, row group g) accumulates a GT x GT block of
//      F_new^T F_new over its row group in f32 registers across the CTA's tiles; at the end the
//      row groups are summed in f64 (fixed order) into one kp x kp slot per CTA.
// With 16 warps per CTA and up to 4 CTAs per SM the per-row dependent chain is hidden by
// occupancy (the previous layouts were latency-bound at 40-55 us for 65536 x 32 —
// tools/fu_bench.cu).
constexpr int kFuRows = kTile;          // rows per tile
constexpr int kFuThreads = 4 * kFuRows;  // 4 threads per row in the update
constexpr int kFuCtasPerSm = 2;
constexpr int kFuMaxParts = 64;          // stream-K partials of one tile summed via smem offsets

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
struct FuCfg {
    static constexpr int FS = KP + 1;                  // padded f32 row stride
    static constexpr int QC = KP / 4;                  // update columns per thread
    static constexpr int GT = KP >= 32 ? 4 : 2;        // Gram thread block GT x GT
    static constexpr int GB = KP / GT;
    static constexpr int NGB = GB * GB;                // Gram blocks (<= 512)
    static constexpr int RG = kFuThreads / NGB;        // row groups
    static_assert(NGB <= kFuThreads && kFuThreads % NGB == 0 && kFuRows % RG == 0, "Gram blocking");
    static constexpr int EPT = kFuRows * KP / kFuThreads;  // staged elements per thread
    // smem: G (f32) | Fs | Ns (f32, padded rows) ; the Gram partials (RG x KP x KP f32) reuse
    // Fs/Ns at the end
    static constexpr size_t ROWS_BYTES = 2 * size_t(kFuRows) * FS * 4;
    static constexpr size_t PART_BYTES = size_t(RG) * KP * KP * 4;
    static_assert(PART_BYTES <= ROWS_BYTES, "Gram partials fit in the row buffers");
    static constexpr size_t SMEM = size_t(KP * KP) * 4 + ROWS_BYTES + size_t(kFuThreads) * 8;
};

template <int KP>
__global__ void __launch_bounds__(kFuThreads, 2)
    k_factor_update(float* __restrict__ F, int64_t tiles, const float* __restrict__ n_plain,
                    const float* __restrict__ n_slots, StreamK sk, const float* __restrict__ G,
                    float eps, int update, double* __restrict__ gram_slots,
                    double* __restrict__ err_slots, int* __restrict__ flag, float* __restrict__ cat_out) {
    using C = FuCfg<KP>;
    constexpr int FS = C::FS, GT = C::GT, QC = C::QC;
    extern __shared__ __align__(16) unsigned char fu_smem[];
    float* Gs = reinterpret_cast<float*>(fu_smem);  // KP x KP
    float* Fs = Gs + KP * KP;                         // kFuRows x FS: old rows
    float* Ns = Fs + kFuRows * FS;                    // kFuRows x FS: numerator, then new rows
    double* red = reinterpret_cast<double*>(Ns + kFuRows * FS);  // kFuThreads (8-byte aligned)
    __shared__ int64_t part_off[kFuMaxParts];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (update)
        for (int e = tid; e < KP * KP; e += kFuThreads) Gs[e] = G[e];
    // update role: warp -> (row block of 32, column quarter)
    const int urow = (warp & 3) * 32 + lane, uc0 = (warp >> 2) * QC;
    // Gram role
    const int gblk = tid % C::NGB, grg = tid / C::NGB;
    const int gi0 = (gblk / C::GB) * GT, gj0 = (gblk % C::GB) * GT;
    float gacc[GT * GT];
#pragma unroll
    for (int q = 0; q < GT * GT; ++q) gacc[q] = 0.f;
    double eacc = 0.0;
    bool bad = false;

    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t base = t * kFuRows * KP;
        int nparts = 0;
        int64_t cfirst = 0;
        if (update && !n_plain) {
            // the tile's partials, ascending CTA order (64-bit divisions once per tile)
            cfirst = sk.cta_of(t * sk.ipt);
            nparts = int(sk.cta_of((t + 1) * sk.ipt - 1) - cfirst + 1);
            for (int q = tid; q < nparts && q < kFuMaxParts; q += kFuThreads)
                part_off[q] = sk.slot(cfirst + q, t) * int64_t(kTile * KP);
            __syncthreads();
        }
        // 1. stage (element e = tid + kFuThreads * i)
        {
            float fv[C::EPT], nv[C::EPT];
#pragma unroll
            for (int i = 0; i < C::EPT; ++i) fv[i] = F[base + tid + i * kFuThreads];
            if (update) {
                if (n_plain) {
#pragma unroll
                    for (int i = 0; i < C::EPT; ++i) nv[i] = n_plain[base + tid + i * kFuThreads];
                } else {
#pragma unroll
                    for (int i = 0; i < C::EPT; ++i) nv[i] = 0.f;
                    for (int q = 0; q < nparts; ++q) {
                        const float* src =
                            n_slots + (q < kFuMaxParts ? part_off[q] : sk.slot(cfirst + q, t) * int64_t(kTile * KP));
                        float pv[C::EPT];
#pragma unroll
                        for (int i = 0; i < C::EPT; ++i) pv[i] = src[tid + i * kFuThreads];
#pragma unroll
                        for (int i = 0; i < C::EPT; ++i) nv[i] += pv[i];
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < C::EPT; ++i) {
                const int e = tid + i * kFuThreads, r = e / KP, j = e % KP;
                Fs[r * FS + j] = fv[i];
                if (update) Ns[r * FS + j] = nv[i];
            }
        }
        __syncthreads();
        // 2. update: lane = row urow, columns [uc0, uc0 + QC)
        if (update) {
            const float* fr = Fs + urow * FS;
            float de[QC];
#pragma unroll
            for (int j = 0; j < QC; ++j) de[j] = 0.f;
#pragma unroll 8
            for (int q = 0; q < KP; ++q) {
                const float fq = fr[q];
                const float* g = Gs + q * KP + uc0;
#pragma unroll
                for (int j = 0; j < QC; ++j) de[j] = fmaf(fq, g[j], de[j]);
            }
            float* nr = Ns + urow * FS + uc0;
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < QC; ++j) {
                const float nu = nr[j];
                const float nf = fr[uc0 + j] * nu / (de[j] + eps);
                bad |= !isfinite(nf);
                e += double(nu) * double(nf);
                nr[j] = nf;  // (row, column quarter) is private to this thread
            }
            eacc += e;
        } else {
            for (int e = tid; e < kFuRows * KP; e += kFuThreads) {
                const int r = e / KP, j = e % KP;
                Ns[r * FS + j] = Fs[r * FS + j];
            }
        }
        __syncthreads();
        // 3. write back (coalesced)
#pragma unroll
        for (int i = 0; i < C::EPT; ++i) {
            const int e = tid + i * kFuThreads, r = e / KP, j = e % KP;
            const float v = Ns[r * FS + j];
            if (update) F[base + e] = v;
            if (cat_out) {
                float* cw = cat_out + (t * kFuRows + r) * 2 * KP;
                cw[j] = v;
                cw[KP + j] = tf32_lo(v);
            }
        }
        // 4. Gram partial of the tile's new rows
#pragma unroll 4
        for (int r = grg; r < kFuRows; r += C::RG) {
            const float* row = Ns + r * FS;
            float fi[GT], fj[GT];
#pragma unroll
            for (int a = 0; a < GT; ++a) fi[a] = row[gi0 + a], fj[a] = row[gj0 + a];
#pragma unroll
            for (int a = 0; a < GT; ++a)
#pragma unroll
                for (int b = 0; b < GT; ++b) gacc[a * GT + b] = fmaf(fi[a], fj[b], gacc[a * GT + b]);
        }
        __syncthreads();  // Fs / Ns are rewritten by the next tile
    }
    // row groups -> f64 CTA sum in fixed order (partials parked in the row buffers)
    float* part = Fs;
#pragma unroll
    for (int a = 0; a < GT; ++a)
#pragma unroll
        for (int b = 0; b < GT; ++b) part[(grg * KP + gi0 + a) * KP + gj0 + b] = gacc[a * GT + b];
    __syncthreads();
    double* gout = gram_slots + int64_t(blockIdx.x) * KP * KP;
    for (int e = tid; e < KP * KP; e += kFuThreads) {
        const int i = e / KP, j = e % KP;
        // mirror the upper triangle so the Gram is symmetric to the bit
        const int src = i <= j ? e : j * KP + i;
        double sum = 0.0;
        for (int g = 0; g < C::RG; ++g) sum += double(part[g * KP * KP + src]);
        gout[e] = sum;
    }
    if (err_slots) {
        const double sum = block_sum_f64(eacc, red);
        if (tid == 0) err_slots[blockIdx.x] = sum;
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
                                 const double* __restrict__ direct_res, double* __restrict__ out,
                                 const int* __restrict__ pred_in, int* __restrict__ pred_out, double threshold) {
    __shared__ double sh[256];
    const int tid = threadIdx.x;
    if (pred_in && *pred_in == 0) return;
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
    if (tid == 0) {
        const double e = sqrt(res > 0.0 ? res : 0.0) / sqrt(*norm_a2);
        *out = e;
        if (pred_out) *pred_out = e < threshold ? 1 : 0;
    }
}

}  // namespace

int factor_grid(int64_t tiles) {
    static int sms = [] {
        int d = 0, n = 148;
        if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
    }();
    static int64_t per_sm = [] {  // OOCNMF_FU_CTAS_PER_SM: developer knob (tools/fu_bench.cu)
        const char* e = std::getenv("OOCNMF_FU_CTAS_PER_SM");
        const int v = e ? std::atoi(e) : 0;
        return int64_t(v > 0 ? v : kFuCtasPerSm);
    }();
    const int64_t cap = int64_t(sms) * per_sm;
    return int(tiles < cap ? (tiles < 1 ? 1 : tiles) : cap);
}

cudaError_t launch_factor_update(int kp, float* F, int64_t rows, const float* n_plain,
                                 const float* n_slots, const StreamK* sk, const float* G,
                                 float eps, bool update, double* gram_slots, double* err_slots,
                                 int* flag, float* cat_out, cudaStream_t s) {
    const int64_t tiles = rows / kTile;
    const int grid = factor_grid(tiles);
    StreamK skv = sk ? *sk : StreamK{};
#define OOC_FU(K)                                                                              \
    case K: {                                                                                  \
        static const cudaError_t attr = cudaFuncSetAttribute(                                  \
            k_factor_update<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(FuCfg<K>::SMEM)); \
        if (attr != cudaSuccess) return attr;                                                  \
        k_factor_update<K><<<grid, kFuThreads, FuCfg<K>::SMEM, s>>>(F, tiles, n_plain, n_slots, skv, G, \
                                                                 eps, update ? 1 : 0, gram_slots, \
                                                                 err_slots, flag, cat_out);    \
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
                                  double* out_err, cudaStream_t s, const int* pred_in, int* pred_out,
                                  double threshold) {
    k_finalize_error<<<1, 256, 0, s>>>(kp, err_slots, n_err, wtw, hht, norm_a2, direct_res, out_err, pred_in,
                                       pred_out, threshold);
    return cudaGetLastError();
}

}  // namespace ooc
