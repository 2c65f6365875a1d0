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

// A CTA of 256 threads owns whole 128-row tiles and loops over them, software-pipelined:
//   0. the next tile's F rows and plain numerator rows are prefetched with cp.async into the
//      other of two shared-memory stages while the current tile is computed (stream-K
//      numerators — the sum of the tile's partials in ascending CTA order — are summed from
//      global memory at the start of the tile instead);
//   1. rows are stored unpadded with the 16-byte chunks of row r XOR-swizzled by swz(r), so
//      the row-broadcast and column reads below are conflict-free and every access is 16 B;
//   2. update: thread (row block rb, column group cg) owns R rows (rb + i * RB) x C columns:
//      per 4 q it reads R float4 of F rows and C/4 float4 of G and issues 4 R C FMAs
//      (8 loads per 64 FMAs at kp 32); then f * n / (de + eps) and the n · f_new term of the
//      trace-form error, written in place over the numerator;
//   3. the new rows go back with 16-byte coalesced stores (and [F | lo(F)] for the
//      tensor-core operand);
//   4. Gram partial of the new rows, upper-triangle 4x4 blocks only (the Gram is mirrored
//      from its upper triangle anyway): thread (block b, row group g) accumulates in f32
//      registers across the CTA's tiles; at the end the row groups are summed in f64 (fixed
//      order) into one kp x kp slot per CTA.
// The FFMA work (kp^2 for the denominator + kp(kp+4)/2 for the Gram per row) is about the
// same time as the 12 kp bytes per row of HBM traffic at kp 32, so both are kept busy
// (3 CTAs / SM at kp <= 32).
#ifndef OOC_FU_CTAS
#define OOC_FU_CTAS 3
#endif
constexpr int kFuRows = kTile;  // rows per tile
constexpr int kFuThreads = 256;
constexpr int kFuMaxParts = 64;  // stream-K partials of one tile summed via smem offsets

template <int KP>
struct FuCfg {
    static constexpr int NCH = KP / 4;                   // 16-byte chunks per row
    static constexpr int TILE = kFuRows * KP;            // floats per tile
    static constexpr int C = KP >= 64 ? 8 : 4;           // update columns per thread
    static constexpr int NCG = KP / C;                   // column groups
    static constexpr int R = TILE / (kFuThreads * C);    // update rows per thread
    static constexpr int RB = kFuRows / R;               // row blocks
    static_assert(RB * NCG == kFuThreads, "update mapping");
    static constexpr int NGB = NCH * (NCH + 1) / 2;      // upper-triangle Gram blocks
    static constexpr int RG0 = kFuThreads / NGB;
    static constexpr int RG = RG0 > 32 ? 32 : RG0;       // Gram row groups
    static constexpr int CTAS = KP >= 64 ? 1 : OOC_FU_CTAS;  // resident CTAs per SM (smem)
    // smem (floats): 2 stages x [F tile | N tile] | G (KP x KP) | f64 reduction scratch
    static constexpr size_t STAGES_F = size_t(4) * TILE;
    static constexpr size_t SMEM = (STAGES_F + size_t(KP) * KP) * 4 + size_t(kFuThreads) * 8;
    static_assert(size_t(RG) * KP * KP <= STAGES_F, "Gram partials fit in the stages");
    // chunk swizzle: rows sharing a 128-byte bank line get distinct chunk offsets
    static __device__ __forceinline__ int swz(int r) {
        constexpr int per_line = KP >= 32 ? 1 : 32 / KP;
        constexpr int mask = NCH - 1 < 7 ? NCH - 1 : 7;
        return (r / per_line) & mask;
    }
    // float offset of chunk ch of row r
    static __device__ __forceinline__ int at(int r, int ch) { return r * KP + ((ch ^ swz(r)) << 2); }
};

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

#ifdef OOC_FU_PROFILE
// developer instrumentation (tools/fu_bench.cu): per-phase SM cycles summed over CTAs (thread 0)
__device__ unsigned long long g_fu_prof[8];
#define FU_MARK(i)                                               \
    if (threadIdx.x == 0) {                                      \
        const long long now_ = clock64();                        \
        prof_acc[i] += now_ - prof_last, prof_last = now_;       \
    }
#else
#define FU_MARK(i)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Copy one 128-row tile (contiguous in global memory) into a swizzled stage.
template <int KP>
__device__ __forceinline__ void stage_tile(float* dst, const float* src) {
    using C = FuCfg<KP>;
#pragma unroll
    for (int i = 0; i < C::TILE / 4 / kFuThreads; ++i) {
        const int c = threadIdx.x + i * kFuThreads, r = c / C::NCH, ch = c % C::NCH;
        cp_async16(dst + C::at(r, ch), src + c * 4);
    }
}

template <int KP>
__global__ void __launch_bounds__(kFuThreads, FuCfg<KP>::CTAS)
    k_factor_update(float* __restrict__ F, int64_t tiles, const float* __restrict__ n_plain,
                    const float* __restrict__ n_slots, StreamK sk, const float* __restrict__ G,
                    float eps, int update, double* __restrict__ gram_slots,
                    double* __restrict__ err_slots, int* __restrict__ flag, float* __restrict__ cat_out) {
    using C = FuCfg<KP>;
    constexpr int TILE = C::TILE, NCH = C::NCH, CC = C::C, R = C::R;
    extern __shared__ __align__(16) unsigned char fu_smem[];
    float* stages = reinterpret_cast<float*>(fu_smem);      // [F0 | N0 | F1 | N1]
    float* Gs = stages + C::STAGES_F;                        // KP x KP
    double* red = reinterpret_cast<double*>(Gs + KP * KP);   // kFuThreads
    __shared__ int64_t part_off[kFuMaxParts];
    const int tid = threadIdx.x;
    const bool plain = update && n_plain;
    if (update)
        for (int e = tid; e < KP * KP; e += kFuThreads) Gs[e] = G[e];
    // update role
    const int cg = tid % C::NCG, rb = tid / C::NCG;
    // Gram role: upper-triangle block (bi <= bj) and row group
    const int gblk = tid % C::NGB, grg = tid / C::NGB;
    int bi = 0, bj = gblk;
    while (bj >= NCH - bi) bj -= NCH - bi, ++bi;
    bj += bi;
    const bool gram_live = grg < C::RG;
    float gacc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) gacc[q] = 0.f;
    double eacc = 0.0;
    bool bad = false;

#ifdef OOC_FU_PROFILE
    long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, prof_last = clock64();
#endif
    if (int64_t(blockIdx.x) < tiles) {
        const int64_t t0 = blockIdx.x;
        stage_tile<KP>(stages, F + t0 * TILE);
        if (plain) stage_tile<KP>(stages + TILE, n_plain + t0 * TILE);
    }
    cp_async_commit();
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        float* Fs = stages + (it & 1) * 2 * TILE;
        float* Ns = Fs + TILE;
        {   // prefetch the next tile into the other stage (freed by the previous iteration's
            // final barrier)
            const int64_t tn = t + gridDim.x;
            if (tn < tiles) {
                float* Fn = stages + ((it + 1) & 1) * 2 * TILE;
                stage_tile<KP>(Fn, F + tn * TILE);
                if (plain) stage_tile<KP>(Fn + TILE, n_plain + tn * TILE);
            }
            cp_async_commit();
        }
        FU_MARK(0)  // prefetch issue
        if (update && !n_plain) {
            // the tile's stream-K partials, ascending CTA order (64-bit divisions once per tile)
            const int64_t cfirst = sk.cta_of(t * sk.ipt);
            const int nparts = int(sk.cta_of((t + 1) * sk.ipt - 1) - cfirst + 1);
            for (int q = tid; q < nparts && q < kFuMaxParts; q += kFuThreads)
                part_off[q] = sk.slot(cfirst + q, t) * int64_t(TILE);
            __syncthreads();
            constexpr int PER = TILE / 4 / kFuThreads;
            float4 acc[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < nparts; ++q) {
                const float4* src = reinterpret_cast<const float4*>(
                    n_slots + (q < kFuMaxParts ? part_off[q] : sk.slot(cfirst + q, t) * int64_t(TILE)));
                float4 pv[PER];
#pragma unroll
                for (int i = 0; i < PER; ++i) pv[i] = src[tid + i * kFuThreads];
#pragma unroll
                for (int i = 0; i < PER; ++i)
                    acc[i].x += pv[i].x, acc[i].y += pv[i].y, acc[i].z += pv[i].z, acc[i].w += pv[i].w;
            }
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int c = tid + i * kFuThreads;
                *reinterpret_cast<float4*>(Ns + C::at(c / NCH, c % NCH)) = acc[i];
            }
        }
        FU_MARK(1)  // stream-K numerator
        cp_async_wait<1>();  // this tile's group (the prefetch may still be in flight)
        FU_MARK(2)  // cp.async wait
        __syncthreads();
        FU_MARK(3)  // barrier
        // 2. update
        if (update) {
            float de[R][CC];
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int j = 0; j < CC; ++j) de[i][j] = 0.f;
#pragma unroll 2
            for (int q4 = 0; q4 < NCH; ++q4) {
                float4 f[R];
#pragma unroll
                for (int i = 0; i < R; ++i) f[i] = *reinterpret_cast<const float4*>(Fs + C::at(rb + i * C::RB, q4));
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    float g[CC];
#pragma unroll
                    for (int j = 0; j < CC; j += 4) {
                        const float4 gv = *reinterpret_cast<const float4*>(Gs + (q4 * 4 + qq) * KP + cg * CC + j);
                        g[j] = gv.x, g[j + 1] = gv.y, g[j + 2] = gv.z, g[j + 3] = gv.w;
                    }
#pragma unroll
                    for (int i = 0; i < R; ++i) {
                        const float fq = qq == 0 ? f[i].x : qq == 1 ? f[i].y : qq == 2 ? f[i].z : f[i].w;
#pragma unroll
                        for (int j = 0; j < CC; ++j) de[i][j] = fmaf(fq, g[j], de[i][j]);
                    }
                }
            }
            // n · f_new: f32 products (round-to-nearest, unbiased) summed over the thread's
            // R x C elements, then one f64 add per tile (f32 -> f64 conversions are slow)
            float e = 0.f;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int r = rb + i * C::RB;
#pragma unroll
                for (int j = 0; j < CC; j += 4) {
                    const int off = C::at(r, (cg * CC + j) >> 2);
                    const float4 fo = *reinterpret_cast<const float4*>(Fs + off);
                    const float4 nu = *reinterpret_cast<const float4*>(Ns + off);
                    // t * nu / (de + eps) as (t * nu) * rcp_rn(de + eps): the denominator is a
                    // normal number (>= eps), so the reciprocal never takes the IEEE-division
                    // slow path that tiny (decaying) numerators would trigger; <= 1.5 ulp
                    float4 nf;
                    nf.x = (fo.x * nu.x) * __frcp_rn(de[i][j] + eps);
                    nf.y = (fo.y * nu.y) * __frcp_rn(de[i][j + 1] + eps);
                    nf.z = (fo.z * nu.z) * __frcp_rn(de[i][j + 2] + eps);
                    nf.w = (fo.w * nu.w) * __frcp_rn(de[i][j + 3] + eps);
                    bad |= !isfinite(nf.x) || !isfinite(nf.y) || !isfinite(nf.z) || !isfinite(nf.w);
                    e = fmaf(nu.x, nf.x, e);
                    e = fmaf(nu.y, nf.y, e);
                    e = fmaf(nu.z, nf.z, e);
                    e = fmaf(nu.w, nf.w, e);
                    *reinterpret_cast<float4*>(Ns + off) = nf;  // (row, chunk) private to this thread
                }
            }
            eacc += double(e);
            FU_MARK(4)  // update
            __syncthreads();
            FU_MARK(5)  // barrier
        }
        const float* src = update ? Ns : Fs;
        // 3. write back (16-byte coalesced)
        if (update || cat_out) {
#pragma unroll
            for (int i = 0; i < TILE / 4 / kFuThreads; ++i) {
                const int c = tid + i * kFuThreads, r = c / NCH, ch = c % NCH;
                const float4 v = *reinterpret_cast<const float4*>(src + C::at(r, ch));
                if (update) reinterpret_cast<float4*>(F + t * TILE)[c] = v;
                if (cat_out) {
                    float* cw = cat_out + (t * kFuRows + r) * 2 * KP + ch * 4;
                    *reinterpret_cast<float4*>(cw) = v;
                    *reinterpret_cast<float4*>(cw + KP) = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
                }
            }
        }
        FU_MARK(6)  // write back
        // 4. Gram partial of the tile's new rows
        if (gram_live) {
#pragma unroll 4
            for (int r = grg; r < kFuRows; r += C::RG) {
                const float4 a = *reinterpret_cast<const float4*>(src + C::at(r, bi));
                const float4 b = *reinterpret_cast<const float4*>(src + C::at(r, bj));
                const float fa[4] = {a.x, a.y, a.z, a.w}, fb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) gacc[x * 4 + y] = fmaf(fa[x], fb[y], gacc[x * 4 + y]);
            }
        }
        FU_MARK(7)  // Gram
        __syncthreads();  // this stage is refilled by the next iteration's prefetch
        FU_MARK(3)
    }
#ifdef OOC_FU_PROFILE
    if (threadIdx.x == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&g_fu_prof[i], (unsigned long long)prof_acc[i]);
#endif
    cp_async_wait<0>();
    __syncthreads();
    // row groups -> f64 CTA sum in fixed order (partials parked in the stages)
    float* part = stages;
    if (gram_live) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) part[(grg * KP + bi * 4 + x) * KP + bj * 4 + y] = gacc[x * 4 + y];
    }
    __syncthreads();
    double* gout = gram_slots + int64_t(blockIdx.x) * KP * KP;
    for (int e = tid; e < KP * KP; e += kFuThreads) {
        const int i = e / KP, j = e % KP;
        // the upper triangle, mirrored, so the Gram is symmetric to the bit
        const int src_e = i <= j ? e : j * KP + i;
        double sum = 0.0;
        for (int g = 0; g < C::RG; ++g) sum += double(part[g * KP * KP + src_e]);
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

#ifdef OOC_FU_PROFILE
void fu_profile_read(unsigned long long* out, bool reset) {
    cudaMemcpyFromSymbol(out, g_fu_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_fu_prof, z, sizeof z);
    }
}
#endif

int factor_grid(int64_t tiles) {
    static int sms = [] {
        int d = 0, n = 148;
        if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
    }();
    static int64_t per_sm = [] {  // OOCNMF_FU_CTAS_PER_SM: developer knob (tools/fu_bench.cu)
        const char* e = std::getenv("OOCNMF_FU_CTAS_PER_SM");
        const int v = e ? std::atoi(e) : 0;
        return int64_t(v > 0 ? v : FuCfg<32>::CTAS);
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
    if (kp > 64) {  // wide factors: plain numerators only (the solver reduces the group passes)
        if (update && !n_plain) return cudaErrorInvalidValue;
        return launch_factor_update_wide(kp, F, rows, n_plain, G, eps, update, gram_slots, grid, err_slots, flag,
                                         cat_out, s);
    }
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
