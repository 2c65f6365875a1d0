// Dense streaming passes over A (the two contractions of one MU iteration).
//
//   pass 1  A·H^T  (reference: matmul_acc dense, src/kernels.cpp:28-45, called from
//                   nmf_serial.cpp:88 / nmf_distributed.cpp:159)
//   pass 2  A^T·W  (reference: matmul_ta_acc dense, src/kernels.cpp:78-101, called from
//                   nmf_serial.cpp:97 / nmf_distributed.cpp:177)
//
// Both are HBM-streaming tall-skinny contractions: every A element is read once per pass
// and used for kp FMAs. Work is split stream-K (common.cuh) over one persistent CTA per
// SM so every SM streams the same number of A bytes; partial tiles go to per-CTA slots
// that the consumer sums in a fixed order (deterministic). A tiles are staged through
// shared memory by a STAGES-deep cp.async ring; the small operand (Ht / W rows) rides in
// the same stage and is read with warp-broadcast 128-bit loads.
//
// This is the CUDA-core (FFMA) path: at kp <= 16 it is HBM-bound (<= 8 flop/B); at
// kp >= 32 FFMA caps it near 70% of the HBM roofline (SURVEY.md §7 hard part 1), which is
// what the tcgen05 path replaces.
#include "kernels.h"

namespace ooc {
namespace {

template <int KP>
struct AhtCfg {
    static constexpr int BM = kTile, BK = 32, STAGES = 4, THREADS = 256, WARPS = 8;
    static constexpr int RG = (KP == 64) ? 2 : 1;  // row groups
    static constexpr int WPG = WARPS / RG;         // warps per row group (split the BK columns)
    static constexpr int TM = 4 / RG;              // rows per thread: lane + 32*i
    static constexpr int CH = RG;                  // 4-column chunks per warp per stage
    static constexpr int AS = BK + 4;              // padded smem row stride: conflict-free LDS.128
    static constexpr int A_STAGE = BM * AS;
    static constexpr int H_STAGE = BK * KP;
    static constexpr int STAGE = A_STAGE + H_STAGE;
    static constexpr int RS = KP + 4;              // reduction scratch row stride
    static constexpr int RED_WARP = 32 * TM * RS;
    static constexpr int RED = (WPG / 2) * RG * RED_WARP;
    static constexpr size_t SMEM = size_t(STAGES * STAGE + RED) * sizeof(float);
};

template <int KP>
__global__ void __launch_bounds__(256, 1)
    k_aht_ffma(const float* __restrict__ A, int64_t lda, const float* __restrict__ Ht,
               float* __restrict__ slots, StreamK sk) {
    using C = AhtCfg<KP>;
    extern __shared__ __align__(16) float smem[];
    float* red = smem + C::STAGES * C::STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp / C::WPG, wl = warp % C::WPG;
    const int rbase = g * 32 * C::TM;

    const int64_t cta = blockIdx.x;
    const int64_t u0 = sk.begin(cta), u1 = sk.begin(cta + 1);

    auto load = [&](int64_t u, int stage) {
        const int64_t tile = u / sk.ipt, it = u % sk.ipt;
        float* As = smem + stage * C::STAGE;
        float* Hs = As + C::A_STAGE;
        const float* src = A + tile * C::BM * lda + it * C::BK;
#pragma unroll
        for (int i = 0; i < (C::BM * C::BK / 4) / C::THREADS; ++i) {
            const int q = tid + i * C::THREADS;
            const int row = q / (C::BK / 4), c4 = q % (C::BK / 4);
            cp_async16(As + row * C::AS + c4 * 4, src + row * lda + c4 * 4);
        }
        const float* hs = Ht + it * C::BK * KP;
        for (int q = tid; q < C::H_STAGE / 4; q += C::THREADS) cp_async16(Hs + q * 4, hs + q * 4);
    };

#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
        if (u0 + s < u1) load(u0 + s, s);
        cp_async_commit();
    }

    float acc[C::TM][KP];
    int64_t u = u0;
    while (u < u1) {
        const int64_t tile = u / sk.ipt;
        const int64_t seg_end = min(u1, (tile + 1) * sk.ipt);
#pragma unroll
        for (int i = 0; i < C::TM; ++i)
#pragma unroll
            for (int j = 0; j < KP; ++j) acc[i][j] = 0.f;

        for (; u < seg_end; ++u) {
            cp_async_wait<C::STAGES - 2>();
            __syncthreads();
            {
                const int64_t nu = u + C::STAGES - 1;
                if (nu < u1) load(nu, int((nu - u0) % C::STAGES));
                cp_async_commit();
            }
            const float* As = smem + int((u - u0) % C::STAGES) * C::STAGE;
            const float* Hs = As + C::A_STAGE;
#pragma unroll
            for (int ch = 0; ch < C::CH; ++ch) {
                const int c = (wl * C::CH + ch) * 4;
                float4 a[C::TM];
#pragma unroll
                for (int i = 0; i < C::TM; ++i)
                    a[i] = *reinterpret_cast<const float4*>(As + (rbase + i * 32 + lane) * C::AS + c);
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const float4* h4 = reinterpret_cast<const float4*>(Hs + (c + cc) * KP);
#pragma unroll
                    for (int j4 = 0; j4 < KP / 4; ++j4) {
                        const float4 hv = h4[j4];
#pragma unroll
                        for (int i = 0; i < C::TM; ++i) {
                            const float av = cc == 0 ? a[i].x : cc == 1 ? a[i].y : cc == 2 ? a[i].z : a[i].w;
                            acc[i][4 * j4 + 0] = fmaf(av, hv.x, acc[i][4 * j4 + 0]);
                            acc[i][4 * j4 + 1] = fmaf(av, hv.y, acc[i][4 * j4 + 1]);
                            acc[i][4 * j4 + 2] = fmaf(av, hv.z, acc[i][4 * j4 + 2]);
                            acc[i][4 * j4 + 3] = fmaf(av, hv.w, acc[i][4 * j4 + 3]);
                        }
                    }
                }
            }
        }
        // Segment done: fixed-shape tree over the WPG warps of each row group.
#pragma unroll
        for (int half = C::WPG / 2; half >= 1; half >>= 1) {
            if (wl >= half && wl < 2 * half) {
                float* dst = red + (g * (C::WPG / 2) + (wl - half)) * C::RED_WARP;
#pragma unroll
                for (int i = 0; i < C::TM; ++i)
#pragma unroll
                    for (int j4 = 0; j4 < KP / 4; ++j4)
                        *reinterpret_cast<float4*>(dst + (i * 32 + lane) * C::RS + 4 * j4) =
                            make_float4(acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2],
                                        acc[i][4 * j4 + 3]);
            }
            __syncthreads();
            if (wl < half) {
                const float* srcp = red + (g * (C::WPG / 2) + wl) * C::RED_WARP;
#pragma unroll
                for (int i = 0; i < C::TM; ++i)
#pragma unroll
                    for (int j4 = 0; j4 < KP / 4; ++j4) {
                        const float4 v =
                            *reinterpret_cast<const float4*>(srcp + (i * 32 + lane) * C::RS + 4 * j4);
                        acc[i][4 * j4] += v.x;
                        acc[i][4 * j4 + 1] += v.y;
                        acc[i][4 * j4 + 2] += v.z;
                        acc[i][4 * j4 + 3] += v.w;
                    }
            }
            __syncthreads();
        }
        if (wl == 0) {
            float* out = slots + sk.slot(cta, tile) * int64_t(C::BM * KP);
#pragma unroll
            for (int i = 0; i < C::TM; ++i) {
                float* orow = out + (rbase + i * 32 + lane) * KP;
#pragma unroll
                for (int j4 = 0; j4 < KP / 4; ++j4)
                    *reinterpret_cast<float4*>(orow + 4 * j4) =
                        make_float4(acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2],
                                    acc[i][4 * j4 + 3]);
            }
        }
    }
    cp_async_wait<0>();
}

template <int KP>
struct WtaCfg {
    static constexpr int BN = kTile, BR = 32, STAGES = 4, THREADS = 256, WARPS = 8;
    static constexpr int JG = (KP == 64) ? 2 : 1;  // j groups (split the kp outputs)
    static constexpr int JW = KP / JG;             // outputs per thread per column
    static constexpr int WPJ = WARPS / JG;         // warps per j group (split the BR rows)
    static constexpr int RPW = BR / WPJ;           // rows per warp per stage
    static constexpr int A_STAGE = BR * BN;
    static constexpr int W_STAGE = BR * KP;
    static constexpr int STAGE = A_STAGE + W_STAGE;
    static constexpr int RED_WARP = JW * BN;
    static constexpr int RED = (WPJ / 2) * JG * RED_WARP;
    static constexpr size_t SMEM = size_t(STAGES * STAGE + RED) * sizeof(float);
};

template <int KP>
__global__ void __launch_bounds__(256, 1)
    k_wta_ffma(const float* __restrict__ A, int64_t lda, const float* __restrict__ W,
               float* __restrict__ slots, StreamK sk) {
    using C = WtaCfg<KP>;
    extern __shared__ __align__(16) float smem[];
    float* red = smem + C::STAGES * C::STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int jg = warp / C::WPJ, wl = warp % C::WPJ;

    const int64_t cta = blockIdx.x;
    const int64_t u0 = sk.begin(cta), u1 = sk.begin(cta + 1);

    auto load = [&](int64_t u, int stage) {
        const int64_t tile = u / sk.ipt, it = u % sk.ipt;
        float* As = smem + stage * C::STAGE;
        float* Ws = As + C::A_STAGE;
        const float* src = A + it * C::BR * lda + tile * C::BN;
#pragma unroll
        for (int i = 0; i < (C::BR * C::BN / 4) / C::THREADS; ++i) {
            const int q = tid + i * C::THREADS;
            const int row = q / (C::BN / 4), c4 = q % (C::BN / 4);
            cp_async16(As + row * C::BN + c4 * 4, src + row * lda + c4 * 4);
        }
        const float* ws = W + it * C::BR * KP;
        for (int q = tid; q < C::W_STAGE / 4; q += C::THREADS) cp_async16(Ws + q * 4, ws + q * 4);
    };

#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
        if (u0 + s < u1) load(u0 + s, s);
        cp_async_commit();
    }

    float acc[C::JW][4];
    int64_t u = u0;
    while (u < u1) {
        const int64_t tile = u / sk.ipt;
        const int64_t seg_end = min(u1, (tile + 1) * sk.ipt);
#pragma unroll
        for (int j = 0; j < C::JW; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

        for (; u < seg_end; ++u) {
            cp_async_wait<C::STAGES - 2>();
            __syncthreads();
            {
                const int64_t nu = u + C::STAGES - 1;
                if (nu < u1) load(nu, int((nu - u0) % C::STAGES));
                cp_async_commit();
            }
            const float* As = smem + int((u - u0) % C::STAGES) * C::STAGE;
            const float* Ws = As + C::A_STAGE;
#pragma unroll
            for (int r = 0; r < C::RPW; ++r) {
                const int row = wl * C::RPW + r;
                const float4 a = *reinterpret_cast<const float4*>(As + row * C::BN + 4 * lane);
                const float4* w4 = reinterpret_cast<const float4*>(Ws + row * KP + jg * C::JW);
#pragma unroll
                for (int j4 = 0; j4 < C::JW / 4; ++j4) {
                    const float4 wv = w4[j4];
                    const float ws[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        acc[4 * j4 + q][0] = fmaf(ws[q], a.x, acc[4 * j4 + q][0]);
                        acc[4 * j4 + q][1] = fmaf(ws[q], a.y, acc[4 * j4 + q][1]);
                        acc[4 * j4 + q][2] = fmaf(ws[q], a.z, acc[4 * j4 + q][2]);
                        acc[4 * j4 + q][3] = fmaf(ws[q], a.w, acc[4 * j4 + q][3]);
                    }
                }
            }
        }
#pragma unroll
        for (int half = C::WPJ / 2; half >= 1; half >>= 1) {
            if (wl >= half && wl < 2 * half) {
                float* dst = red + (jg * (C::WPJ / 2) + (wl - half)) * C::RED_WARP;
#pragma unroll
                for (int j = 0; j < C::JW; ++j)
                    *reinterpret_cast<float4*>(dst + j * C::BN + 4 * lane) =
                        make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
            }
            __syncthreads();
            if (wl < half) {
                const float* srcp = red + (jg * (C::WPJ / 2) + wl) * C::RED_WARP;
#pragma unroll
                for (int j = 0; j < C::JW; ++j) {
                    const float4 v = *reinterpret_cast<const float4*>(srcp + j * C::BN + 4 * lane);
                    acc[j][0] += v.x;
                    acc[j][1] += v.y;
                    acc[j][2] += v.z;
                    acc[j][3] += v.w;
                }
            }
            __syncthreads();
        }
        if (wl == 0) {
            float* out = slots + sk.slot(cta, tile) * int64_t(C::BN * KP);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float* orow = out + (4 * lane + q) * KP + jg * C::JW;
#pragma unroll
                for (int j4 = 0; j4 < C::JW / 4; ++j4)
                    *reinterpret_cast<float4*>(orow + 4 * j4) =
                        make_float4(acc[4 * j4][q], acc[4 * j4 + 1][q], acc[4 * j4 + 2][q],
                                    acc[4 * j4 + 3][q]);
            }
        }
    }
    cp_async_wait<0>();
}

template <class K>
cudaError_t launch_sk(K kernel, size_t smem, const StreamK& sk, cudaStream_t s, const float* A,
                      int64_t lda, const float* B, float* slots) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    kernel<<<dim3(unsigned(sk.G)), dim3(256), smem, s>>>(A, lda, B, slots, sk);
    return cudaGetLastError();
}

}  // namespace

void plan_aht(StreamK& sk, int64_t mp, int64_t np, int num_sms, int step) {
    sk.plan(mp / kTile, np / step, num_sms);
}
void plan_wta(StreamK& sk, int64_t mp, int64_t np, int num_sms, int step) {
    sk.plan(np / kTile, mp / step, num_sms);
}

cudaError_t launch_aht(int kp, const float* A, int64_t lda, const float* Ht, float* slots,
                       const StreamK& sk, cudaStream_t s) {
    switch (kp) {
        case 8: return launch_sk(k_aht_ffma<8>, AhtCfg<8>::SMEM, sk, s, A, lda, Ht, slots);
        case 16: return launch_sk(k_aht_ffma<16>, AhtCfg<16>::SMEM, sk, s, A, lda, Ht, slots);
        case 32: return launch_sk(k_aht_ffma<32>, AhtCfg<32>::SMEM, sk, s, A, lda, Ht, slots);
        case 64: return launch_sk(k_aht_ffma<64>, AhtCfg<64>::SMEM, sk, s, A, lda, Ht, slots);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_wta(int kp, const float* A, int64_t lda, const float* W, float* slots,
                       const StreamK& sk, cudaStream_t s) {
    switch (kp) {
        case 8: return launch_sk(k_wta_ffma<8>, WtaCfg<8>::SMEM, sk, s, A, lda, W, slots);
        case 16: return launch_sk(k_wta_ffma<16>, WtaCfg<16>::SMEM, sk, s, A, lda, W, slots);
        case 32: return launch_sk(k_wta_ffma<32>, WtaCfg<32>::SMEM, sk, s, A, lda, W, slots);
        case 64: return launch_sk(k_wta_ffma<64>, WtaCfg<64>::SMEM, sk, s, A, lda, W, slots);
    }
    return cudaErrorInvalidValue;
}

}  // namespace ooc
