// Developer probe: sustained rate of the kind::tf32 MMA patterns the split-precision passes
// can use (one CTA per SM, garbage operands), alone and with concurrent tcgen05.st / ld
// traffic from other warps. Prints cycles per 64-deep K step ("unit"). Not part of the
// product. build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 tools/tc_rate.cu -o tools/tc_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
           (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ts16(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss16(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t p = 0;
    asm volatile("{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n selp.u32 %0, 1, 0, q;\n}" : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    } while (!ok);
}

// pattern: 0 = 8 x [SS N=64 + TS N=32]   (A_hi from smem, [B_hi|B_lo] in one MMA)
//          1 = 8 x [TS N=64 + TS N=32]   (A_hi from TMEM)
//          2 = 8 x [TS N=32 x 3]         (separate hi / lo chains, A from TMEM)
//          3 = 8 x [SS N=32 x 2 + TS N=32]
//          4 = 8 x [TS N=128 + TS N=64]  (kp = 64, one N = 2kp MMA)
//          5 = 8 x [TS N=32 + TS N=16]   (kp = 16)
// st_warps: warps doing 2 x tcgen05.st.32x32b.x32 per unit (8 = the split warpgroups)
// ld_warps: warps doing 1 x tcgen05.ld.32x32b.x32 per unit (4 = the drain warpgroup)
template <int pattern>
__global__ void __launch_bounds__(512, 1) k_rate(int units, int st_warps, int ld_warps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f800000u;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    const long long t0 = clock64();
    if (warp == 1) {
        const uint32_t a_s = su32(sm), b_s = su32(sm + 32768);
        const uint64_t da0 = sdesc(a_s, 16, 1024, 2);
        const uint64_t db0 = sdesc(b_s, 8192, 512, 1);
        const uint32_t acc = tm, a_hi = tm + 384, a_lo = tm + 448;
        for (int u = 0; u < units; ++u) {
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t da = da0 + uint64_t((((kk >> 2) * 16384 + (kk & 3) * 32) >> 4));
                    const uint64_t db = db0 + uint64_t(kk * 64);
                    switch (pattern) {  // compile-time: operands stay in uniform registers
                        case 0: mma_ss(acc, da, db, idesc(64, 0, 1), kk); mma_ts(acc + 32, a_lo + 8 * kk, db, idesc(32, 0, 1), 1); break;
                        case 1: mma_ts(acc, a_hi + 8 * kk, db, idesc(64, 0, 1), kk); mma_ts(acc + 32, a_lo + 8 * kk, db, idesc(32, 0, 1), 1); break;
                        case 2:
                            mma_ts(acc, a_hi + 8 * kk, db, idesc(32, 0, 1), kk);
                            mma_ts(acc + 64, a_hi + 8 * kk, db + 512, idesc(32, 0, 1), 1);
                            mma_ts(acc + 64, a_lo + 8 * kk, db, idesc(32, 0, 1), 1);
                            break;
                        case 3:
                            mma_ss(acc, da, db, idesc(32, 0, 1), kk);
                            mma_ss(acc + 64, da, db + 512, idesc(32, 0, 1), 1);
                            mma_ts(acc + 64, a_lo + 8 * kk, db, idesc(32, 0, 1), 1);
                            break;
                        case 4: mma_ts(acc, a_hi + 8 * kk, db, idesc(128, 0, 1), kk); mma_ts(acc + 128, a_lo + 8 * kk, db, idesc(64, 0, 1), 1); break;
                        case 5: mma_ts(acc, a_hi + 8 * kk, db, idesc(32, 0, 1), kk); mma_ts(acc + 16, a_lo + 8 * kk, db, idesc(16, 0, 1), 1); break;
                        case 6: {  // kp = 32, two interleaved [H|L] accumulators
                            const uint32_t dd = acc + 64 * (kk & 1);
                            mma_ts(dd, a_hi + 8 * kk, db, idesc(64, 0, 1), kk > 1);
                            mma_ts(dd + 32, a_lo + 8 * kk, db, idesc(32, 0, 1), 1);
                            break;
                        }
                        case 7: {  // kp = 32, four interleaved [H|L] accumulators
                            const uint32_t dd = acc + 64 * (kk & 3);
                            mma_ts(dd, a_hi + 8 * kk, db, idesc(64, 0, 1), kk > 3);
                            mma_ts(dd + 32, a_lo + 8 * kk, db, idesc(32, 0, 1), 1);
                            break;
                        }
                        case 8: {  // kp = 32, [H|L] then A_lo into a separate L2 (no overlap)
                            mma_ts(acc, a_hi + 8 * kk, db, idesc(64, 0, 1), kk);
                            mma_ts(acc + 64, a_lo + 8 * kk, db, idesc(32, 0, 1), kk);
                            break;
                        }
                        case 9: {  // kp = 32, pattern 8 with two interleaved sets
                            const uint32_t dd = acc + 96 * (kk & 1);
                            mma_ts(dd, a_hi + 8 * kk, db, idesc(64, 0, 1), kk > 1);
                            mma_ts(dd + 64, a_lo + 8 * kk, db, idesc(32, 0, 1), kk > 1);
                            break;
                        }
                        case 10: {  // kp = 64, two interleaved sets, separate L2
                            const uint32_t dd = acc + 0;
                            mma_ts(dd + 192 * (kk & 1) - 0, a_hi + 8 * kk, db, idesc(128, 0, 1), kk > 1);
                            mma_ts(dd + 192 * (kk & 1) + 128, a_lo + 8 * kk, db, idesc(64, 0, 1), kk > 1);
                            break;
                        }
                        case 12:  // bf16x6, kp = 32: per K=16 step A0·[c0|c1|c2], A1·[c0|c1], A2·c0
                            if (kk < 4) {
                                mma_ts16(acc, a_hi + 8 * kk, db, idesc_bf16(96), kk);
                                mma_ts16(acc + 32, a_hi + 32 + 8 * kk, db, idesc_bf16(64), 1);
                                mma_ts16(acc + 64, a_lo + 8 * kk, db, idesc_bf16(32), 1);
                            }
                            break;
                        case 13:  // bf16x6, kp = 64
                            if (kk < 4) {
                                mma_ts16(acc, a_hi + 8 * kk, db, idesc_bf16(192), kk);
                                mma_ts16(acc + 64, a_hi + 32 + 8 * kk, db, idesc_bf16(128), 1);
                                mma_ts16(acc + 128, a_lo + 8 * kk, db, idesc_bf16(64), 1);
                            }
                            break;
                        case 14:  // bf16 K-stacked: 8 x N=96 + 4 x N=32
                            mma_ts16(acc, a_hi + 8 * kk, db, idesc_bf16(96), kk);
                            if (kk & 1) mma_ts16(acc + 64, a_lo + 4 * kk, db, idesc_bf16(32), 1);
                            break;
                        case 15:  // bf16x6 SS, kp = 32
                            if (kk < 4) {
                                mma_ss16(acc, da, db, idesc_bf16(96), kk);
                                mma_ss16(acc + 32, da + 64, db, idesc_bf16(64), 1);
                                mma_ss16(acc + 64, da + 128, db, idesc_bf16(32), 1);
                            }
                            break;
                        case 16:  // tf32 kp = 32 with 4 products in N=64 twice (16 instr, control)
                            mma_ts(acc, a_hi + 8 * kk, db, idesc(64, 0, 1), kk);
                            mma_ts(acc, a_lo + 8 * kk, db, idesc(64, 0, 1), 1);
                            break;
                        case 11: {  // kp = 16, [H|L] + separate L2, two interleaved sets
                            const uint32_t dd = acc + 48 * (kk & 1);
                            mma_ts(dd, a_hi + 8 * kk, db, idesc(32, 0, 1), kk > 1);
                            mma_ts(dd + 32, a_lo + 8 * kk, db, idesc(16, 0, 1), kk > 1);
                            break;
                        }
                        default: break;
                    }
                }
                if (u == units - 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
            }
            __syncwarp();
        }
        wait_bar(&bar[0], 0);
        if ((tid & 31) == 0) out[blockIdx.x * 3 + 0] = clock64() - t0;
    } else if (warp >= 4 && warp < 4 + st_warps && warp < 12) {
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = 0x3f800000u + j;
        const uint32_t dst = tm + 384 + (uint32_t(32 * (warp & 3)) << 16) + 32 * ((warp - 4) >> 2);
        for (int u = 0; u < units; ++u) {
            for (int h = 0; h < 2; ++h)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                             ::"r"(dst + 64 * h), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            r[u & 31] += 1;
        }
        if ((tid & 31) == 0 && warp == 4) out[blockIdx.x * 3 + 1] = clock64() - t0;
    } else if (warp >= 12 && warp < 12 + ld_warps) {
        uint32_t s = 0;
        const uint32_t src = tm + 128 + (uint32_t(32 * (warp & 3)) << 16);
        for (int u = 0; u < units; ++u) {
            uint32_t v[32];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\ttcgen05.wait::ld.sync.aligned;"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                         : "r"(src) : "memory");
            for (int j = 0; j < 32; ++j) s += v[j];
        }
        if ((tid & 31) == 0 && warp == 12) out[blockIdx.x * 3 + 2] = clock64() - t0 + (s == 12345u);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
    }
}

int main() {
    const int G = 148, U = 4000;
    unsigned long long* d;
    cudaMalloc(&d, G * 3 * sizeof(unsigned long long));
    void (*kern[17])(int, int, int, unsigned long long*) = {k_rate<0>, k_rate<1>, k_rate<2>, k_rate<3>, k_rate<4>, k_rate<5>,
                                                            k_rate<6>, k_rate<7>, k_rate<8>, k_rate<9>, k_rate<10>, k_rate<11>,
                                                            k_rate<12>, k_rate<13>, k_rate<14>, k_rate<15>, k_rate<16>};
    for (auto k : kern) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char* names[] = {"SS64+TS32", "TS64+TS32", "TS32x3", "SS32x2+TS32", "TS128+TS64", "TS32+TS16",
                           "2x[TS64+TS32]", "4x[TS64+TS32]", "TS64|TS32sep", "2x[64|32sep]", "2x[128|64sep]", "2x[32|16sep]",
                           "bf16x6 kp32", "bf16x6 kp64", "bf16 kstack", "bf16x6 SS", "tf32 2xTS64"};
    for (int p = 0; p < 17; ++p)
        for (int cfg = 0; cfg < 4; cfg += 3) {
            const int st = (cfg & 1) ? 8 : 0, ld = (cfg & 2) ? 4 : 0;
            cudaMemset(d, 0, G * 3 * sizeof(unsigned long long));
            kern[p]<<<G, 512, 100 * 1024>>>(U, st, ld, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h[G * 3];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m = 0, s = 0, l = 0;
            for (int i = 0; i < G; ++i) m += h[3 * i], s += h[3 * i + 1], l += h[3 * i + 2];
            printf("%-12s st_warps %d ld_warps %d : mma %.0f  st %.0f  ld %.0f cycles/unit\n", names[p], st, ld,
                   m / G / U, s / G / U, l / G / U);
        }
    return 0;
}
