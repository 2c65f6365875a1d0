// Tensor-core (tcgen05, kind::tf32) streaming passes for kp in {32, 64}.
//
// At k = 32 an A-pass needs 16 flop per byte of A; CUDA-core FFMA tops out near 70% of the
// HBM roofline there (SURVEY.md §7 hard part 1), so the contractions move to the 5th-gen
// tensor cores. Single-pass TF32 fails the 1e-4 trace parity, so each tile runs the
// split-precision "3xTF32" scheme
//     A·B ≈ A_hi·B_hi + A_hi·B_lo + A_lo·B_hi,   x_hi = tf32(x) (hardware truncation),
//                                                x_lo = x - x_hi (exact in f32)
// arranged so the streamed A tile is read from shared memory only once per K step:
//   MMA 1 (SS): D'[:, 0:2kp] += A_hi(smem) · [B_hi | B_lo](smem)     one N = 2kp MMA
//   MMA 2 (TS): D'[:, 0:kp]  += A_lo(TMEM) · B_hi(smem)              A_lo never touches smem
//   epilogue:   D = D'[:, 0:kp] + D'[:, kp:2kp]
// A_hi is the raw f32 tile TMA lands in shared memory (the MMA reads only its tf32 bits);
// A_lo is produced by four "split" warps that read the tile and tcgen05.st the low halves
// straight into TMEM in the K-major operand layout (transposing for pass 2); B_lo
// (Ht_lo / W_lo) is written by the factor-update kernel that produced B.
//
// Pipeline (one persistent CTA per SM, stream-K split as the FFMA path):
//   warp 0      TMA producer: A tile + B_hi + B_lo per stage                 -> full[s]
//   warps 4..7  split: A_lo[s] -> TMEM                                        -> split[s]
//   warp 1      MMA issuer; commit -> empty[s] (smem stage + TMEM A_lo slot free) and, at
//               a tile end, -> accfull[b]
//   warps 4..7  epilogue at tile ends: tcgen05.ld the 128 x 2kp accumulator -> slot -> accempty[b]
//
// pass 1 (A·Ht):  D[128 rows x kp] += A[rows, 32 cols] · Ht[32 cols, kp]
//                 A K-major (row-major A tile), B MN-major (Ht is n x kp).
// pass 2 (A^T·W): D[128 cols x kp] += A^T[128 cols, 32 rows] · W[32 rows, kp]
//                 A MN-major (4 atoms of 32 columns), B MN-major.
// Swizzles (verified on B200 with tools/tc_micro*.cu): K-major tf32 operands use
// SWIZZLE_128B (TMA SWIZZLE_128B); MN-major tf32 operands must use SWIZZLE_128B_BASE32B
// (TMA SWIZZLE_128B_ATOM_32B) — with the plain 128B swizzle the MMA reads zeros.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.h"

namespace ooc {
namespace {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
// L2 eviction policies (the encodings CUTLASS uses for TMA cache hints).
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull, kEvictLast = 0x14F0000000000000ull;
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "l"(policy)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t p = 0;
    asm volatile("{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n selp.u32 %0, 1, 0, q;\n}" : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, version 1 (sm_100). Layout 2 = SWIZZLE_128B (16-byte
// granules XOR row%8), layout 1 = SWIZZLE_128B_BASE32B (32-byte granules XOR row%4).
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW128B32 = 1;
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}
// K-major, 128-byte rows of K, 8-row swizzle groups; one MMA K step (8 x f32) = +32 B.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int kk) {
    return sdesc(base + kk * 32, 16, 1024, kLayoutSW128);
}
// MN-major, 128-byte rows of MN (32 f32), one row per K index, 4-row swizzle groups (512 B),
// MN atoms of 32 elements every `atom_stride` bytes; one MMA K step (8 rows) = +1024 B.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int kk, uint32_t atom_stride) {
    return sdesc(base + kk * 1024, atom_stride, 512, kLayoutSW128B32);
}
// Instruction descriptor: kind::tf32, f32 accumulate, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
           (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(
            d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

#define OOC_R32(r)                                                                                               \
    "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),  \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),   \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),  \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define OOC_W32(r)                                                                                               \
    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), \
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),          \
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),          \
        "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])

// 32 consecutive 32-bit TMEM columns of this warp's 32 lanes <-> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
    // wait::ld inside the same asm: the destination registers are only defined after it.
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
        "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : OOC_R32(r)
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%"
        "18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\t"
        "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
        OOC_W32(r)
        : "memory");
}

__device__ __forceinline__ uint32_t lo_bits(float x) {
    return __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}

// ------------------------------------------------------------------ kernel
// One pipeline stage covers kTcStep (= 64) K indices: 64 columns of A (pass 1) or 64 rows
// (pass 2). Every stage arrives in two TMA operations (A tile, [B_hi | B_lo] tile) — TMA
// operations, not bytes, bound a single-issuer ring with small boxes (tools/tma_stream_bench.cu).
template <int KP, int PASS>
struct TcCfg {
    static constexpr int BK = kTcStep;                          // K per stage
    static constexpr int KSTEPS = BK / 8;                       // tf32 MMA K = 8
    static constexpr int A_BYTES = 128 * BK * 4;                // 32 KB
    static constexpr int B_BYTES = BK * 2 * KP * 4;             // [B_hi | B_lo], 16 / 32 KB
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = KP == 32 ? 4 : 3;
    static constexpr uint32_t TX_BYTES = STAGE_BYTES;
    static constexpr uint32_t ATOM_STRIDE = BK * 128;           // MN-major atoms: BK rows x 128 B
    static constexpr int ACC_COLS = 2 * KP;                     // D' = [hi | lo] per accumulator
    static constexpr int ALO_COL0 = 2 * ACC_COLS;               // A_lo slots after 2 accumulators
    static constexpr int TMEM_COLS = (ALO_COL0 + STAGES * BK) <= 256 ? 256 : 512;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr uint32_t IDESC_SS = idesc_tf32(2 * KP, PASS == 2 ? 1 : 0, 1);  // A_hi · [B_hi|B_lo]
    static constexpr uint32_t IDESC_TS = idesc_tf32(KP, 0, 1);                       // A_lo(TMEM) · B_hi
};

template <int KP, int PASS>
__global__ void __launch_bounds__(256, 1)
    k_pass_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              float* __restrict__ slots, StreamK sk) {
    using C = TcCfg<KP, PASS>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t* full = bars;                     // [STAGES]
    uint64_t* split = bars + C::STAGES;        // [STAGES]
    uint64_t* empty = bars + 2 * C::STAGES;    // [STAGES]
    uint64_t* accfull = bars + 3 * C::STAGES;  // [2]
    uint64_t* accempty = accfull + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t cta = blockIdx.x;
    const int64_t u0 = sk.begin(cta), u1 = sk.begin(cta + 1);

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(split + s, 4);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accfull + b, 1);
            mbar_init(accempty + b, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto stage_ptr = [&](int s) { return smem + s * C::STAGE_BYTES; };
    // Loop-carried ring / tile counters instead of 64-bit divisions per unit.
    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            int64_t tile = u0 / sk.ipt, it = u0 % sk.ipt;
            for (int64_t u = u0; u < u1; ++u) {
                mbar_wait(empty + s, ph ^ 1u);
                uint8_t* sA = stage_ptr(s);
                mbar_expect_tx(full + s, C::TX_BYTES);
                if (PASS == 1)  // rows [tile*128, +128), K-atoms [2 it, 2 it + 2): atom j -> +16 KB
                    tma_load_3d(sA, &tmA, full + s, 0, int(tile * 128), int(it * (C::BK / 32)), kEvictFirst);
                else            // rows [it*64, +64), column atoms [4 tile, +4): atom j -> +8 KB
                    tma_load_3d(sA, &tmA, full + s, 0, int(it * C::BK), int(tile * 4), kEvictFirst);
                // factor rows [it*64, +64) of [F | F_lo]: 2kp/32 atoms of 8 KB
                tma_load_3d(sA + C::A_BYTES, &tmB, full + s, 0, int(it * C::BK), 0, kEvictLast);
                if (++s == C::STAGES) s = 0, ph ^= 1u;
                if (++it == sk.ipt) it = 0, ++tile;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int s = 0;
        uint32_t ph = 0;
        int64_t sg = 0;
        int64_t u = u0;
        int64_t tile = u0 / sk.ipt;
        while (u < u1) {
            const int64_t seg_end = min(u1, (tile + 1) * sk.ipt);
            const int b = int(sg & 1);
            mbar_wait(accempty + b, (uint32_t(sg >> 1) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem + uint32_t(b * C::ACC_COLS);
            for (bool first = true; u < seg_end; ++u, first = false) {
                mbar_wait(split + s, ph);  // implies full[s]: the split warps waited on it
                tc_fence_after();
                // Descriptors are built warp-uniformly (uniform registers) once per stage; the
                // K steps only add the start-address offset (>> 4) to the low word.
                const uint32_t a0 = smem_u32(stage_ptr(s));
                const uint64_t da0 = PASS == 1 ? desc_kmajor(a0, 0) : desc_mnmajor(a0, 0, C::ATOM_STRIDE);
                const uint64_t db0 = desc_mnmajor(a0 + C::A_BYTES, 0, C::ATOM_STRIDE);  // [hi atoms | lo atoms]
                const uint32_t alo = tmem + uint32_t(C::ALO_COL0 + C::BK * s);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < C::KSTEPS; ++kk) {
                        const uint64_t da =
                            da0 + uint64_t(PASS == 1 ? (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4) : kk * 64);
                        const uint64_t db = db0 + uint64_t(kk * 64);
                        mma_ss(d, da, db, C::IDESC_SS, (first && kk == 0) ? 0u : 1u);
                        mma_ts(d, alo + 8 * kk, db, C::IDESC_TS, 1u);
                    }
                    mma_commit(empty + s);
                    if (u + 1 == seg_end) mma_commit(accfull + b);
                }
                __syncwarp();
                if (++s == C::STAGES) s = 0, ph ^= 1u;
            }
            ++sg;
            ++tile;
        }
    } else if (warp >= 4) {
        // ---------------- split (A_lo -> TMEM) + epilogue warpgroup
        const int t = tid - 128;  // TMEM lane / D row owned by this thread
        const int q = warp - 4;   // this warp's TMEM lane quarter [32q, 32q+32)
        const uint32_t lane_bits = uint32_t(32 * q) << 16;
        int s = 0;
        uint32_t ph = 0;
        int64_t sg = 0;
        int64_t tile = u0 / sk.ipt, it = u0 % sk.ipt;
        for (int64_t u = u0; u < u1; ++u) {
            mbar_wait(full + s, ph);
            const uint8_t* sA = stage_ptr(s);
            const uint32_t dst = tmem + lane_bits + uint32_t(C::ALO_COL0 + C::BK * s);
#pragma unroll
            for (int h = 0; h < C::BK / 32; ++h) {
                uint32_t r[32];
                if (PASS == 1) {
                    // row t of K-atom h (K-major SW128): 8 chunks of 16 B, chunk c at (c ^ t%8)
                    const float4* row = reinterpret_cast<const float4*>(sA + h * 16384 + t * 128);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 v = row[c ^ (t & 7)];
                        r[4 * c] = lo_bits(v.x), r[4 * c + 1] = lo_bits(v.y), r[4 * c + 2] = lo_bits(v.z),
                        r[4 * c + 3] = lo_bits(v.w);
                    }
                } else {
                    // column t of the MN-major BASE32B tile (atom t/32, element e = t%32), rows
                    // 32h..32h+31: 32-byte granule (e/8) ^ (k%4) of 128-byte row k
                    const float* atom = reinterpret_cast<const float*>(sA + (t >> 5) * C::ATOM_STRIDE);
                    const int e = t & 31;
#pragma unroll
                    for (int kr = 0; kr < 32; ++kr) {
                        const int k = 32 * h + kr;
                        r[kr] = lo_bits(atom[k * 32 + (((e >> 3) ^ (k & 3)) << 3) + (e & 7)]);
                    }
                }
                tmem_st32(dst + 32 * h, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(split + s);
            if (++s == C::STAGES) s = 0, ph ^= 1u;

            if (u + 1 == min(u1, (tile + 1) * sk.ipt)) {
                const int b = int(sg & 1);
                mbar_wait(accfull + b, uint32_t(sg >> 1) & 1u);
                tc_fence_after();
                float* out = slots + sk.slot(cta, tile) * int64_t(128 * KP) + int64_t(t) * KP;
#pragma unroll
                for (int h = 0; h < KP / 32; ++h) {
                    uint32_t hi[32], lo[32];
                    tmem_ld32(tmem + lane_bits + uint32_t(b * C::ACC_COLS + h * 32), hi);
                    tmem_ld32(tmem + lane_bits + uint32_t(b * C::ACC_COLS + KP + h * 32), lo);
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4)
                        reinterpret_cast<float4*>(out + h * 32)[j4] =
                            make_float4(__uint_as_float(hi[4 * j4]) + __uint_as_float(lo[4 * j4]),
                                        __uint_as_float(hi[4 * j4 + 1]) + __uint_as_float(lo[4 * j4 + 1]),
                                        __uint_as_float(hi[4 * j4 + 2]) + __uint_as_float(lo[4 * j4 + 2]),
                                        __uint_as_float(hi[4 * j4 + 3]) + __uint_as_float(lo[4 * j4 + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(accempty + b);
                ++sg;
            }
            if (++it == sk.ipt) it = 0, ++tile;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
    }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// View a row-major f32 matrix [rows][cols] (ld floats) as 3-D (32 columns of an atom, rows,
// cols/32 atoms) and box (32, box_rows, box_atoms): one TMA operation lands box_atoms
// atoms of box_rows x 128 B, atom j at j * box_rows * 128 B in shared memory. K-major tiles
// use the 16-byte-granule 128B swizzle, MN-major ones the 32-byte-granule variant that
// matches UMMA's SWIZZLE_128B_BASE32B layout.
cudaError_t make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int box_atoms, bool mn_major) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {32u, cuuint64_t(rows), cuuint64_t(cols / 32)};
    const cuuint64_t strides[2] = {cuuint64_t(ld) * 4, 128u};
    const cuuint32_t box[3] = {32u, cuuint32_t(box_rows), cuuint32_t(box_atoms)};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int KP, int PASS>
cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, float* slots, const StreamK& sk, cudaStream_t s) {
    using C = TcCfg<KP, PASS>;
    auto kern = k_pass_tc<KP, PASS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<unsigned(sk.G), 256, C::SMEM, s>>>(a, b, slots, sk);
    return cudaGetLastError();
}

}  // namespace

bool tc_supported(int kp) { return (kp == 32 || kp == 64) && encode_fn() != nullptr; }

// Pass 1 on the tensor cores: A (mp x np, ld lda) K-major, Ht_cat (np x 2kp) MN-major.
cudaError_t launch_aht_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np, const float* Ht_cat,
                          float* slots, const StreamK& sk, cudaStream_t s) {
    CUtensorMap ma, mb;
    cudaError_t e;
    if ((e = make_map(&ma, A, mp, np, lda, 128, kTcStep / 32, false)) != cudaSuccess) return e;
    if ((e = make_map(&mb, Ht_cat, np, 2 * kp, 2 * kp, kTcStep, 2 * kp / 32, true)) != cudaSuccess) return e;
    return kp == 32 ? launch_tc<32, 1>(ma, mb, slots, sk, s) : launch_tc<64, 1>(ma, mb, slots, sk, s);
}

// Pass 2 on the tensor cores: A MN-major (4 column atoms per 128-column tile), W_cat (mp x 2kp).
cudaError_t launch_wta_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np, const float* W_cat,
                          float* slots, const StreamK& sk, cudaStream_t s) {
    CUtensorMap ma, mb;
    cudaError_t e;
    if ((e = make_map(&ma, A, mp, np, lda, kTcStep, 4, true)) != cudaSuccess) return e;
    if ((e = make_map(&mb, W_cat, mp, 2 * kp, 2 * kp, kTcStep, 2 * kp / 32, true)) != cudaSuccess) return e;
    return kp == 32 ? launch_tc<32, 2>(ma, mb, slots, sk, s) : launch_tc<64, 2>(ma, mb, slots, sk, s);
}

}  // namespace ooc
