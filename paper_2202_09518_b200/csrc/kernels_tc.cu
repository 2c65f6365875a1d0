// Tensor-core (tcgen05, kind::tf32) streaming passes for kp in {16, 32, 64}.
//
// At k = 32 an A-pass needs 16 flop per byte of A; CUDA-core FFMA tops out near 70% of the
// HBM roofline there (SURVEY.md §7 hard part 1), so the contractions move to the 5th-gen
// tensor cores. Single-pass TF32 fails the 1e-4 trace parity, so each tile runs the
// split-precision "3xTF32" scheme
//     A·B ≈ A_hi·B_hi + A_hi·B_lo + A_lo·B_hi,   x_hi = tf32(x) (hardware truncation),
//                                                x_lo = rna_tf32(x - x_hi) (common.cuh tf32_lo)
// with both A halves in TMEM (the split warps tcgen05.st them there, transposing for pass 2)
// and [B_hi | B_lo] in shared memory (B_lo written by the factor-update kernel):
//   kp <= 32:  D' = [H | L]: one N = 2kp MMA A_hi · [B_hi | B_lo], plus A_lo · B_hi into L
//   kp = 64:   hi chain  H  += A_hi · B_hi              (N = kp)
//              lo chain  L  += A_hi · B_lo + A_lo · B_hi (2 x N = kp)
//
// Numerics (tools/bias_probe.py, signed mean relative error of A·Ht vs f64): the tensor
// core's f32 accumulation truncates once per MMA, so one TMEM accumulator carried through a
// tile's whole K range biased the products by -1e-5..-4e-5 — enough to drift low-rank
// trajectories past the 1e-4 parity bar. The hi chain therefore restarts every two K steps
// (128, 16 MMAs) in a fresh TMEM buffer that drain warps add into round-to-nearest f32 register
// sums (kp = 64: the lo chain, values ~2^-11 of H so its own truncation is negligible,
// restarts every LO_UNITS steps). The remaining bias is a constant ~-6e-7 for any K with the
// default 2-step chains (~-3e-7 with 1; FFMA path: unbiased, rms 5e-8..1.3e-7);
// OOCNMF_TC_DRAIN=n sets the hi chain to n steps (developer knob).
//
// Pipeline (one persistent CTA per SM, 16 warps, stream-K split as the FFMA path):
//   warp 0       TMA producer: A ring (32 KB stages, freed by the split warps as soon as the
//                tile is in TMEM) and B ring ([B_hi | B_lo] rows, freed by the MMAs)
//   warps 4..11  split: A tile -> [A_hi | A_lo] TMEM slot (two warpgroups, one K half each)
//   warp 1       MMA issuer (elect.sync, uniform descriptors); commits free B stages and
//                A slots and signal closed hi / lo chains
//   warps 12..15 drain: closed chains -> f32 row sums; at a tile end, row sums -> slot
//
// pass 1 (A·Ht):  D[128 rows x kp] += A[rows, 64 cols] · Ht[64 cols, kp]
//                 A tile row-major (TMA 128B swizzle), B MN-major (Ht is n x kp).
// pass 2 (A^T·W): D[128 cols x kp] += A^T[128 cols, 64 rows] · W[64 rows, kp]
//                 A tile as 4 MN atoms of 32 columns, B MN-major.
// Swizzles (verified on B200 with tools/tc_micro*.cu): MN-major tf32 operands must use
// SWIZZLE_128B_BASE32B (TMA SWIZZLE_128B_ATOM_32B) — with the plain 128B swizzle the MMA
// reads zeros.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "tc_ptx.cuh"

namespace ooc {
using namespace tc;
namespace {

// ------------------------------------------------------------------ kernel
// One pipeline stage covers kTcStep (= 64) K indices: 64 columns of A (pass 1) or 64 rows
// (pass 2). Every stage arrives in two TMA operations (A tile, [B_hi | B_lo] tile) — TMA
// operations, not bytes, bound a single-issuer ring with small boxes (tools/tma_stream_bench.cu).
template <int KP, int PASS>
struct TcCfg {
    static constexpr int BK = kTcStep;                          // K per stage
    static constexpr int KSTEPS = BK / 8;                       // tf32 MMA K = 8
    static constexpr uint32_t ATOM_STRIDE = BK * 128;           // MN-major atoms: BK rows x 128 B
    // Two shared-memory rings. A stages (the streamed 128 x 64 tile) are consumed by the split
    // warps alone — the MMAs read A_hi / A_lo from TMEM — and are released as soon as they are
    // split, so a stage's lifetime is HBM latency + split and the ring keeps enough bytes in
    // flight; B stages ([B_hi | B_lo] factor rows, L2-resident) live until their MMAs retire.
    static constexpr int A_BYTES = 128 * BK * 4;                // 32 KB
    static constexpr int B_BYTES = BK * 2 * KP * 4;             // 8 / 16 / 32 KB
    static constexpr int A_STAGES = KP == 64 ? 4 : (KP == 32 ? 5 : 6);
    static constexpr int B_STAGES = KP == 64 ? 3 : 4;
    // kp <= 32: one N = 2kp MMA writes D' = [H | L] = A_hi · [B_hi | B_lo], a second adds
    // A_lo · B_hi into L, and the drain reads both halves every chunk (16 MMAs per K step).
    // SEP (kp = 64): H and L are separate chains (3 MMAs of N = kp per 8-deep K step); the
    // per-unit drain reads only H's kp columns and L is drained every LO_UNITS units, which
    // halves the drain traffic where D' would be 128 columns. (The tensor pipe is far from
    // bound either way — tools/tc_rate.cu: ~400 cycles per K step at kp = 32 against ~1100
    // for the HBM stream — but under the board's power cap every SM-side byte and
    // instruction costs clock, so the layouts minimise both.)
    static constexpr bool SEP = KP >= 64;
    static constexpr int LO_UNITS = 16;
    static constexpr int ACC_COLS = SEP ? KP : 2 * KP;
    static constexpr int NBUF = KP == 16 ? 3 : 2;               // H (or D') buffers
    static constexpr int NLO = SEP ? 2 : 0;                     // lo buffers
    static constexpr int ASLOTS = KP == 64 ? 2 : 3;             // [A_hi | A_lo] operand slots
    static constexpr int ASLOT_COLS = 2 * BK;
    static constexpr int LO_COL0 = NBUF * ACC_COLS;
    static constexpr int A_COL0 = LO_COL0 + NLO * KP;
    static_assert(A_COL0 + ASLOTS * ASLOT_COLS <= 512, "TMEM budget");
    static_assert(BK == 64, "two split warpgroups, one 32-wide K half each");
    static constexpr int TMEM_COLS = (A_COL0 + ASLOTS * ASLOT_COLS) <= 256 ? 256 : 512;
    static constexpr size_t RING_BYTES = size_t(A_STAGES) * A_BYTES + size_t(B_STAGES) * B_BYTES;
    static constexpr size_t SMEM = RING_BYTES + 1024 /*align*/ + 512 /*barriers*/;
    static_assert(SMEM <= 232448, "shared memory budget");
    // A(TMEM, K-major) · B(MN-major): the hi-chain MMA (N = 2kp writes D' when !SEP) and
    // the N = kp lo-chain MMAs
    static constexpr uint32_t IDESC_HI = idesc_tf32(SEP ? KP : 2 * KP, 0, 1);
    static constexpr uint32_t IDESC_KP = idesc_tf32(KP, 0, 1);
    static constexpr uint32_t LO_DESC_OFF = SEP ? (KP / 32) * ATOM_STRIDE >> 4 : 0;  // B_lo atoms
};

// Unit bookkeeping shared by the MMA issuer and the drain warps: which chains close after
// this unit. Hi chunks are `drain_units` long, lo chunks LO_UNITS; both are cut at tile ends
// and at the CTA's last unit.
struct ChainClock {
    int64_t it;
    int hu = 0, lu = 0;
    __device__ void step(int64_t u, int64_t u1, int64_t ipt, int du, int lo_units, bool& tile_end, bool& hi_close,
                         bool& lo_close) {
        tile_end = ++it == ipt;
        if (tile_end) it = 0;
        const bool cut = tile_end || u + 1 == u1;
        hi_close = cut || ++hu == du;
        lo_close = cut || ++lu == lo_units;
        if (hi_close) hu = 0;
        if (lo_close) lu = 0;
    }
};

template <int KP, int PASS>
__global__ void __launch_bounds__(512, 1)
    k_pass_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              float* __restrict__ slots, StreamK sk, int drain_units, float* __restrict__ out_final,
              unsigned* __restrict__ flags, unsigned epoch) {
    using C = TcCfg<KP, PASS>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned, derived from the __shared__ array so loads compile to LDS, not LD
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::RING_BYTES);
    uint64_t* fullA = bars;                      // [A_STAGES]  TMA -> split
    uint64_t* emptyA = fullA + C::A_STAGES;      // [A_STAGES]  split -> TMA
    uint64_t* fullB = emptyA + C::A_STAGES;      // [B_STAGES]  TMA -> split / MMA
    uint64_t* emptyB = fullB + C::B_STAGES;      // [B_STAGES]  MMA -> TMA
    uint64_t* split = emptyB + C::B_STAGES;      // [ASLOTS]    split -> MMA (A slot + B_lo ready)
    uint64_t* accfull = split + C::ASLOTS;       // [NBUF]
    uint64_t* accempty = accfull + C::NBUF;    // [NBUF]
    uint64_t* afree = accempty + C::NBUF;      // [ASLOTS]
    uint64_t* lofull = afree + C::ASLOTS;      // [NLO]
    uint64_t* loempty = lofull + C::NLO;       // [NLO]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(loempty + C::NLO);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t cta = blockIdx.x;
    const int64_t u0 = sk.begin(cta), u1 = sk.begin(cta + 1);

    if (tid == 0) {
        for (int s = 0; s < C::A_STAGES; ++s) {
            mbar_init(fullA + s, 1);
            mbar_init(emptyA + s, 8);
        }
        for (int s = 0; s < C::B_STAGES; ++s) {
            mbar_init(fullB + s, 1);
            mbar_init(emptyB + s, 1);
        }
        for (int r = 0; r < C::ASLOTS; ++r) mbar_init(split + r, 8);
        for (int b = 0; b < C::NBUF; ++b) {
            mbar_init(accfull + b, 1);
            mbar_init(accempty + b, 4);
        }
        for (int r = 0; r < C::ASLOTS; ++r) mbar_init(afree + r, 1);
        for (int b = 0; b < C::NLO; ++b) {
            mbar_init(lofull + b, 1);
            mbar_init(loempty + b, 4);
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
#ifdef OOC_TC_PROFILE
    long long prof[16] = {};
    const long long t_start = clock64();
#endif

    auto a_stage = [&](int s) { return smem + s * C::A_BYTES; };
    auto b_stage = [&](int s) { return smem + C::A_STAGES * C::A_BYTES + s * C::B_BYTES; };
    // Loop-carried ring / tile counters instead of 64-bit divisions per unit.
    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int sa = 0, sb = 0;
            uint32_t pha = 0, phb = 0;
            int64_t tile = u0 / sk.ipt, it = u0 % sk.ipt;
            for (int64_t u = u0; u < u1; ++u) {
                TC_WAIT(0, mbar_wait(emptyA + sa, pha ^ 1u));
                uint8_t* sA = a_stage(sa);
                mbar_expect_tx(fullA + sa, C::A_BYTES);
                if (PASS == 1)  // rows [tile*128, +128), K-atoms [2 it, 2 it + 2): atom j -> +16 KB
                    tma_load_3d(sA, &tmA, fullA + sa, 0, int(tile * 128), int(it * (C::BK / 32)), kEvictFirst);
                else            // rows [it*64, +64), column atoms [4 tile, +4): atom j -> +8 KB
                    tma_load_3d(sA, &tmA, fullA + sa, 0, int(it * C::BK), int(tile * 4), kEvictFirst);
                if (++sa == C::A_STAGES) sa = 0, pha ^= 1u;
                // factor rows [it*64, +64) of [F | F_lo]: 2kp/32 atoms of 8 KB
                TC_WAIT(1, mbar_wait(emptyB + sb, phb ^ 1u));
                mbar_expect_tx(fullB + sb, C::B_BYTES);
                tma_load_3d(b_stage(sb), &tmB, fullB + sb, 0, int(it * C::BK), 0, kEvictLast);
                if (++sb == C::B_STAGES) sb = 0, phb ^= 1u;
                if (++it == sk.ipt) it = 0, ++tile;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (header: numerics for the chain lengths)
        int sb = 0, r = 0, b = 0, lb = 0;
        uint32_t phb = 0, rph = 0, aph = 0, lph = 0;
        bool hi_open = true, lo_open = true;
        ChainClock clk{u0 % sk.ipt};
        for (int64_t u = u0; u < u1; ++u) {
            if (hi_open) TC_WAIT(5, mbar_wait(accempty + b, aph ^ 1u));
            if (C::SEP && lo_open) TC_WAIT(5, mbar_wait(loempty + lb, lph ^ 1u));
            TC_WAIT(6, mbar_wait(fullB + sb, phb));
            TC_WAIT(7, mbar_wait(split + r, rph));  // A slot r written
            tc_fence_after();
            const uint32_t d = tmem + uint32_t(b * C::ACC_COLS);
            const uint32_t dlo = tmem + uint32_t(C::LO_COL0 + lb * KP);
            // The B descriptor is built warp-uniformly (uniform registers) once per stage; the
            // K steps only add the start-address offset (>> 4) to the low word.
            const uint64_t db0 = desc_mnmajor(smem_u32(b_stage(sb)), 0, C::ATOM_STRIDE);
            const uint32_t ahi = tmem + uint32_t(C::A_COL0 + r * C::ASLOT_COLS), alo = ahi + C::BK;
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < C::KSTEPS; ++kk) {
                    const uint64_t db = db0 + uint64_t(kk * 64);  // [hi atoms | lo atoms]
                    const uint64_t dbl = db + C::LO_DESC_OFF;     // B_lo atoms (SEP)
                    mma_ts(d, ahi + 8 * kk, db, C::IDESC_HI, (hi_open && kk == 0) ? 0u : 1u);
                    if constexpr (C::SEP) {
                        mma_ts(dlo, ahi + 8 * kk, dbl, C::IDESC_KP, (lo_open && kk == 0) ? 0u : 1u);
                        mma_ts(dlo, alo + 8 * kk, db, C::IDESC_KP, 1u);
                    } else {
                        (void)dbl;
                        mma_ts(d + KP, alo + 8 * kk, db, C::IDESC_KP, 1u);
                    }
                }
                mma_commit(emptyB + sb);
                mma_commit(afree + r);
            }
            if (++r == C::ASLOTS) r = 0, rph ^= 1u;
            if (++sb == C::B_STAGES) sb = 0, phb ^= 1u;
            bool tile_end, hi_close, lo_close;
            clk.step(u, u1, sk.ipt, drain_units, C::LO_UNITS, tile_end, hi_close, lo_close);
            if (hi_close) {
                if (elect_one()) mma_commit(accfull + b);
                if (++b == C::NBUF) b = 0, aph ^= 1u;
            }
            if (C::SEP && lo_close) {
                if (elect_one()) mma_commit(lofull + lb);
                if (++lb == C::NLO) lb = 0, lph ^= 1u;
            }
            hi_open = hi_close, lo_open = lo_close;
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 12) {
        // ---------------- split warps: A tile -> [A_hi | A_lo] in TMEM slot r. Two warpgroups:
        // warp w owns TMEM lane quarter w % 4 (tile rows t) and K half h = (w - 4) / 4.
        const int t = 32 * (warp & 3) + lane;  // TMEM lane / tile row owned by this thread
        const int h = (warp - 4) >> 2;
        const uint32_t lane_bits = uint32_t(32 * (warp & 3)) << 16;
        int sa = 0, rs = 0;
        uint32_t pha = 0, rph = 0;
        for (int64_t u = u0; u < u1; ++u) {
            TC_WAIT(2, mbar_wait(fullA + sa, pha));
            TC_WAIT(3, mbar_wait(afree + rs, rph ^ 1u));
            tc_fence_after();
            const uint8_t* sA = a_stage(sa);
            const uint32_t dst = tmem + lane_bits + uint32_t(C::A_COL0 + rs * C::ASLOT_COLS);
            {
                uint32_t r[32], x[32];
                if (PASS == 1) {
                    // row t of K-atom h (K-major SW128): 8 chunks of 16 B, chunk c at (c ^ t%8)
                    const float4* row = reinterpret_cast<const float4*>(sA + h * 16384 + t * 128);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 v = row[c ^ (t & 7)];
                        x[4 * c] = __float_as_uint(v.x), x[4 * c + 1] = __float_as_uint(v.y),
                        x[4 * c + 2] = __float_as_uint(v.z), x[4 * c + 3] = __float_as_uint(v.w);
                        lo_bits2(v.x, v.y, r[4 * c], r[4 * c + 1]);
                        lo_bits2(v.z, v.w, r[4 * c + 2], r[4 * c + 3]);
                    }
                } else {
                    // column t of the MN-major BASE32B tile (atom t/32, element e = t%32), rows
                    // 32h..32h+31: 32-byte granule (e/8) ^ (k%4) of 128-byte row k
                    const float* atom = reinterpret_cast<const float*>(sA + (t >> 5) * C::ATOM_STRIDE);
                    const int e = t & 31;
#pragma unroll
                    for (int kr = 0; kr < 32; kr += 2) {
                        const int k = 32 * h + kr;
                        const float v0 = atom[k * 32 + (((e >> 3) ^ (k & 3)) << 3) + (e & 7)];
                        const float v1 = atom[(k + 1) * 32 + (((e >> 3) ^ ((k + 1) & 3)) << 3) + (e & 7)];
                        x[kr] = __float_as_uint(v0), x[kr + 1] = __float_as_uint(v1);
                        lo_bits2(v0, v1, r[kr], r[kr + 1]);
                    }
                }
                tmem_st32(dst + 32 * h, x);         // A_hi: raw bits, the MMA truncates to tf32
                tmem_st32(dst + C::BK + 32 * h, r);  // A_lo
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(emptyA + sa);  // the tile is in registers / TMEM now
            if (++sa == C::A_STAGES) sa = 0, pha ^= 1u;
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(split + rs);
            if (++rs == C::ASLOTS) rs = 0, rph ^= 1u;
        }
    } else if (warp >= 12) {
        // ---------------- drain warpgroup: closed chains -> f32 row sums; at a tile end (or
        // the CTA's last unit) the tile's row t -> its stream-K slot
        const int t = tid - 384;
        const uint32_t lane_bits = uint32_t(32 * (warp & 3)) << 16;
        float acc[KP];
#pragma unroll
        for (int j = 0; j < KP; ++j) acc[j] = 0.f;
        int64_t tile = u0 / sk.ipt;
        int b = 0, lb = 0;
        uint32_t aph = 0, lph = 0;
        ChainClock clk{u0 % sk.ipt};
        // add one closed chain (D' = [H | L] folded, or one SEP chain) into the row sums
        auto add_cols = [&](uint32_t src) {
            if constexpr (KP == 16) {
                uint32_t v[32];  // D' = [hi(16) | lo(16)] in one 32-column load
                tmem_ld32(src, v);
                acc_add2<16>(acc, v, v + 16);
            } else if constexpr (C::SEP) {  // one chain's kp columns
#pragma unroll
                for (int h = 0; h < KP / 32; ++h) {
                    uint32_t v[32];
                    tmem_ld32(src + h * 32, v);
#pragma unroll
                    for (int j = 0; j < 32; j += 2) add2(acc[32 * h + j], acc[32 * h + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                }
            } else {  // D' = [H | L]
#pragma unroll
                for (int h = 0; h < KP / 32; ++h) {
                    uint32_t hi[32], lo[32];
                    tmem_ld32(src + h * 32, hi);
                    tmem_ld32(src + KP + h * 32, lo);
                    acc_add2<32>(acc + 32 * h, hi, lo);
                }
            }
        };
        for (int64_t u = u0; u < u1; ++u) {
            bool tile_end, hi_close, lo_close;
            clk.step(u, u1, sk.ipt, drain_units, C::LO_UNITS, tile_end, hi_close, lo_close);
            if (hi_close) {
                TC_WAIT(8, mbar_wait(accfull + b, aph));
                tc_fence_after();
                add_cols(tmem + lane_bits + uint32_t(b * C::ACC_COLS));
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(accempty + b);
                if (++b == C::NBUF) b = 0, aph ^= 1u;
            }
            if (C::SEP && lo_close) {
                TC_WAIT(8, mbar_wait(lofull + lb, lph));
                tc_fence_after();
                add_cols(tmem + lane_bits + uint32_t(C::LO_COL0 + lb * KP));
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(loempty + lb);
                if (++lb == C::NLO) lb = 0, lph ^= 1u;
            }
            if (tile_end || u + 1 == u1) {
                // In-kernel stream-K fix-up (out_final set): the CTA holding a tile's FIRST unit
                // finishes that tile last (it reaches it at the end of its range, while the CTAs
                // holding the later units started their ranges with it), so it adds the peers'
                // published partials in ascending CTA order — the order k_streamk_reduce uses —
                // and writes the reduced rows; peers publish their slot and a per-warp flag.
                const bool owner = out_final && tile * sk.ipt >= u0;
                if (owner) {
                    const int64_t c_last = sk.cta_of((tile + 1) * sk.ipt - 1);
                    for (int64_t c = cta + 1; c <= c_last; ++c) {
                        const int64_t sl = sk.slot(c, tile);
                        const unsigned* fl = flags + sl * 4 + (warp & 3);
                        unsigned v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
                        } while (v != epoch);
                        const float4* src = reinterpret_cast<const float4*>(slots + sl * int64_t(128 * KP) +
                                                                            int64_t(t) * KP);
#pragma unroll
                        for (int j4 = 0; j4 < KP / 4; ++j4) {
                            const float4 p = src[j4];
                            acc[4 * j4] += p.x, acc[4 * j4 + 1] += p.y, acc[4 * j4 + 2] += p.z, acc[4 * j4 + 3] += p.w;
                        }
                        // consumed: re-arm the flag for the next launch (graph replays reuse the
                        // same epoch value)
                        __syncwarp();
                        if (lane == 0) *const_cast<unsigned*>(fl) = 0u;
                    }
                }
                float* out = owner ? out_final + (tile * 128 + t) * int64_t(KP)
                                   : slots + sk.slot(cta, tile) * int64_t(128 * KP) + int64_t(t) * KP;
#pragma unroll
                for (int j4 = 0; j4 < KP / 4; ++j4) {
                    reinterpret_cast<float4*>(out)[j4] =
                        make_float4(acc[4 * j4], acc[4 * j4 + 1], acc[4 * j4 + 2], acc[4 * j4 + 3]);
                    acc[4 * j4] = acc[4 * j4 + 1] = acc[4 * j4 + 2] = acc[4 * j4 + 3] = 0.f;
                }
                if (out_final && !owner) {
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) {
                        unsigned* fl = flags + sk.slot(cta, tile) * 4 + (warp & 3);
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl), "r"(epoch) : "memory");
                    }
                }
                ++tile;
            }
        }
    }
#ifdef OOC_TC_PROFILE
    // per role: lane 0 of warp 0 (producer), warp 1 (MMA), warp 4 (split), warp 12 (drain)
    if (lane == 0 && (warp == 0 || warp == 1 || warp == 4 || warp == 12)) {
        for (int j = 0; j < 9; ++j)
            if (prof[j]) atomicAdd(&g_tc_prof[j], (unsigned long long)prof[j]);
        atomicAdd(&g_tc_prof[9 + (warp == 0 ? 0 : warp == 1 ? 1 : warp == 4 ? 2 : 3)],
                  (unsigned long long)(clock64() - t_start));
    }
#endif
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
    }
}

}  // namespace

// ------------------------------------------------------------------ host side
namespace tc {
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

// K steps (64 each) per TMEM accumulation chain; OOCNMF_TC_DRAIN overrides (developer knob).
// 2 steps (16 MMAs, 128 deep): signed bias ≈ -6e-7 relative (tools/bias_probe.py: 1 step
// -3e-7, 4 steps -1.3e-6; 8 steps fails the low-rank 1e-4 trajectory test), half the drain
// work of 1 step — ≈ +3% at config 2 under the power cap.
int tc_drain_units() {
    static int du = [] {
        const char* e = getenv("OOCNMF_TC_DRAIN");
        const int v = e ? atoi(e) : 0;
        return v > 0 ? v : 2;
    }();
    return du;
}
}  // namespace tc
namespace {

template <int KP, int PASS>
cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, float* slots, const StreamK& sk, cudaStream_t s,
                      float* out_final = nullptr, unsigned* flags = nullptr, unsigned epoch = 0) {
    using C = TcCfg<KP, PASS>;
    auto kern = k_pass_tc<KP, PASS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    if (!out_final) {
        kern<<<unsigned(sk.G), 512, C::SMEM, s>>>(a, b, slots, sk, tc_drain_units(), nullptr, nullptr, 0u);
        return cudaGetLastError();
    }
    // The in-kernel fix-up has owner CTAs wait for peers' partials, so every CTA must be
    // resident at once: a cooperative launch guarantees that or fails (MPS SM limits, green
    // contexts, a concurrent kernel holding SMs). On failure the pass runs without the fix-up
    // and the partials go through k_streamk_reduce (same ascending-CTA order, same result).
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(sk.G));
    lc.blockDim = dim3(512);
    lc.dynamicSmemBytes = C::SMEM;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, kern, a, b, slots, sk, tc_drain_units(), out_final, flags, epoch);
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
        cudaGetLastError();
        kern<<<unsigned(sk.G), 512, C::SMEM, s>>>(a, b, slots, sk, tc_drain_units(), nullptr, nullptr, 0u);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        return launch_streamk_reduce(KP, slots, sk, out_final, false, s);
    }
    return e;
}

}  // namespace

#ifdef OOC_TC_PROFILE
void tc_profile_read(unsigned long long* out16, bool reset) {
    cudaMemcpyFromSymbol(out16, g_tc_prof, 16 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
    }
}
#endif

bool tc_supported(int kp) { return (kp == 16 || kp == 32 || kp == 64) && encode_fn() != nullptr; }

// Pass 1 on the tensor cores: A (mp x np, ld lda) K-major, Ht_cat (np x 2kp) MN-major.
cudaError_t launch_aht_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np, const float* Ht_cat,
                          float* slots, const StreamK& sk, cudaStream_t s, int64_t ldb) {
    CUtensorMap ma, mb;
    cudaError_t e;
    if ((e = make_map(&ma, A, mp, np, lda, 128, kTcStep / 32, false)) != cudaSuccess) return e;
    if ((e = make_map(&mb, Ht_cat, np, 2 * kp, ldb ? ldb : 2 * kp, kTcStep, 2 * kp / 32, true)) != cudaSuccess) return e;
    return kp == 16   ? launch_tc<16, 1>(ma, mb, slots, sk, s)
           : kp == 32 ? launch_tc<32, 1>(ma, mb, slots, sk, s)
                      : launch_tc<64, 1>(ma, mb, slots, sk, s);
}

// Pass 2 on the tensor cores: A MN-major (4 column atoms per 128-column tile), W_cat (mp x 2kp).
cudaError_t launch_wta_tc(int kp, const float* A, int64_t lda, int64_t mp, int64_t np, const float* W_cat,
                          float* slots, const StreamK& sk, cudaStream_t s, float* out_final,
                          unsigned* flags, unsigned epoch, int64_t ldb) {
    CUtensorMap ma, mb;
    cudaError_t e;
    if ((e = make_map(&ma, A, mp, np, lda, kTcStep, 4, true)) != cudaSuccess) return e;
    if ((e = make_map(&mb, W_cat, mp, 2 * kp, ldb ? ldb : 2 * kp, kTcStep, 2 * kp / 32, true)) != cudaSuccess) return e;
    return kp == 16   ? launch_tc<16, 2>(ma, mb, slots, sk, s, out_final, flags, epoch)
           : kp == 32 ? launch_tc<32, 2>(ma, mb, slots, sk, s, out_final, flags, epoch)
                      : launch_tc<64, 2>(ma, mb, slots, sk, s, out_final, flags, epoch);
}

}  // namespace ooc
