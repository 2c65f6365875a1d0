// One-pass dense MU W-half (tcgen05, kind::tf32, 3xTF32): A crosses HBM once per iteration.
//
// The reference's RNMF worker (src/nmf_distributed.cpp:151-185) and nmf_serial
// (src/nmf_serial.cpp:84-101) run two contractions over A per iteration: A·H^T for the W update,
// then W^T·A with the NEW W for the H update. Done as two streaming passes (kernels_tc.cu) that
// is 2|A| of HBM traffic. Both contractions of a 128-row block of A only need that block and the
// block's new W rows, so this persistent kernel walks the row blocks once:
//
//   P1(b)  A[b, :]·Ht partials       (A block read from HBM; lands in L2)
//   U(b)   W[b] <- W[b] * (A·Ht)[b] / (W[b]·HH^T + eps), [W | W_lo][b]   (updater warps)
//   P2(b)  W^T A[:, cols] += W[b]^T · A[b, cols]   (the same block re-read from L2)
//
// with P2 running D blocks behind P1, so the A bytes of a block stay L2-resident (D + 1 blocks
// of 32 MB at n = 65536) between their two uses and HBM only sees the first.
//
// Work split (148 persistent CTAs, cooperative launch: every CTA waits on others):
//   * P2 is column-owned: CTA c owns the 128-column tiles [t0(c), t1(c)) of W^T A for the whole
//     iteration and accumulates them over the blocks in TMEM (f32, one two-step chain per block,
//     the same drained-chain numerics as kernels_tc.cu), so W^T A needs no cross-CTA reduction.
//   * P1 is column-chunked: CTA c computes the partial A[b, q-chunks]·Ht of its 64-column chunks
//     [q0(c), q1(c)) (chosen so every CTA has the same P1 + P2 unit count per block), drains it
//     into f32 registers and publishes it to a slot ring.
//   * U is row-distributed: row r of block b is gathered (one TMA operation over the 148 slots),
//     reduced (partials in a fixed order: deterministic) and updated by the updater warp of CTA
//     (128 b + r) mod G, which then bumps the block's half-block done-counter; the B producer of
//     every CTA waits for it before loading the block's two [W | W_lo] halves for P2 (once per
//     block, reused for all the CTA's owned tiles). The gathered partial lines are discarded
//     from L2 (dead data must not be written back to HBM), and the updater accumulates the new
//     rows' W^T W in f64 (one slot per CTA) after the release.
// Pipeline per CTA: warp 0 A producer (TMA), warp 3 B producer, warp 1 tcgen05 MMA issuer,
// warps 4-11 split A into [A_hi | A_lo] TMEM slots, warps 12-15 drain, warp 2 the updater; one
// unit sequence
//   for s in [0, NB + D):  P1 units of block s (if s < NB), then P2 units of block s - D.
#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"

namespace ooc {
using namespace tc;
namespace {

template <int KP>
struct FzCfg {
    static constexpr int BK = kTcStep;                 // K per unit (64)
    static constexpr int KSTEPS = BK / 8;
    static constexpr uint32_t ATOM_STRIDE = BK * 128;  // MN-major atoms: BK rows x 128 B
    static constexpr int A_BYTES = 128 * BK * 4;       // 32 KB (P1: 128 rows x 64 cols, P2: 64 x 128)
    static constexpr int B_BYTES = BK * 2 * KP * 4;    // [F | F_lo] rows
    static constexpr int A_STAGES = KP == 32 ? 4 : 5;
    static constexpr int B_STAGES = 4;
    static constexpr int ACC_COLS = 2 * KP;            // D' = [H | L]
    static constexpr int NBUF = 2;
    static constexpr int MAXT = KP == 16 ? 8 : 4;      // owned W^T A tiles (TMEM running sums)
    static constexpr int RUN_COL0 = NBUF * ACC_COLS;
    static constexpr int A_COL0 = RUN_COL0 + MAXT * KP;
    static constexpr int ASLOT_COLS = 2 * BK;
    static constexpr int ASLOTS = (512 - A_COL0) / ASLOT_COLS;
    static_assert(ASLOTS >= 2, "TMEM budget");
    static constexpr int TMEM_COLS = 512;
    static constexpr int MAX_G = 192;                  // CTAs (smem list of P1 publishers)
    static constexpr int RS = KP < 32 ? 32 : KP;       // P1 slot row stride: a whole 128-byte line
    static constexpr size_t RING_BYTES = size_t(A_STAGES) * A_BYTES + size_t(B_STAGES) * B_BYTES;
    static constexpr size_t BAR_BYTES = 512;
    // updater gather buffer: one row of every CTA's published P1 partial (TMA, G x kp floats)
    static constexpr size_t GATHER_OFF = RING_BYTES + BAR_BYTES + MAX_G * 4 + 64 * 4;  // 128-aligned
    static constexpr size_t WGRAM_OFF = GATHER_OFF + size_t(MAX_G) * KP * 4;             // [KP][KP] f64
    static constexpr size_t SMEM = WGRAM_OFF + size_t(KP) * KP * 8 + 1024;
    static_assert(SMEM <= 232448, "shared memory budget");
    static constexpr uint32_t IDESC_HI = idesc_tf32(2 * KP, 0, 1);
    static constexpr uint32_t IDESC_KP = idesc_tf32(KP, 0, 1);
};

// Spin on a device-scope counter (all lanes load with acquire; nanosleep between polls). A
// counter that never arrives (a bug, never a correct run) traps after ~4 s instead of hanging.
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
#ifndef OOC_FZ_SPIN
        __nanosleep(64);
#endif
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) return;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 4000000000ull) asm volatile("trap;");
    }
}
// Publish: after the warp's stores (__syncwarp orders them before lane 0's release), one
// gpu-scope release add on the counter (no separate membar.gl).
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
#ifdef OOC_FZ_AB_FENCE  // developer A/B: membar.gl + relaxed add
    __threadfence();
    atomicAdd(p, v);
#else
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Developer stall profile (tools/fz_stall.cu, -DOOC_FZ_PROFILE): cycles each role spends in
// each wait, summed over CTAs. Compiled out of the product.
#ifdef OOC_FZ_PROFILE
__device__ unsigned long long g_fz_prof[24];
#define FZ_WAIT(idx, call)              \
    do {                                \
        const long long t_ = clock64(); \
        call;                           \
        prof[idx] += clock64() - t_;    \
    } while (0)
#else
#define FZ_WAIT(idx, call) call
#endif
// Latency trace of the first kFzTraceBlocks blocks (profile builds): globaltimer ns at each
// CTA's P1 publish, at each row's updater seeing the count / finishing, at each CTA's B producer
// seeing the block's rows 0-63 ready, at each row's gather landing. [5][kFzTraceBlocks][128 or G]
#ifdef OOC_FZ_PROFILE
constexpr int kFzTraceBlocks = 64;
__device__ unsigned long long* g_fz_trace = nullptr;
__device__ __forceinline__ void fz_trace(int kind, int b, int i) {
    if (g_fz_trace && b < kFzTraceBlocks) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_fz_trace[(size_t(kind) * kFzTraceBlocks + b) * 256 + i] = t;
    }
}
#define FZ_TRACE(kind, b, i) fz_trace(kind, b, i)
#else
#define FZ_TRACE(kind, b, i)
#endif

template <int KP>
__global__ void __launch_bounds__(512, 1)
    k_mu_fused(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2,
               const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmB2,
               const __grid_constant__ CUtensorMap tmS, const __grid_constant__ FusedArgs p) {
    using C = FzCfg<KP>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::RING_BYTES);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + C::A_STAGES;
    uint64_t* fullB = emptyA + C::A_STAGES;
    uint64_t* emptyB = fullB + C::B_STAGES;
    uint64_t* split = emptyB + C::B_STAGES;   // [ASLOTS]
    uint64_t* afree = split + C::ASLOTS;      // [ASLOTS]
    uint64_t* accfull = afree + C::ASLOTS;    // [NBUF]
    uint64_t* accempty = accfull + C::NBUF;   // [NBUF]
    uint64_t* gbar = accempty + C::NBUF;       // updater gather (TMA -> updaters)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbar + 1);
    int* act = reinterpret_cast<int*>(smem + C::RING_BYTES + C::BAR_BYTES);  // [G1] P1 publishers
    float* red = reinterpret_cast<float*>(act + C::MAX_G);                   // [64] updater scratch
    float* gbuf = reinterpret_cast<float*>(smem + C::GATHER_OFF);            // [G][kp] gathered partials
    double* wg = reinterpret_cast<double*>(smem + C::WGRAM_OFF);             // [kp][kp] Gram of the new W rows

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta = blockIdx.x, G = gridDim.x;
    const int q0 = p.q0[cta], q1 = p.q0[cta + 1], t0 = p.t0[cta], t1 = p.t0[cta + 1];
    const int NB = p.NB, D = p.D;

    if (tid == 0) {
        for (int s = 0; s < C::A_STAGES; ++s) mbar_init(fullA + s, 1), mbar_init(emptyA + s, 8);
        for (int s = 0; s < C::B_STAGES; ++s) mbar_init(fullB + s, 1), mbar_init(emptyB + s, 1);
        for (int r = 0; r < C::ASLOTS; ++r) mbar_init(split + r, 8), mbar_init(afree + r, 1);
        for (int b = 0; b < C::NBUF; ++b) mbar_init(accfull + b, 1), mbar_init(accempty + b, 4);
        mbar_init(gbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < p.G1; i += blockDim.x) act[i] = p.act[i];
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
#ifdef OOC_FZ_PROFILE
    long long prof[24] = {};
    const long long t_start = clock64();
#endif
    auto a_stage = [&](int s) { return smem + s * C::A_BYTES; };
    auto b_stage = [&](int s) { return smem + C::A_STAGES * C::A_BYTES + s * C::B_BYTES; };
    const int du = p.drain_units;

    if (warp == 0) {
        // ---------------- A producer (never waits on other CTAs: P2's A tiles load ahead)
        if (lane == 0) {
            int sa = 0;
            uint32_t pha = 0;
            auto load_a = [&](const CUtensorMap* m, int y, int z, uint64_t pol) {
                FZ_WAIT(0, mbar_wait(emptyA + sa, pha ^ 1u));
                mbar_expect_tx(fullA + sa, C::A_BYTES);
                tma_load_3d(a_stage(sa), m, fullA + sa, 0, y, z, pol);
                if (++sa == C::A_STAGES) sa = 0, pha ^= 1u;
            };
            auto p1 = [&](int s) {
                if (s < NB)
                    for (int q = q0; q < q1; ++q)  // block s, K-atoms 2q..
                        load_a(&tmA1, s * 128, 2 * q, (q >> 1) % p.keep_den < p.keep_num ? p.pol_p1 : p.pol_p1s);
            };
            auto p2 = [&](int s) {
                if (s >= D)
                    for (int j = t0; j < t1; ++j)
                        for (int h = 0; h < 2; ++h) load_a(&tmA2, (s - D) * 128 + 64 * h, 4 * j, p.pol_p2);
            };
            for (int s = 0; s < NB + D; ++s) p.p2_first ? (p2(s), p1(s)) : (p1(s), p2(s));
        }
    } else if (warp == 3) {
        // ---------------- B producer: [Ht | Ht_lo] chunk rows for P1; for P2 the block's new
        // [W | W_lo] rows, each 64-row half once its updaters are done (wdone[2 b + h] = 64)
        if (lane == 0) {
            int sb = 0;
            uint32_t phb = 0;
            auto load_b = [&](const CUtensorMap* m, int y, uint64_t pol) {
                FZ_WAIT(1, mbar_wait(emptyB + sb, phb ^ 1u));
                mbar_expect_tx(fullB + sb, C::B_BYTES);
                tma_load_3d(b_stage(sb), m, fullB + sb, 0, y, 0, pol);
                if (++sb == C::B_STAGES) sb = 0, phb ^= 1u;
            };
            auto p1 = [&](int s) {
                if (s < NB)
                    for (int q = q0; q < q1; ++q) load_b(&tmB1, q * C::BK, kEvictLast);
            };
            auto p2 = [&](int s) {
                if (s >= D && t1 == t0) {
                    // no owned tiles: still wait for block s - D's update, which throttles this
                    // CTA's P1 publishing to the slot ring (the MMA runs P1(s + 1) after these
                    // loads; blocks reuse slots NS = D + 2 apart)
                    FZ_WAIT(2, wait_count(p.wdone + 2 * (s - D), 64u));
                    FZ_WAIT(2, wait_count(p.wdone + 2 * (s - D) + 1, 64u));
                } else if (s >= D) {
                    // the two 64-row halves once per block: the MMA reuses them for every
                    // owned tile (one 16 KB TMA load per half instead of one per tile)
                    const int b = s - D;
                    for (int h = 0; h < 2; ++h) {
                        FZ_WAIT(2, wait_count(p.wdone + 2 * b + h, 64u));
                        fence_proxy_async_global();
                        if (h == 0) FZ_TRACE(3, b, cta);
                        load_b(&tmB2, b * 128 + 64 * h, kEvictNormal);
                    }
                }
            };
            for (int s = 0; s < NB + D; ++s) p.p2_first ? (p2(s), p1(s)) : (p1(s), p2(s));
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int sb = 0, r = 0, buf = 0;
        uint32_t phb = 0, rph = 0, aph = 0;
        bool open = true;
        // one unit on B stage st: wait for it to fill (wait_b) and release it when its MMAs
        // are done (release_b); P2 holds a block's two W stages across all its tiles
        auto unit_on = [&](bool close, int st, uint32_t ph, bool wait_b, bool release_b) {
            if (open) FZ_WAIT(5, mbar_wait(accempty + buf, aph ^ 1u));
            if (wait_b) FZ_WAIT(6, mbar_wait(fullB + st, ph));
            FZ_WAIT(7, mbar_wait(split + r, rph));
            tc_fence_after();
            const uint32_t d = tmem + uint32_t(buf * C::ACC_COLS);
            const uint64_t db0 = desc_mnmajor(smem_u32(b_stage(st)), 0, C::ATOM_STRIDE);
            const uint32_t ahi = tmem + uint32_t(C::A_COL0 + r * C::ASLOT_COLS), alo = ahi + C::BK;
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < C::KSTEPS; ++kk) {
                    const uint64_t db = db0 + uint64_t(kk * 64);
                    mma_ts(d, ahi + 8 * kk, db, C::IDESC_HI, (open && kk == 0) ? 0u : 1u);
                    mma_ts(d + KP, alo + 8 * kk, db, C::IDESC_KP, 1u);
                }
                if (release_b) mma_commit(emptyB + st);
                mma_commit(afree + r);
            }
            if (++r == C::ASLOTS) r = 0, rph ^= 1u;
            if (close) {
                if (elect_one()) mma_commit(accfull + buf);
                if (++buf == C::NBUF) buf = 0, aph ^= 1u;
            }
            open = close;
            __syncwarp();
        };
        auto next_b = [&]() {
            if (++sb == C::B_STAGES) sb = 0, phb ^= 1u;
        };
        auto p1 = [&](int s) {
            if (s < NB) {
                int cu = 0;
                for (int q = q0; q < q1; ++q) {
                    const bool close = ++cu == du || q + 1 == q1;
                    if (close) cu = 0;
                    unit_on(close, sb, phb, true, true);
                    next_b();
                }
            }
        };
        auto p2 = [&](int s) {
            if (s >= D && t1 > t0) {
                const int s0 = sb;
                const uint32_t ph0 = phb;
                next_b();
                const int s1 = sb;
                const uint32_t ph1 = phb;
                next_b();
                for (int j = t0; j < t1; ++j) {
                    const bool first = j == t0, last = j + 1 == t1;
                    unit_on(false, s0, ph0, first, last);
                    unit_on(true, s1, ph1, first, last);
                }
            }
        };
        for (int s = 0; s < NB + D; ++s) p.p2_first ? (p2(s), p1(s)) : (p1(s), p2(s));
    } else if (warp == 2) {
        // ---------------- updater: row r of block b -> CTA (128 b + r) mod G
        constexpr int P = 32 / KP;  // parts of the CTA range (kp 16: two), summed in fixed order
        const int j = lane % KP, part = lane / KP;
        const int c_lo = part * G / P, c_hi = (part + 1) * G / P;
        float hcol[KP];  // column j of HH^T
#pragma unroll
        for (int q = 0; q < KP; ++q) hcol[q] = p.HHt[q * KP + j];
        for (int e = lane; e < KP * KP; e += 32) wg[e] = 0.0;
        __syncwarp();
        const unsigned target = 4u * unsigned(p.G1);
        bool bad = false;
        uint32_t gph = 0;
        for (int64_t g = cta; g < int64_t(NB) * 128; g += G) {
            const int b = int(g >> 7), row = int(g & 127);
            float* wrow = p.W + g * KP;
            const float wold = wrow[j];  // last iteration's row: load it while P1 of the block runs
            FZ_WAIT(9, wait_count(p.count + b, target));
            if (lane == 0) FZ_TRACE(1, b, row);
            // one TMA operation gathers row `row` of every CTA's partial (G x kp floats, CTAs
            // without P1 work hold zeros); each lane sums its column over the CTAs in order
            if (lane == 0) {
                fence_proxy_async_global();  // the partials were written by generic stores
                mbar_expect_tx(gbar, uint32_t(G * KP * 4));
                tma_load_3d(gbuf, &tmS, gbar, 0, row, (b % p.NS) * G, kEvictFirst);
            }
            FZ_WAIT(10, mbar_wait(gbar, gph));
            gph ^= 1u;
            if (lane == 0) FZ_TRACE(4, b, row);
#ifndef OOC_FZ_KEEP_SLOTS
            {
                // The gathered partials are dead (their slot is rewritten NS blocks later, after
                // this row's W-ready release): drop the G dirty lines (one per CTA: slot rows are
                // a whole 128-byte line) from L2 instead of letting the A stream evict them to HBM
                // (≈ 1.2 GB of writes per iteration at config 2).
                const float* sb = p.p1slots + (int64_t(b % p.NS) * G) * (128 * C::RS) + row * C::RS;
                for (int c = lane; c < G; c += 32)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(sb + int64_t(c) * 128 * C::RS) : "memory");
            }
#endif
            // four interleaved partial sums (CTAs c = c_lo + 4 i + l), combined in a fixed order:
            // deterministic, and a quarter of the dependent-add chain of one running sum
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
            int c = c_lo;
#pragma unroll 2
            for (; c + 4 <= c_hi; c += 4)
#pragma unroll
                for (int l = 0; l < 4; ++l) s4[l] += gbuf[(c + l) * KP + j];
            for (int l = 0; c < c_hi; ++c, ++l) s4[l] += gbuf[c * KP + j];
            float nu = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            if constexpr (P == 2) nu += __shfl_down_sync(0xffffffffu, nu, 16);  // part 0 + part 1
            float d4[4] = {0.f, 0.f, 0.f, 0.f};  // W_old · HH^T column j, four interleaved chains
#pragma unroll
            for (int q = 0; q < KP; ++q) d4[q & 3] = fmaf(__shfl_sync(0xffffffffu, wold, q), hcol[q], d4[q & 3]);
            const float de = (d4[0] + d4[1]) + (d4[2] + d4[3]);
            float wn = 0.f;
            if (lane < KP) {
                // t * nu / (de + eps) as (t * nu) * rcp_rn(de + eps), the factor-update
                // kernel's formula (kernels_factor.cu)
                wn = (wold * nu) * __frcp_rn(de + p.eps);
                bad |= !isfinite(wn);
                wrow[lane] = wn;
                float* cw = p.Wcat + g * (2 * KP);
                cw[lane] = wn;
                cw[KP + lane] = tf32_lo(wn);
            }
            __syncwarp();  // (also: gbuf is refilled by the next row's TMA)
            if (lane == 0) {
                fence_proxy_async_global();  // read by the B producers' TMA
                red_release_add(p.wdone + 2 * b + (row >> 6), 1u);
                FZ_TRACE(2, b, row);
            }
            if (p.wgram) {
                // the row's contribution to W^T W (column `lane`), exact f32 products summed in
                // f64 in row order, off the W-ready path (after the release)
#pragma unroll 8
                for (int i = 0; i < KP; ++i) {
                    const float wi = __shfl_sync(0xffffffffu, wn, i);
                    if (lane < KP) wg[i * KP + lane] += double(wi) * double(wn);
                }
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.flag, 1);
        if (p.wgram) {  // this CTA's slot (zeros if it updated no row)
            __syncwarp();
            for (int e = lane; e < KP * KP; e += 32) p.wgram[int64_t(cta) * KP * KP + e] = wg[e];
        }
    } else if (warp >= 4 && warp < 12) {
        // ---------------- split warps: A tile -> [A_hi | A_lo] in TMEM slot
        const int t = 32 * (warp & 3) + lane;
        const int h = (warp - 4) >> 2;
        const uint32_t lane_bits = uint32_t(32 * (warp & 3)) << 16;
        int sa = 0, rs = 0;
        uint32_t pha = 0, rph = 0;
        auto unit = [&](bool p1) {
            FZ_WAIT(3, mbar_wait(fullA + sa, pha));
            FZ_WAIT(4, mbar_wait(afree + rs, rph ^ 1u));
            tc_fence_after();
            const uint8_t* sA = a_stage(sa);
            const uint32_t dst = tmem + lane_bits + uint32_t(C::A_COL0 + rs * C::ASLOT_COLS);
            uint32_t r[32], x[32];
            if (p1) {
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
            tmem_st32(dst + 32 * h, x);
            tmem_st32(dst + C::BK + 32 * h, r);
            __syncwarp();
            if (lane == 0) mbar_arrive(emptyA + sa);
            if (++sa == C::A_STAGES) sa = 0, pha ^= 1u;
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(split + rs);
            if (++rs == C::ASLOTS) rs = 0, rph ^= 1u;
        };
        auto p1 = [&](int s) {
            if (s < NB)
                for (int q = q0; q < q1; ++q) unit(true);
        };
        auto p2 = [&](int s) {
            if (s >= D)
                for (int j = t0; j < t1; ++j) unit(false), unit(false);
        };
        for (int s = 0; s < NB + D; ++s) p.p2_first ? (p2(s), p1(s)) : (p1(s), p2(s));
    } else if (warp >= 12) {
        // ---------------- drain: P1 chains -> f32 row sums -> published partial; P2 chains
        // (one per block and owned tile) -> TMEM running sums of W^T A
        const int t = tid - 384;
        const uint32_t lane_bits = uint32_t(32 * (warp & 3)) << 16;
        float acc[KP];
#pragma unroll
        for (int jj = 0; jj < KP; ++jj) acc[jj] = 0.f;
        int buf = 0;
        uint32_t aph = 0;
        // fold one closed chain D' = [H | L] into acc
        auto take = [&]() {
            FZ_WAIT(8, mbar_wait(accfull + buf, aph));
            tc_fence_after();
            const uint32_t src = tmem + lane_bits + uint32_t(buf * C::ACC_COLS);
            if constexpr (KP == 16) {
                uint32_t v[32];
                tmem_ld32(src, v);
                acc_add2<16>(acc, v, v + 16);
            } else {
                uint32_t hi[32], lo[32];
                tmem_ld32(src, hi);
                tmem_ld32(src + KP, lo);
                acc_add2<32>(acc, hi, lo);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty + buf);
            if (++buf == C::NBUF) buf = 0, aph ^= 1u;
        };
        auto p1 = [&](int s) {
            if (s < NB && q1 > q0) {
                int cu = 0;
                for (int q = q0; q < q1; ++q) {
                    const bool close = ++cu == du || q + 1 == q1;
                    if (close) cu = 0, take();
                }
                // publish this CTA's partial of block s: row t
                float* out = p.p1slots + (int64_t(s % p.NS) * G + cta) * (128 * C::RS) + t * C::RS;
#pragma unroll
                for (int j4 = 0; j4 < KP / 4; ++j4) {
                    __stcg(reinterpret_cast<float4*>(out) + j4,
                           make_float4(acc[4 * j4], acc[4 * j4 + 1], acc[4 * j4 + 2], acc[4 * j4 + 3]));
                    acc[4 * j4] = acc[4 * j4 + 1] = acc[4 * j4 + 2] = acc[4 * j4 + 3] = 0.f;
                }
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_global();  // read back by the updaters' TMA (async proxy)
                    red_release_add(p.count + s, 1u);
                    if (warp == 15) FZ_TRACE(0, s, cta);
                }
            }
        };
        auto p2 = [&](int s) {
            if (s >= D) {
                const int b = s - D;
                for (int j = t0; j < t1; ++j) {
                    take();  // the chain of (b, j): acc = its 128-row product
                    const uint32_t run = tmem + lane_bits + uint32_t(C::RUN_COL0 + (j - t0) * KP);
#pragma unroll
                    for (int h = 0; h < (KP + 31) / 32; ++h) {
                        constexpr int WD = KP < 32 ? KP : 32;
                        uint32_t v[32];
                        if (b > 0) {  // running sum += this block's chain (ascending blocks)
                            if constexpr (WD == 16) tmem_ld16(run, v);
                            else tmem_ld32(run + 32 * h, v);
#pragma unroll
                            for (int jj = 0; jj < WD; jj += 2)
                                add2(acc[WD * h + jj], acc[WD * h + jj + 1], __uint_as_float(v[jj]),
                                     __uint_as_float(v[jj + 1]));
                        }
#pragma unroll
                        for (int jj = 0; jj < WD; ++jj) v[jj] = __float_as_uint(acc[WD * h + jj]);
                        if constexpr (WD == 16) tmem_st16(run, v);
                        else tmem_st32(run + 32 * h, v);
                    }
                    tmem_st_wait();
#pragma unroll
                    for (int jj = 0; jj < KP; ++jj) acc[jj] = 0.f;
                }
            }
        };
        for (int s = 0; s < NB + D; ++s) p.p2_first ? (p2(s), p1(s)) : (p1(s), p2(s));
        // the owned tiles of W^T A (np x kp, row = column of A)
        for (int j = t0; j < t1; ++j) {
            const uint32_t run = tmem + lane_bits + uint32_t(C::RUN_COL0 + (j - t0) * KP);
            float4* out = reinterpret_cast<float4*>(p.wta + (int64_t(j) * 128 + t) * KP);
            uint32_t v[32];
#pragma unroll
            for (int h = 0; h < (KP + 31) / 32; ++h) {
                if constexpr (KP == 16) tmem_ld16(run, v);
                else tmem_ld32(run + 32 * h, v);
#pragma unroll
                for (int j4 = 0; j4 < (KP < 32 ? KP : 32) / 4; ++j4)
                    out[h * 8 + j4] = make_float4(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1]),
                                                  __uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3]));
            }
        }
    }
#ifdef OOC_FZ_PROFILE
    // per role: lane 0 of warp 0 (A producer), 1 (MMA), 2 (updater), 3 (B producer), 4 (split),
    // 12 (drain); the B producer's waits go to slots 11 (emptyB) and 12 (W ready)
    if (lane == 0 && (warp <= 4 || warp == 12)) {
        for (int j = 0; j < 11; ++j)
            if (prof[j]) atomicAdd(&g_fz_prof[warp == 3 && (j == 1 || j == 2) ? 10 + j : j], (unsigned long long)prof[j]);
        atomicAdd(&g_fz_prof[16 + (warp == 12 ? 5 : warp)], (unsigned long long)(clock64() - t_start));
    }
#endif
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
    }
}

template <int KP>
cudaError_t launch_fused_t(const FusedPlan& fp, const float* A, int64_t mp, int64_t np, const float* Ht_cat,
                           const FusedArgs& args, cudaStream_t s) {
    using C = FzCfg<KP>;
    CUtensorMap a1, a2, b1, b2;
    cudaError_t e;
    if ((e = make_map(&a1, A, mp, np, np, 128, kTcStep / 32, false)) != cudaSuccess) return e;
    if ((e = make_map(&a2, A, mp, np, np, kTcStep, 4, true)) != cudaSuccess) return e;
    if ((e = make_map(&b1, Ht_cat, np, 2 * KP, 2 * KP, kTcStep, 2 * KP / 32, true)) != cudaSuccess) return e;
    if ((e = make_map(&b2, args.Wcat, mp, 2 * KP, 2 * KP, kTcStep, 2 * KP / 32, true)) != cudaSuccess) return e;
    CUtensorMap sm;  // P1 slots [NS * G][128][kp]: box (kp, 1 row, G slots) = one row of every CTA
    {
        auto fn = encode_fn();
        if (!fn) return cudaErrorNotSupported;
        const cuuint64_t dims[3] = {cuuint64_t(KP), 128u, cuuint64_t(fp.NS) * fp.G};
        const cuuint64_t strides[2] = {cuuint64_t(C::RS) * 4, cuuint64_t(128) * C::RS * 4};
        const cuuint32_t box[3] = {cuuint32_t(KP), 1u, cuuint32_t(fp.G)};
        const cuuint32_t estr[3] = {1u, 1u, 1u};
        if (fn(&sm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, args.p1slots, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    auto kern = k_mu_fused<KP>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM))) != cudaSuccess)
        return e;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(unsigned(fp.G));
    lc.blockDim = dim3(512);
    lc.dynamicSmemBytes = C::SMEM;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // CTAs wait on each other: all must be resident
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, a1, a2, b1, b2, sm, args);
}

}  // namespace

size_t fused_slot_bytes(int kp, const FusedPlan& fp) {
    return size_t(fp.NS) * fp.G * 128 * size_t(kp < 32 ? 32 : kp) * 4;
}

bool fused_supported(int kp, int64_t mp, int64_t np, int num_sms) {
    if (!(kp == 16 || kp == 32) || !tc_supported(kp)) return false;
    if (mp % kTile || np % kTile || mp < kTile || np < kTile || num_sms < 1) return false;
    const int64_t nt = np / kTile, maxt = kp == 16 ? FzCfg<16>::MAXT : FzCfg<32>::MAXT;
    return (nt + num_sms - 1) / num_sms <= maxt && num_sms <= FzCfg<32>::MAX_G;
}

// Static work split of one launch (host). Per row block every CTA gets the same number of
// units: tiles t0(c) = floor(c NT / G) (2 P2 units each), then P1 chunks filling each CTA up
// to its share round(c U / G) of the U = NQ + 2 NT units of the block.
void plan_fused(FusedPlan& fp, int64_t mp, int64_t np, int num_sms, int lookahead) {
    fp.G = num_sms;
    fp.NB = int(mp / kTile);
    fp.NT = int(np / kTile);
    fp.NQ = int(np / kTcStep);
    fp.D = std::max(1, std::min(lookahead, fp.NB));
    fp.NS = fp.D + 2;
    const int G = fp.G;
    const int64_t U = int64_t(fp.NQ) + 2 * int64_t(fp.NT);
    fp.q0.assign(G + 1, 0);
    fp.t0.assign(G + 1, 0);
    for (int c = 0; c <= G; ++c) fp.t0[c] = int(int64_t(c) * fp.NT / G);
    const char* pm = std::getenv("OOCNMF_FUSED_PLAN");  // developer knob: 1 = even P1 ranges
    if (pm && pm[0] == '1') {
        for (int c = 0; c <= G; ++c) fp.q0[c] = int(int64_t(c) * fp.NQ / G);
    } else {
    int prev = 0;
    for (int c = 0; c <= G; ++c) {
        const int64_t share = (int64_t(c) * U + G / 2) / G;
        int q = int(share - 2 * int64_t(fp.t0[c]));
        q = std::max(prev, std::min(q, fp.NQ));
        if (c == G) q = fp.NQ;
        fp.q0[c] = q;
        prev = q;
    }
    }
    fp.act.clear();
    for (int c = 0; c < G; ++c)
        if (fp.q0[c + 1] > fp.q0[c]) fp.act.push_back(c);
    fp.G1 = int(fp.act.size());
}

void fused_policies(FusedArgs& a) {
    const char* e = std::getenv("OOCNMF_FUSED_POL");  // 0 normal/first, 1 last/first, 2 normal/normal
    const int pol = e && *e ? std::atoi(e) : 0;
    a.pol_p1 = pol == 1 ? kEvictLast : kEvictNormal;
    a.pol_p2 = pol == 2 ? kEvictNormal : kEvictFirst;
    a.pol_p1s = kEvictFirst;
    a.keep_num = a.keep_den = 1;
    if (const char* k = std::getenv("OOCNMF_FUSED_KEEP"); k && *k) {  // "num/den"
        int n = 1, d = 1;
        if (std::sscanf(k, "%d/%d", &n, &d) == 2 && d >= 1 && n >= 0 && n <= d) a.keep_num = n, a.keep_den = d;
    }
}

#ifdef OOC_FZ_PROFILE
void fz_trace_set(unsigned long long* buf) { cudaMemcpyToSymbol(g_fz_trace, &buf, sizeof(buf)); }
void fz_profile_read(unsigned long long* out24, bool reset) {
    cudaMemcpyFromSymbol(out24, g_fz_prof, 24 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[24] = {};
        cudaMemcpyToSymbol(g_fz_prof, z, sizeof(z));
    }
}
#endif

cudaError_t launch_mu_fused(int kp, const FusedPlan& fp, const float* A, int64_t mp, int64_t np, const float* Ht_cat,
                            const FusedArgs& args, cudaStream_t s) {
    return kp == 16 ? launch_fused_t<16>(fp, A, mp, np, Ht_cat, args, s)
                    : launch_fused_t<32>(fp, A, mp, np, Ht_cat, args, s);
}

}  // namespace ooc
