// tcgen05 / TMA / mbarrier PTX wrappers shared by the tensor-core kernels (kernels_tc.cu:
// the two streaming passes; kernels_fused.cu: the one-pass MU iteration). sm_100a only.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.h"

namespace ooc {
namespace tc {

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
// The suspend-time hint lets a waiting warp sleep until the phase flips instead of spinning:
// without it the producer / drain / MMA warps' try_wait loops took ~30% of all issued
// instructions (ncu source page) from the split warps that share their SM sub-partitions.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity), "r"(0x989680u)
            : "memory");
    } while (!ok);
}
// Developer stall profile (tools/tc_stall.cu, -DOOC_TC_PROFILE): cycles each role spends in
// each wait, summed over CTAs. Compiled out of the product.
#ifdef OOC_TC_PROFILE
__device__ unsigned long long g_tc_prof[16];
#define TC_WAIT(idx, call)                          \
    do {                                            \
        const long long t_ = clock64();             \
        call;                                       \
        prof[idx] += clock64() - t_;                \
    } while (0)
#else
#define TC_WAIT(idx, call) call
#endif

// L2 eviction policies (the encodings CUTLASS uses for TMA cache hints).
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull, kEvictLast = 0x14F0000000000000ull,
                   kEvictNormal = 0x1000000000000000ull;
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

// UMMA shared-memory descriptor, version 1 (sm_100). Layout 1 = SWIZZLE_128B_BASE32B
// (32-byte granules XOR row%4); (layout 2 = SWIZZLE_128B, 16-byte granules XOR row%8, is
// what K-major operands would use — A now reaches the MMA through TMEM instead).
constexpr uint32_t kLayoutSW128B32 = 1;
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
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
// K-major SWIZZLE_128B operand (layout 2): 8-row x 128-byte swizzle atoms, 1024 B apart (SBO);
// an MMA's 8-deep tf32 K slice is +32 B inside the atom row. (LBO is unused for swizzled K-major.)
constexpr uint32_t kLayoutSW128 = 2;
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t addr) { return sdesc(addr, 16, 1024, kLayoutSW128); }
// both operands from shared memory
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
// (no wait: the caller issues tmem_st_wait() once after its last store)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%"
        "18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        OOC_W32(r)
        : "memory");
}
// 16 consecutive 32-bit TMEM columns <-> 16 registers (kp = 16 running sums)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// (a0, a1) += (b0, b1) as one packed FADD2 (sm_100 f32x2): two IEEE round-to-nearest adds,
// bit-identical to the scalar pair at half the issue slots (the split and drain warps'
// adds are ~20% of the pass's instructions, and under the power cap issue costs clock)
__device__ __forceinline__ void add2(float& a0, float& a1, float b0, float b1) {
    asm("{\n.reg .b64 ra, rb;\nmov.b64 ra, {%0, %1};\nmov.b64 rb, {%2, %3};\n"
        "add.rn.f32x2 ra, ra, rb;\nmov.b64 {%0, %1}, ra;\n}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1));
}
// tf32_lo(x) of two values as the MMA will read them: adding half a tf32 ulp to the bits of
// the remainder x - trunc(x) and letting the tensor core's truncation drop the low 13 bits is
// round-to-nearest (ties away) — one integer add instead of cvt.rna (a 4-instruction
// emulation) — and the two remainders come from one FADD2.
__device__ __forceinline__ void lo_bits2(float x0, float x1, uint32_t& r0, uint32_t& r1) {
    float d0 = x0, d1 = x1;
    add2(d0, d1, -__uint_as_float(__float_as_uint(x0) & 0xFFFFE000u), -__uint_as_float(__float_as_uint(x1) & 0xFFFFE000u));
    r0 = __float_as_uint(d0) + 0x1000u;
    r1 = __float_as_uint(d1) + 0x1000u;
}
// acc[j] += a[j] + b[j] for an even-length run, in pairs
template <int N>
__device__ __forceinline__ void acc_add2(float* acc, const uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        float s0 = __uint_as_float(a[j]), s1 = __uint_as_float(a[j + 1]);
        add2(s0, s1, __uint_as_float(b[j]), __uint_as_float(b[j + 1]));
        add2(acc[j], acc[j + 1], s0, s1);
    }
}

// View a row-major f32 matrix [rows][cols] (ld floats) as 3-D (32 columns of an atom, rows,
// cols/32 atoms) and box (32, box_rows, box_atoms): one TMA operation lands box_atoms
// atoms of box_rows x 128 B, atom j at j * box_rows * 128 B in shared memory. K-major tiles
// use the 16-byte-granule 128B swizzle, MN-major ones the 32-byte-granule variant that
// matches UMMA's SWIZZLE_128B_BASE32B layout. (kernels_tc.cu)
cudaError_t make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int box_atoms, bool mn_major);
// K steps per TMEM accumulation chain (OOCNMF_TC_DRAIN, default 2). (kernels_tc.cu)
int tc_drain_units();
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

}  // namespace tc
}  // namespace ooc
