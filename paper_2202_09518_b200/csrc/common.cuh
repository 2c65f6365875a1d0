// Shared device-side definitions of the B200 MU-NMF backend.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ooc {

// ---------------------------------------------------------------------------
// SplitMix64 counter RNG — the same pure function of (seed, stream, index) as the
// reference's CounterRng (include/oocnmf/rng.hpp:11-40), usable on host and device.
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += kGolden;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
    return splitmix(seed ^ splitmix(stream + 0x632BE59BD9B4E019ULL));
}
__host__ __device__ __forceinline__ uint64_t rng_bits53(uint64_t key, uint64_t index) {
    return splitmix(key + (index + 1) * kGolden) >> 11;
}
__host__ __device__ __forceinline__ double rng_u01(uint64_t key, uint64_t index) {
    return static_cast<double>(rng_bits53(key, index)) * 0x1.0p-53;
}

// Streams used by the reference (src/nmf_serial.cpp:17-18, src/synth.cpp:12-15,
// bench/kernels_bench.cpp:14).
constexpr uint64_t kStreamW = 1, kStreamH = 2, kStreamSparseMask = 14, kStreamSparseVal = 15;
constexpr uint64_t kStreamPerturb = 21;  // src/model_selection.cpp:17

// ---------------------------------------------------------------------------
// Stream-K work split. A pass over A is `tiles` output tiles x `ipt` reduction steps;
// CTA c of G owns the contiguous unit range [begin(c), begin(c+1)) of the flattened
// (tile, step) space, so every CTA streams the same number of A bytes. A tile touched by
// several CTAs gets one partial per CTA in slot c*smax + (tile - first_tile(c)); the
// consumer sums a tile's partials in ascending c, so results are deterministic.
// ---------------------------------------------------------------------------
struct StreamK {
    int64_t tiles = 0, ipt = 0, G = 0, smax = 0;

    __host__ __device__ int64_t total() const { return tiles * ipt; }
    __host__ __device__ int64_t begin(int64_t c) const { return c * total() / G; }
    __host__ __device__ int64_t cta_of(int64_t u) const {
        return ((u + 1) * G + total() - 1) / total() - 1;
    }
    __host__ __device__ int64_t first_tile(int64_t c) const { return begin(c) / ipt; }
    __host__ __device__ int64_t slot(int64_t c, int64_t t) const {
        return c * smax + (t - first_tile(c));
    }
    __host__ void plan(int64_t tiles_, int64_t ipt_, int64_t g_max) {
        tiles = tiles_;
        ipt = ipt_;
        G = g_max < total() ? g_max : total();
        if (G < 1) G = 1;
        smax = 0;
        for (int64_t c = 0; c < G; ++c) {
            const int64_t s = (begin(c + 1) - 1) / ipt - begin(c) / ipt + 1;
            if (s > smax) smax = s;
        }
    }
};

// ---------------------------------------------------------------------------
// 3xTF32 split: x = hi + lo + r with hi = trunc_tf32(x) (what the tensor core reads from a
// raw f32 operand) and lo = rna_tf32(x - hi). Rounding lo to nearest (instead of letting the
// MMA truncate it) keeps the residual r (|r| <= 2^-21 |x|) unbiased, so it averages out over
// the long K reductions instead of accumulating a one-signed bias.
__device__ __forceinline__ float tf32_lo(float x) {
    const float rem = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(rem));
    return __uint_as_float(r);
}

// ---------------------------------------------------------------------------
// small PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace ooc
