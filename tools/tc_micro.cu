// Developer micro-probes for tcgen05 building blocks (TMEM st/ld, one UMMA tf32 from
// hand-filled SW128 smem). Not part of the product.
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_tmem_roundtrip(float* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&slot)), "r"(64) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
    uint32_t v0 = __float_as_uint(float(threadIdx.x) + 0.5f), v1 = __float_as_uint(float(threadIdx.x) + 0.25f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" :: "r"(taddr), "r"(v0), "r"(v1) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n\ttcgen05.wait::ld.sync.aligned;" : "=r"(r0), "=r"(r1) : "r"(taddr) : "memory");
    out[threadIdx.x * 2] = __uint_as_float(r0);
    out[threadIdx.x * 2 + 1] = __uint_as_float(r1);
    if (threadIdx.x == 0) out[256] = __uint_as_float(tmem);
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(64) : "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}

// D[128 x 32] = A[128 x 32 (K)] · B[32 (K) x 32 (N)], A K-major SW128, B MN-major SW128.
__global__ void k_one_mma(const float* A, const float* B, float* D, int a_mn, float* dbg) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    float* sA = (float*)sm;              // 16 KB
    float* sB = (float*)(sm + 16384);    // 4 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    // fill A: K-major SW128: (r, c) -> r*128 + ((c/4) ^ (r%8))*16 + (c%4)*4 bytes
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        const int r = e / 32, c = e % 32;
        const int off = r * 32 + (((c / 4) ^ (r % 8)) * 4) + (c % 4);
        sA[off] = A[r * 32 + c];
    }
    // fill B (K x N, N contiguous): MN-major SW128: (k, n) -> k*128 + ((n/4) ^ (k%8))*16 + (n%4)*4
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
        const int k = e / 32, n = e % 32;
        const int off = k * 32 + (((n / 4) ^ (k % 8)) * 4) + (n % 4);
        sB[off] = B[k * 32 + n];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(&slot)), "r"(64) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 1 && lane == 0) {
        for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = sdesc(su32(sA) + kk * 32, 16, 1024, 2);
            const uint64_t db = sdesc(su32(sB) + kk * 1024, 4096, 1024, 2);
            const uint32_t acc = kk > 0;
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                         :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
        if (dbg) { dbg[0] = (float)(sdesc(su32(sA), 16, 1024, 2) & 0xFFFFFFFF); }
    }
    if (warp < 4) {
        uint32_t ok = 0;
        do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
        } while (!ok);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t r[8];
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
        for (int c8 = 0; c8 < 4; ++c8) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\ttcgen05.wait::ld.sync.aligned;"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr + c8 * 8) : "memory");
            for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * 32 + c8 * 8 + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(64) : "memory");
}

int main() {
    float* d; cudaMalloc(&d, 4096); cudaMemset(d, 0, 4096);
    k_tmem_roundtrip<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[257]; cudaMemcpy(h, d, 257 * 4, cudaMemcpyDeviceToHost);
    int bad = 0; for (int t = 0; t < 128; ++t) if (h[2*t] != t + 0.5f || h[2*t+1] != t + 0.25f) ++bad;
    printf("tmem roundtrip: err=%s bad=%d tmem_base=%u sample %g %g\n", cudaGetErrorString(e), bad, *(unsigned*)&h[256], h[0], h[3]);

    float hA[128 * 32], hB[32 * 32], hD[128 * 32];
    for (int i = 0; i < 128 * 32; ++i) hA[i] = float((i * 7) % 13) * 0.25f;   // exact in tf32
    for (int i = 0; i < 32 * 32; ++i) hB[i] = float((i * 5) % 11) * 0.5f;
    float *dA, *dB, *dD, *dg; cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD); cudaMalloc(&dg, 64);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, sizeof hD);
    cudaFuncSetAttribute(k_one_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024);
    k_one_mma<<<1, 128, 24 * 1024>>>(dA, dB, dD, 0, dg);
    e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0; int shown = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 32; ++j) {
        double ref = 0; for (int k = 0; k < 32; ++k) ref += double(hA[i * 32 + k]) * hB[k * 32 + j];
        double err = std::abs(hD[i * 32 + j] - ref);
        if (!(err <= maxerr)) maxerr = err;
        if (!(err < 1e-3) && shown < 8) { printf("  D[%d][%d] = %g want %g\n", i, j, hD[i * 32 + j], ref); ++shown; }
    }
    printf("one mma: err=%s max abs err %g\n", cudaGetErrorString(e), maxerr);
    return 0;
}
