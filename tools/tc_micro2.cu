// Developer micro-probe: one 128xNx(KSTEPS*kstep) UMMA from host-built SW128 smem images,
// for kind::tf32 and kind::f16 (bf16), K-major / MN-major B. Not part of the product.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t version) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(version) << 46) | (uint64_t(layout) << 61);
}

struct P { int kind; int a_mn, b_mn; uint32_t a_step, b_step, a_lbo, b_lbo; int ksteps; int version; };

__global__ void k_mma(const uint8_t* imgA, int bytesA, const uint8_t* imgB, int bytesB, float* D, P p) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < bytesA; i += blockDim.x) sA[i] = imgA[i];
    for (int i = tid; i < bytesB; i += blockDim.x) sB[i] = imgB[i];
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
    const uint32_t fmt = p.kind == 0 ? 2u : 1u;  // tf32 : bf16
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(p.a_mn) << 15) | (uint32_t(p.b_mn) << 16) |
                           ((32u >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 1 && lane == 0) {
        for (int kk = 0; kk < p.ksteps; ++kk) {
            const uint64_t da = sdesc(su32(sA) + kk * p.a_step, p.a_lbo, 1024, 2, p.version);
            const uint64_t db = sdesc(su32(sB) + kk * p.b_step, p.b_lbo, 1024, 2, p.version);
            const uint32_t acc = kk > 0;
            if (p.kind == 0)
                asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n}"
                             :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
            else
                asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}"
                             :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
    }
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}" : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
    } while (!ok);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
    for (int c8 = 0; c8 < 4; ++c8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\ttcgen05.wait::ld.sync.aligned;"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr + c8 * 8) : "memory");
        for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * 32 + c8 * 8 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(64) : "memory");
}

// SW128 images. K-major: row r (M or N index), 128 B per row of K. MN-major: row = K index,
// 128 B of MN per row (only MN <= 128 B / e here).
static void put(std::vector<uint8_t>& img, int row, int byte_in_row, const void* v, int e) {
    const int ch = byte_in_row / 16, w = byte_in_row % 16;
    memcpy(&img[row * 128 + ((ch ^ (row % 8)) * 16) + w], v, e);
}

int run(int kind, int b_mn, int version) {
    const int e = kind == 0 ? 4 : 2;
    const int K = 128 / e;  // one 128-B swizzle row of K
    const int M = 128, N = 32;
    std::vector<float> A(M * K), B(K * N);
    for (int i = 0; i < M * K; ++i) A[i] = float((i * 7) % 13) * 0.25f;
    for (int i = 0; i < K * N; ++i) B[i] = float((i * 5) % 11) * 0.5f;
    std::vector<uint8_t> iA(M * 128, 0), iB(std::max(N, K) * 128 * 2, 0);
    for (int r = 0; r < M; ++r)
        for (int k = 0; k < K; ++k) {
            if (kind == 0) put(iA, r, k * 4, &A[r * K + k], 4);
            else { __nv_bfloat16 b = __float2bfloat16(A[r * K + k]); put(iA, r, k * 2, &b, 2); }
        }
    for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) {
            const float x = B[k * N + n];
            if (kind == 0) {
                if (b_mn) put(iB, k, n * 4, &x, 4); else put(iB, n, k * 4, &x, 4);
            } else {
                __nv_bfloat16 b = __float2bfloat16(x);
                if (b_mn) put(iB, k, n * 2, &b, 2); else put(iB, n, k * 2, &b, 2);
            }
        }
    uint8_t *dA, *dB; float* dD;
    cudaMalloc(&dA, iA.size()); cudaMalloc(&dB, iB.size()); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, iA.data(), iA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, iB.data(), iB.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, M * N * 4);
    const int kstep = 32 / e;  // elements per MMA K step (32 B)
    P p{kind, 0, b_mn, 32, uint32_t(b_mn ? 8 * 128 * (kstep / 8) : 32), 16, uint32_t(b_mn ? 4096 : 16), K / kstep, version};
    // MN-major B: one MMA consumes kstep K-rows: tf32 kstep=8 -> 1024 B; bf16 kstep=16 -> 2048 B
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    k_mma<<<1, 128, 48 * 1024>>>(dA, (int)iA.size(), dB, (int)iB.size(), dD, p);
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
        double ref = 0; for (int k = 0; k < K; ++k) ref += double(A[i * K + k]) * B[k * N + j];
        double d = std::fabs(D[i * N + j] - ref); if (!(d <= maxerr)) maxerr = d;
    }
    printf("kind=%s b_mn=%d version=%d: %s max abs err %g  D[0][0..3]=%g %g %g %g\n", kind == 0 ? "tf32" : "bf16", b_mn, version,
           cudaGetErrorString(err), maxerr, D[0], D[1], D[2], D[3]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return 0;
}

int main() {
    for (int version : {1, 0})
        for (int kind : {1, 0})
            for (int bmn : {0, 1}) run(kind, bmn, version);
    return 0;
}
