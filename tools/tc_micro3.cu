// Developer probe: (1) UMMA kind::tf32 with MN-major B in the SWIZZLE_128B_BASE32B layout
// (layout type 1: 32-byte granules XOR (row % 4) inside 128-byte rows, 4-row groups);
// (2) what TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes to smem. Not part of the product.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(layout) << 61);
}

__global__ void k_mma(const uint8_t* imgA, int bytesA, const uint8_t* imgB, int bytesB, float* D, uint32_t b_layout,
                      uint32_t b_sbo, uint32_t b_step) {
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 1 && lane == 0) {
        for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = sdesc(su32(sA) + kk * 32, 16, 1024, 2);
            const uint64_t db = sdesc(su32(sB) + kk * b_step, 4096, b_sbo, b_layout);
            asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n}"
                         :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)(kk > 0)) : "memory");
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

__global__ void k_tma_dump(const __grid_constant__ CUtensorMap m, float* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar)), "r"(4096) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     :: "r"(su32(sm)), "l"(&m), "r"(su32(&bar)), "r"(0), "r"(0) : "memory");
    }
    __syncthreads();
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}" : "=r"(ok) : "r"(su32(&bar)), "r"(0) : "memory");
    } while (!ok);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = ((float*)sm)[i];
}

static void put(std::vector<uint8_t>& img, int row, int byte_in_row, const void* v, int gran, int period) {
    const int ch = byte_in_row / gran, w = byte_in_row % gran;
    memcpy(&img[row * 128 + ((ch ^ (row % period)) * gran) + w], v, 4);
}

int main() {
    const int M = 128, K = 32, N = 32;
    std::vector<float> A(M * K), B(K * N);
    for (int i = 0; i < M * K; ++i) A[i] = float((i * 7) % 13) * 0.25f;
    for (int i = 0; i < K * N; ++i) B[i] = float((i * 5) % 11) * 0.5f;
    std::vector<uint8_t> iA(M * 128, 0), iB(K * 128, 0);
    for (int r = 0; r < M; ++r) for (int k = 0; k < K; ++k) put(iA, r, k * 4, &A[r * K + k], 16, 8);
    for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) put(iB, k, n * 4, &B[k * N + n], 32, 4);
    uint8_t *dA, *dB; float* dD;
    cudaMalloc(&dA, iA.size()); cudaMalloc(&dB, iB.size()); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, iA.data(), iA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, iB.data(), iB.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    for (uint32_t sbo : {512u, 1024u}) {
        cudaMemset(dD, 0xFF, M * N * 4);
        k_mma<<<1, 128, 48 * 1024>>>(dA, (int)iA.size(), dB, (int)iB.size(), dD, 1, sbo, 1024);
        cudaError_t err = cudaDeviceSynchronize();
        std::vector<float> D(M * N);
        cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
            double ref = 0; for (int k = 0; k < K; ++k) ref += double(A[i * K + k]) * B[k * N + j];
            double d = std::fabs(D[i * N + j] - ref); if (!(d <= maxerr)) maxerr = d;
        }
        printf("tf32 MN-major B, layout BASE32B, SBO %u: %s max abs err %g D[0][0..3]=%g %g %g %g\n", sbo,
               cudaGetErrorString(err), maxerr, D[0], D[1], D[2], D[3]);
    }
    // TMA ATOM_32B dump: 32 rows x 32 floats, value = row*100 + col
    std::vector<float> G(32 * 32);
    for (int r = 0; r < 32; ++r) for (int c = 0; c < 32; ++c) G[r * 32 + c] = r * 100 + c;
    float *dG, *dO; cudaMalloc(&dG, 4096); cudaMalloc(&dO, 4096);
    cudaMemcpy(dG, G.data(), 4096, cudaMemcpyHostToDevice);
    void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    for (auto sw : {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B}) {
        CUtensorMap m;
        cuuint64_t dims[2] = {32, 32}, strides[1] = {128};
        cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dG, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k_tma_dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
        k_tma_dump<<<1, 128, 8192>>>(m, dO);
        cudaError_t err = cudaDeviceSynchronize();
        std::vector<float> O(1024);
        cudaMemcpy(O.data(), dO, 4096, cudaMemcpyDeviceToHost);
        int bad16 = 0, bad32 = 0;
        for (int r = 0; r < 32; ++r) for (int c = 0; c < 32; ++c) {
            const int o16 = r * 32 + (((c / 4) ^ (r % 8)) * 4) + c % 4;
            const int o32 = r * 32 + (((c / 8) ^ (r % 4)) * 8) + c % 8;
            bad16 += O[o16] != G[r * 32 + c];
            bad32 += O[o32] != G[r * 32 + c];
        }
        printf("TMA swizzle %d (encode %d, %s): mismatches vs 16B/row%%8 = %d, vs 32B/row%%4 = %d; smem row1: %g %g %g %g %g %g %g %g %g\n",
               int(sw), int(r), cudaGetErrorString(err), bad16, bad32, O[32], O[33], O[34], O[35], O[36], O[40], O[48], O[56], O[63]);
    }
    return 0;
}
