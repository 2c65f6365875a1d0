// Developer probe (not part of the product): TMA streaming rate from L2 versus HBM on B200.
// A persistent 148-CTA ring (5 x 32 KB stages, 3-D boxes of 128 rows x 2 atoms of 32 f32, the
// pass-1 box of kernels_tc.cu) streams a rows x 8192 f32 matrix `reps` times; when the matrix
// fits in L2 every pass after the first is served from L2. Prints TB/s per size, which bounds
// a fused iteration's second (L2) pass over a row block and the B-operand re-reads.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/l2_probe.cu -lcuda -o tools/l2_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);            \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(par)
            : "memory");
    } while (!ok);
}

constexpr int kStages = 5, kStage = 32768;

// tiles: 128 rows x 64 cols; CTA c streams tiles [c T / G, (c + 1) T / G) `reps` times
__global__ void k_stream(const __grid_constant__ CUtensorMap m, int64_t n_tiles, int tiles_per_row, int reps,
                         uint64_t policy, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint64_t* full = (uint64_t*)(sm + kStages * kStage);
    uint64_t* empty = full + kStages;
    const int64_t c = blockIdx.x, G = gridDim.x;
    const int64_t t0 = c * n_tiles / G, t1 = (c + 1) * n_tiles / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + s)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t total = (t1 - t0) * reps;
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t u = 0; u < total; ++u) {
            const int64_t t = t0 + u % (t1 - t0);
            mbar_wait(empty + s, ph ^ 1u);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(kStage)
                         : "memory");
            const int row = int(t / tiles_per_row) * 128, atom = int(t % tiles_per_row) * 2;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(su32(sm + s * kStage)),
                "l"(&m), "r"(su32(full + s)), "r"(0), "r"(row), "r"(atom), "l"(policy)
                : "memory");
            if (++s == kStages) s = 0, ph ^= 1u;
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        float acc = 0.f;
        for (int64_t u = 0; u < total; ++u) {
            mbar_wait(full + s, ph);
            acc += *(volatile float*)(sm + s * kStage);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
            if (++s == kStages) s = 0, ph ^= 1u;
        }
        if (acc == 12345.f) *sink = acc;
    }
}

int main(int argc, char** argv) {
    const int64_t n = 8192;
    const long sizes_mb[] = {16, 32, 48, 64, 80, 96, 112, 128, 192, 256, 2048};
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *A, *sink;
    const size_t max_bytes = size_t(2048) << 20;
    CK(cudaMalloc(&A, max_bytes));
    CK(cudaMemset(A, 0, max_bytes));
    CK(cudaMalloc(&sink, 4));
    const size_t smem = kStages * kStage + 1024 + 256;
    CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const uint64_t pols[2] = {0x1000000000000000ull /*evict_normal*/, 0x14F0000000000000ull /*evict_last*/};
    const char* pn[2] = {"normal", "last"};
    for (int pi = 0; pi < 2; ++pi)
        for (long mb : sizes_mb) {
            const int64_t rows = (int64_t(mb) << 20) / (n * 4) / 128 * 128;
            CUtensorMap m;
            const cuuint64_t dims[3] = {32u, cuuint64_t(rows), cuuint64_t(n / 32)};
            const cuuint64_t strides[2] = {cuuint64_t(n) * 4, 128u};
            const cuuint32_t box[3] = {32u, 128u, 2u};
            const cuuint32_t estr[3] = {1u, 1u, 1u};
            if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, A, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("encode failed\n");
                return 1;
            }
            const int64_t tiles = rows / 128 * (n / 64);
            const int reps = int(std::max<long>(2, 8192 / mb));
            k_stream<<<sms, 64, smem>>>(m, tiles, int(n / 64), 2, pols[pi], sink);  // warm L2
            CK(cudaDeviceSynchronize());
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0), cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_stream<<<sms, 64, smem>>>(m, tiles, int(n / 64), reps, pols[pi], sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = double(rows) * n * 4 * reps;
            printf("policy %-6s %5ld MB x %4d reps: %.3f ms  %.2f TB/s\n", pn[pi], mb, reps, ms, bytes / ms / 1e9);
        }
    return 0;
}
