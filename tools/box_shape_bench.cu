// Developer microbenchmark (not part of the product): does the A·Hᵀ pass's TMA box shape cost
// HBM rate on random data? Streams a 65536² f32 matrix (hash-filled, not zeros) through a
// persistent 5-stage TMA ring of 32 KB stages, each stage ONE 3-D operation of (32 floats,
// R rows, 8192/(32R) atoms) — R = 128 is pass 1's layout (256 B per row), R = 64 pass 2's
// (512 B per row), R = 32 1 KB per row. Each CTA walks its contiguous range of row-block-major
// stages (the pass's stream-K order). Configs alternate over several rounds so board power state
// is shared; each timing covers 200 passes (≈0.5 s) and reads NVML's energy counter around
// them (mJ per pass: a pattern that activates more DRAM rows costs more energy at equal speed,
// which is what matters under the board's power cap).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/box_shape_bench tools/box_shape_bench.cu -lcuda \
//   -L/usr/local/cuda/lib64/stubs -lnvidia-ml
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvml.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
                     : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
    } while (!ok);
}

__global__ void k_fill(float* a, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32) * 40503u;
        x ^= x >> 15, x *= 2246822519u, x ^= x >> 13;
        a[i] = float(x >> 8) * (1.f / 16777216.f);
    }
}

constexpr int kStages = 5, kStageBytes = 32768;

// stage t: row block t / spr (R rows), atom block t % spr (A atoms of 32 floats)
__global__ void k_stream(const __grid_constant__ CUtensorMap m, int64_t n_stages, int spr, int R, int A, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint64_t* full = (uint64_t*)(sm + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    const int64_t c = blockIdx.x, G = gridDim.x;
    const int64_t t0 = c * n_stages / G, t1 = (c + 1) * n_stages / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + s)) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(empty + s, ph ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(kStageBytes)
                         : "memory");
            const int rb = int(t / spr), ab = int(t % spr);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
                    su32(sm + s * kStageBytes)),
                "l"(&m), "r"(su32(full + s)), "r"(0), "r"(rb * R), "r"(ab * A), "l"(0x12F0000000000000ull)
                : "memory");
            if (++s == kStages) s = 0, ph ^= 1;
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        float acc = 0.f;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(full + s, ph);
            acc += ((float*)(sm + s * kStageBytes))[t & 255];
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
            if (++s == kStages) s = 0, ph ^= 1;
        }
        if (acc == 12345.f) sink[0] = acc;
    }
}

int main() {
    const int64_t M = 65536, N = 65536;
    float* a;
    if (cudaMalloc(&a, M * N * 4) != cudaSuccess) return 1;
    k_fill<<<148 * 8, 256>>>(a, M * N);
    float* sink;
    cudaMalloc(&sink, 4);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = size_t(kStages) * kStageBytes + 1024 + 256;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int Rs[3] = {128, 64, 32};
    CUtensorMap maps[3];
    for (int i = 0; i < 3; ++i) {
        const int R = Rs[i], A = kStageBytes / (R * 128);
        cuuint64_t dims[3] = {32u, cuuint64_t(M), cuuint64_t(N / 32)}, strides[2] = {cuuint64_t(N) * 4, 128u};
        cuuint32_t box[3] = {32u, cuuint32_t(R), cuuint32_t(A)}, es[3] = {1, 1, 1};
        if (fn(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode failed R=%d\n", R);
            return 1;
        }
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    const int passes = 200;
    nvmlDevice_t dev;
    const bool nv = nvmlInit() == NVML_SUCCESS && nvmlDeviceGetHandleByIndex(0, &dev) == NVML_SUCCESS;
    for (int round = 0; round < 4; ++round)
        for (int i = 0; i < 3; ++i) {
            const int R = Rs[i], A = kStageBytes / (R * 128);
            const int spr = int(N / 32 / A);
            const int64_t n_stages = (M / R) * spr;
            k_stream<<<sms, 64, smem>>>(maps[i], n_stages, spr, R, A, sink);
            cudaDeviceSynchronize();
            unsigned long long en0 = 0, en1 = 0;
            if (nv) nvmlDeviceGetTotalEnergyConsumption(dev, &en0);
            cudaEventRecord(e0);
            for (int p = 0; p < passes; ++p) k_stream<<<sms, 64, smem>>>(maps[i], n_stages, spr, R, A, sink);
            cudaEventRecord(e1);
            const cudaError_t err = cudaEventSynchronize(e1);
            if (nv) nvmlDeviceGetTotalEnergyConsumption(dev, &en1);
            unsigned sm_mhz = 0;
            if (nv) nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &sm_mhz);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("round %d box %3d rows x %d atoms (%4d B/row): %s %.3f ms/pass %.1f GB/s, %.1f mJ/pass, %.0f W, SM %u MHz\n",
                   round, R, A, A * 128, cudaGetErrorString(err), ms / passes, M * N * 4.0 * passes / (ms * 1e-3) / 1e9,
                   double(en1 - en0) / passes, double(en1 - en0) / ms, sm_mhz);
        }
    return 0;
}
