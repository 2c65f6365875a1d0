// Developer microbenchmark: how fast can a persistent TMA ring stream a row-major f32 matrix
// through shared memory on B200, as a function of box shape / stages / CTAs per SM?
// (No compute: consumers release a stage as soon as it lands.) Not part of the product.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
    } while (!ok);
}

// Each CTA streams tiles (tile_rows x tile_cols, as nbox boxes of box_cols columns) of its
// contiguous share of the tile sequence (tiles ordered row-block-major).
__global__ void k_stream(const __grid_constant__ CUtensorMap m, int64_t n_tiles, int tiles_per_row, int tile_rows,
                         int tile_cols, int box_cols, int stages, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int stage_bytes = tile_rows * tile_cols * 4;
    uint64_t* full = (uint64_t*)(sm + stages * stage_bytes);
    uint64_t* empty = full + stages;
    const int64_t c = blockIdx.x, G = gridDim.x;
    const int64_t t0 = c * n_tiles / G, t1 = (c + 1) * n_tiles / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(full + s)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(empty + s)) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (threadIdx.x == 0) {
        int s = 0; uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(empty + s, ph ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(full + s)), "r"(stage_bytes) : "memory");
            const int rb = int(t / tiles_per_row), cb = int(t % tiles_per_row);
            for (int j = 0; j < tile_cols / box_cols; ++j) {
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
                    :: "r"(su32(sm + s * stage_bytes + j * tile_rows * box_cols * 4)), "l"(&m), "r"(su32(full + s)),
                       "r"(cb * tile_cols + j * box_cols), "r"(rb * tile_rows), "l"(0x12F0000000000000ull) : "memory");
            }
            if (++s == stages) s = 0, ph ^= 1;
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(full + s, ph);
            acc += ((float*)(sm + s * stage_bytes))[t & 255];
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(empty + s)) : "memory");
            if (++s == stages) s = 0, ph ^= 1;
        }
        if (acc == 12345.f) sink[0] = acc;
    }
}

int main() {
    const int64_t M = 65536, N = 65536;
    float* A; cudaMalloc(&A, M * N * 4); cudaMemset(A, 0, M * N * 4);
    float* sink; cudaMalloc(&sink, 4);
    void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    struct Cfg { int tr, tc, bc, st, cps; bool sw32; };
    std::vector<Cfg> cfgs = {
        {128, 32, 32, 6, 1, false}, {128, 32, 32, 12, 1, false}, {128, 64, 32, 6, 1, false}, {128, 128, 32, 3, 1, false},
        {32, 128, 32, 6, 1, true}, {32, 128, 32, 12, 1, true}, {64, 128, 32, 6, 1, true}, {16, 256, 32, 12, 1, true},
        {128, 32, 32, 6, 2, false}, {32, 128, 32, 6, 2, true}, {8, 512, 32, 12, 1, true}, {128, 32, 32, 4, 3, false}};
    for (auto c : cfgs) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M}, strides[1] = {(cuuint64_t)N * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.bc, (cuuint32_t)c.tr}, es[2] = {1, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        c.sw32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int64_t tiles_per_row = N / c.tc, n_tiles = (M / c.tr) * tiles_per_row;
        const size_t smem = (size_t)c.st * c.tr * c.tc * 4 + 1024 + 256;
        const int grid = sms * c.cps;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) k_stream<<<grid, 64, smem>>>(m, n_tiles, (int)tiles_per_row, c.tr, c.tc, c.bc, c.st, sink);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int rep = 0; rep < reps; ++rep) k_stream<<<grid, 64, smem>>>(m, n_tiles, (int)tiles_per_row, c.tr, c.tc, c.bc, c.st, sink);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        printf("tile %3dx%3d box_cols %2d stages %2d ctas/SM %d smem %6zu: %s %.1f GB/s\n", c.tr, c.tc, c.bc, c.st, c.cps, smem,
               cudaGetErrorString(err), M * N * 4.0 * reps / (ms * 1e-3) / 1e9);
    }
    return 0;
}
