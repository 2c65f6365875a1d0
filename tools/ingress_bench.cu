// Developer microbenchmark: does a small L2-resident operand loaded next to every streamed A
// tile (the factor rows B of the MU passes) slow the HBM stream? One persistent CTA per SM,
// TMA ring of (A 128 x 64 f32 tile + B bytes of 64-row x 32-col boxes), consumers release a
// stage as soon as it lands. Not part of the product.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 tools/ingress_bench.cu -lcuda -o tools/ingress_bench
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
                     : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
                 ::"r"(su32(dst)), "l"(m), "r"(su32(bar)), "r"(x), "r"(y), "l"(pol) : "memory");
}

__global__ void k_stream(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int64_t n_tiles,
                         int tiles_per_row, int b_boxes, int b_rows_total, int stages, float* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
    const int a_bytes = 128 * 64 * 4, stage_bytes = a_bytes + b_boxes * 8192;
    uint64_t* full = (uint64_t*)(sm + stages * stage_bytes);
    uint64_t* empty = full + stages;
    const int64_t c = blockIdx.x, G = gridDim.x;
    const int64_t t0 = c * n_tiles / G, t1 = (c + 1) * n_tiles / G;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
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
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(stage_bytes) : "memory");
            const int rb = int(t / tiles_per_row), cb = int(t % tiles_per_row);
            uint8_t* st = sm + s * stage_bytes;
            for (int j = 0; j < 2; ++j) tma2d(st + j * 16384, &ma, full + s, cb * 64 + j * 32, rb * 128, 0x12F0000000000000ull);
            const int brow = int((cb * 64) % b_rows_total);
            for (int j = 0; j < b_boxes; ++j)
                tma2d(st + a_bytes + j * 8192, &mb, full + s, j * 32, brow, 0x14F0000000000000ull);
            if (++s == stages) s = 0, ph ^= 1;
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        float acc = 0.f;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(full + s, ph);
            acc += ((float*)(sm + s * stage_bytes))[t & 255];
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
            if (++s == stages) s = 0, ph ^= 1;
        }
        if (acc == 12345.f) sink[0] = acc;
    }
}

int main() {
    const int64_t M = 65536, N = 65536, BR = 65536, BC = 128;
    float *A, *B, *sink;
    cudaMalloc(&A, M * N * 4);
    cudaMemset(A, 0, M * N * 4);
    cudaMalloc(&B, BR * BC * 4);
    cudaMemset(B, 0, BR * BC * 4);
    cudaMalloc(&sink, 4);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    CUtensorMap ma, mb;
    cuuint64_t da[2] = {(cuuint64_t)N, (cuuint64_t)M}, sa[1] = {(cuuint64_t)N * 4};
    cuuint32_t ba[2] = {32, 128}, es[2] = {1, 1};
    fn(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t db[2] = {(cuuint64_t)BC, (cuuint64_t)BR}, sb[1] = {(cuuint64_t)BC * 4};
    cuuint32_t bb[2] = {32, 64};
    fn(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int bboxes = 0; bboxes <= 4; ++bboxes) {
        const int stage_bytes = 32768 + bboxes * 8192;
        const int stages = (220 * 1024) / stage_bytes;
        const size_t smem = (size_t)stages * stage_bytes + 1024 + 512;
        const int64_t tiles_per_row = N / 64, n_tiles = (M / 128) * tiles_per_row;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep)
            k_stream<<<sms, 64, smem>>>(ma, mb, n_tiles, (int)tiles_per_row, bboxes, (int)BR, stages, sink);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int rep = 0; rep < reps; ++rep)
            k_stream<<<sms, 64, smem>>>(ma, mb, n_tiles, (int)tiles_per_row, bboxes, (int)BR, stages, sink);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ms * 1e-3 / reps;
        printf("B per A tile %2d KB (%d boxes) stages %d: %s  pass %.3f ms  A %.1f GB/s  SM ingress %.1f GB/s\n",
               bboxes * 8, bboxes, stages, cudaGetErrorString(err), t * 1e3, M * N * 4.0 / t / 1e9,
               M * N * 4.0 * stage_bytes / 32768.0 / t / 1e9);
    }
    return 0;
}
