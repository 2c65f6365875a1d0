// Developer probe (not part of the product): NVLink SHARP (NVLS) multicast through NCCL 2.28's
// symmetric-memory device API, for a fused "reduce-scatter -> row update -> all-gather" of a
// config-3-sized W^T A / H (n = 2^22 rows x kp = 32 f32, 537 MB) on the GPUs of one box.
// One host thread per GPU (ncclCommInitAll). Per launch of k_rs_update_ag:
//   cross-rank barrier (multimem.red on a symmetric counter), each rank ld_reduce's its n/N rows
//   of the partial buffer (the switch sums the N ranks' copies), applies a stand-in update
//   (x 0.5), multimem.st's the rows into every rank's output, barrier.
// Checks the result on every rank and times it against NCCL's ReduceScatter + AllGather.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I$NCCL/include
//        tools/nvls_probe.cu -L$NCCL/lib -lnccl -Xlinker -rpath -Xlinker $NCCL/lib -o tools/nvls_probe
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include <nccl.h>
#include <nccl_device.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)
#define NK(x)                                                                                  \
    do {                                                                                       \
        ncclResult_t r_ = (x);                                                                 \
        if (r_ != ncclSuccess) {                                                               \
            std::printf("NCCL %s at %s:%d\n", ncclGetErrorString(r_), __FILE__, __LINE__); \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

__global__ void k_mc_ptrs(ncclWindow_t a, ncclWindow_t b, ncclWindow_t c, ncclDevComm dc, void** out) {
    out[0] = ncclGetLsaMultimemPointer(a, 0, dc);
    out[1] = ncclGetLsaMultimemPointer(b, 0, dc);
    out[2] = ncclGetLsaMultimemPointer(c, 0, dc);
}

__device__ __forceinline__ void mc_barrier(unsigned* mc_ctr, const unsigned* local_ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_ctr), "r"(1u) : "memory");
        unsigned v;
        long long t0 = clock64();
        while (true) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(local_ctr) : "memory");
            if (int(v - target) >= 0) break;
            if (clock64() - t0 > 20000000000ll) asm volatile("trap;");
        }
    }
    __syncthreads();
}

// rows [row0, row0 + rows) of the N-rank sum of `part` (kp = 32 floats a row), halved, stored
// to every rank's `out` (all multicast addresses).
__global__ void __launch_bounds__(256) k_rs_update_ag(const float* mc_part, float* mc_out, unsigned* mc_bar,
                                                     const unsigned* bar, unsigned epoch, int nranks, long row0,
                                                     long rows, const float* out_local, int* stale) {
    const float scale = 0.5f + float(epoch);
    const unsigned tgt = unsigned(nranks) * (2u * epoch + 1u);
    mc_barrier(mc_bar + blockIdx.x, bar + blockIdx.x, tgt);
    const long nvec = rows * 8;  // float4s
    const long base = row0 * 8;
    // U independent ld_reduce's in flight per thread, then their stores
    constexpr int U = 4;
    const long stride = long(gridDim.x) * blockDim.x;
    for (long i0 = blockIdx.x * long(blockDim.x) + threadIdx.x; i0 < nvec; i0 += U * stride) {
        float v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = i0 + u * stride;
            if (i < nvec)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3])
                             : "l"(mc_part + (base + i) * 4)
                             : "memory");
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = i0 + u * stride;
            if (i < nvec)
                asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_out + (base + i) * 4),
                             "f"(scale * v[u][0]), "f"(scale * v[u][1]), "f"(scale * v[u][2]), "f"(scale * v[u][3])
                             : "memory");
        }
    }
    mc_barrier(mc_bar + blockIdx.x, bar + blockIdx.x, tgt + unsigned(nranks));
    // ordering check: after the exit barrier, rows that other ranks stored must be visible here
    // (the value depends on the epoch, so a stale read is caught)
    const long total = rows * nranks;
    const float s = scale * float(nranks * (nranks + 1) / 2);
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total * 32; i += long(gridDim.x) * blockDim.x * 97) {
        if (out_local[i] != s * float((i % 1000) + 1)) atomicAdd(stale, 1);
    }
}

__global__ void k_fill(float* p, long n, int rank) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        p[i] = float(rank + 1) * float((i % 1000) + 1);
}
__global__ void k_check(const float* p, long n, int nranks, int* bad) {
    const float s = 0.5f * float(nranks * (nranks + 1) / 2);  // epoch 0
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        if (p[i] != s * float((i % 1000) + 1)) atomicAdd(bad, 1);
}

int main(int argc, char** argv) {
    int N = 0;
    CK(cudaGetDeviceCount(&N));
    if (argc > 1) N = std::min(N, std::atoi(argv[1]));
    const long n = 1l << 22, kp = 32, elems = n * kp;
    const size_t bytes = size_t(elems) * 4;
    std::vector<int> devs(N);
    for (int i = 0; i < N; ++i) devs[i] = i;
    std::vector<ncclComm_t> comms(N);
    NK(ncclCommInitAll(comms.data(), N, devs.data()));
    std::vector<std::thread> th;
    for (int r = 0; r < N; ++r)
        th.emplace_back([&, r] {
            CK(cudaSetDevice(r));
            ncclComm_t comm = comms[r];
            float *part, *out, *tmp;
            unsigned* bar;
            NK(ncclMemAlloc((void**)&part, bytes));
            NK(ncclMemAlloc((void**)&out, bytes));
            NK(ncclMemAlloc((void**)&bar, 4096));
            CK(cudaMalloc(&tmp, bytes));
            ncclWindow_t wp, wo, wb;
            NK(ncclCommWindowRegister(comm, part, bytes, &wp, NCCL_WIN_COLL_SYMMETRIC));
            NK(ncclCommWindowRegister(comm, out, bytes, &wo, NCCL_WIN_COLL_SYMMETRIC));
            NK(ncclCommWindowRegister(comm, bar, 4096, &wb, NCCL_WIN_COLL_SYMMETRIC));
            ncclDevCommRequirements req = {};
            req.lsaMultimem = true;
            ncclDevComm dc;
            NK(ncclDevCommCreate(comm, &req, &dc));
            void** dptr;
            CK(cudaMalloc(&dptr, 3 * sizeof(void*)));
            k_mc_ptrs<<<1, 1>>>(wp, wo, wb, dc, dptr);
            void* mc[3];
            CK(cudaMemcpy(mc, dptr, sizeof mc, cudaMemcpyDeviceToHost));
            k_fill<<<1184, 256>>>(part, elems, r);
            CK(cudaMemset(bar, 0, 4096));
            CK(cudaMemset(out, 0, bytes));
            CK(cudaDeviceSynchronize());
            // all ranks' counters zeroed before anyone arrives
            int* one;
            CK(cudaMalloc(&one, 4));
            NK(ncclAllReduce(one, one, 1, ncclInt, ncclSum, comm, 0));
            CK(cudaDeviceSynchronize());
            const long hr = n / N;
            const int G = argc > 2 ? std::atoi(argv[2]) : 148 * 4;
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            unsigned epoch = 0;
            int* stale;
            CK(cudaMalloc(&stale, 4));
            CK(cudaMemset(stale, 0, 4));
            k_rs_update_ag<<<G, 256>>>((const float*)mc[0], (float*)mc[1], (unsigned*)mc[2], bar, epoch++, N,
                                       r * hr, hr, out, stale);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            int* bad;
            CK(cudaMalloc(&bad, 4));
            CK(cudaMemset(bad, 0, 4));
            k_check<<<1184, 256>>>(out, elems, N, bad);
            int hbad = 0;
            CK(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
            const int reps = 20;
            CK(cudaEventRecord(e0));
            for (int i = 0; i < reps; ++i)
                k_rs_update_ag<<<G, 256>>>((const float*)mc[0], (float*)mc[1], (unsigned*)mc[2], bar, epoch++, N,
                                           r * hr, hr, out, stale);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            // NCCL baseline: reduce-scatter + all-gather of the same buffers
            CK(cudaEventRecord(e0));
            for (int i = 0; i < reps; ++i) {
                NK(ncclReduceScatter(part, tmp + r * hr * kp, hr * kp, ncclFloat, ncclSum, comm, 0));
                NK(ncclAllGather(tmp + r * hr * kp, tmp, hr * kp, ncclFloat, comm, 0));
            }
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms2 = 0;
            CK(cudaEventElapsedTime(&ms2, e0, e1));
            int hstale = 0;
            CK(cudaMemcpy(&hstale, stale, 4, cudaMemcpyDeviceToHost));
            std::printf("rank %d/%d: fused NVLS rs+update+ag %.3f ms, NCCL RS+AG %.3f ms, mismatches %d, stale reads %d\n",
                        r, N, ms / reps, ms2 / reps, hbad, hstale);
            CK(cudaDeviceSynchronize());
            NK(ncclDevCommDestroy(comm, &dc));
            NK(ncclCommWindowDeregister(comm, wp));
            NK(ncclCommWindowDeregister(comm, wo));
            NK(ncclCommWindowDeregister(comm, wb));
            NK(ncclMemFree(part));
            NK(ncclMemFree(out));
            NK(ncclMemFree(bar));
        });
    for (auto& t : th) t.join();
    for (auto c : comms) ncclCommDestroy(c);
    return 0;
}
