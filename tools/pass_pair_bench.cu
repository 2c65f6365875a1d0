// Developer probe (not part of the product): are the two tcgen05 passes equally fast on REAL
// (non-zero) data? Config-2 shape (65536², kp = 32), A and the factors hash-filled. Times
// (a) each pass alone, 10 back-to-back launches, and (b) the two passes interleaved as in an MU
// iteration (pass 1, pass 2, pass 1, ...), each launch bracketed by its own events; 4 rounds.
// build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include -I paper_2202_09518_b200/csrc \
//     tools/pass_pair_bench.cu paper_2202_09518_b200/csrc/kernels_tc.cu \
//     paper_2202_09518_b200/csrc/kernels_dense.cu -lcuda -o tools/pass_pair_bench
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

using namespace ooc;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__global__ void k_fill(float* a, int64_t n, uint32_t salt, float scale) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32) * 40503u ^ salt;
        x ^= x >> 15, x *= 2246822519u, x ^= x >> 13;
        a[i] = float(x >> 8) * (scale / 16777216.f);
    }
}

int main() {
    const int kp = 32;
    const int64_t mp = 65536, np = 65536;
    float *A, *Hc, *Wc, *slots1, *slots2;
    CK(cudaMalloc(&A, size_t(mp) * np * 4));
    CK(cudaMalloc(&Hc, size_t(np) * 2 * kp * 4));
    CK(cudaMalloc(&Wc, size_t(mp) * 2 * kp * 4));
    k_fill<<<148 * 8, 256>>>(A, mp * np, 1u, 1.f);
    k_fill<<<148 * 8, 256>>>(Hc, np * 2 * kp, 2u, 0.01f);
    k_fill<<<148 * 8, 256>>>(Wc, mp * 2 * kp, 3u, 0.01f);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    StreamK sk1, sk2;
    plan_aht(sk1, mp, np, sms, kTcStep);
    plan_wta(sk2, mp, np, sms, kTcStep);
    CK(cudaMalloc(&slots1, size_t(sk1.G * sk1.smax) * 128 * kp * 4));
    CK(cudaMalloc(&slots2, size_t(sk2.G * sk2.smax) * 128 * kp * 4));
    auto run = [&](int pass) {
        if (pass == 1) CK(launch_aht_tc(kp, A, np, mp, np, Hc, slots1, sk1, 0));
        else CK(launch_wta_tc(kp, A, np, mp, np, Wc, slots2, sk2, 0));
    };
    run(1), run(2);
    CK(cudaDeviceSynchronize());
    const int n = 10;
    cudaEvent_t ev[2 * n + 1];
    for (auto& e : ev) cudaEventCreate(&e);
    for (int round = 0; round < 4; ++round) {
        for (int pass = 1; pass <= 2; ++pass) {
            cudaEventRecord(ev[0]);
            for (int r = 0; r < n; ++r) run(pass);
            cudaEventRecord(ev[1]);
            CK(cudaEventSynchronize(ev[1]));
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[0], ev[1]);
            printf("round %d alone  pass %d: %.3f ms per launch\n", round, pass, ms / n);
        }
        cudaEventRecord(ev[0]);
        for (int r = 0; r < 2 * n; ++r) {
            run(1 + (r & 1));
            cudaEventRecord(ev[r + 1]);
        }
        CK(cudaEventSynchronize(ev[2 * n]));
        double t[2] = {0, 0};
        for (int r = 0; r < 2 * n; ++r) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[r], ev[r + 1]);
            t[r & 1] += ms;
        }
        printf("round %d interleaved: pass 1 %.3f ms, pass 2 %.3f ms per launch\n", round, t[0] / n, t[1] / n);
    }
    return 0;
}
