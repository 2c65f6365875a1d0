// Developer microbenchmark: the MU factor-update kernel (kernels_factor.cu) at config-2 shape
// (65536 rows, kp = 32), through the product launchers, in its W form (numerator from
// stream-K slots) and H form (plain numerator, error slots). Not part of the product. build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include -I paper_2202_09518_b200/csrc \
//     tools/fu_bench.cu paper_2202_09518_b200/csrc/kernels_factor.cu paper_2202_09518_b200/csrc/kernels_dense.cu \
//     -o tools/fu_bench
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

using namespace ooc;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

int main(int argc, char** argv) {
    const int kp = argc > 1 ? atoi(argv[1]) : 32;
    const int64_t rows = argc > 2 ? atoll(argv[2]) : 65536, cols = 65536;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    StreamK sk;
    plan_aht(sk, rows, cols, sms, kTcStep);
    float *F, *N, *slots, *G, *cat, *o32;
    double *gram, *err, *o64;
    int* flag;
    const int fg = factor_grid(rows / kTile);
    CK(cudaMalloc(&F, rows * kp * 4));
    CK(cudaMalloc(&N, rows * kp * 4));
    CK(cudaMalloc(&cat, rows * 2 * kp * 4));
    CK(cudaMalloc(&slots, size_t(sk.G * sk.smax) * kTile * kp * 4));
    CK(cudaMalloc(&G, kp * kp * 4));
    CK(cudaMalloc(&gram, size_t(fg) * kp * kp * 8));
    CK(cudaMalloc(&err, size_t(fg) * 8));
    CK(cudaMalloc(&o32, kp * kp * 4));
    CK(cudaMalloc(&o64, kp * kp * 8));
    CK(cudaMalloc(&flag, 4));
    CK(cudaMemset(F, 0, rows * kp * 4));
    CK(cudaMemset(N, 0, rows * kp * 4));
    CK(cudaMemset(slots, 0, size_t(sk.G * sk.smax) * kTile * kp * 4));
    CK(cudaMemset(G, 0, kp * kp * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 50;
    for (int form = 0; form < 2; ++form) {
        auto run = [&] {
            if (form == 0)
                CK(launch_factor_update(kp, F, rows, nullptr, slots, &sk, G, 1e-16f, true, gram, nullptr, flag, cat, 0));
            else
                CK(launch_factor_update(kp, F, rows, N, nullptr, nullptr, G, 1e-16f, true, gram, err, flag, cat, 0));
            CK(launch_reduce_slots(gram, fg, int64_t(kp) * kp, o32, o64, 0));
        };
        for (int i = 0; i < 3; ++i) run();
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("kp %d rows %ld %s: update + gram reduce %.1f us (grid %d)\n", kp, long(rows),
               form == 0 ? "W form (slots)" : "H form (plain, err)", ms * 1e3 / reps, fg);
    }
    return 0;
}
