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

// positive pseudo-random fill (zeros would send every division down its slow path)
__global__ void fill(float* p, int64_t n, uint32_t seed, float lo, float hi) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ seed;
        x ^= x >> 15, x *= 2246822519u, x ^= x >> 13;
        p[i] = lo + (hi - lo) * (x >> 8) * (1.0f / 16777216.0f);
    }
}
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

#ifdef OOC_FU_PROFILE
namespace ooc { void fu_profile_read(unsigned long long* out, bool reset); }
#endif

int main(int argc, char** argv) {
    const int kp = argc > 1 ? atoi(argv[1]) : 32;
    const int64_t rows = argc > 2 ? atoll(argv[2]) : 65536, cols = 65536;
    const bool with_cat = argc > 3 ? atoi(argv[3]) != 0 : true;  // [F | lo(F)] copy (dense TC path)
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
    fill<<<1184, 256>>>(F, rows * kp, 1, 0.5f, 1.5f);
    fill<<<1184, 256>>>(N, rows * kp, 2, 0.5f, 1.5f);
    fill<<<1184, 256>>>(slots, int64_t(sk.G * sk.smax) * kTile * kp, 3, 0.2f, 0.6f);
    fill<<<1, 256>>>(G, kp * kp, 4, 1.0f / kp, 2.0f / kp);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 50;
    for (int form = 0; form < 2; ++form) {
        auto run = [&] {
            if (form == 0)
                CK(launch_factor_update(kp, F, rows, nullptr, slots, &sk, G, 1e-16f, true, gram, nullptr, flag, with_cat ? cat : nullptr, 0));
            else
                CK(launch_factor_update(kp, F, rows, N, nullptr, nullptr, G, 1e-16f, true, gram, err, flag, with_cat ? cat : nullptr, 0));
            CK(launch_reduce_slots(gram, fg, int64_t(kp) * kp, o32, o64, 0));
        };
        for (int i = 0; i < 3; ++i) run();
#ifdef OOC_FU_PROFILE
        unsigned long long pr[8];
        CK(cudaDeviceSynchronize());
        fu_profile_read(pr, true);
#endif
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
#ifdef OOC_FU_PROFILE
        fu_profile_read(pr, true);
        const char* nm[8] = {"prefetch", "streamk", "cpwait", "barrier", "update", "barrier2", "writeback", "gram"};
        double tot = 0;
        for (int i = 0; i < 8; ++i) tot += double(pr[i]);
        for (int i = 0; i < 8; ++i) printf("  %-9s %5.1f%%\n", nm[i], 100.0 * double(pr[i]) / tot);
#endif
        printf("kp %d rows %ld %s%s: update + gram reduce %.1f us (grid %d)\n", kp, long(rows),
               form == 0 ? "W form (slots)" : "H form (plain, err)", with_cat ? " +cat" : "", ms * 1e3 / reps, fg);
    }
    return 0;
}
