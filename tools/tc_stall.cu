// Developer probe: where the tcgen05 pass spends its time. Runs pass 1 / pass 2 at a full
// config-2 shape with kernels_tc.cu built with -DOOC_TC_PROFILE and prints, per role, the
// cycles spent in each barrier wait (averaged over CTAs, per 64-deep K step). Not part of the
// product. build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DOOC_TC_PROFILE -I include \
//     -I paper_2202_09518_b200/csrc tools/tc_stall.cu paper_2202_09518_b200/csrc/kernels_tc.cu \
//     paper_2202_09518_b200/csrc/kernels_dense.cu paper_2202_09518_b200/csrc/kernels_factor.cu paper_2202_09518_b200/csrc/kernels_wide.cu paper_2202_09518_b200/csrc/kernels_setup.cu -lcuda -o tools/tc_stall
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace ooc {
void tc_profile_read(unsigned long long* out16, bool reset);
}
using namespace ooc;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__global__ void k_fill(float* a, int64_t n, uint32_t salt, float scale) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32) * 40503u ^ salt;
        x ^= x >> 15, x *= 2246822519u, x ^= x >> 13;
        a[i] = float(x >> 8) * (scale / 16777216.f);
    }
}

// argv: kp mp np [random=0|1] [reps] (random: hash-filled A and factors instead of zeros)
int main(int argc, char** argv) {
    const int kp = argc > 1 ? atoi(argv[1]) : 32;
    const int64_t mp = argc > 2 ? atoll(argv[2]) : 65536, np = argc > 3 ? atoll(argv[3]) : 65536;
    const int reps = argc > 5 ? atoi(argv[5]) : 5;
    float *A, *Hc, *Wc, *slots;
    CK(cudaMalloc(&A, size_t(mp) * np * 4));
    CK(cudaMemset(A, 0, size_t(mp) * np * 4));
    CK(cudaMalloc(&Hc, size_t(np) * 2 * kp * 4));
    CK(cudaMalloc(&Wc, size_t(mp) * 2 * kp * 4));
    CK(cudaMemset(Hc, 0, size_t(np) * 2 * kp * 4));
    CK(cudaMemset(Wc, 0, size_t(mp) * 2 * kp * 4));
    if (argc > 4 && atoi(argv[4])) {
        k_fill<<<148 * 8, 256>>>(A, mp * np, 1u, 1.f);
        k_fill<<<148 * 8, 256>>>(Hc, np * 2 * kp, 2u, 0.01f);
        k_fill<<<148 * 8, 256>>>(Wc, mp * 2 * kp, 3u, 0.01f);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int pass_i = 0; pass_i < 4; ++pass_i) {
        const int pass = 1 + (pass_i & 1);
        StreamK sk;
        if (pass == 1) plan_aht(sk, mp, np, sms, kTcStep); else plan_wta(sk, mp, np, sms, kTcStep);
        CK(cudaMalloc(&slots, size_t(sk.G * sk.smax) * 128 * kp * 4));
        auto run = [&] {
            if (pass == 1) CK(launch_aht_tc(kp, A, np, mp, np, Hc, slots, sk, 0));
            else CK(launch_wta_tc(kp, A, np, mp, np, Wc, slots, sk, 0));
        };
        run();
        CK(cudaDeviceSynchronize());
        unsigned long long p[16];
        tc_profile_read(p, true);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) run();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        tc_profile_read(p, true);
        const double units = double(sk.total()) * reps;  // all CTAs
        const double per = 1.0 / units;                   // summed-over-CTAs cycles per unit
        const char* names[9] = {"producer wait emptyA", "producer wait emptyB", "split wait fullA", "split wait afree",
                                "-", "mma wait accempty", "mma wait fullB", "mma wait split", "drain wait accfull"};
        printf("pass %d kp %d %ldx%ld: %.3f ms per pass, %.0f units per CTA\n", pass, kp, long(mp), long(np), ms / reps,
               double(sk.total()) / sk.G);
        printf("  total cycles per unit: producer %.0f  mma %.0f  split %.0f  drain %.0f\n", p[9] * per, p[10] * per,
               p[11] * per, p[12] * per);
        for (int j = 0; j < 9; ++j)
            if (j != 4) printf("  %-22s %7.0f cycles/unit\n", names[j], p[j] * per);
        cudaFree(slots);
    }
    return 0;
}
