// Developer probe for the tcgen05 passes: runs pass 1 / pass 2 on small random inputs and
// prints max relative error vs a host f64 reference, plus a few entries. Not part of the
// product; build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I include \
//   -I paper_2202_09518_b200/csrc tools/tc_probe.cu paper_2202_09518_b200/csrc/kernels_tc.cu \
//   paper_2202_09518_b200/csrc/kernels_factor.cu paper_2202_09518_b200/csrc/kernels_dense.cu -lcuda -o tools/tc_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"

using namespace ooc;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

static float lo_part(float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float h; memcpy(&h, &u, 4); return x - h; }

int run(int pass, int kp, int mp, int np, int sms) {
    std::vector<float> A(size_t(mp) * np), B(size_t(pass == 1 ? np : mp) * kp), Bl(B.size() * 2);
    srand(1);
    for (auto& x : A) x = rand() / float(RAND_MAX);
    for (size_t i = 0; i < B.size(); ++i) { B[i] = rand() / float(RAND_MAX); }
    for (size_t r = 0; r < B.size() / kp; ++r) for (int j = 0; j < kp; ++j) { Bl[r * 2 * kp + j] = B[r * kp + j]; Bl[r * 2 * kp + kp + j] = lo_part(B[r * kp + j]); }
    float *dA, *dB, *dBl, *dS, *dO;
    StreamK sk;
    if (pass == 1) plan_aht(sk, mp, np, sms, kTcStep); else plan_wta(sk, mp, np, sms, kTcStep);
    const int64_t out_rows = pass == 1 ? mp : np;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dBl, Bl.size() * 4));
    CK(cudaMalloc(&dS, size_t(sk.G * sk.smax) * 128 * kp * 4)); CK(cudaMalloc(&dO, size_t(out_rows) * kp * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dBl, Bl.data(), Bl.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dS, 0xFF, size_t(sk.G * sk.smax) * 128 * kp * 4));  // NaN fill: unwritten slots show up
    if (pass == 1) CK(launch_aht_tc(kp, dA, np, mp, np, dBl, dS, sk, 0));
    else CK(launch_wta_tc(kp, dA, np, mp, np, dBl, dS, sk, 0));
    CK(launch_streamk_reduce(kp, dS, sk, dO, false, 0));
    CK(cudaDeviceSynchronize());
    std::vector<float> O(size_t(out_rows) * kp);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0; int shown = 0;
    for (int64_t r = 0; r < out_rows; ++r)
        for (int j = 0; j < kp; ++j) {
            double ref = 0;
            if (pass == 1) for (int c = 0; c < np; ++c) ref += double(A[size_t(r) * np + c]) * B[size_t(c) * kp + j];
            else for (int i = 0; i < mp; ++i) ref += double(A[size_t(i) * np + r]) * B[size_t(i) * kp + j];
            const double got = O[size_t(r) * kp + j];
            const double rel = std::fabs(got - ref) / std::fabs(ref);
            if (!(rel <= maxrel)) maxrel = rel;
            if (!(rel < 1e-5) && shown < 6) { printf("  [%ld,%d] got %.7g want %.7g\n", long(r), j, got, ref); ++shown; }
        }
    printf("pass %d kp %d mp %d np %d G %ld: max rel err %.3e\n", pass, kp, mp, np, long(sk.G), maxrel);
    cudaFree(dA); cudaFree(dB); cudaFree(dBl); cudaFree(dS); cudaFree(dO);
    return maxrel < 1e-5 ? 0 : 1;
}

int main() {
    int bad = 0;
    bad += run(1, 16, 256, 256, 148);
    bad += run(2, 16, 256, 384, 148);
    bad += run(1, 32, 128, 128, 1);
    bad += run(1, 32, 256, 256, 148);
    bad += run(1, 64, 256, 256, 148);
    bad += run(2, 32, 128, 128, 1);
    bad += run(2, 32, 256, 256, 148);
    bad += run(2, 64, 256, 384, 148);
    bad += run(1, 32, 1024, 4096, 148);
    bad += run(2, 32, 1024, 4096, 148);
    printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
    return bad;
}
