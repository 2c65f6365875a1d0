// Developer probe (not part of the product): the one-pass kernel (kernels_fused.cu) alone at a
// config-2 shape on hash-filled data, timed with CUDA events, with per-role wait cycles when
// built with -DOOC_FZ_PROFILE. build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DOOC_FZ_PROFILE -I include \
//     -I paper_2202_09518_b200/csrc tools/fz_stall.cu paper_2202_09518_b200/csrc/kernels_fused.cu \
//     paper_2202_09518_b200/csrc/kernels_tc.cu paper_2202_09518_b200/csrc/kernels_factor.cu paper_2202_09518_b200/csrc/kernels_wide.cu paper_2202_09518_b200/csrc/kernels_setup.cu -lcuda -o tools/fz_stall
// argv: kp mp np lookahead reps pol drain_units p2_first
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "kernels.h"

#ifdef OOC_FZ_PROFILE
namespace ooc {
void fz_profile_read(unsigned long long* out24, bool reset);
void fz_trace_set(unsigned long long* buf);
}
#else
static void fz_profile_read(unsigned long long* out24, bool) {
    for (int i = 0; i < 24; ++i) out24[i] = 0;
}
#endif
using namespace ooc;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);            \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

__global__ void k_fill(float* a, int64_t n, uint32_t salt, float scale) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32) * 40503u ^ salt;
        x ^= x >> 15, x *= 2246822519u, x ^= x >> 13;
        a[i] = float(x >> 8) * (scale / 16777216.f) + 1e-3f;
    }
}

int main(int argc, char** argv) {
    const int kp = argc > 1 ? atoi(argv[1]) : 32;
    const int64_t mp = argc > 2 ? atoll(argv[2]) : 65536, np = argc > 3 ? atoll(argv[3]) : 65536;
    const int D = argc > 4 ? atoi(argv[4]) : 2;
    const int reps = argc > 5 ? atoi(argv[5]) : 10;
    const int pol = argc > 6 ? atoi(argv[6]) : 0;
    const int du = argc > 7 ? atoi(argv[7]) : 2;
    const int p2f = argc > 8 ? atoi(argv[8]) : 0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *A, *W, *Wc, *Hc, *HHt, *wta, *slots;
    unsigned* cnt;
    int *flag, *idx;
    CK(cudaMalloc(&A, size_t(mp) * np * 4));
    CK(cudaMalloc(&W, size_t(mp) * kp * 4));
    CK(cudaMalloc(&Wc, size_t(mp) * 2 * kp * 4));
    CK(cudaMalloc(&Hc, size_t(np) * 2 * kp * 4));
    CK(cudaMalloc(&HHt, size_t(kp) * kp * 4));
    CK(cudaMalloc(&wta, size_t(np) * kp * 4));
    CK(cudaMalloc(&flag, 4));
    k_fill<<<sms * 8, 256>>>(A, mp * np, 1u, 1.f);
    k_fill<<<sms * 8, 256>>>(W, mp * kp, 2u, 0.5f);
    k_fill<<<sms * 8, 256>>>(Hc, np * 2 * kp, 3u, 0.01f);
    k_fill<<<sms * 8, 256>>>(HHt, kp * kp, 4u, 100.f);
    FusedPlan fp;
    plan_fused(fp, mp, np, sms, D);
    std::vector<int> h;
    h.insert(h.end(), fp.q0.begin(), fp.q0.end());
    h.insert(h.end(), fp.t0.begin(), fp.t0.end());
    h.insert(h.end(), fp.act.begin(), fp.act.end());
    CK(cudaMalloc(&idx, h.size() * 4));
    CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&slots, fused_slot_bytes(kp, fp)));
    CK(cudaMemset(slots, 0, fused_slot_bytes(kp, fp)));
    CK(cudaMalloc(&cnt, size_t(3) * fp.NB * 4));
    FusedArgs a{};
    a.NB = fp.NB, a.D = fp.D, a.NS = fp.NS, a.G1 = fp.G1, a.drain_units = du;
    a.p2_first = p2f;
    a.q0 = idx, a.t0 = idx + fp.G + 1, a.act = idx + 2 * (fp.G + 1);
    a.p1slots = slots, a.count = cnt, a.wdone = cnt + fp.NB;
    a.W = W, a.Wcat = Wc, a.HHt = HHt, a.eps = 1e-12f, a.flag = flag, a.wta = wta;
    setenv("OOCNMF_FUSED_POL", std::to_string(pol).c_str(), 0);
    fused_policies(a);
    printf("plan: G %d NB %d NT %d NQ %d D %d NS %d G1 %d; CTA 0: q [%d,%d) t [%d,%d)\n", fp.G, fp.NB, fp.NT, fp.NQ,
           fp.D, fp.NS, fp.G1, fp.q0[0], fp.q0[1], fp.t0[0], fp.t0[1]);
    auto run = [&] {
        CK(cudaMemsetAsync(cnt, 0, size_t(3) * fp.NB * 4, 0));
        CK(launch_mu_fused(kp, fp, A, mp, np, Hc, a, 0));
    };
    run();
    CK(cudaDeviceSynchronize());
    unsigned long long p[24];
    fz_profile_read(p, true);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    fz_profile_read(p, true);
    const double units = double(fp.NB) * (fp.NQ + 2.0 * fp.NT) / fp.G * reps;  // per CTA
    const double ctas = fp.G;
    printf("p2_first %d kp %d %ldx%ld D %d pol %d: %.3f ms per launch (%.2f TB/s of A once)\n", p2f, kp, long(mp), long(np), D, pol,
           ms / reps, double(mp) * np * 4 / (ms / reps) / 1e9);
    const char* role[6] = {"producerA", "mma", "updater", "producerB", "split", "drain"};
    printf("  total cycles per unit:");
    for (int r = 0; r < 6; ++r) printf(" %s %.0f", role[r], p[16 + r] / ctas / units);
    printf("\n");
    const char* name[13] = {"prodA wait emptyA",  "(unused)",          "(unused)",          "split wait fullA",
                            "split wait afree",   "mma wait accempty", "mma wait fullB",    "mma wait split",
                            "drain wait accfull", "updater wait count", "updater wait gather", "prodB wait emptyB",
                            "prodB wait W ready"};
    for (int j = 0; j < 13; ++j) printf("  %-22s %8.0f cycles/unit\n", name[j], p[j] / ctas / units);
#ifdef OOC_FZ_PROFILE
    // latency trace of blocks 8..63 of one more launch (ns, relative to the block's first publish)
    {
        const int TB = 64;
        unsigned long long* tr;
        CK(cudaMalloc(&tr, size_t(6) * TB * 256 * 8));
        CK(cudaMemset(tr, 0, size_t(6) * TB * 256 * 8));
        fz_trace_set(tr);
        run();
        CK(cudaDeviceSynchronize());
        fz_trace_set(nullptr);
        std::vector<unsigned long long> h(size_t(6) * TB * 256);
        CK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
        auto at = [&](int kind, int b, int i) { return h[(size_t(kind) * TB + b) * 256 + i]; };
        double s_last = 0, s_cnt = 0, s_upd_med = 0, s_upd = 0, s_wr = 0, s_wr_max = 0, s_step = 0;
        int nb = 0;
        for (int b = 8; b < TB && b < fp.NB; ++b) {
            unsigned long long p0 = ~0ull, p1 = 0, c0 = ~0ull, u1 = 0, w0 = ~0ull, w1 = 0;
            std::vector<unsigned long long> ups;
            for (int c = 0; c < fp.G; ++c)
                if (at(0, b, c)) p0 = std::min(p0, at(0, b, c)), p1 = std::max(p1, at(0, b, c));
            for (int r = 0; r < 128; ++r) {
                if (at(1, b, r)) c0 = std::min(c0, at(1, b, r));
                if (at(2, b, r) && r < 64) u1 = std::max(u1, at(2, b, r)), ups.push_back(at(2, b, r));
            }
            for (int c = 0; c < fp.G; ++c)
                if (at(3, b, c)) w0 = std::min(w0, at(3, b, c)), w1 = std::max(w1, at(3, b, c));
            std::sort(ups.begin(), ups.end());
            s_last += double(p1 - p0), s_cnt += double(c0 - p1), s_upd += double(u1 - c0);
            s_upd_med += double(ups[ups.size() / 2] - c0);
            s_wr += double(w0 - u1), s_wr_max += double(w1 - u1);
            if (b > 8) s_step += double(p1 - at(0, b - 1, 0));
            ++nb;
        }
        // per-CTA publish offset vs the block's median publish (us), averaged over blocks
        std::vector<double> off(fp.G, 0.0);
        for (int b = 8; b < TB && b < fp.NB; ++b) {
            std::vector<unsigned long long> v;
            for (int c = 0; c < fp.G; ++c) v.push_back(at(0, b, c));
            std::vector<unsigned long long> srt = v;
            std::sort(srt.begin(), srt.end());
            const double med = double(srt[srt.size() / 2]);
            for (int c = 0; c < fp.G; ++c) off[c] += (double(v[c]) - med) / 1e3 / nb;
        }
        std::vector<int> idx(fp.G);
        for (int c = 0; c < fp.G; ++c) idx[c] = c;
        std::sort(idx.begin(), idx.end(), [&](int x, int y) { return off[x] < off[y]; });
        printf("  earliest CTAs (cta:offset_us:n1:n2):");
        for (int i = 0; i < 6; ++i)
            printf(" %d:%.2f:%d:%d", idx[i], off[idx[i]], fp.q0[idx[i] + 1] - fp.q0[idx[i]],
                   2 * (fp.t0[idx[i] + 1] - fp.t0[idx[i]]));
        printf("\n  latest CTAs:");
        for (int i = fp.G - 6; i < fp.G; ++i)
            printf(" %d:%.2f:%d:%d", idx[i], off[idx[i]], fp.q0[idx[i] + 1] - fp.q0[idx[i]],
                   2 * (fp.t0[idx[i] + 1] - fp.t0[idx[i]]));
        double by_n1[16] = {}, cnt_n1[16] = {};
        for (int c = 0; c < fp.G; ++c) {
            const int n1 = fp.q0[c + 1] - fp.q0[c];
            if (n1 < 16) by_n1[n1] += off[c], cnt_n1[n1] += 1;
        }
        printf("\n  mean offset by P1 units:");
        for (int k = 0; k < 16; ++k)
            if (cnt_n1[k]) printf(" n1=%d:%.2f(%d)", k, by_n1[k] / cnt_n1[k], int(cnt_n1[k]));
        printf("\n");
        {   // per row (first half): count seen - first count seen, gather latency, compute + publish
            double d1 = 0, d2 = 0, d3 = 0, d4 = 0;
            int nr = 0;
            for (int b = 8; b < TB && b < fp.NB; ++b) {
                unsigned long long c0 = ~0ull;
                for (int r = 0; r < 64; ++r)
                    if (at(1, b, r)) c0 = std::min(c0, at(1, b, r));
                for (int r = 0; r < 64; ++r)
                    if (at(1, b, r) && at(4, b, r) && at(2, b, r)) {
                        d1 += double(at(1, b, r) - c0), d2 += double(at(4, b, r) - at(1, b, r));
                        d3 += double(at(5, b, r) - at(4, b, r)), d4 += double(at(2, b, r) - at(5, b, r)), ++nr;
                    }
            }
            printf("  per row (us): count seen after the first %.2f | gather %.2f | sum + update + stores %.2f | "
                   "publish %.2f\n", d1 / nr / 1e3, d2 / nr / 1e3, d3 / nr / 1e3, d4 / nr / 1e3);
        }
        printf("  latency (us, mean over %d blocks): publish spread %.2f | last publish -> first updater sees count "
               "%.2f | -> all 64 rows updated %.2f (median row %.2f) | -> first B producer sees W %.2f, last %.2f\n",
               nb, s_last / nb / 1e3, s_cnt / nb / 1e3, s_upd / nb / 1e3, s_upd_med / nb / 1e3, s_wr / nb / 1e3,
               s_wr_max / nb / 1e3);
    }
#endif
    return 0;
}
