// The sharded H update of the row-partitioned solve as ONE kernel over NVLink SHARP (NVLS)
// multicast: reduce-scatter of W^T A, the MU update of this rank's H rows and the all-gather of
// the new rows, fused.
//
// The reference (src/nmf_distributed.cpp:171-185) all-reduces the packed [W^T A | W^T W] and
// every rank repeats the whole H update. The NCCL path of this backend (solver.cu h_update)
// reduce-scatters W^T A, updates n/N rows and all-gathers H: two collectives around a small
// kernel (config 3 at N = 4: 537 MB each way, 1.45 ms of NCCL time per iteration). Here the
// partial W^T A of every rank and Ht live in NCCL symmetric memory (ncclMemAlloc +
// ncclCommWindowRegister) with a multicast mapping (ncclDevCommCreate, lsaMultimem), and
//   1. a cross-rank barrier (per CTA index: multimem.red.release on a symmetric counter, spin
//      with acquire; traps after 2x the group timeout instead of hanging) orders this launch after every rank's
//      A^T W SpMM;
//   2. each warp lane group reads its rows' reduced W^T A with multimem.ld_reduce (the switch
//      sums the N ranks' partials), the old H row locally, computes
//      h <- h * nu * rcp_rn(h . W^T W + eps) (the factor-update kernel's formula) and
//      multimem.st's the new row into every rank's Ht;
//   3. a second barrier: when any rank's kernel has finished, every rank's stores have landed.
// Requires NCCL >= 2.28 (the device API) and NVLS on the box; solver.cu falls back to the NCCL
// collectives otherwise. Developer probe with NCCL's own RS + AG for scale: tools/nvls_probe.cu.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.h"

#if defined(NCCL_VERSION_CODE) && NCCL_VERSION_CODE >= NCCL_VERSION(2, 28, 0)
#define OOC_HAVE_NVLS 1
#include <nccl_device.h>
#endif

namespace ooc {
namespace {

#ifdef OOC_HAVE_NVLS
__global__ void k_nvls_resolve(ncclWindow_t wp, ncclWindow_t ht, ncclWindow_t bar, ncclDevComm dc, void** out) {
    out[0] = ncclGetLsaMultimemPointer(wp, 0, dc);
    out[1] = ncclGetLsaMultimemPointer(ht, 0, dc);
    out[2] = ncclGetLsaMultimemPointer(bar, 0, dc);
}
#endif

// all CTAs with this index on every rank arrive, then wait for the count of this phase
__device__ __forceinline__ void mc_barrier(unsigned* mc_ctr, const unsigned* ctr, unsigned target, uint64_t limit) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_ctr), "r"(1u) : "memory");
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (true) {
            unsigned v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (int(v - target) >= 0) break;
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > limit) asm volatile("trap;");  // a peer that never arrives
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void mc_ld_reduce4(const float* p, float (&v)[4]) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void mc_st4(float* p, const float (&v)[4]) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
}

// KP / 4 lanes per row, each owning 4 columns; U rows per lane group in flight.
template <int KP, int U>
__global__ void __launch_bounds__(256) k_h_update_nvls(NvlsArgs a) {
    constexpr int L = KP / 4, RPW = 32 / L;
    __shared__ float wtw[KP * KP];
    const unsigned tgt = unsigned(a.nranks) * (2u * a.epoch + 1u);
    mc_barrier(a.mc_bar + blockIdx.x, a.bar + blockIdx.x, tgt, a.timeout_ns);
    for (int i = threadIdx.x; i < KP * KP; i += blockDim.x) wtw[i] = a.wtw[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, sub = lane / L, j0 = 4 * (lane % L);
    const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u) << (sub * L));
    const int64_t groups_per_cta = int64_t(blockDim.x / 32) * RPW;
    const int64_t gstride = int64_t(gridDim.x) * groups_per_cta;
    bool bad = false;
    for (int64_t g0 = int64_t(blockIdx.x) * groups_per_cta + (threadIdx.x >> 5) * RPW + sub; g0 < a.rows;
         g0 += U * gstride) {
        float nu[U][4], h[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = g0 + u * gstride;
            if (r < a.rows) {
                const int64_t off = (a.row0 + r) * KP + j0;
                mc_ld_reduce4(a.mc_wp + off, nu[u]);
                const float4 o = *reinterpret_cast<const float4*>(a.ht + off);
                h[u][0] = o.x, h[u][1] = o.y, h[u][2] = o.z, h[u][3] = o.w;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = g0 + u * gstride;
            if (r >= a.rows) continue;  // (uniform across the lane group)
            // de_j = sum_q h_q W^T W[q][j], q ascending (the whole old row through shuffles)
            float de[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const float hq = __shfl_sync(gmask, h[u][q & 3], sub * L + (q >> 2));
#pragma unroll
                for (int t = 0; t < 4; ++t) de[t] = fmaf(hq, wtw[q * KP + j0 + t], de[t]);
            }
            float w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                w[t] = (h[u][t] * nu[u][t]) * __frcp_rn(de[t] + a.eps);
                bad |= !isfinite(w[t]);
            }
            mc_st4(a.mc_ht + (a.row0 + r) * KP + j0, w);
        }
    }
    if (bad) atomicOr(a.flag, 1);
    mc_barrier(a.mc_bar + blockIdx.x, a.bar + blockIdx.x, tgt + unsigned(a.nranks), a.timeout_ns);
}

}  // namespace

bool nvls_compiled() {
#ifdef OOC_HAVE_NVLS
    return true;
#else
    return false;
#endif
}

#ifdef OOC_HAVE_NVLS
namespace {
cudaError_t nvls_resolve(NvlsState& st, cudaStream_t s) {
    void** d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, 3 * sizeof(void*), s);
    if (e != cudaSuccess) return e;
    k_nvls_resolve<<<1, 1, 0, s>>>(static_cast<ncclWindow_t>(st.win[0]), static_cast<ncclWindow_t>(st.win[1]),
                                   static_cast<ncclWindow_t>(st.win[2]), *static_cast<ncclDevComm*>(st.devcomm), d);
    if ((e = cudaGetLastError()) == cudaSuccess)
        e = cudaMemcpyAsync(st.mc, d, 3 * sizeof(void*), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    return e;
}
}  // namespace
#endif

bool nvls_setup(NvlsState& st, ncclComm_t comm, size_t wp_bytes, size_t ht_bytes, int nbar, cudaStream_t s,
                std::string* why) {
#ifndef OOC_HAVE_NVLS
    (void)st, (void)comm, (void)wp_bytes, (void)ht_bytes, (void)nbar, (void)s;
    if (why) *why = "built without NCCL >= 2.28 (device API)";
    return false;
#else
    st = NvlsState{};
    st.wp_bytes = wp_bytes, st.ht_bytes = ht_bytes;
    st.bar_bytes = std::max<size_t>(4096, size_t(nbar) * 4);
    auto bad = [&](const char* what, const char* msg) {
        if (why) *why = std::string(what) + ": " + msg;
        nvls_teardown(st, comm);
        return false;
    };
    ncclResult_t r;
    if ((r = ncclMemAlloc(&st.wp, wp_bytes)) != ncclSuccess) return bad("ncclMemAlloc", ncclGetErrorString(r));
    if ((r = ncclMemAlloc(&st.ht, ht_bytes)) != ncclSuccess) return bad("ncclMemAlloc", ncclGetErrorString(r));
    if ((r = ncclMemAlloc(&st.bar, st.bar_bytes)) != ncclSuccess) return bad("ncclMemAlloc", ncclGetErrorString(r));
    cudaError_t e;
    if ((e = cudaMemsetAsync(st.bar, 0, st.bar_bytes, s)) != cudaSuccess) return bad("memset", cudaGetErrorString(e));
    if ((e = cudaMemsetAsync(st.wp, 0, wp_bytes, s)) != cudaSuccess) return bad("memset", cudaGetErrorString(e));
    void* bufs[3] = {st.wp, st.ht, st.bar};
    const size_t sizes[3] = {wp_bytes, ht_bytes, st.bar_bytes};
    for (int i = 0; i < 3; ++i) {
        ncclWindow_t w = nullptr;
        if ((r = ncclCommWindowRegister(comm, bufs[i], sizes[i], &w, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)
            return bad("ncclCommWindowRegister", ncclGetErrorString(r));
        st.win[i] = w;
    }
    auto* dc = new ncclDevComm{};
    ncclDevCommRequirements req = {};
    req.lsaMultimem = true;
    if ((r = ncclDevCommCreate(comm, &req, dc)) != ncclSuccess) {
        delete dc;
        return bad("ncclDevCommCreate (lsa multimem)", ncclGetErrorString(r));
    }
    st.devcomm = dc;
    if ((e = nvls_resolve(st, s)) != cudaSuccess) return bad("multicast addresses", cudaGetErrorString(e));
    if (!st.mc[0] || !st.mc[1] || !st.mc[2]) return bad("multicast addresses", "no NVLS multicast on this group");
    return true;
#endif
}

void nvls_teardown(NvlsState& st, ncclComm_t comm) {
#ifdef OOC_HAVE_NVLS
    if (st.devcomm) {
        ncclDevCommDestroy(comm, static_cast<ncclDevComm*>(st.devcomm));
        delete static_cast<ncclDevComm*>(st.devcomm);
    }
    for (void*& w : st.win)
        if (w) ncclCommWindowDeregister(comm, static_cast<ncclWindow_t>(w)), w = nullptr;
    for (void* p : {st.wp, st.ht, st.bar})
        if (p) ncclMemFree(p);
#else
    (void)comm;
#endif
    st = NvlsState{};
}

cudaError_t launch_h_update_nvls(int kp, const NvlsArgs& a, int grid, cudaStream_t s) {
    static const int u = [] {  // developer knob: rows in flight per lane group (2 or 4)
        const char* e = std::getenv("OOCNMF_NVLS_U");
        return e && e[0] == '4' ? 4 : 2;
    }();
    switch (kp * 10 + u) {
        case 162: k_h_update_nvls<16, 2><<<grid, 256, 0, s>>>(a); break;
        case 322: k_h_update_nvls<32, 2><<<grid, 256, 0, s>>>(a); break;
        case 642: k_h_update_nvls<64, 2><<<grid, 256, 0, s>>>(a); break;
        case 164: k_h_update_nvls<16, 4><<<grid, 256, 0, s>>>(a); break;
        case 324: k_h_update_nvls<32, 4><<<grid, 256, 0, s>>>(a); break;
        case 644: k_h_update_nvls<64, 4><<<grid, 256, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace ooc
