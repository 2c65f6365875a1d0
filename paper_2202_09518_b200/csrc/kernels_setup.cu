// Setup-time and check-time kernels: on-device synthetic inputs and seeded init with the
// reference's counter RNG, f64->f32 staging, ||A||^2 and the direct residual (f64 sums).
#include "kernels.h"

namespace ooc {
namespace {

constexpr int kRedGrid = 4 * 148;

// A[i][j] = (float) U(seed, stream, (row0 + i) * n + j)   (bench/kernels_bench.cpp:12-18)
__global__ void k_gen_dense_uniform(float* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                    int64_t row0, int64_t n, uint64_t key) {
    const int64_t c4n = (cols + 3) / 4;
    const int64_t total = rows * c4n;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = q / c4n, j = (q % c4n) * 4;
        const uint64_t base = uint64_t(row0 + i) * uint64_t(n) + uint64_t(j);
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            v[t] = (j + t < cols) ? __double2float_rn(rng_u01(key, base + t)) : 0.f;
        *reinterpret_cast<float4*>(A + i * lda + j) = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// W[i][j] = U(seed,1,(row0+i)*k + j), H[r][c] = U(seed,2,r*n_global + col0 + c) stored as
// Ht[c][r] (src/nmf_serial.cpp:31-48; init_w_rows / init_h_cols windows), rounded to f32;
// padding stays zero (caller memsets).
__global__ void k_init_factors(float* __restrict__ W, float* __restrict__ Ht, int kp, int64_t k,
                               int64_t rows, int64_t row0, int64_t n, int64_t n_global, int64_t col0,
                               uint64_t kw, uint64_t kh) {
    const int64_t nw = rows * k, nh = n * k;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nw + nh;
         q += int64_t(gridDim.x) * blockDim.x) {
        if (q < nw) {
            const int64_t i = q / k, j = q % k;
            W[i * kp + j] = __double2float_rn(rng_u01(kw, uint64_t(row0 + i) * k + j));
        } else {
            const int64_t e = q - nw, r = e / n, c = e % n;
            Ht[c * kp + r] = __double2float_rn(rng_u01(kh, uint64_t(r) * n_global + uint64_t(col0 + c)));
        }
    }
}

__global__ void k_cast_pad_f64(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                               int64_t cols, float* __restrict__ dst, int64_t ld_dst) {
    const int64_t total = rows * cols;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = q / cols, j = q % cols;
        dst[i * ld_dst + j] = __double2float_rn(src[i * ld_src + j]);
    }
}

// Layout conversion for the copy-in / copy-out calls of the C-ABI: out(r, c) = in(r, c) for an
// R x C block with arbitrary element strides, converting the element type; the loop runs along
// the output's unit-stride axis so the writes coalesce.
template <class Tin, class Tout>
__global__ void k_strided_cast(const Tin* __restrict__ in, int64_t is_r, int64_t is_c, Tout* __restrict__ out,
                               int64_t os_r, int64_t os_c, int64_t R, int64_t C, bool rows_fast) {
    const int64_t total = R * C;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = rows_fast ? q % R : q / C, c = rows_fast ? q / R : q % C;
        out[r * os_r + c * os_c] = Tout(in[r * is_r + c * is_c]);
    }
}

__device__ double block_sum(double v) {
    __shared__ double sh[256];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    return sh[0];
}

__global__ void __launch_bounds__(256) k_sq_norm_dense(const float* __restrict__ A, int64_t lda,
                                                       int64_t rows, int64_t cols4,
                                                       double* __restrict__ out) {
    double acc = 0.0;
    const int64_t total = rows * cols4;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = q / cols4, j = (q % cols4) * 4;
        const float4 v = *reinterpret_cast<const float4*>(A + i * lda + j);
        acc += double(v.x) * v.x + double(v.y) * v.y + double(v.z) * v.z + double(v.w) * v.w;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_sq_norm_vals(const float* __restrict__ v, int64_t nnz,
                                                      double* __restrict__ out) {
    double acc = 0.0;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
         q += int64_t(gridDim.x) * blockDim.x)
        acc += double(v[q]) * v[q];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_reduce_f64(const double* __restrict__ in, int64_t n,
                                                    double* __restrict__ out) {
    double acc = 0.0;
    for (int64_t q = threadIdx.x; q < n; q += 256) acc += in[q];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) *out = s;
}

// sum over the window of (A - W Ht^T)^2; thread = one column j for 4 consecutive rows.
template <int KP>
__global__ void __launch_bounds__(256) k_residual_dense(const float* __restrict__ A, int64_t lda,
                                                        int64_t rows, int64_t cols,
                                                        const float* __restrict__ W,
                                                        const float* __restrict__ Ht,
                                                        double* __restrict__ out, const int* __restrict__ pred) {
    if (pred && *pred == 0) return;  // device-side predication (error_mode auto)
    __shared__ float Ws[4][KP];
    double acc = 0.0;
    const int64_t rblocks = (rows + 3) / 4, cblocks = (cols + 255) / 256;
    for (int64_t b = blockIdx.x; b < rblocks * cblocks; b += gridDim.x) {
        const int64_t rb = b / cblocks, cb = b % cblocks;
        __syncthreads();
        for (int e = threadIdx.x; e < 4 * KP; e += 256) {
            const int64_t r = rb * 4 + e / KP;
            Ws[e / KP][e % KP] = r < rows ? W[r * KP + e % KP] : 0.f;
        }
        __syncthreads();
        const int64_t j = cb * 256 + threadIdx.x;
        if (j >= cols) continue;
        float h[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) h[q] = Ht[j * KP + q];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t r = rb * 4 + t;
            if (r >= rows) break;
            // (WH)_rj in f64 from the f32 factors (products exact): the residual keeps its
            // relative accuracy even when ||A - WH|| << ||A|| (where the trace form cancels).
            double wh = 0.0;
#pragma unroll
            for (int q = 0; q < KP; ++q) wh = fma(double(Ws[t][q]), double(h[q]), wh);
            const double d = double(A[r * lda + j]) - wh;
            acc += d * d;
        }
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void k_check_finite(const float* __restrict__ x, int64_t n, int* flag) {
    bool bad = false;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x)
        bad |= !isfinite(x[q]);
    if (bad) atomicOr(flag, 1);
}

// [F_g | F_lo_g] per group of gw = min(kp, 64) columns (one group for kp <= 64: [F | F_lo])
__global__ void k_split_cat(const float* __restrict__ F, float* __restrict__ cat, int64_t rows, int kp) {
    const int64_t n = rows * kp;
    const int gw = kp < 64 ? kp : 64;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = q / kp;
        const int j = int(q % kp);
        const float v = F[q];
        float* c = cat + r * 2 * kp + 2 * gw * (j / gw) + j % gw;
        c[0] = v;
        c[gw] = tf32_lo(v);
    }
}

// Model-selection perturbation (src/model_selection.cpp:35-60): every stored entry times an
// i.i.d. factor 1 - delta + 2 delta U(seed, 21, i * n + j) in f64, rounded to f32.
__global__ void k_perturb_dense(const float* __restrict__ in, float* __restrict__ out, int64_t lda,
                                int64_t rows, int64_t cols, int64_t row0, int64_t n, uint64_t key,
                                double delta) {
    const int64_t total = rows * cols;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = q / cols, j = q % cols;
        const double f = 1.0 - delta + 2.0 * delta * rng_u01(key, uint64_t(row0 + i) * uint64_t(n) + uint64_t(j));
        out[i * lda + j] = __double2float_rn(double(in[i * lda + j]) * f);
    }
}

// CSR values (one thread per stored row). transposed: stored row r is column r of A and the
// column indices are slab rows.
__global__ void k_perturb_csr(const float* __restrict__ in, float* __restrict__ out,
                              const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t rows,
                              int64_t row0, int64_t n, uint64_t key, double delta, int transposed) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x)
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
            const uint64_t flat = transposed ? uint64_t(row0 + ci[p]) * uint64_t(n) + uint64_t(r)
                                             : uint64_t(row0 + r) * uint64_t(n) + uint64_t(ci[p]);
            const double f = 1.0 - delta + 2.0 * delta * rng_u01(key, flat);
            out[p] = __double2float_rn(double(in[p]) * f);
        }
}

unsigned grid_for(int64_t work, int per_thread = 1) {
    const int64_t b = (work / per_thread + 255) / 256;
    return unsigned(b < 1 ? 1 : (b > 65535 * 16 ? 65535 * 16 : b));
}

}  // namespace

int sqnorm_grid() { return kRedGrid; }

cudaError_t launch_gen_dense_uniform(float* A, int64_t lda, int64_t rows, int64_t cols, int64_t row0,
                                     int64_t n_global, uint64_t seed, uint64_t stream, cudaStream_t s) {
    k_gen_dense_uniform<<<grid_for(rows * ((cols + 3) / 4), 8), 256, 0, s>>>(
        A, lda, rows, cols, row0, n_global, rng_key(seed, stream));
    return cudaGetLastError();
}

cudaError_t launch_init_factors(float* W, float* Ht, int kp, int64_t k, int64_t rows, int64_t row0,
                                int64_t n, int64_t n_global, int64_t col0, uint64_t seed, cudaStream_t s) {
    k_init_factors<<<grid_for((rows + n) * k, 4), 256, 0, s>>>(
        W, Ht, kp, k, rows, row0, n, n_global, col0, rng_key(seed, kStreamW), rng_key(seed, kStreamH));
    return cudaGetLastError();
}

cudaError_t launch_cast_pad_f64(const double* src, int64_t ld_src, int64_t rows, int64_t cols,
                                float* dst, int64_t ld_dst, cudaStream_t s) {
    k_cast_pad_f64<<<grid_for(rows * cols, 4), 256, 0, s>>>(src, ld_src, rows, cols, dst, ld_dst);
    return cudaGetLastError();
}

cudaError_t launch_strided_cast(CastKind kind, const void* in, int64_t is_r, int64_t is_c, void* out, int64_t os_r,
                                int64_t os_c, int64_t R, int64_t C, cudaStream_t s) {
    if (R <= 0 || C <= 0) return cudaSuccess;
    const bool rows_fast = os_r == 1 && os_c != 1;
    const int g = grid_for(R * C, 4);
    switch (kind) {
        case CastKind::f32_f64:
            k_strided_cast<<<g, 256, 0, s>>>(static_cast<const float*>(in), is_r, is_c, static_cast<double*>(out),
                                             os_r, os_c, R, C, rows_fast);
            break;
        case CastKind::f64_f32:
            k_strided_cast<<<g, 256, 0, s>>>(static_cast<const double*>(in), is_r, is_c, static_cast<float*>(out),
                                             os_r, os_c, R, C, rows_fast);
            break;
        case CastKind::i32_u64:
            k_strided_cast<<<g, 256, 0, s>>>(static_cast<const int32_t*>(in), is_r, is_c,
                                             static_cast<unsigned long long*>(out), os_r, os_c, R, C, rows_fast);
            break;
    }
    return cudaGetLastError();
}

cudaError_t launch_sq_norm_dense(const float* A, int64_t lda, int64_t rows, int64_t cols,
                                 double* out_slots, cudaStream_t s) {
    k_sq_norm_dense<<<kRedGrid, 256, 0, s>>>(A, lda, rows, (cols + 3) / 4, out_slots);
    return cudaGetLastError();
}

cudaError_t launch_sq_norm_vals(const float* v, int64_t nnz, double* out_slots, cudaStream_t s) {
    k_sq_norm_vals<<<kRedGrid, 256, 0, s>>>(v, nnz, out_slots);
    return cudaGetLastError();
}

cudaError_t launch_reduce_f64(const double* slots, int64_t n, double* out, cudaStream_t s) {
    k_reduce_f64<<<1, 256, 0, s>>>(slots, n, out);
    return cudaGetLastError();
}

cudaError_t launch_residual_dense(int kp, const float* A, int64_t lda, int64_t rows, int64_t cols,
                                  const float* W, const float* Ht, double* out_slots, cudaStream_t s,
                                  const int* pred) {
    if (kp > 64) return launch_residual_dense_wide(kp, A, lda, rows, cols, W, Ht, out_slots, kRedGrid, s, pred);
    switch (kp) {
        case 8: k_residual_dense<8><<<kRedGrid, 256, 0, s>>>(A, lda, rows, cols, W, Ht, out_slots, pred); break;
        case 16: k_residual_dense<16><<<kRedGrid, 256, 0, s>>>(A, lda, rows, cols, W, Ht, out_slots, pred); break;
        case 32: k_residual_dense<32><<<kRedGrid, 256, 0, s>>>(A, lda, rows, cols, W, Ht, out_slots, pred); break;
        case 64: k_residual_dense<64><<<kRedGrid, 256, 0, s>>>(A, lda, rows, cols, W, Ht, out_slots, pred); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t s) {
    k_check_finite<<<grid_for(n, 8), 256, 0, s>>>(x, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_perturb_dense(const float* in, float* out, int64_t lda, int64_t rows, int64_t cols,
                                 int64_t row0, int64_t n, uint64_t seed, double delta, cudaStream_t s) {
    k_perturb_dense<<<grid_for(rows * cols, 8), 256, 0, s>>>(in, out, lda, rows, cols, row0, n,
                                                             rng_key(seed, kStreamPerturb), delta);
    return cudaGetLastError();
}

cudaError_t launch_perturb_csr(const float* in, float* out, const int64_t* rp, const int32_t* ci, int64_t rows,
                               int64_t row0, int64_t n, uint64_t seed, double delta, bool transposed,
                               cudaStream_t s) {
    k_perturb_csr<<<grid_for(rows, 1), 256, 0, s>>>(in, out, rp, ci, rows, row0, n, rng_key(seed, kStreamPerturb),
                                                    delta, transposed ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_split_cat(const float* F, float* cat, int64_t rows, int kp, cudaStream_t s) {
    k_split_cat<<<grid_for(rows * kp, 8), 256, 0, s>>>(F, cat, rows, kp);
    return cudaGetLastError();
}

}  // namespace ooc
