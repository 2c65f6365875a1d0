// Synthetic inputs of the reference (include/oocnmf/synth.hpp, src/synth.cpp), for the oocnmf
// CLI's `gen` and `bench` and for user code that builds test problems.
//   gen_lowrank       host, OpenMP over rows; compiled with -ffp-contract=off so W0·H0 is summed
//                     in the reference's order without fused multiply-adds (bit-identical).
//   gen_sparse_random the O(m n) presence draws run on GPU 0 (k_gen_csr_*, the same generator the
//                     solver uses for config 3); the f64 values of the present entries are then
//                     drawn here from the value stream (O(nnz)), so the result is bit-identical
//                     to the reference's f64 CSR, not only to its f32 rounding.
#include <cmath>
#include <vector>

#include "oocnmf_b200/oocnmf.hpp"

namespace oocnmf {
namespace {
constexpr std::uint64_t kStreamW0 = 11, kStreamH0 = 12, kStreamNoise = 13, kStreamSparse = 14;

void check(int st) {
    if (st == 0) return;
    const std::string msg = oocnmf_last_error();
    switch (st) {
        case OOCNMF_ERR_SHAPE: throw ShapeError(msg);
        case OOCNMF_ERR_DATA: throw DataError(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace

LowrankData gen_lowrank(const LowrankSpec& spec) {
    if (spec.m == 0 || spec.n == 0 || spec.k_true == 0)
        throw ShapeError("gen_lowrank: m, n and k_true must be positive");
    if (spec.k_true > spec.m || spec.k_true > spec.n)
        throw ShapeError("gen_lowrank: k_true must not exceed min(m, n)");
    if (spec.noise < 0.0 || spec.noise >= 1.0) throw ShapeError("gen_lowrank: noise must lie in [0, 1)");
    const index_t m = spec.m, n = spec.n, kt = spec.k_true;
    LowrankData out{DenseMatrix(m, n), DenseMatrix(m, kt), DenseMatrix(kt, n)};

    const CounterRng wrng(spec.seed, kStreamW0), hrng(spec.seed, kStreamH0), nrng(spec.seed, kStreamNoise);
    const double width = double(m) / (4.0 * double(kt));
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(m); ++i)
        for (index_t c = 0; c < kt; ++c) {
            const double mu = (double(c) + 0.5) * double(m) / double(kt);
            const double d = (double(i) - mu) / width;
            out.w0.at(index_t(i), c) = std::exp(-0.5 * d * d) + 0.01 * wrng.uniform(index_t(i) * kt + c);
        }
#pragma omp parallel for schedule(static)
    for (std::int64_t r = 0; r < std::int64_t(kt); ++r)
        for (index_t j = 0; j < n; ++j) out.h0.at(index_t(r), j) = hrng.uniform(index_t(r) * n + j);

    // a(i, j) = sum_q w0(i, q) h0(q, j), q ascending from 0.0 (src/kernels.cpp:33-44)
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(m); ++i) {
        double* row = out.a.data() + index_t(i) * n;
        for (index_t q = 0; q < kt; ++q) {
            const double wv = out.w0.at(index_t(i), q);
            const double* h = out.h0.data() + q * n;
            for (index_t j = 0; j < n; ++j) row[j] += wv * h[j];
        }
        if (spec.noise > 0.0)
            for (index_t j = 0; j < n; ++j)
                row[j] *= 1.0 + spec.noise * (2.0 * nrng.uniform(index_t(i) * n + j) - 1.0);
    }
    return out;
}

CsrMatrix gen_sparse_random(const SparseSpec& spec) {
    if (spec.m == 0 || spec.n == 0) throw ShapeError("gen_sparse_random: m and n must be positive");
    if (spec.density < 0.0 || spec.density > 1.0) throw ShapeError("gen_sparse_random: density must lie in [0, 1]");
    oocnmf_ctx* c = nullptr;
    check(oocnmf_ctx_create(0, &c));
    std::vector<index_t> rp(spec.m + 1), ci;
    std::vector<double> v;
    try {
        check(oocnmf_set_problem(c, spec.m, spec.n, 1, 0, spec.m));
        check(oocnmf_generate_csr_uniform(c, spec.density, spec.seed));
        std::uint64_t nnz = 0;
        check(oocnmf_csr_nnz(c, &nnz));
        ci.resize(nnz), v.resize(nnz);
        check(oocnmf_download_csr(c, reinterpret_cast<std::uint64_t*>(rp.data()),
                                  reinterpret_cast<std::uint64_t*>(ci.data()), v.data()));
    } catch (...) {
        oocnmf_ctx_destroy(c);
        throw;
    }
    oocnmf_ctx_destroy(c);
    const CounterRng vals(spec.seed, kStreamSparse + 1);
#pragma omp parallel for schedule(dynamic, 1024)
    for (std::int64_t i = 0; i < std::int64_t(spec.m); ++i)
        for (index_t p = rp[index_t(i)]; p < rp[index_t(i) + 1]; ++p) v[p] = vals.uniform(index_t(i) * spec.n + ci[p]);
    return CsrMatrix(spec.m, spec.n, std::move(rp), std::move(ci), std::move(v));
}

}  // namespace oocnmf
