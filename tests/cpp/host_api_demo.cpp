// A reference-style caller, compiled unchanged against the B200 host core: it includes the
// reference header names and calls oocnmf::nmf_serial exactly as the reference's CLI does
// (tools/oocnmf_cli.cpp:201) — the drop-in check for the C++ boundary. Prints one JSON line
// per trace entry and the factor norms; tests/test_gpu_parity.py compares them with the oracle.
#include <cmath>
#include <cstdio>

#include "oocnmf/matrix.hpp"
#include "oocnmf/nmf.hpp"
#include "oocnmf/rng.hpp"

int main(int argc, char** argv) {
    using namespace oocnmf;
    const index_t m = argc > 1 ? std::atoi(argv[1]) : 300, n = argc > 2 ? std::atoi(argv[2]) : 200;
    const index_t k = argc > 3 ? std::atoi(argv[3]) : 8;
    DenseMatrix a(m, n);
    CounterRng rng(42, 99);
    for (index_t i = 0; i < m; ++i)
        for (index_t j = 0; j < n; ++j) a.at(i, j) = double(float(rng.uniform(i * n + j)));
    NmfConfig cfg;
    cfg.k = k;
    cfg.max_iters = 30;
    cfg.error_check_interval = 10;
    cfg.eta = 0;
    try {
        NmfResult r = nmf_serial(MatrixRef(a), cfg);
        for (auto& [it, err] : r.error_trace) std::printf("{\"iter\": %zu, \"err\": %.17g}\n", it, err);
        double wn = 0, hn = 0;
        for (index_t i = 0; i < r.w.size(); ++i) wn += r.w.data()[i] * r.w.data()[i];
        for (index_t i = 0; i < r.h.size(); ++i) hn += r.h.data()[i] * r.h.data()[i];
        std::printf("{\"w_fro\": %.17g, \"h_fro\": %.17g, \"iterations_run\": %zu}\n", std::sqrt(wn), std::sqrt(hn),
                    r.iterations_run);
    } catch (const DeviceError& e) {
        std::printf("{\"device_error\": \"%s\"}\n", e.what());
        return 3;
    }
    // Error mapping: an invalid config throws ShapeError like the reference.
    try {
        NmfConfig bad = cfg;
        bad.max_iters = 0;
        nmf_serial(MatrixRef(a), bad);
    } catch (const ShapeError&) {
        std::printf("{\"shape_error\": true}\n");
    }
    return 0;
}
