// A reference-style caller, compiled unchanged against the B200 host core: it includes the
// reference header names and calls oocnmf::nmf_serial exactly as the reference's CLI does
// (tools/oocnmf_cli.cpp:201) — the drop-in check for the C++ boundary. Prints one JSON line
// per trace entry and the factor norms; tests/test_gpu_parity.py compares them with the oracle.
#include <cmath>
#include <cstdio>

#include "oocnmf/matrix.hpp"
#include "oocnmf/model_selection.hpp"
#include "oocnmf/nmf.hpp"
#include "oocnmf/partition.hpp"
#include "oocnmf/rng.hpp"

#include <string>

static std::string jesc(const std::string& s) {
    std::string o;
    for (char ch : s) {
        if (ch == '\n') o += "\\n";
        else if (ch == '"') o += "\\\"";
        else o += ch;
    }
    return o;
}

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
    // Model selection driven as the reference CLI drives it (tools/oocnmf_cli.cpp:298-318) on an
    // exactly rank-2 input: the largest k with a stable ensemble is 2.
    {
        DenseMatrix lr(60, 40);
        CounterRng ra(7, 1), rb(7, 2);
        for (index_t i = 0; i < 60; ++i)
            for (index_t j = 0; j < 40; ++j) {
                double v = 0;
                for (index_t t = 0; t < 2; ++t) v += ra.uniform(i * 2 + t) * rb.uniform(t * 40 + j);
                lr.at(i, j) = double(float(v));
            }
        SelectionConfig sc;
        sc.k_min = 1;
        sc.k_max = 3;
        sc.n_perturbations = 4;
        sc.nmf.max_iters = 200;
        sc.nmf.eta = 1e-6;
        SelectionReport rep = select_k(MatrixRef(lr), sc);
        std::printf("{\"select_chosen\": %lld, \"select_records\": %zu}\n",
                    rep.chosen_k ? (long long)*rep.chosen_k : -1LL, rep.records.size());
    }
    // The plan / memory-report JSON of the reference (src/partition.cpp:89,199)
    {
        const std::string pj = make_plan(1000, 900, 8, 4, 3, Strategy::rnmf).to_json();
        MemoryReport mr;
        mr.a_slab_bytes = 1, mr.store_peak_bytes = 2, mr.factor_bytes = 3, mr.intermediate_bytes = 4;
        mr.peak_bytes = 5, mr.min_n_b = 6, mr.feasible = true;
        std::printf("{\"plan_json\": \"%s\", \"report_json\": \"%s\"}\n", jesc(pj).c_str(), jesc(mr.to_json()).c_str());
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
