// A reference-style caller of the distributed path, compiled unchanged against the B200 host
// core: it uses only the reference header names and the calls a reference user makes —
// make_plan (include/oocnmf/partition.hpp:45), run_distributed_threads
// (include/oocnmf/nmf_distributed.hpp:40), spawn_group + CommHandle::all_reduce_sum / barrier /
// stats (include/oocnmf/comm.hpp:48-82) and nmf_distributed over a threads-backend group
// (src/nmf_distributed.cpp:291-319). argv: n_workers m n k. Prints JSON lines that
// tests/test_gpu_distributed.py compares with the CPU oracle.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "oocnmf/comm.hpp"
#include "oocnmf/matrix.hpp"
#include "oocnmf/nmf.hpp"
#include "oocnmf/nmf_distributed.hpp"
#include "oocnmf/partition.hpp"
#include "oocnmf/rng.hpp"

using namespace oocnmf;

int main(int argc, char** argv) {
    const int workers = argc > 1 ? std::atoi(argv[1]) : 1;
    const index_t m = argc > 2 ? std::atoi(argv[2]) : 700, n = argc > 3 ? std::atoi(argv[3]) : 500;
    const index_t k = argc > 4 ? std::atoi(argv[4]) : 8;
    DenseMatrix a(m, n);
    CounterRng rng(42, 99);
    for (index_t i = 0; i < m; ++i)
        for (index_t j = 0; j < n; ++j) a.at(i, j) = double(float(rng.uniform(i * n + j)));
    NmfConfig cfg;
    cfg.k = k;
    cfg.max_iters = 30;
    cfg.error_check_interval = 10;
    cfg.eta = 0;
    PartitionPlan plan = make_plan(m, n, k, workers, 1, Strategy::rnmf);

    // 1. the convenience driver: every rank on its own thread and GPU
    std::vector<CollectiveStats> stats;
    std::vector<NmfResult> res = run_distributed_threads(ASource::memory(MatrixRef(a)), cfg, plan, {}, &stats);
    for (auto& [it, err] : res[0].error_trace) std::printf("{\"iter\": %zu, \"err\": %.17g}\n", it, err);
    double wn = 0, hn = 0;
    for (index_t i = 0; i < res[0].w.size(); ++i) wn += res[0].w.data()[i] * res[0].w.data()[i];
    for (index_t i = 0; i < res[0].h.size(); ++i) hn += res[0].h.data()[i] * res[0].h.data()[i];
    bool same = true;  // the result is identical on every rank (nmf_distributed.hpp:28)
    for (auto& r : res) same = same && r.w == res[0].w && r.h == res[0].h && r.error_trace == res[0].error_trace;
    std::printf("{\"w_fro\": %.17g, \"h_fro\": %.17g, \"ranks\": %zu, \"identical\": %s}\n", std::sqrt(wn),
                std::sqrt(hn), res.size(), same ? "true" : "false");
    const auto& s0 = stats[0];
    std::printf("{\"h_update_calls\": %zu, \"h_update_bytes\": %zu, \"gather_calls\": %zu, \"error_check_calls\": %zu, "
                "\"total_calls\": %zu}\n",
                s0[PhaseTag::h_update].calls, s0[PhaseTag::h_update].bytes, s0[PhaseTag::gather].calls,
                s0[PhaseTag::error_check].calls, s0.total_calls());

    // 2. the group itself: all_reduce_sum / barrier / stats from worker threads
    CommGroup group = spawn_group(workers, workers == 1 ? Backend::loopback : Backend::threads);
    std::vector<double> sums(workers);
    std::vector<std::thread> th;
    for (int r = 0; r < workers; ++r)
        th.emplace_back([&, r] {
            DenseMatrix buf(2, 3);
            for (index_t i = 0; i < 6; ++i) buf.data()[i] = double(r + 1) * double(i + 1);
            group.handles[r].all_reduce_sum(buf, PhaseTag::generic);
            group.handles[r].barrier();
            sums[r] = buf.at(1, 2);  // 6 * (1 + 2 + ... + workers)
        });
    for (auto& t : th) t.join();
    std::printf("{\"allreduce_last\": %.17g, \"generic_calls\": %zu, \"barrier_calls\": %zu}\n", sums[workers - 1],
                group.handles[0].stats()[PhaseTag::generic].calls, group.handles[0].stats()[PhaseTag::barrier].calls);

    // 3. errors map to the reference's exception types
    try {
        PartitionPlan bad = plan;
        bad.n_workers = workers + 1;
        nmf_distributed(ASource::memory(MatrixRef(a)), cfg, bad, group.handles[0]);
    } catch (const ShapeError&) {
        std::printf("{\"shape_error\": true}\n");
    }
    return 0;
}
