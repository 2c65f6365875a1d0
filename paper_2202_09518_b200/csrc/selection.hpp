// Model selection (NMFk) host core — the ensemble clustering and scoring that consume the MU
// path (reference: include/oocnmf/model_selection.hpp, src/model_selection.cpp). Private to
// liboocnmf_b200.so: the C-ABI (oocnmf_select_k, oocnmf_cluster_silhouette,
// oocnmf_pearson_correlation) and the C++ host core (host_api.cpp) are built on it.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace ooc_sel {

// One W factor of an ensemble: m x k, row-major.
struct Factor {
    const double* w;
};

struct Clusters {
    uint64_t m = 0, k = 0;
    // cluster c: its members as (run, column) and their unit-normalized columns (m each)
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> member_ids;
    std::vector<std::vector<std::vector<double>>> points;
    std::vector<double> medians;  // m x k row-major
    uint64_t dropped_zero_columns = 0;
};

struct Silhouette {
    double min_sil = 0.0, mean_sil = 0.0;
    std::vector<double> per_cluster;
};

// cluster_columns (model_selection.cpp:163-231): anchors = run 0's columns, later runs matched
// one-to-one by maximal total cosine similarity (exact bitmask DP for k <= 16, greedy above),
// elementwise medians of each cluster. Throws std::invalid_argument on bad shapes.
Clusters cluster_columns(const std::vector<Factor>& runs, uint64_t m, uint64_t k);
// silhouette (model_selection.cpp:233-281), cosine distance; k = 1 scores 1.0 by convention.
// Throws std::invalid_argument("silhouette: empty cluster") like the reference.
Silhouette silhouette(const Clusters& c);
// pearson_correlation_matrix (model_selection.cpp:283-314); throws std::domain_error on a
// zero-variance column.
std::vector<double> pearson(const double* w_true, uint64_t m, uint64_t k1, const double* w_est, uint64_t k2);

// The selection rule of select_k (model_selection.cpp:372-404) over per-k records.
struct KScore {
    uint64_t k = 0;
    bool valid = false;
    uint64_t runs_used = 0;
    double min_sil = 0.0, mean_sil = 0.0, mean_err = 0.0;
};
// Returns chosen k (or -1) and the rationale text.
std::pair<int64_t, std::string> choose_k(const std::vector<KScore>& recs, double sil_threshold);

}  // namespace ooc_sel
