// Model selection (NMFk) on the B200 MU path: select_k drives P perturbed GPU factorizations
// per candidate k (perturbation generated in HBM from the counter RNG, stream 21), then scores
// the W ensemble on the host exactly as the reference does (src/model_selection.cpp):
// unit-normalized columns, one-to-one matching to run 0's columns (bitmask DP up to k = 16,
// greedy above), elementwise medians, cosine silhouette, and the "largest k with min
// silhouette >= threshold and error <= 1.5 x the best k's error" rule.
//
// Every cosine is the same left-to-right f64 dot product the reference evaluates, computed
// once per pair (the silhouette reads them from a cached Gram of all ensemble columns, filled
// in parallel), so the host scores are bit-identical to the reference's for identical W's.
#include "selection.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "oocnmf_b200.h"

namespace ooc {
void set_last_error(const std::string& msg);
}

namespace ooc_sel {
namespace {

constexpr double kZeroColumnNorm = 1e-300;   // model_selection.cpp:18
constexpr uint64_t kExactAssignmentMaxK = 16;  // model_selection.cpp:19
constexpr uint64_t kNpos = ~uint64_t(0);

double dot(const std::vector<double>& x, const std::vector<double>& y) {
    double d = 0.0;
    for (size_t i = 0; i < x.size(); ++i) d += x[i] * y[i];
    return d;
}

// Column c of W (m x k row-major), unit-normalized; alive = false for a ~zero column.
std::vector<std::vector<double>> unit_columns(const double* w, uint64_t m, uint64_t k, std::vector<bool>& alive) {
    std::vector<std::vector<double>> cols(k, std::vector<double>(m));
    alive.assign(k, true);
    for (uint64_t c = 0; c < k; ++c) {
        double sq = 0.0;
        for (uint64_t i = 0; i < m; ++i) {
            const double v = w[i * k + c];
            cols[c][i] = v;
            sq += v * v;
        }
        const double norm = std::sqrt(sq);
        if (norm < kZeroColumnNorm) {
            alive[c] = false;
            continue;
        }
        for (double& v : cols[c]) v /= norm;
    }
    return cols;
}

// One-to-one assignment of `cols` to `anchors` maximizing the total cosine similarity
// (model_selection.cpp:94-159 semantics: DP over anchor subsets taking columns in order,
// strict improvements only; greedy global-best pairs above kExactAssignmentMaxK anchors).
std::vector<uint64_t> assign_columns(const std::vector<std::vector<double>>& anchors,
                                     const std::vector<const std::vector<double>*>& cols) {
    const uint64_t na = anchors.size(), nc = cols.size();
    std::vector<double> sim(nc * na);
    for (uint64_t c = 0; c < nc; ++c)
        for (uint64_t a = 0; a < na; ++a) sim[c * na + a] = dot(*cols[c], anchors[a]);
    std::vector<uint64_t> out(nc, kNpos);
    if (na <= kExactAssignmentMaxK) {
        const uint64_t nmask = uint64_t(1) << na;
        const double neg = -std::numeric_limits<double>::infinity();
        std::vector<double> best(nmask, neg);
        std::vector<int> last(nmask, -1);
        best[0] = 0.0;
        for (uint64_t mask = 0; mask < nmask; ++mask) {
            if (best[mask] == neg) continue;
            const uint64_t c = uint64_t(std::popcount(mask));
            if (c >= nc) continue;
            for (uint64_t a = 0; a < na; ++a) {
                const uint64_t bit = uint64_t(1) << a;
                if (mask & bit) continue;
                const double v = best[mask] + sim[c * na + a];
                if (v > best[mask | bit]) best[mask | bit] = v, last[mask | bit] = int(a);
            }
        }
        uint64_t top = 0;
        double top_v = neg;
        for (uint64_t mask = 0; mask < nmask; ++mask)
            if (uint64_t(std::popcount(mask)) == nc && best[mask] > top_v) top_v = best[mask], top = mask;
        for (uint64_t mask = top; mask != 0;) {
            const uint64_t a = uint64_t(last[mask]);
            mask &= ~(uint64_t(1) << a);
            out[uint64_t(std::popcount(mask))] = a;
        }
    } else {
        std::vector<bool> cu(nc, false), au(na, false);
        for (uint64_t step = 0; step < std::min(na, nc); ++step) {
            double bv = -std::numeric_limits<double>::infinity();
            uint64_t bc = kNpos, ba = kNpos;
            for (uint64_t c = 0; c < nc; ++c) {
                if (cu[c]) continue;
                for (uint64_t a = 0; a < na; ++a)
                    if (!au[a] && sim[c * na + a] > bv) bv = sim[c * na + a], bc = c, ba = a;
            }
            cu[bc] = au[ba] = true;
            out[bc] = ba;
        }
    }
    return out;
}

}  // namespace

Clusters cluster_columns(const std::vector<Factor>& runs, uint64_t m, uint64_t k) {
    if (runs.size() < 2) throw std::invalid_argument("cluster_columns: need at least 2 runs");
    if (m < 1 || k < 1) throw std::invalid_argument("cluster_columns: all runs must be m x k");
    Clusters out;
    out.m = m, out.k = k;
    out.member_ids.resize(k);
    out.points.resize(k);
    std::vector<bool> alive0;
    auto cols0 = unit_columns(runs[0].w, m, k, alive0);
    std::vector<std::vector<double>> anchors;
    std::vector<uint64_t> anchor_cluster;
    for (uint64_t c = 0; c < k; ++c) {
        if (!alive0[c]) {
            ++out.dropped_zero_columns;
            continue;
        }
        anchors.push_back(cols0[c]);
        anchor_cluster.push_back(c);
        out.member_ids[c].push_back({0, c});
        out.points[c].push_back(std::move(cols0[c]));
    }
    for (uint64_t r = 1; r < runs.size(); ++r) {
        std::vector<bool> alive;
        auto cols = unit_columns(runs[r].w, m, k, alive);
        std::vector<const std::vector<double>*> live;
        std::vector<uint64_t> live_id;
        for (uint64_t c = 0; c < k; ++c) {
            if (!alive[c]) {
                ++out.dropped_zero_columns;
                continue;
            }
            live.push_back(&cols[c]);
            live_id.push_back(c);
        }
        const auto assign = assign_columns(anchors, live);
        for (uint64_t i = 0; i < live.size(); ++i) {
            if (assign[i] == kNpos) continue;
            const uint64_t cl = anchor_cluster[assign[i]];
            out.member_ids[cl].push_back({r, live_id[i]});
            out.points[cl].push_back(*live[i]);
        }
    }
    // elementwise medians (average of the two middle values for an even count)
    out.medians.assign(m * k, 0.0);
    std::vector<double> v;
    for (uint64_t c = 0; c < k; ++c) {
        const auto& mem = out.points[c];
        if (mem.empty()) continue;
        for (uint64_t i = 0; i < m; ++i) {
            v.clear();
            for (const auto& col : mem) v.push_back(col[i]);
            std::sort(v.begin(), v.end());
            const size_t h = v.size() / 2;
            out.medians[i * k + c] = v.size() % 2 ? v[h] : 0.5 * (v[h - 1] + v[h]);
        }
    }
    return out;
}

Silhouette silhouette(const Clusters& cl) {
    const uint64_t k = cl.points.size();
    Silhouette out;
    out.per_cluster.assign(k, 0.0);
    if (k == 1) {
        out.min_sil = out.mean_sil = 1.0;
        out.per_cluster[0] = 1.0;
        return out;
    }
    for (uint64_t c = 0; c < k; ++c)
        if (cl.points[c].empty()) throw std::invalid_argument("silhouette: empty cluster");
    // all ensemble columns, cluster-major; cosine Gram computed once per pair
    std::vector<const std::vector<double>*> pts;
    std::vector<uint64_t> first(k + 1, 0);
    for (uint64_t c = 0; c < k; ++c) {
        first[c] = pts.size();
        for (const auto& p : cl.points[c]) pts.push_back(&p);
    }
    first[k] = pts.size();
    const int64_t np = int64_t(pts.size());
    std::vector<double> g(size_t(np) * np, 0.0);
#pragma omp parallel for schedule(dynamic)
    for (int64_t a = 0; a < np; ++a)
        for (int64_t b = a + 1; b < np; ++b) {
            const double d = dot(*pts[a], *pts[b]);
            g[a * np + b] = g[b * np + a] = d;
        }
    auto dist = [&](uint64_t a, uint64_t b) { return 1.0 - g[a * np + b]; };
    double total = 0.0;
    uint64_t count = 0;
    out.min_sil = 1.0;
    for (uint64_t c = 0; c < k; ++c) {
        const uint64_t n_c = first[c + 1] - first[c];
        double csum = 0.0;
        for (uint64_t s = first[c]; s < first[c + 1]; ++s) {
            double sil = 0.0;
            if (n_c > 1) {
                double a = 0.0;
                for (uint64_t t = first[c]; t < first[c + 1]; ++t)
                    if (t != s) a += dist(s, t);
                a /= double(n_c - 1);
                double b = std::numeric_limits<double>::infinity();
                for (uint64_t o = 0; o < k; ++o) {
                    if (o == c || first[o + 1] == first[o]) continue;
                    double d = 0.0;
                    for (uint64_t y = first[o]; y < first[o + 1]; ++y) d += dist(s, y);
                    b = std::min(b, d / double(first[o + 1] - first[o]));
                }
                const double den = std::max(a, b);
                sil = den > 0.0 ? (b - a) / den : 0.0;
            }
            csum += sil;
            total += sil;
            ++count;
            out.min_sil = std::min(out.min_sil, sil);
        }
        out.per_cluster[c] = csum / double(n_c);
    }
    out.mean_sil = count > 0 ? total / double(count) : 0.0;
    return out;
}

std::vector<double> pearson(const double* wt, uint64_t m, uint64_t k1, const double* we, uint64_t k2) {
    auto standardize = [m](const double* w, uint64_t k) {
        std::vector<std::vector<double>> cols(k, std::vector<double>(m));
        for (uint64_t c = 0; c < k; ++c) {
            double mean = 0.0;
            for (uint64_t i = 0; i < m; ++i) mean += w[i * k + c];
            mean /= double(m);
            double sq = 0.0;
            for (uint64_t i = 0; i < m; ++i) {
                cols[c][i] = w[i * k + c] - mean;
                sq += cols[c][i] * cols[c][i];
            }
            if (sq <= 0.0) throw std::domain_error("pearson_correlation_matrix: zero-variance column");
            const double inv = 1.0 / std::sqrt(sq);
            for (double& v : cols[c]) v *= inv;
        }
        return cols;
    };
    const auto a = standardize(wt, k1), b = standardize(we, k2);
    std::vector<double> corr(k1 * k2);
    for (uint64_t i = 0; i < k1; ++i)
        for (uint64_t j = 0; j < k2; ++j) corr[i * k2 + j] = dot(a[i], b[j]);
    return corr;
}

std::pair<int64_t, std::string> choose_k(const std::vector<KScore>& recs, double thr) {
    const KScore* best = nullptr;
    for (const auto& r : recs) {
        if (!r.valid) continue;
        if (!best || r.min_sil > best->min_sil || (r.min_sil == best->min_sil && r.mean_err < best->mean_err))
            best = &r;
    }
    if (!best) return {-1, "no candidate k produced at least two successful runs"};
    const double cap = 1.5 * best->mean_err;
    int64_t chosen = -1;
    for (const auto& r : recs)
        if (r.valid && r.min_sil >= thr && r.mean_err <= cap) chosen = int64_t(r.k);  // ascending: keep largest
    // the reference streams doubles with the default ostream format (%g, 6 digits)
    char buf[256];
    if (chosen >= 0)
        std::snprintf(buf, sizeof buf,
                      "k=%lld is the largest candidate with min silhouette >= %g and mean relative error <= %g",
                      (long long)chosen, thr, cap);
    else
        std::snprintf(buf, sizeof buf, "no candidate met min silhouette >= %g with mean relative error <= %g", thr,
                      cap);
    return {chosen, buf};
}

}  // namespace ooc_sel

// =============================================================================== C-ABI
namespace {

uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// derive_seed (include/oocnmf/rng.hpp:43-45)
uint64_t derive_seed(uint64_t seed, uint64_t a, uint64_t b) { return mix(seed ^ mix(a ^ mix(b))); }

struct Status {
    int code;
};

template <class F>
int host_guard(F&& f) {
    try {
        f();
        return OOCNMF_OK;
    } catch (const Status& s) {
        return s.code;  // message already set by the failing C-ABI call
    } catch (const std::invalid_argument& e) {
        ooc::set_last_error(e.what());
        return OOCNMF_ERR_SHAPE;
    } catch (const std::domain_error& e) {
        ooc::set_last_error(e.what());
        return OOCNMF_ERR_DATA;
    } catch (const std::bad_alloc&) {
        ooc::set_last_error("host allocation failed");
        return OOCNMF_ERR_DEVICE;
    } catch (const std::exception& e) {
        ooc::set_last_error(e.what());
        return OOCNMF_ERR_DEVICE;
    }
}
void chk(int st) {
    if (st != OOCNMF_OK) throw Status{st};
}

}  // namespace

extern "C" {

int oocnmf_cluster_silhouette(const double* runs, uint64_t nruns, uint64_t m, uint64_t k, double* medians,
                              double* per_cluster, double* min_sil, double* mean_sil, uint64_t* dropped,
                              int64_t* member_cluster) {
    return host_guard([&] {
        std::vector<ooc_sel::Factor> f;
        for (uint64_t r = 0; r < nruns; ++r) f.push_back({runs + r * m * k});
        const auto cl = ooc_sel::cluster_columns(f, m, k);
        if (member_cluster) {
            std::fill(member_cluster, member_cluster + nruns * k, int64_t(-1));
            for (uint64_t c = 0; c < k; ++c)
                for (const auto& [r, col] : cl.member_ids[c]) member_cluster[r * k + col] = int64_t(c);
        }
        if (medians) std::copy(cl.medians.begin(), cl.medians.end(), medians);
        if (dropped) *dropped = cl.dropped_zero_columns;
        const auto s = ooc_sel::silhouette(cl);
        if (per_cluster) std::copy(s.per_cluster.begin(), s.per_cluster.end(), per_cluster);
        if (min_sil) *min_sil = s.min_sil;
        if (mean_sil) *mean_sil = s.mean_sil;
    });
}

int oocnmf_pearson_correlation(const double* w_true, uint64_t m, uint64_t k1, const double* w_est, uint64_t k2,
                               double* corr) {
    return host_guard([&] {
        const auto c = ooc_sel::pearson(w_true, m, k1, w_est, k2);
        std::copy(c.begin(), c.end(), corr);
    });
}

int oocnmf_select_k(oocnmf_ctx* ctx, const oocnmf_selection_config* cfg, oocnmf_k_record* records, uint64_t cap,
                    double* medians, int64_t* chosen_k, char* rationale, uint64_t rationale_cap) {
    int rank = 0, nranks = 1;
    bool local_set = false, perturbed = false;
    const int st = host_guard([&] {
        if (!cfg) throw std::invalid_argument("select_k: null config");
        uint64_t m, n, k0, row0, rows;
        chk(oocnmf_problem_dims(ctx, &m, &n, &k0, &row0, &rows));
        // SelectionConfig::validate (model_selection.cpp:22-33)
        if (cfg->k_min < 1 || cfg->k_max < cfg->k_min)
            throw std::invalid_argument("SelectionConfig: need 1 <= k_min <= k_max");
        if (cfg->k_max >= std::min(m, n)) throw std::invalid_argument("SelectionConfig: k_max must be below min(m, n)");
        if (cfg->n_perturbations < 2) throw std::invalid_argument("SelectionConfig: need at least 2 perturbations");
        if (!(cfg->delta > 0.0 && cfg->delta < 1.0))
            throw std::invalid_argument("SelectionConfig: delta must lie in (0, 1)");
        if (!(cfg->sil_threshold >= -1.0 && cfg->sil_threshold <= 1.0))
            throw std::invalid_argument("SelectionConfig: sil_threshold must lie in [-1, 1]");
        if (row0 != 0 || rows != m)
            throw std::invalid_argument("select_k: the context must hold the full A (row0 = 0, rows = m)");
        const uint64_t nk = cfg->k_max - cfg->k_min + 1;
        if (!records || cap < nk) throw std::invalid_argument("select_k: records capacity below k_max - k_min + 1");
        chk(oocnmf_ctx_rank(ctx, &rank, &nranks));
        if (nranks > 1) chk(oocnmf_set_local(ctx, 1)), local_set = true;

        const uint64_t P = cfg->n_perturbations;
        const uint64_t interval = std::max<uint64_t>(cfg->nmf.error_check_interval, 1);
        const uint64_t tcap = cfg->nmf.max_iters / interval + 2;
        std::vector<uint64_t> ti(tcap);
        std::vector<double> te(tcap), hbuf;
        std::vector<ooc_sel::KScore> scores;
        double* med_out = medians;
        for (uint64_t k = cfg->k_min; k <= cfg->k_max; ++k) {
            chk(oocnmf_set_rank(ctx, k));
            // per-perturbation slots, filled by the owning rank, summed over ranks
            std::vector<double> wall(P * m * k, 0.0), err(P, 0.0), ok(P, 0.0), iters(P, 0.0);
            hbuf.assign(k * n, 0.0);
            for (uint64_t p = uint64_t(rank); p < P; p += uint64_t(nranks)) {
                for (uint64_t attempt = 0; attempt < 2 && ok[p] == 0.0; ++attempt) {
                    const uint64_t pert_seed = derive_seed(cfg->seed, k, 2 * p + attempt * 1000003);
                    const uint64_t run_seed = derive_seed(cfg->seed, k, 2 * p + 1 + attempt * 1000003);
                    chk(oocnmf_perturb(ctx, cfg->delta, pert_seed));
                    perturbed = true;
                    oocnmf_config rc = cfg->nmf;
                    rc.k = k;
                    rc.seed = run_seed;
                    oocnmf_info info{};
                    const int s = oocnmf_solve(ctx, &rc, ti.data(), te.data(), tcap, &info);
                    if (s == OOCNMF_ERR_DATA || s == OOCNMF_ERR_SHAPE) continue;  // failed run: excluded / retried
                    chk(s);
                    chk(oocnmf_get_factors_f64(ctx, wall.data() + p * m * k, hbuf.data()));
                    err[p] = te[std::min<uint64_t>(info.n_trace, tcap) - 1];
                    ok[p] = 1.0;
                    iters[p] = double(info.iterations_run);
                }
            }
            if (nranks > 1) {
                chk(oocnmf_allreduce_sum_f64(ctx, wall.data(), wall.size()));
                chk(oocnmf_allreduce_sum_f64(ctx, err.data(), P));
                chk(oocnmf_allreduce_sum_f64(ctx, ok.data(), P));
                chk(oocnmf_allreduce_sum_f64(ctx, iters.data(), P));
            }
            std::vector<ooc_sel::Factor> ws;
            double err_sum = 0.0;
            for (uint64_t p = 0; p < P; ++p)
                if (ok[p] != 0.0) ws.push_back({wall.data() + p * m * k}), err_sum += err[p];
            ooc_sel::KScore sc;
            sc.k = k;
            sc.runs_used = ws.size();
            oocnmf_k_record& rec = records[k - cfg->k_min];
            rec = oocnmf_k_record{};
            rec.k = k;
            rec.runs_used = ws.size();
            for (uint64_t p = 0; p < P; ++p) rec.iterations += uint64_t(iters[p]);
            if (ws.size() >= 2) {
                const auto cl = ooc_sel::cluster_columns(ws, m, k);
                const auto sil = ooc_sel::silhouette(cl);
                sc.valid = true;
                sc.min_sil = sil.min_sil;
                sc.mean_sil = sil.mean_sil;
                sc.mean_err = err_sum / double(ws.size());
                rec.valid = 1;
                rec.min_silhouette = sil.min_sil;
                rec.mean_silhouette = sil.mean_sil;
                rec.mean_relative_error = sc.mean_err;
                if (med_out) std::copy(cl.medians.begin(), cl.medians.end(), med_out);
            } else if (med_out) {
                std::fill(med_out, med_out + m * k, 0.0);
            }
            if (med_out) med_out += m * k;
            scores.push_back(sc);
        }
        const auto [chosen, why] = ooc_sel::choose_k(scores, cfg->sil_threshold);
        if (chosen_k) *chosen_k = chosen;
        if (rationale && rationale_cap > 0) {
            const size_t len = std::min<size_t>(why.size(), rationale_cap - 1);
            std::memcpy(rationale, why.data(), len);
            rationale[len] = '\0';
        }
    });
    // leave the context as found: pristine A, collective solves
    if (perturbed) oocnmf_perturb(ctx, 0.0, 0);
    if (local_set) oocnmf_set_local(ctx, 0);
    return st;
}

}  // extern "C"
