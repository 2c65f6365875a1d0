// C++ host core over the C-ABI (include/oocnmf_b200.h): the reference's oocnmf:: API for
// the MU path, implemented as validation + f64<->f32 staging + status->exception mapping.
#include <algorithm>
#include <cmath>

#include "oocnmf_b200/oocnmf.hpp"

#include <chrono>
#include <exception>
#include <thread>
#include "json_out.hpp"
#include "selection.hpp"

namespace oocnmf {

void throw_status(int st) {
    if (st == OOCNMF_OK) return;
    const std::string msg = oocnmf_last_error();
    switch (st) {
        case OOCNMF_ERR_SHAPE: throw ShapeError(msg);
        case OOCNMF_ERR_DATA: throw DataError(msg);
        case OOCNMF_ERR_IO: throw IoError(msg);
        case OOCNMF_ERR_COMM: throw CommError(msg);
        case OOCNMF_ERR_STORE: throw StoreError(msg);
        default: throw DeviceError(msg);
    }
}

// ------------------------------------------------------------------------- matrices
DenseMatrix::DenseMatrix(index_t r, index_t c, std::vector<double> data) : r_(r), c_(c), v_(std::move(data)) {
    if (v_.size() != r_ * c_)
        throw ShapeError("DenseMatrix: data length " + std::to_string(v_.size()) + " != " + shape_str());
}

CsrMatrix::CsrMatrix(index_t rows, index_t cols, std::vector<index_t> rp, std::vector<index_t> ci,
                     std::vector<double> v)
    : r_(rows), c_(cols), rp_(std::move(rp)), ci_(std::move(ci)), val_(std::move(v)) {
    validate_structure();
}

void CsrMatrix::validate_structure() const {
    if (rp_.size() != r_ + 1) throw ShapeError("CsrMatrix: row_ptr must have rows+1 entries");
    if (rp_.front() != 0) throw ShapeError("CsrMatrix: row_ptr[0] != 0");
    if (rp_.back() != val_.size() || ci_.size() != val_.size())
        throw ShapeError("CsrMatrix: row_ptr[rows] disagrees with nnz");
    for (index_t i = 0; i < r_; ++i) {
        if (rp_[i] > rp_[i + 1]) throw ShapeError("CsrMatrix: row_ptr decreases at row " + std::to_string(i));
        for (index_t p = rp_[i]; p < rp_[i + 1]; ++p) {
            if (ci_[p] >= c_) throw ShapeError("CsrMatrix: column index out of range in row " + std::to_string(i));
            if (p > rp_[i] && ci_[p] <= ci_[p - 1])
                throw ShapeError("CsrMatrix: column indices not strictly increasing in row " + std::to_string(i));
        }
    }
}

DenseMatrix CsrMatrix::to_dense() const {
    DenseMatrix d(r_, c_);
    for (index_t i = 0; i < r_; ++i)
        for (index_t p = rp_[i]; p < rp_[i + 1]; ++p) d.at(i, ci_[p]) = val_[p];
    return d;
}

CsrMatrix CsrMatrix::from_dense(const DenseMatrix& d, double tol) {
    std::vector<index_t> rp{0}, ci;
    std::vector<double> v;
    for (index_t i = 0; i < d.rows(); ++i) {
        for (index_t j = 0; j < d.cols(); ++j)
            if (std::abs(d.at(i, j)) > tol) ci.push_back(j), v.push_back(d.at(i, j));
        rp.push_back(v.size());
    }
    return CsrMatrix(d.rows(), d.cols(), std::move(rp), std::move(ci), std::move(v));
}

MatrixRef MatrixRef::window(IndexRange r, IndexRange c) const {
    if (r.begin > r.end || r.end > rows() || c.begin > c.end || c.end > cols())
        throw ShapeError("MatrixRef::window: window out of bounds for " + shape_str());
    MatrixRef o = *this;
    o.rr_ = {rr_.begin + r.begin, rr_.begin + r.end};
    o.cr_ = {cr_.begin + c.begin, cr_.begin + c.end};
    return o;
}

double MatrixRef::at(index_t i, index_t j) const {
    const index_t gi = rr_.begin + i, gj = cr_.begin + j;
    if (d_) return d_->at(gi, gj);
    const auto& rp = s_->row_ptr();
    const auto& ci = s_->col_idx();
    const auto b = ci.begin() + std::ptrdiff_t(rp[gi]), e = ci.begin() + std::ptrdiff_t(rp[gi + 1]);
    const auto it = std::lower_bound(b, e, gj);
    return (it != e && *it == gj) ? s_->values()[index_t(it - ci.begin())] : 0.0;
}

// ------------------------------------------------------------------------- rng
std::uint64_t CounterRng::mix(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
CounterRng::CounterRng(std::uint64_t seed, std::uint64_t stream) : key_(mix(seed ^ mix(stream + 0x632BE59BD9B4E019ULL))) {}
std::uint64_t CounterRng::bits(std::uint64_t index) const { return mix(key_ + (index + 1) * 0x9E3779B97F4A7C15ULL); }
double CounterRng::uniform(std::uint64_t index) const { return double(bits(index) >> 11) * 0x1.0p-53; }
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
    return CounterRng::mix(seed ^ CounterRng::mix(a ^ CounterRng::mix(b)));
}

// ------------------------------------------------------------------------- solver API
void NmfConfig::validate() const {
    if (k < 1) throw ShapeError("NmfConfig: k must be >= 1");
    if (!(eta >= 0)) throw ShapeError("NmfConfig: eta must be >= 0");
    if (max_iters < 1) throw ShapeError("NmfConfig: max_iters must be >= 1");
    if (error_check_interval < 1) throw ShapeError("NmfConfig: error_check_interval must be >= 1");
    if (!(epsilon > 0)) throw ShapeError("NmfConfig: epsilon must be > 0");
    if (init == FactorInit::from_files && (!init_w || !init_h))
        throw ShapeError("NmfConfig: init=from_files requires both factors");
}

DenseMatrix init_w_rows(index_t m, index_t k, std::uint64_t seed, IndexRange rows) {
    (void)m;
    DenseMatrix w(rows.extent(), k);
    throw_status(oocnmf_counter_uniform(seed, 1, rows.begin * k, rows.extent() * k, w.data()));
    return w;
}

DenseMatrix init_h_cols(index_t n, index_t k, std::uint64_t seed, IndexRange cols) {
    DenseMatrix h(k, cols.extent());
    for (index_t r = 0; r < k; ++r)
        throw_status(oocnmf_counter_uniform(seed, 2, r * n + cols.begin, cols.extent(), h.row(r)));
    return h;
}

std::pair<DenseMatrix, DenseMatrix> init_factors(index_t m, index_t n, index_t k, std::uint64_t seed) {
    if (m < 1 || n < 1 || k < 1) throw ShapeError("init_factors: dimensions must be >= 1");
    return {init_w_rows(m, k, seed, {0, m}), init_h_cols(n, k, seed, {0, n})};
}

namespace {

struct Ctx {
    oocnmf_ctx* c = nullptr;
    bool own = true;
    ~Ctx() {
        if (own && c) oocnmf_ctx_destroy(c);
    }
};

oocnmf_config to_c(const NmfConfig& cfg) {
    oocnmf_config c{};
    c.k = cfg.k;
    c.eta = cfg.eta;
    c.max_iters = cfg.max_iters;
    c.error_check_interval = cfg.error_check_interval;
    c.epsilon = cfg.epsilon;
    c.seed = cfg.seed;
    c.init = cfg.init == FactorInit::from_files ? 1 : 0;
    c.error_mode = int32_t(cfg.error_mode);
    return c;
}

// Uploads the row window [r0, r1) of `a` (all of its columns) as this context's A slab.
void upload(oocnmf_ctx* c, MatrixRef a, index_t r0, index_t r1) {
    const index_t rows = r1 - r0, n = a.cols();
    if (a.is_dense()) {
        const DenseMatrix& d = a.dense();
        const double* base = d.row(a.row_range().begin + r0) + a.col_range().begin;
        throw_status(oocnmf_load_dense_f64(c, base, d.cols()));
        return;
    }
    // CSR window: keep entries inside the column window, rebase to local coordinates.
    const CsrMatrix& s = a.sparse();
    const index_t c0 = a.col_range().begin, c1 = a.col_range().end;
    std::vector<std::uint64_t> rp(rows + 1, 0), ci;
    std::vector<double> v;
    for (index_t i = 0; i < rows; ++i) {
        const index_t gi = a.row_range().begin + r0 + i;
        for (index_t p = s.row_ptr()[gi]; p < s.row_ptr()[gi + 1]; ++p) {
            const index_t j = s.col_idx()[p];
            if (j < c0 || j >= c1) continue;
            ci.push_back(j - c0);
            v.push_back(s.values()[p]);
        }
        rp[i + 1] = v.size();
    }
    (void)n;
    throw_status(oocnmf_load_csr_f64(c, rp.data(), ci.data(), v.data()));
}

void fill_result(NmfResult& res, const oocnmf_info& info, const std::vector<std::uint64_t>& ti,
                 const std::vector<double>& te) {
    const index_t nt = std::min<index_t>(info.n_trace, ti.size());
    for (index_t i = 0; i < nt; ++i) res.error_trace.emplace_back(ti[i], te[i]);
    res.iterations_run = info.iterations_run;
    res.converged = info.converged != 0;
    auto& k = res.counters;
    k.h_update_s = info.h_update_s;
    k.w_update_s = info.w_update_s;
    k.allreduce_s = info.allreduce_s;
    k.error_check_s = info.error_check_s;
    k.io_s = info.io_s;
    k.total_s = info.total_s;
    k.flops = info.flops;
    k.peak_resident_bytes = info.peak_resident_bytes;
}

}  // namespace

NmfResult nmf_serial(MatrixRef a, const NmfConfig& cfg) {
    cfg.validate();
    const index_t m = a.rows(), n = a.cols(), k = cfg.k;
    if (m < 1 || n < 1) throw ShapeError("nmf_serial: empty input " + a.shape_str());
    if (cfg.init == FactorInit::from_files &&
        (cfg.init_w->rows() != m || cfg.init_w->cols() != k || cfg.init_h->rows() != k || cfg.init_h->cols() != n))
        throw ShapeError("nmf_serial: provided factors do not match A and k");
    Ctx ctx;
    throw_status(oocnmf_ctx_create(cfg.device, &ctx.c));
    throw_status(oocnmf_set_problem(ctx.c, m, n, k, 0, m));
    upload(ctx.c, a, 0, m);
    if (cfg.init == FactorInit::from_files)
        throw_status(oocnmf_set_factors_f64(ctx.c, cfg.init_w->data(), cfg.init_h->data()));
    const oocnmf_config cc = to_c(cfg);
    std::vector<std::uint64_t> ti(cfg.max_iters / cfg.error_check_interval + 2);
    std::vector<double> te(ti.size());
    oocnmf_info info{};
    throw_status(oocnmf_solve(ctx.c, &cc, ti.data(), te.data(), ti.size(), &info));
    NmfResult res;
    res.w = DenseMatrix(m, k);
    res.h = DenseMatrix(k, n);
    throw_status(oocnmf_get_factors_f64(ctx.c, res.w.data(), res.h.data()));
    fill_result(res, info, ti, te);
    return res;
}

// ------------------------------------------------------------------------- partition
std::string to_string(Strategy s) { return s == Strategy::cnmf ? "cnmf" : "rnmf"; }
Strategy choose_strategy(index_t m, index_t n) { return n > m ? Strategy::cnmf : Strategy::rnmf; }

namespace {
std::vector<IndexRange> split(index_t extent, index_t parts) {
    std::vector<std::uint64_t> b(parts + 1);
    throw_status(oocnmf_split_even(extent, parts, b.data()));
    std::vector<IndexRange> out;
    for (index_t p = 0; p < parts; ++p) out.push_back({b[p], b[p + 1]});
    return out;
}
}  // namespace

index_t PartitionPlan::max_slab_extent() const {
    index_t best = 0;
    for (const auto& s : slabs) best = std::max(best, strategy == Strategy::cnmf ? s.a_cols.extent() : s.a_rows.extent());
    return best;
}
index_t PartitionPlan::max_batch_extent() const {
    index_t best = 0;
    for (const auto& b : batches) best = std::max(best, b.extent());
    return best;
}

PartitionPlan make_plan(index_t m, index_t n, index_t k, int n_workers, index_t n_b, Strategy strategy) {
    if (m < 1 || n < 1 || k < 1) throw ShapeError("make_plan: dimensions must be >= 1");
    if (n_workers < 1) throw ShapeError("make_plan: need at least one worker");
    if (n_b < 1) throw ShapeError("make_plan: need at least one batch");
    const bool col = strategy == Strategy::cnmf;
    const index_t part_axis = col ? n : m, batch_axis = col ? m : n;
    if (index_t(n_workers) > part_axis)
        throw ShapeError("make_plan: " + std::to_string(n_workers) + " workers exceed the " + std::to_string(part_axis) +
                         " slabs available under " + to_string(strategy));
    if (n_b > batch_axis) throw ShapeError("make_plan: batches exceed the batched axis");
    PartitionPlan p;
    p.strategy = strategy;
    p.n_workers = n_workers;
    p.m = m, p.n = n, p.k = k, p.n_b = n_b;
    const auto sl = split(part_axis, index_t(n_workers));
    for (int r = 0; r < n_workers; ++r)
        p.slabs.push_back({r, col ? IndexRange{0, m} : sl[r], col ? sl[r] : IndexRange{0, n}});
    p.batches = split(batch_axis, n_b);
    return p;
}

namespace {
// Minimal writer for the reference's nlohmann::json::dump(2) output (2-space indent, objects one
// member per line, arrays of numbers on one line, keys emitted in sorted order by the callers).
std::string jpad(int d) { return std::string(size_t(2 * d), ' '); }
std::string jrange(const IndexRange& r, int) {  // (numeric arrays stay on one line)
    return "[" + std::to_string(r.begin) + "," + std::to_string(r.end) + "]";
}
}  // namespace

std::string PartitionPlan::to_json() const {
    const bool col = strategy == Strategy::cnmf;
    std::string o = "{\n";
    if (!batches.empty()) {
        o += jpad(1) + "\"batches\": [\n";
        for (size_t i = 0; i < batches.size(); ++i)
            o += jpad(2) + jrange(batches[i], 2) + (i + 1 < batches.size() ? ",\n" : "\n");
        o += jpad(1) + "],\n";
    }
    o += jpad(1) + "\"h_role\": \"" + (col ? "slab" : "replicated") + "\",\n";
    o += jpad(1) + "\"k\": " + std::to_string(k) + ",\n";
    o += jpad(1) + "\"m\": " + std::to_string(m) + ",\n";
    o += jpad(1) + "\"n\": " + std::to_string(n) + ",\n";
    o += jpad(1) + "\"n_b\": " + std::to_string(n_b) + ",\n";
    o += jpad(1) + "\"n_workers\": " + std::to_string(n_workers) + ",\n";
    o += jpad(1) + "\"strategy\": \"" + (col ? "cnmf" : "rnmf") + "\",\n";
    o += jpad(1) + "\"w_role\": \"" + (col ? "replicated" : "slab") + "\"";
    if (!slabs.empty()) {
        o += ",\n" + jpad(1) + "\"workers\": [\n";
        for (size_t i = 0; i < slabs.size(); ++i) {
            const auto& w = slabs[i];
            o += jpad(2) + "{\n" + jpad(3) + "\"a_cols\": " + jrange(w.a_cols, 3) + ",\n" + jpad(3) +
                 "\"a_rows\": " + jrange(w.a_rows, 3) + ",\n" + jpad(3) + "\"rank\": " + std::to_string(w.rank) +
                 "\n" + jpad(2) + "}" + (i + 1 < slabs.size() ? ",\n" : "\n");
        }
        o += jpad(1) + "]";
    }
    return o + "\n}";
}

std::string MemoryReport::to_json() const {
    return "{\n" + jpad(1) + "\"a_slab_bytes\": " + std::to_string(a_slab_bytes) + ",\n" + jpad(1) +
           "\"factor_bytes\": " + std::to_string(factor_bytes) + ",\n" + jpad(1) + "\"feasible\": " +
           (feasible ? "true" : "false") + ",\n" + jpad(1) + "\"intermediate_bytes\": " +
           std::to_string(intermediate_bytes) + ",\n" + jpad(1) + "\"min_n_b\": " + std::to_string(min_n_b) +
           ",\n" + jpad(1) + "\"peak_bytes\": " + std::to_string(peak_bytes) + ",\n" + jpad(1) +
           "\"store_peak_bytes\": " + std::to_string(store_peak_bytes) + "\n}";
}

MemoryReport memory_estimate(const PartitionPlan& plan, double density, index_t budget_bytes, index_t n_cb) {
    if (n_cb < 1) throw ShapeError("memory_estimate: n_cb must be >= 1");
    oocnmf_memory_report r{};
    throw_status(oocnmf_memory_estimate(plan.m, plan.n, plan.k, plan.n_workers, plan.strategy == Strategy::cnmf ? 1 : 2,
                                        density, budget_bytes, 0, &r));
    MemoryReport out;
    out.a_slab_bytes = r.a_slab_bytes, out.store_peak_bytes = r.store_peak_bytes, out.factor_bytes = r.factor_bytes;
    out.intermediate_bytes = r.intermediate_bytes, out.peak_bytes = r.peak_bytes, out.min_n_b = r.min_n_b;
    out.feasible = r.feasible != 0, out.in_core = r.in_core != 0;
    return out;
}

// ------------------------------------------------------------------------- distributed
CommHandle::UniqueId CommHandle::new_unique_id() {
    UniqueId id{};
    throw_status(oocnmf_comm_unique_id(id.data()));
    return id;
}

CommHandle::CommHandle(int rank, int size, int device, const UniqueId& id, double timeout_s)
    : rank_(rank), size_(size), device_(device) {
    oocnmf_ctx* c = nullptr;
    throw_status(oocnmf_ctx_create_comm(device, rank, size, id.data(), &c));
    ctx_ = std::shared_ptr<oocnmf_ctx>(c, [](oocnmf_ctx* p) { oocnmf_ctx_destroy(p); });
    set_timeout(timeout_s);
}

CommHandle::CommHandle(oocnmf_ctx* ctx, int rank, int size, int device)
    : rank_(rank), size_(size), device_(device), ctx_(ctx, [](oocnmf_ctx* p) { oocnmf_ctx_destroy(p); }) {}

void CommHandle::all_reduce_sum(DenseMatrix& buffer, PhaseTag tag) {
    if (!ctx_) throw CommError("all_reduce_sum: CommHandle has no device context");
    throw_status(oocnmf_allreduce_f64(ctx_.get(), buffer.data(), buffer.size(), int(tag)));
}

void CommHandle::barrier() {
    if (!ctx_) throw CommError("barrier: CommHandle has no device context");
    throw_status(oocnmf_barrier(ctx_.get()));
}

const CollectiveStats& CommHandle::stats() const {
    if (ctx_) {
        std::uint64_t b[kNumPhaseTags], c[kNumPhaseTags];
        double sec[kNumPhaseTags];
        throw_status(oocnmf_comm_stats(ctx_.get(), b, c, sec));
        for (std::size_t t = 0; t < kNumPhaseTags; ++t)
            stats_->per_tag[t] = {index_t(b[t]), index_t(c[t]), sec[t]};
    }
    return *stats_;
}

void CommHandle::reset_stats() {
    if (ctx_) throw_status(oocnmf_comm_reset_stats(ctx_.get()));
    *stats_ = CollectiveStats{};
}

void CommHandle::set_timeout(double seconds) {
    if (ctx_) throw_status(oocnmf_set_comm_timeout(ctx_.get(), seconds));
}

index_t CollectiveStats::total_bytes() const {
    index_t s = 0;
    for (const auto& t : per_tag) s += t.bytes;
    return s;
}
index_t CollectiveStats::total_calls() const {
    index_t s = 0;
    for (const auto& t : per_tag) s += t.calls;
    return s;
}
double CollectiveStats::total_seconds() const {
    double s = 0;
    for (const auto& t : per_tag) s += t.seconds;
    return s;
}

Backend backend_from_string(const std::string& s) {
    if (s == "loopback") return Backend::loopback;
    if (s == "threads") return Backend::threads;
    if (s == "tcp") return Backend::tcp;
    throw ShapeError("unknown comm backend '" + s + "' (expected loopback|threads|tcp)");
}

CommGroup spawn_group(int n, Backend backend, double timeout_s) {
    if (n < 1) throw ShapeError("spawn_group: need at least one rank");
    if (backend == Backend::loopback && n != 1) throw ShapeError("spawn_group: loopback needs n == 1");
    if (backend == Backend::tcp)
        throw ShapeError("spawn_group: the tcp backend is one process per rank; use connect_tcp");
    std::vector<int> devs(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r) devs[std::size_t(r)] = r;
    std::vector<oocnmf_ctx*> cs(static_cast<std::size_t>(n), nullptr);
    throw_status(oocnmf_ctx_create_group(n, devs.data(), cs.data()));
    CommGroup g;
    for (int r = 0; r < n; ++r) {
        g.handles.emplace_back(cs[std::size_t(r)], r, n, r);
        g.handles.back().set_timeout(timeout_s);
    }
    return g;
}

namespace {
// This rank's window of A (rows for RNMF, columns for CNMF) from memory or from a PDN1 /
// Matrix Market file (ASource::file: a PDN1 file is read window-only, like the reference's
// ChunkStore over a file).
void upload_slab(oocnmf_ctx* c, const ASource& a, const PartitionPlan& plan, const WorkerSlab& slab) {
    const bool col = plan.strategy == Strategy::cnmf;
    auto put = [&](MatrixRef full_or_win, bool is_window) {
        if (is_window) {
            upload(c, full_or_win, 0, full_or_win.rows());
            return;
        }
        if (full_or_win.rows() != plan.m || full_or_win.cols() != plan.n)
            throw ShapeError("nmf_distributed: A does not match the plan");
        if (col)
            upload(c, full_or_win.window({0, plan.m}, slab.a_cols), 0, plan.m);
        else
            upload(c, full_or_win, slab.a_rows.begin, slab.a_rows.end);
    };
    if (a.pdn1_path.empty()) {
        if (a.mem.empty()) throw ShapeError("nmf_distributed: empty A source");
        put(a.mem, false);
        return;
    }
    const std::string& p = a.pdn1_path;
    if (p.size() >= 4 && p.compare(p.size() - 4, 4, ".mtx") == 0) {
        const AnyMatrix full = read_mtx(p);
        put(full.ref(), false);
        return;
    }
    Pdn1File f(p);
    if (f.rows() != plan.m || f.cols() != plan.n) throw ShapeError("nmf_distributed: file A does not match the plan");
    if (f.is_dense()) {
        const DenseMatrix win = f.read_dense_window(slab.a_rows, slab.a_cols);
        put(MatrixRef(win), true);
    } else if (col) {
        const CsrMatrix all = f.read_csr_rows({0, plan.m});
        put(MatrixRef(all).window({0, plan.m}, slab.a_cols), true);
    } else {
        const CsrMatrix rows = f.read_csr_rows(slab.a_rows);
        put(MatrixRef(rows), true);
    }
}
}  // namespace

NmfResult nmf_distributed(const ASource& a, const NmfConfig& cfg, const PartitionPlan& plan, CommHandle& comm,
                          const StoreConfig& store_cfg, StoreCounters* store_counters_out) {
    cfg.validate();
    if (cfg.k != plan.k)
        throw ShapeError("nmf_distributed: cfg.k=" + std::to_string(cfg.k) + " disagrees with plan.k=" +
                         std::to_string(plan.k));
    if (comm.size() != plan.n_workers)
        throw ShapeError("nmf_distributed: group size " + std::to_string(comm.size()) + " != plan workers " +
                         std::to_string(plan.n_workers));
    if (!comm.context()) throw CommError("nmf_distributed: CommHandle has no device context");
    oocnmf_ctx* c = comm.context();
    const WorkerSlab& slab = plan.slabs[std::size_t(comm.rank())];
    if (plan.strategy == Strategy::cnmf) {
        // column partition (src/nmf_distributed.cpp:112-149): W replicated, H column slabs
        if (a.host_f32) throw ShapeError("nmf_distributed: out-of-core streaming is row-partitioned (RNMF) only");
        const index_t m = plan.m, n = plan.n, k = plan.k, c0 = slab.a_cols.begin, cols = slab.a_cols.extent();
        throw_status(oocnmf_set_problem_cols(c, m, n, k, c0, cols));
        upload_slab(c, a, plan, slab);
        if (cfg.init == FactorInit::from_files) {
            if (cfg.init_w->rows() != m || cfg.init_w->cols() != k || cfg.init_h->rows() != k ||
                cfg.init_h->cols() != n)
                throw ShapeError("nmf_distributed: provided factors do not match plan");
            DenseMatrix hs(k, cols);
            for (index_t r = 0; r < k; ++r)
                for (index_t j = 0; j < cols; ++j) hs.at(r, j) = cfg.init_h->at(r, c0 + j);
            throw_status(oocnmf_set_factors_f64(c, cfg.init_w->data(), hs.data()));
        }
        const oocnmf_config cc = to_c(cfg);
        std::vector<std::uint64_t> ti(cfg.max_iters / cfg.error_check_interval + 2);
        std::vector<double> te(ti.size());
        oocnmf_info info{};
        throw_status(oocnmf_solve(c, &cc, ti.data(), te.data(), ti.size(), &info));
        NmfResult res;
        res.w = DenseMatrix(m, k);
        res.h = DenseMatrix(k, n);
        throw_status(oocnmf_get_factors_f64(c, res.w.data(), nullptr));
        throw_status(oocnmf_gather_h_f64(c, res.h.data()));
        fill_result(res, info, ti, te);
        if (store_counters_out) *store_counters_out = StoreCounters{};
        return res;
    }
    const index_t m = plan.m, n = plan.n, k = plan.k, r0 = slab.a_rows.begin, rows = slab.a_rows.extent();
    throw_status(oocnmf_set_problem(c, m, n, k, r0, rows));
    const index_t per_row = ((n + 127) / 128 * 128) * 4;  // one padded f32 row of the device layout
    const index_t batch = store_cfg.budget_bytes ? std::max<index_t>(128, store_cfg.budget_bytes / 2 / per_row) : 0;
    StoreCounters sc{};
    // ASource::file under a budget the dense window does not fit (the reference's ChunkStore over
    // a PDN1 file, src/chunk_store.cpp:106-168): the window is read from the file once into
    // page-locked host memory and streamed to the GPU in budget-sized row batches every
    // iteration (out-of-core mode), instead of re-reading the file every iteration.
    std::vector<float> host_window;
    bool registered = false;
    const bool pdn1 = !a.pdn1_path.empty() &&
                      !(a.pdn1_path.size() >= 4 && a.pdn1_path.compare(a.pdn1_path.size() - 4, 4, ".mtx") == 0);
    bool file_ooc = false;
    if (pdn1 && store_cfg.budget_bytes) {
        Pdn1File f(a.pdn1_path);
        file_ooc = f.is_dense() && rows * per_row > store_cfg.budget_bytes;
        if (file_ooc && (f.rows() != m || f.cols() != n))
            throw ShapeError("nmf_distributed: file A does not match the plan");
    }
    if (a.host_f32) {
        throw_status(oocnmf_attach_host_dense_f32(c, a.host_f32, a.host_ld ? a.host_ld : n, batch));
    } else if (file_ooc) {
        const auto t_io = std::chrono::steady_clock::now();
        host_window.resize(rows * n);
        throw_status(oocnmf_pdn1_read_dense_f32(a.pdn1_path.c_str(), r0, r0 + rows, 0, n, host_window.data()));
        sc.io_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_io).count();
        sc.bytes_read = rows * n * index_t(Pdn1File(a.pdn1_path).dtype() == 1 ? 4 : 8);
        throw_status(oocnmf_host_register(host_window.data(), host_window.size() * sizeof(float)));
        registered = true;
        throw_status(oocnmf_attach_host_dense_f32(c, host_window.data(), n, batch));
    } else {
        const auto t_io = std::chrono::steady_clock::now();
        upload_slab(c, a, plan, slab);
        if (!a.pdn1_path.empty()) {
            sc.io_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_io).count();
            if (pdn1) {
                Pdn1File f(a.pdn1_path);
                sc.bytes_read = f.is_dense() ? rows * n * index_t(f.dtype() == 1 ? 4 : 8) : f.window_bytes(slab.a_rows, {0, n});
            }
        }
        sc.loads = 1;  // the slab is resident in HBM for the whole solve
        sc.resident_bytes = sc.peak_resident_bytes = rows * per_row;
    }
    struct Unregister {
        bool on;
        void* p;
        ~Unregister() {
            if (on) oocnmf_host_unregister(p);
        }
    } unreg{registered, host_window.data()};
    if (cfg.init == FactorInit::from_files) {
        if (cfg.init_w->rows() != m || cfg.init_w->cols() != k || cfg.init_h->rows() != k || cfg.init_h->cols() != n)
            throw ShapeError("nmf_distributed: provided factors do not match plan");
        throw_status(oocnmf_set_factors_f64(c, cfg.init_w->row(r0), cfg.init_h->data()));
    }
    const oocnmf_config cc = to_c(cfg);
    std::vector<std::uint64_t> ti(cfg.max_iters / cfg.error_check_interval + 2);
    std::vector<double> te(ti.size());
    oocnmf_info info{};
    throw_status(oocnmf_solve(c, &cc, ti.data(), te.data(), ti.size(), &info));
    NmfResult res;
    res.w = DenseMatrix(m, k);
    res.h = DenseMatrix(k, n);
    throw_status(oocnmf_get_factors_f64(c, nullptr, res.h.data()));
    throw_status(oocnmf_gather_w_f64(c, res.w.data()));
    fill_result(res, info, ti, te);
    if (a.host_f32 || file_ooc) {
        // every streamed row batch is a load into one of the two staging buffers, reclaimed by the
        // batch two after it (the reference's load / evict counting, chunk_store.cpp:65-104)
        sc.loads = info.h2d_batches;
        sc.evictions = info.h2d_batches > 2 ? info.h2d_batches - 2 : 0;
        sc.resident_bytes = sc.peak_resident_bytes = info.peak_resident_bytes;
        res.counters.io_s = sc.io_seconds;
    }
    if (store_counters_out) *store_counters_out = sc;
    return res;
}

std::vector<NmfResult> run_distributed_threads(const ASource& a, const NmfConfig& cfg, const PartitionPlan& plan,
                                               const StoreConfig& store_cfg, std::vector<CollectiveStats>* stats_out) {
    auto group = spawn_group(plan.n_workers, plan.n_workers == 1 ? Backend::loopback : Backend::threads);
    const std::size_t n = std::size_t(plan.n_workers);
    std::vector<NmfResult> results(n);
    std::vector<std::exception_ptr> errors(n);
    std::vector<std::thread> threads;
    for (std::size_t r = 0; r < n; ++r)
        threads.emplace_back([&, r] {
            try {
                NmfConfig c = cfg;
                c.device = group.handles[r].device();
                results[r] = nmf_distributed(a, c, plan, group.handles[r], store_cfg);
            } catch (...) {
                errors[r] = std::current_exception();
            }
        });
    for (auto& t : threads) t.join();
    if (stats_out) {
        stats_out->clear();
        for (auto& h : group.handles) stats_out->push_back(h.stats());
    }
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
    return results;
}

// ------------------------------------------------------------------------- model selection
void SelectionConfig::validate(index_t m, index_t n) const {
    if (k_min < 1 || k_max < k_min) throw ShapeError("SelectionConfig: need 1 <= k_min <= k_max");
    if (k_max >= std::min(m, n)) throw ShapeError("SelectionConfig: k_max must be below min(m, n)");
    if (n_perturbations < 2) throw ShapeError("SelectionConfig: need at least 2 perturbations");
    if (delta <= 0.0 || delta >= 1.0) throw ShapeError("SelectionConfig: delta must lie in (0, 1)");
    if (sil_threshold < -1.0 || sil_threshold > 1.0)
        throw ShapeError("SelectionConfig: sil_threshold must lie in [-1, 1]");
}

namespace {

SelectionReport run_select(oocnmf_ctx* c, index_t m, const SelectionConfig& cfg) {
    oocnmf_selection_config sc{};
    sc.k_min = cfg.k_min, sc.k_max = cfg.k_max, sc.n_perturbations = cfg.n_perturbations;
    sc.delta = cfg.delta, sc.sil_threshold = cfg.sil_threshold, sc.seed = cfg.seed;
    sc.nmf = to_c(cfg.nmf);
    const index_t nk = cfg.k_max - cfg.k_min + 1;
    std::vector<oocnmf_k_record> recs(nk);
    index_t med_total = 0;
    for (index_t k = cfg.k_min; k <= cfg.k_max; ++k) med_total += m * k;
    std::vector<double> med(med_total);
    std::int64_t chosen = -1;
    char why[512] = {0};
    throw_status(oocnmf_select_k(c, &sc, recs.data(), nk, med.data(), &chosen, why, sizeof why));
    SelectionReport rep;
    const double* mp = med.data();
    for (const auto& r : recs) {
        KRecord kr;
        kr.k = r.k, kr.valid = r.valid != 0, kr.runs_used = r.runs_used;
        kr.min_silhouette = r.min_silhouette, kr.mean_silhouette = r.mean_silhouette;
        kr.mean_relative_error = r.mean_relative_error;
        if (kr.valid) kr.medians = DenseMatrix(m, r.k, std::vector<double>(mp, mp + m * r.k));
        mp += m * r.k;
        rep.records.push_back(std::move(kr));
    }
    if (chosen >= 0) rep.chosen_k = index_t(chosen);
    rep.rationale = why;
    return rep;
}

std::string fmt_g(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%g", v);
    return b;
}

}  // namespace

SelectionReport select_k(MatrixRef a, const SelectionConfig& cfg) {
    cfg.validate(a.rows(), a.cols());
    Ctx ctx;
    throw_status(oocnmf_ctx_create(cfg.nmf.device, &ctx.c));
    throw_status(oocnmf_set_problem(ctx.c, a.rows(), a.cols(), cfg.k_min, 0, a.rows()));
    upload(ctx.c, a, 0, a.rows());
    return run_select(ctx.c, a.rows(), cfg);
}

SelectionReport select_k(MatrixRef a, const SelectionConfig& cfg, CommHandle& comm) {
    cfg.validate(a.rows(), a.cols());
    if (!comm.context()) throw CommError("select_k: CommHandle has no device context");
    throw_status(oocnmf_set_problem(comm.context(), a.rows(), a.cols(), cfg.k_min, 0, a.rows()));
    upload(comm.context(), a, 0, a.rows());
    return run_select(comm.context(), a.rows(), cfg);
}

std::string SelectionReport::to_json() const {  // model_selection.cpp:408-424
    jsonout::Json j;
    j["chosen_k"] = chosen_k ? jsonout::Json(std::uint64_t(*chosen_k)) : jsonout::Json("none");
    j["rationale"] = rationale;
    j["records"] = jsonout::Json::array();
    for (const KRecord& r : records) {
        jsonout::Json rec;
        rec["k"] = std::uint64_t(r.k);
        rec["valid"] = r.valid;
        rec["runs_used"] = std::uint64_t(r.runs_used);
        rec["min_silhouette"] = r.min_silhouette;
        rec["mean_silhouette"] = r.mean_silhouette;
        rec["mean_relative_error"] = r.mean_relative_error;
        j["records"].push_back(std::move(rec));
    }
    return j.dump(2);
}

std::string SelectionReport::to_csv() const {
    std::string out = "k,valid,runs_used,min_silhouette,mean_silhouette,mean_relative_error\n";
    for (const auto& r : records)
        out += std::to_string(r.k) + ',' + (r.valid ? "1" : "0") + ',' + std::to_string(r.runs_used) + ',' +
               fmt_g(r.min_silhouette) + ',' + fmt_g(r.mean_silhouette) + ',' + fmt_g(r.mean_relative_error) + '\n';
    return out;
}

DenseMatrix perturb_dense(MatrixRef a, double delta, std::uint64_t seed) {
    if (delta < 0.0 || delta >= 1.0) throw ShapeError("perturb: delta must lie in [0, 1)");
    if (!a.is_dense()) throw ShapeError("perturb_dense: dense input required");
    Ctx ctx;
    throw_status(oocnmf_ctx_create(0, &ctx.c));
    throw_status(oocnmf_set_problem(ctx.c, a.rows(), a.cols(), 1, 0, a.rows()));
    upload(ctx.c, a, 0, a.rows());
    throw_status(oocnmf_perturb(ctx.c, delta, seed));
    std::vector<float> f(a.rows() * a.cols());
    throw_status(oocnmf_download_dense_f32(ctx.c, f.data()));
    return DenseMatrix(a.rows(), a.cols(), std::vector<double>(f.begin(), f.end()));
}

CsrMatrix perturb_sparse(const CsrMatrix& a, double delta, std::uint64_t seed) {
    if (delta < 0.0 || delta >= 1.0) throw ShapeError("perturb: delta must lie in [0, 1)");
    Ctx ctx;
    throw_status(oocnmf_ctx_create(0, &ctx.c));
    throw_status(oocnmf_set_problem(ctx.c, a.rows(), a.cols(), 1, 0, a.rows()));
    upload(ctx.c, MatrixRef(a), 0, a.rows());
    throw_status(oocnmf_perturb(ctx.c, delta, seed));
    std::uint64_t nnz = 0;
    throw_status(oocnmf_csr_nnz(ctx.c, &nnz));
    std::vector<std::uint64_t> rp(a.rows() + 1), ci(nnz);
    std::vector<double> v(nnz);
    throw_status(oocnmf_download_csr(ctx.c, rp.data(), ci.data(), v.data()));
    return CsrMatrix(a.rows(), a.cols(), std::vector<index_t>(rp.begin(), rp.end()),
                     std::vector<index_t>(ci.begin(), ci.end()), std::move(v));
}

ColumnClusters cluster_columns(const std::vector<DenseMatrix>& runs, index_t k) {
    if (runs.size() < 2) throw ShapeError("cluster_columns: need at least 2 runs");
    const index_t m = runs[0].rows();
    std::vector<ooc_sel::Factor> f;
    for (const auto& w : runs) {
        if (w.rows() != m || w.cols() != k) throw ShapeError("cluster_columns: all runs must be m x k");
        f.push_back({w.data()});
    }
    try {
        ooc_sel::Clusters cl = ooc_sel::cluster_columns(f, m, k);
        ColumnClusters out;
        out.member_ids.resize(k);
        for (index_t c = 0; c < k; ++c)
            for (const auto& [r, col] : cl.member_ids[c]) out.member_ids[c].push_back({index_t(r), index_t(col)});
        out.points = std::move(cl.points);
        out.medians = DenseMatrix(m, k, std::move(cl.medians));
        out.dropped_zero_columns = cl.dropped_zero_columns;
        return out;
    } catch (const std::invalid_argument& e) {
        throw ShapeError(e.what());
    }
}

SilhouetteScore silhouette(const ColumnClusters& clusters) {
    ooc_sel::Clusters cl;
    cl.k = clusters.points.size();
    cl.m = clusters.medians.rows();
    cl.points = clusters.points;
    try {
        const ooc_sel::Silhouette s = ooc_sel::silhouette(cl);
        return {s.min_sil, s.mean_sil, s.per_cluster};
    } catch (const std::invalid_argument& e) {
        throw ShapeError(e.what());
    }
}

DenseMatrix pearson_correlation_matrix(const DenseMatrix& w_true, const DenseMatrix& w_est) {
    if (w_true.rows() != w_est.rows()) throw ShapeError("pearson_correlation_matrix: row counts differ");
    try {
        return DenseMatrix(w_true.cols(), w_est.cols(),
                           ooc_sel::pearson(w_true.data(), w_true.rows(), w_true.cols(), w_est.data(), w_est.cols()));
    } catch (const std::domain_error& e) {
        throw DataError(e.what());
    }
}

// ------------------------------------------------------------------------- matrix files
namespace {
std::vector<std::uint64_t> u64s(const std::vector<index_t>& v) { return {v.begin(), v.end()}; }
}  // namespace

void write_pdn1(const std::string& path, const DenseMatrix& m) {
    throw_status(oocnmf_pdn1_write_dense(path.c_str(), m.data(), m.rows(), m.cols(), 0));
}
void write_pdn1_f32(const std::string& path, const DenseMatrix& m) {
    throw_status(oocnmf_pdn1_write_dense(path.c_str(), m.data(), m.rows(), m.cols(), 1));
}
void write_pdn1(const std::string& path, const CsrMatrix& m) {
    const auto rp = u64s(m.row_ptr()), ci = u64s(m.col_idx());
    throw_status(oocnmf_pdn1_write_csr(path.c_str(), m.rows(), m.cols(), rp.data(), ci.data(), m.values().data(), 0));
}
void write_pdn1_f32(const std::string& path, const CsrMatrix& m) {
    const auto rp = u64s(m.row_ptr()), ci = u64s(m.col_idx());
    throw_status(oocnmf_pdn1_write_csr(path.c_str(), m.rows(), m.cols(), rp.data(), ci.data(), m.values().data(), 1));
}

Pdn1File::Pdn1File(const std::string& path) : path_(path) {
    std::int32_t kind = 0, dtype = 0;
    std::uint64_t r = 0, c = 0, z = 0;
    throw_status(oocnmf_pdn1_info(path.c_str(), &kind, &dtype, &r, &c, &z));
    kind_ = kind, dtype_ = dtype, rows_ = r, cols_ = c, nnz_ = z;
}

DenseMatrix Pdn1File::read_dense_window(IndexRange r, IndexRange c) const {
    DenseMatrix out(r.extent(), c.extent());
    throw_status(oocnmf_pdn1_read_dense(path_.c_str(), r.begin, r.end, c.begin, c.end, out.data()));
    return out;
}

CsrMatrix Pdn1File::read_csr_rows(IndexRange r) const {
    std::uint64_t nnz = 0;
    throw_status(oocnmf_pdn1_csr_rows_nnz(path_.c_str(), r.begin, r.end, &nnz));
    std::vector<std::uint64_t> rp(r.extent() + 1), ci(nnz);
    std::vector<double> v(nnz);
    throw_status(oocnmf_pdn1_read_csr_rows(path_.c_str(), r.begin, r.end, rp.data(), ci.data(), v.data()));
    return CsrMatrix(r.extent(), cols_, std::vector<index_t>(rp.begin(), rp.end()),
                     std::vector<index_t>(ci.begin(), ci.end()), std::move(v));
}

index_t Pdn1File::window_bytes(IndexRange r, IndexRange c) const {
    const index_t vb = dtype_ == 1 ? 4 : 8;
    if (kind_ == 0) return r.extent() * c.extent() * vb;
    std::uint64_t nnz = 0;
    throw_status(oocnmf_pdn1_csr_rows_nnz(path_.c_str(), r.begin, r.end, &nnz));
    return (r.extent() + 1) * 8 + nnz * (8 + vb);
}

AnyMatrix read_pdn1(const std::string& path) {
    Pdn1File f(path);
    if (f.is_dense()) return AnyMatrix{f.read_dense_window({0, f.rows()}, {0, f.cols()})};
    return AnyMatrix{f.read_csr_rows({0, f.rows()})};
}

void write_mtx(const std::string& path, const DenseMatrix& m) {
    throw_status(oocnmf_mtx_write_dense(path.c_str(), m.data(), m.rows(), m.cols()));
}
void write_mtx(const std::string& path, const CsrMatrix& m) {
    const auto rp = u64s(m.row_ptr()), ci = u64s(m.col_idx());
    throw_status(oocnmf_mtx_write_csr(path.c_str(), m.rows(), m.cols(), rp.data(), ci.data(), m.values().data()));
}

AnyMatrix read_mtx(const std::string& path) {
    std::int32_t kind = 0;
    std::uint64_t r = 0, c = 0, z = 0;
    throw_status(oocnmf_mtx_info(path.c_str(), &kind, &r, &c, &z));
    if (kind == 0) {
        DenseMatrix d(r, c);
        throw_status(oocnmf_mtx_read(path.c_str(), d.data(), nullptr, nullptr, nullptr));
        return AnyMatrix{std::move(d)};
    }
    std::vector<std::uint64_t> rp(r + 1), ci(z);
    std::vector<double> v(z);
    throw_status(oocnmf_mtx_read(path.c_str(), nullptr, rp.data(), ci.data(), v.data()));
    return AnyMatrix{CsrMatrix(r, c, std::vector<index_t>(rp.begin(), rp.end()),
                               std::vector<index_t>(ci.begin(), ci.end()), std::move(v))};
}

AnyMatrix read_matrix(const std::string& path) {
    if (path.size() >= 4 && path.compare(path.size() - 4, 4, ".mtx") == 0) return read_mtx(path);
    return read_pdn1(path);
}

}  // namespace oocnmf
