// C++ host core of the B200 MU-NMF backend — source-compatible with the reference's
// `oocnmf` API for the MU path, so a caller of
//     oocnmf::nmf_serial(MatrixRef, const NmfConfig&)          (include/oocnmf/nmf.hpp:64)
//     oocnmf::nmf_distributed(ASource, NmfConfig, PartitionPlan, CommHandle&, StoreConfig)
//                                                  (include/oocnmf/nmf_distributed.hpp:34-36)
// recompiles against these headers unchanged. Everything here is host plumbing (types,
// validation, f64<->f32 at the boundary, exception mapping); all arithmetic runs on the
// GPU behind the C-ABI in include/oocnmf_b200.h. The reference header names
// (oocnmf/matrix.hpp, nmf.hpp, ...) are thin forwarders to this file.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "oocnmf_b200.h"

namespace oocnmf {

using index_t = std::size_t;

// ---- errors (reference: include/oocnmf/error.hpp:9-36) ----
struct ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CommError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StoreError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// New: CUDA / device failures of the B200 backend (no CPU fallback exists).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Throws the exception type matching an oocnmf_status (OOCNMF_OK is a no-op).
void throw_status(int status);

// ---- matrices (reference: include/oocnmf/matrix.hpp:15-151) ----
struct IndexRange {
    index_t begin = 0, end = 0;
    index_t extent() const { return end - begin; }
    bool contains(index_t i) const { return begin <= i && i < end; }
    bool operator==(const IndexRange&) const = default;
};

class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(index_t r, index_t c, double fill = 0.0) : r_(r), c_(c), v_(r * c, fill) {}
    DenseMatrix(index_t r, index_t c, std::vector<double> data);
    index_t rows() const { return r_; }
    index_t cols() const { return c_; }
    index_t size() const { return v_.size(); }
    double& at(index_t i, index_t j) { return v_[i * c_ + j]; }
    double at(index_t i, index_t j) const { return v_[i * c_ + j]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double* row(index_t i) { return v_.data() + i * c_; }
    const double* row(index_t i) const { return v_.data() + i * c_; }
    std::string shape_str() const { return std::to_string(r_) + "x" + std::to_string(c_); }
    bool operator==(const DenseMatrix&) const = default;

private:
    index_t r_ = 0, c_ = 0;
    std::vector<double> v_;
};

class CsrMatrix {
public:
    CsrMatrix() = default;
    CsrMatrix(index_t rows, index_t cols, std::vector<index_t> row_ptr, std::vector<index_t> col_idx,
              std::vector<double> values);
    index_t rows() const { return r_; }
    index_t cols() const { return c_; }
    index_t nnz() const { return val_.size(); }
    const std::vector<index_t>& row_ptr() const { return rp_; }
    const std::vector<index_t>& col_idx() const { return ci_; }
    const std::vector<double>& values() const { return val_; }
    std::vector<double>& values() { return val_; }
    std::string shape_str() const { return std::to_string(r_) + "x" + std::to_string(c_); }
    void validate_structure() const;
    DenseMatrix to_dense() const;
    static CsrMatrix from_dense(const DenseMatrix& d, double zero_tol = 0.0);
    bool operator==(const CsrMatrix&) const = default;

private:
    index_t r_ = 0, c_ = 0;
    std::vector<index_t> rp_{0}, ci_;
    std::vector<double> val_;
};

/// Non-owning window over a dense or CSR matrix (local coordinates [0,rows) x [0,cols)).
class MatrixRef {
public:
    MatrixRef() = default;
    explicit MatrixRef(const DenseMatrix& m) : d_(&m), rr_{0, m.rows()}, cr_{0, m.cols()} {}
    explicit MatrixRef(const CsrMatrix& m) : s_(&m), rr_{0, m.rows()}, cr_{0, m.cols()} {}
    MatrixRef window(IndexRange r, IndexRange c) const;
    index_t rows() const { return rr_.extent(); }
    index_t cols() const { return cr_.extent(); }
    IndexRange row_range() const { return rr_; }
    IndexRange col_range() const { return cr_; }
    bool is_dense() const { return d_ != nullptr; }
    bool is_sparse() const { return s_ != nullptr; }
    bool empty() const { return !d_ && !s_; }
    const DenseMatrix& dense() const { return *d_; }
    const CsrMatrix& sparse() const { return *s_; }
    double at(index_t i, index_t j) const;
    std::string shape_str() const { return std::to_string(rows()) + "x" + std::to_string(cols()); }

private:
    const DenseMatrix* d_ = nullptr;
    const CsrMatrix* s_ = nullptr;
    IndexRange rr_, cr_;
};

// ---- counter RNG (reference: include/oocnmf/rng.hpp:11-45) ----
class CounterRng {
public:
    CounterRng(std::uint64_t seed, std::uint64_t stream);
    std::uint64_t bits(std::uint64_t index) const;
    double uniform(std::uint64_t index) const;
    double uniform(std::uint64_t index, double lo, double hi) const { return lo + (hi - lo) * uniform(index); }
    static std::uint64_t mix(std::uint64_t z);

private:
    std::uint64_t key_;
};
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b = 0);

// ---- solver config / result (reference: include/oocnmf/nmf.hpp:11-66) ----
inline constexpr double kDefaultEpsilon = 1e-12;
enum class FactorInit { uniform01, from_files };
/// B200 extension: how the relative error is evaluated at check iterations.
enum class ErrorMode { automatic = 0, direct = 1, trace = 2 };

struct NmfConfig {
    index_t k = 1;
    double eta = 1e-4;
    index_t max_iters = 1000;
    index_t error_check_interval = 10;
    double epsilon = kDefaultEpsilon;
    std::uint64_t seed = 0;
    FactorInit init = FactorInit::uniform01;
    std::optional<DenseMatrix> init_w;
    std::optional<DenseMatrix> init_h;
    // B200 extensions (defaults reproduce the reference's behaviour on GPU 0)
    int device = 0;
    ErrorMode error_mode = ErrorMode::automatic;
    void validate() const;
};

struct PhaseCounters {
    double h_update_s = 0, w_update_s = 0, allreduce_s = 0, error_check_s = 0, io_s = 0, total_s = 0;
    double flops = 0;
    index_t peak_resident_bytes = 0;
};

struct NmfResult {
    DenseMatrix w;
    DenseMatrix h;
    std::vector<std::pair<index_t, double>> error_trace;
    index_t iterations_run = 0;
    bool converged = false;
    PhaseCounters counters;
};

std::pair<DenseMatrix, DenseMatrix> init_factors(index_t m, index_t n, index_t k, std::uint64_t seed);
DenseMatrix init_w_rows(index_t m, index_t k, std::uint64_t seed, IndexRange rows);
DenseMatrix init_h_cols(index_t n, index_t k, std::uint64_t seed, IndexRange cols);

/// W-then-H multiplicative updates of A ≈ WH on one B200 (A dense or CSR).
NmfResult nmf_serial(MatrixRef a, const NmfConfig& cfg);

// ---- partition (reference: include/oocnmf/partition.hpp:10-46) ----
enum class Strategy { cnmf, rnmf };
std::string to_string(Strategy s);
Strategy choose_strategy(index_t m, index_t n);
struct WorkerSlab {
    int rank = 0;
    IndexRange a_rows, a_cols;
};
struct PartitionPlan {
    Strategy strategy = Strategy::rnmf;
    int n_workers = 1;
    index_t m = 0, n = 0, k = 0;
    index_t n_b = 1;
    std::vector<WorkerSlab> slabs;
    std::vector<IndexRange> batches;
    index_t max_slab_extent() const;
    index_t max_batch_extent() const;
    /// The reference's JSON (src/partition.cpp:89-104: nlohmann dump(2), sorted keys).
    std::string to_json() const;
};
PartitionPlan make_plan(index_t m, index_t n, index_t k, int n_workers, index_t n_b, Strategy strategy);

/// Per-rank device bytes of the B200 layout (f32, padded, tensor-core operand copies, stream-K
/// slots) for the plan's largest slab; min_n_b: 1 = in-core fits, > 1 = out-of-core row batches
/// (dense RNMF), 0 = infeasible (reference: partition.hpp:51-64).
struct MemoryReport {
    index_t a_slab_bytes = 0;
    index_t store_peak_bytes = 0;
    index_t factor_bytes = 0;
    index_t intermediate_bytes = 0;
    index_t peak_bytes = 0;
    index_t min_n_b = 0;
    bool feasible = false;
    bool in_core = false;
    /// The reference's JSON (src/partition.cpp:199-209; in_core is this backend's extra field
    /// and, like the reference, not serialised).
    std::string to_json() const;
};
MemoryReport memory_estimate(const PartitionPlan& plan, double density, index_t budget_bytes, index_t n_cb = 1);

// ---- distributed (reference: include/oocnmf/nmf_distributed.hpp, comm.hpp) ----
/// Group transports (comm.hpp:10). B200: loopback (one rank), threads (one process, one GPU
/// per rank thread, NCCL clique) and tcp (one process per rank: connect_tcp, a TCP rendezvous
/// that hands out an NCCL unique id; the collectives themselves run over NCCL).
enum class Backend { loopback, threads, tcp };
Backend backend_from_string(const std::string& s);

/// Tags collectives so stats can be attributed to algorithm phases (comm.hpp:13-20).
enum class PhaseTag : std::uint32_t {
    generic = 0,
    w_update = 1,
    h_update = 2,
    error_check = 3,
    gather = 4,
    barrier = 5,
};
inline constexpr std::size_t kNumPhaseTags = 6;

/// comm.hpp:28-43. seconds = device time of the collectives (NCCL over NVLink).
struct CollectiveStats {
    struct PerTag {
        index_t bytes = 0;
        index_t calls = 0;
        double seconds = 0;
    };
    std::array<PerTag, kNumPhaseTags> per_tag{};
    PerTag& operator[](PhaseTag t) { return per_tag[static_cast<std::size_t>(t)]; }
    const PerTag& operator[](PhaseTag t) const { return per_tag[static_cast<std::size_t>(t)]; }
    index_t total_bytes() const;
    index_t total_calls() const;
    double total_seconds() const;
};

/// One rank of an NCCL group (one process or host thread per GPU). Multi-process: rank 0
/// calls new_unique_id(), ships it to the others, every rank constructs a handle. In one
/// process: spawn_group(n, Backend::threads). Collectives are blocking; a collective that makes
/// no progress for timeout_s (default 60 s, comm.cpp:89-111) throws CommError and poisons the
/// group (the communicator is aborted, every later collective throws).
class CommHandle {
public:
    using UniqueId = std::array<unsigned char, 128>;
    static UniqueId new_unique_id();
    CommHandle() = default;
    CommHandle(int rank, int size, int device, const UniqueId& id, double timeout_s = 60.0);
    /// Adopt a context made by oocnmf_ctx_create_group (takes ownership).
    CommHandle(oocnmf_ctx* ctx, int rank, int size, int device);
    int rank() const { return rank_; }
    int size() const { return size_; }
    int device() const { return device_; }
    oocnmf_ctx* context() const { return ctx_.get(); }
    /// In-place elementwise sum across all ranks (comm.hpp:61).
    void all_reduce_sum(DenseMatrix& buffer, PhaseTag tag);
    /// Returns once every rank has entered.
    void barrier();
    /// This rank's collective statistics, the solver's own collectives included.
    const CollectiveStats& stats() const;
    void reset_stats();
    void set_timeout(double seconds);

private:
    int rank_ = 0, size_ = 1, device_ = 0;
    std::shared_ptr<oocnmf_ctx> ctx_;
    std::shared_ptr<CollectiveStats> stats_ = std::make_shared<CollectiveStats>();
};

/// All handles of an in-process group (comm.hpp:75-77).
struct CommGroup {
    std::vector<CommHandle> handles;
};
/// loopback: n must be 1. threads: n handles on GPUs 0..n-1 sharing one NCCL clique, one per
/// worker thread (comm.hpp:80-82).
CommGroup spawn_group(int n, Backend backend, double timeout_s = 60.0);
/// tcp backend (comm.hpp:84-87): rank 0 listens on peers[0] ("host:port"), the other ranks
/// connect to it (retrying until timeout_s) and receive an NCCL unique id; every rank then
/// joins one NCCL communicator on its GPU (OOCNMF_DEVICE, else LOCAL_RANK, else rank modulo the
/// visible GPUs). One handle per process.
CommHandle connect_tcp(int n, int rank, const std::vector<std::string>& peers, std::uint64_t group_id = 0,
                       double timeout_s = 60.0);

struct ASource {
    MatrixRef mem;
    std::string pdn1_path;  // PDN1 (.pdn1) or Matrix Market (.mtx) file; PDN1 is read window-wise
    const float* host_f32 = nullptr;  // B200 extension: out-of-core host slab (rows of this rank)
    index_t host_ld = 0;
    static ASource memory(MatrixRef a) { return {a, {}, nullptr, 0}; }
    static ASource file(std::string path) { return {{}, std::move(path), nullptr, 0}; }
    static ASource host_slab(const float* p, index_t ld) { return {{}, {}, p, ld}; }
};
struct StoreConfig {
    index_t budget_bytes = 0;  // out-of-core: HBM staging budget for the two row-batch buffers
    int n_cb = 1;
    bool prefetch = false;
};
struct StoreCounters {
    index_t loads = 0, evictions = 0, bytes_read = 0, resident_bytes = 0, peak_resident_bytes = 0;
    double io_seconds = 0;
};

/// Row-partitioned (RNMF) MU on this rank's GPU; collective over the CommHandle's group.
/// Returns the gathered W (m x k) and replicated H on every rank.
NmfResult nmf_distributed(const ASource& a, const NmfConfig& cfg, const PartitionPlan& plan, CommHandle& comm,
                          const StoreConfig& store_cfg = {}, StoreCounters* store_counters_out = nullptr);
/// Convenience driver: runs all ranks of a threads-backend group on worker threads, one GPU
/// each, and returns the per-rank results (index = rank) (nmf_distributed.hpp:40-43).
std::vector<NmfResult> run_distributed_threads(const ASource& a, const NmfConfig& cfg, const PartitionPlan& plan,
                                               const StoreConfig& store_cfg = {},
                                               std::vector<CollectiveStats>* stats_out = nullptr);

// ---- matrix files (reference: include/oocnmf/io.hpp) ----
struct AnyMatrix {
    std::variant<DenseMatrix, CsrMatrix> value;
    bool is_dense() const { return std::holds_alternative<DenseMatrix>(value); }
    const DenseMatrix& dense() const { return std::get<DenseMatrix>(value); }
    const CsrMatrix& sparse() const { return std::get<CsrMatrix>(value); }
    MatrixRef ref() const { return is_dense() ? MatrixRef(dense()) : MatrixRef(sparse()); }
    index_t rows() const { return is_dense() ? dense().rows() : sparse().rows(); }
    index_t cols() const { return is_dense() ? dense().cols() : sparse().cols(); }
};

void write_pdn1(const std::string& path, const DenseMatrix& m);
void write_pdn1(const std::string& path, const CsrMatrix& m);
/// B200 extension: PDN1 dtype 1 (f32 values), the byte the reference reserves.
void write_pdn1_f32(const std::string& path, const DenseMatrix& m);
void write_pdn1_f32(const std::string& path, const CsrMatrix& m);
AnyMatrix read_pdn1(const std::string& path);

/// Random-access reader over a PDN1 file (f64 or f32 payload).
class Pdn1File {
public:
    explicit Pdn1File(const std::string& path);
    bool is_dense() const { return kind_ == 0; }
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    index_t nnz() const { return nnz_; }
    int dtype() const { return dtype_; }
    DenseMatrix read_dense_window(IndexRange r, IndexRange c) const;
    CsrMatrix read_csr_rows(IndexRange r) const;  // global column indices
    index_t window_bytes(IndexRange r, IndexRange c) const;

private:
    std::string path_;
    int kind_ = 0, dtype_ = 0;
    index_t rows_ = 0, cols_ = 0, nnz_ = 0;
};

void write_mtx(const std::string& path, const DenseMatrix& m);
void write_mtx(const std::string& path, const CsrMatrix& m);
AnyMatrix read_mtx(const std::string& path);
/// Dispatch on extension: .mtx -> Matrix Market, anything else -> PDN1.
AnyMatrix read_matrix(const std::string& path);

// ---- synthetic inputs (reference: include/oocnmf/synth.hpp) ----
struct LowrankSpec {
    index_t m = 0;
    index_t n = 0;
    index_t k_true = 0;
    double noise = 0.0;  ///< multiplicative noise amplitude (0 disables)
    std::uint64_t seed = 0;
};
struct LowrankData {
    DenseMatrix a;   // m x n
    DenseMatrix w0;  // m x k_true
    DenseMatrix h0;  // k_true x n
};
/// A = W0 H0 with Gaussian-bump columns of W0 (plus a 0.01 U floor) and U(0,1) H0, optionally
/// scaled entrywise by U(1 - noise, 1 + noise) (src/synth.cpp:18-57). Host-side, bit-identical
/// to the reference (same CounterRng streams, same f64 summation order).
LowrankData gen_lowrank(const LowrankSpec& spec);
struct SparseSpec {
    index_t m = 0;
    index_t n = 0;
    double density = 0.0;  ///< independent per-entry Bernoulli probability
    std::uint64_t seed = 0;
};
/// m x n CSR, entry (i, j) present iff U(seed, 14, i n + j) < density, value U(seed, 15, i n + j)
/// (src/synth.cpp:59-86). Evaluated on GPU 0 (the reference generator, O(m n) draws, runs
/// there at HBM speed) and downloaded; bit-identical to the reference.
CsrMatrix gen_sparse_random(const SparseSpec& spec);

// ---- model selection (reference: include/oocnmf/model_selection.hpp) ----
struct SelectionConfig {
    index_t k_min = 1;
    index_t k_max = 1;
    index_t n_perturbations = 16;  ///< P: runs per candidate k
    double delta = 0.03;           ///< perturbation amplitude, in (0,1)
    double sil_threshold = 0.75;   ///< min-silhouette acceptance bar
    NmfConfig nmf;                 ///< per-run template (k and seed are overridden); nmf.device = GPU
    std::uint64_t seed = 0;
    void validate(index_t m, index_t n) const;
};

struct KRecord {
    index_t k = 0;
    bool valid = false;
    index_t runs_used = 0;
    double min_silhouette = 0.0;
    double mean_silhouette = 0.0;
    double mean_relative_error = 0.0;
    DenseMatrix medians;  ///< m x k elementwise-median cluster columns
};

struct SelectionReport {
    std::vector<KRecord> records;
    std::optional<index_t> chosen_k;
    std::string rationale;
    std::string to_json() const;
    std::string to_csv() const;
};

/// perturb_dense / perturb_sparse, evaluated on the GPU (cfg device 0): every stored entry
/// times 1 - delta + 2 delta U(seed, 21, i * n + j); values come back f32-rounded.
DenseMatrix perturb_dense(MatrixRef a, double delta, std::uint64_t seed);
CsrMatrix perturb_sparse(const CsrMatrix& a, double delta, std::uint64_t seed);

struct ColumnClusters {
    std::vector<std::vector<std::pair<index_t, index_t>>> member_ids;
    std::vector<std::vector<std::vector<double>>> points;
    DenseMatrix medians;  // m x k
    index_t dropped_zero_columns = 0;
};
ColumnClusters cluster_columns(const std::vector<DenseMatrix>& runs, index_t k);

struct SilhouetteScore {
    double min_sil = 0.0;
    double mean_sil = 0.0;
    std::vector<double> per_cluster;
};
SilhouetteScore silhouette(const ColumnClusters& clusters);

DenseMatrix pearson_correlation_matrix(const DenseMatrix& w_true, const DenseMatrix& w_est);

/// P perturbed GPU factorizations per k in [k_min, k_max], W-column clustering, silhouettes,
/// errors, and the largest qualifying k (src/model_selection.cpp:316-406).
SelectionReport select_k(MatrixRef a, const SelectionConfig& cfg);
/// B200 extension: the same sweep spread over an NCCL group as replicas (every rank passes the
/// full A); collective, every rank returns the same report.
SelectionReport select_k(MatrixRef a, const SelectionConfig& cfg, CommHandle& comm);

}  // namespace oocnmf
