// mbstab_b200.hpp -- C++ API mirroring the reference's operator interface for
// the multi-RHS BiCGStab hot path, implemented over the C ABI (mbstab_b200.h).
//
// A reference user swaps
//     #include "mbstab/core/spmv.hpp"      (proj/include/mbstab/core/spmv.hpp:16-17)
//     #include "mbstab/kernels/execute.hpp" (proj/include/mbstab/kernels/execute.hpp:26-30)
// for this header and the namespace mbstab:: for mbstab_b200::.  Container
// layouts are the reference's (types.hpp:13-83, csr.hpp:13-30); errors are
// rethrown as std::invalid_argument / std::runtime_error like the reference.
//
// Performance note: the free functions below upload their operands on every
// call (drop-in semantics).  For the hot path keep data resident with
// Device / DeviceMatrix / DeviceVector and call solve() on them.
#pragma once

#include <cstdint>
#include <memory>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "mbstab_b200.h"

namespace mbstab_b200 {

inline void check(int rc) {
    if (rc == MBG_OK) return;
    const std::string msg = mbg_last_error();
    if (rc == MBG_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

namespace core {

using index_t = std::int64_t;

struct MultiVector {  // types.hpp:13-35
    index_t n_rows = 0;
    int n_cols = 0;
    std::vector<double> data;
    MultiVector() = default;
    MultiVector(index_t rows, int cols)
        : n_rows(rows), n_cols(cols), data(static_cast<std::size_t>(rows) * cols, 0.0) {}
    double& operator()(index_t i, int c) { return data[static_cast<std::size_t>(i) * n_cols + c]; }
    double operator()(index_t i, int c) const { return data[static_cast<std::size_t>(i) * n_cols + c]; }
    bool same_shape(const MultiVector& o) const { return n_rows == o.n_rows && n_cols == o.n_cols; }
    void fill(double v) { data.assign(data.size(), v); }
};

struct ColumnScalars {  // types.hpp:39-50
    std::vector<double> values;
    ColumnScalars() = default;
    explicit ColumnScalars(int cols, double v = 0.0) : values(cols, v) {}
    static ColumnScalars constant(int cols, double v) { return ColumnScalars(cols, v); }
    int cols() const { return static_cast<int>(values.size()); }
    double& operator[](int c) { return values[c]; }
    double operator[](int c) const { return values[c]; }
};

struct ReductionEvent {
    int dots = 0;
    int cols = 0;
};

struct TrafficCounter {  // types.hpp:95-109
    std::int64_t vector_reads = 0;
    std::int64_t vector_writes = 0;
    double spmv_bytes = 0.0;
    std::vector<ReductionEvent> reductions;
    std::int64_t precond_applications = 0;
    std::int64_t vector_transfers() const { return vector_reads + vector_writes; }
};

struct CsrMatrix {  // csr.hpp:13-30
    index_t n_rows = 0;
    std::vector<std::int64_t> row_offsets;
    std::vector<std::int32_t> col_indices;
    std::vector<double> values;
    std::int64_t nnz() const { return row_offsets.empty() ? 0 : row_offsets.back(); }
    double avg_row_nnz() const { return n_rows > 0 ? double(nnz()) / double(n_rows) : 0.0; }
    void validate() const {
        if (row_offsets.size() != static_cast<std::size_t>(n_rows) + 1)
            throw std::invalid_argument("csr: row_offsets length must be n_rows+1");
        if (col_indices.size() != values.size())
            throw std::invalid_argument("csr: col_indices and values length mismatch");
        check(mbg_csr_validate(n_rows, row_offsets.data(), col_indices.data(),
                               static_cast<std::int64_t>(col_indices.size())));
    }
};

inline double spmv_traffic_bytes(const CsrMatrix& A, int m) {  // spmv.cpp:10-16
    return mbg_spmv_traffic_bytes(A.n_rows, A.nnz(), m);
}

inline CsrMatrix gen_poisson_7pt(int nx, int ny, int nz) {  // generators.cpp:37-67
    CsrMatrix A;
    A.n_rows = static_cast<index_t>(nx) * ny * nz;
    std::int64_t nnz = 0;
    A.row_offsets.resize(A.n_rows + 1);
    check(mbg_gen_stencil(0, nx, ny, nz, 0, &nnz, A.row_offsets.data(), nullptr, nullptr));
    A.col_indices.resize(nnz);
    A.values.resize(nnz);
    check(mbg_gen_stencil(0, nx, ny, nz, 0, &nnz, A.row_offsets.data(), A.col_indices.data(), A.values.data()));
    return A;
}

inline CsrMatrix gen_poisson_5pt(int nx, int ny) {  // generators.cpp:69-91
    CsrMatrix A;
    A.n_rows = static_cast<index_t>(nx) * ny;
    std::int64_t nnz = 0;
    A.row_offsets.resize(A.n_rows + 1);
    check(mbg_gen_stencil(3, nx, ny, 1, 0, &nnz, A.row_offsets.data(), nullptr, nullptr));
    A.col_indices.resize(nnz);
    A.values.resize(nnz);
    check(mbg_gen_stencil(3, nx, ny, 1, 0, &nnz, A.row_offsets.data(), A.col_indices.data(), A.values.data()));
    return A;
}

// core::read_matrix_market / write_matrix_market (matrix_market.hpp:15-20)
inline CsrMatrix read_matrix_market(const std::string& path) {
    void* h = nullptr;
    std::int64_t n = 0, nnz = 0;
    const int rc = mbg_mm_read(path.c_str(), &h, &n, &nnz);
    if (rc != MBG_OK) throw std::runtime_error(mbg_last_error());
    CsrMatrix A;
    A.n_rows = n;
    A.row_offsets.resize(n + 1);
    A.col_indices.resize(nnz);
    A.values.resize(nnz);
    mbg_mm_copy(h, A.row_offsets.data(), A.col_indices.data(), A.values.data());
    mbg_mm_free(h);
    return A;
}

inline void write_matrix_market(const CsrMatrix& A, const std::string& path) {
    const int rc = mbg_mm_write(path.c_str(), A.n_rows, A.row_offsets.data(), A.col_indices.data(), A.values.data());
    if (rc != MBG_OK) throw std::runtime_error(mbg_last_error());
}

}  // namespace core

// ---- device-resident objects ------------------------------------------------
class Device {
public:
    explicit Device(int device = 0) { check(mbg_ctx_create(device, &ctx_)); }
    ~Device() { if (ctx_) mbg_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    mbg_ctx* get() const { return ctx_; }
    // small classical solves in one cooperative launch (default on; same bits)
    void set_small_path(bool enable) { check(mbg_ctx_set_small_path(ctx_, enable ? 1 : 0)); }
    // leave `count` SMs to concurrent kernels (same bits)
    void reserve_sms(int count) { check(mbg_ctx_reserve_sms(ctx_, count)); }
    static Device& default_device() {
        static Device d(0);
        return d;
    }

private:
    mbg_ctx* ctx_ = nullptr;
};

class DeviceMatrix {
public:
    DeviceMatrix(Device& dev, const core::CsrMatrix& A) : dev_(&dev) {
        check(mbg_csr_upload(dev.get(), A.n_rows, A.row_offsets.data(), A.col_indices.data(), A.values.data(), &h_));
    }
    // Structured-grid hint (mbg_csr_set_grid): a grid-neighbour operator gets the
    // stencil twin (implicit columns, TMA-staged x planes); same bits.  Returns
    // the stencil kind (7, 27) or 0.
    int set_grid(int nx, int ny, int nz) {
        check(mbg_csr_set_grid(dev_->get(), h_, nx, ny, nz));
        return mbg_csr_stencil_kind(h_);
    }
    // The upload detects a lexicographic 7- / 27-point grid operator itself
    // (mbstab_b200.h); stencil_kind() tells, clear_grid() drops the twin.
    int stencil_kind() const { return mbg_csr_stencil_kind(h_); }
    void clear_grid() { check(mbg_csr_clear_grid(h_)); }
    ~DeviceMatrix() { if (h_) mbg_csr_free(h_); }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    const mbg_csr* get() const { return h_; }

private:
    Device* dev_ = nullptr;
    mbg_csr* h_ = nullptr;
};

class DeviceVector {
public:
    DeviceVector(Device& dev, core::index_t n, int m) : n_(n), m_(m) { check(mbg_mv_alloc(dev.get(), n, m, &h_)); }
    DeviceVector(Device& dev, const core::MultiVector& v) : DeviceVector(dev, v.n_rows, v.n_cols) { upload(v); }
    ~DeviceVector() { if (h_) mbg_mv_free(h_); }
    DeviceVector(const DeviceVector&) = delete;
    DeviceVector& operator=(const DeviceVector&) = delete;
    void upload(const core::MultiVector& v) { check(mbg_mv_upload(h_, v.data.data())); }
    void download(core::MultiVector& v) const {
        v.n_rows = n_;
        v.n_cols = m_;
        v.data.resize(static_cast<std::size_t>(n_) * m_);
        check(mbg_mv_download(h_, v.data.data()));
    }
    mbg_mv* get() const { return h_; }

private:
    mbg_mv* h_ = nullptr;
    core::index_t n_;
    int m_;
};

namespace core {

// core::spmv (spmv.hpp:16-17).  `threads` is accepted for signature
// compatibility; the GPU decides its own parallelism.
inline void spmv(const CsrMatrix& A, const MultiVector& x, MultiVector& y, TrafficCounter* counter = nullptr,
                 int threads = 1) {
    (void)threads;
    if (x.n_rows != A.n_rows || y.n_rows != A.n_rows || x.n_cols != y.n_cols)
        throw std::invalid_argument("spmv: dimension mismatch");
    if (x.data.data() == y.data.data()) throw std::invalid_argument("spmv: x and y must be distinct storage");
    Device& dev = Device::default_device();
    DeviceMatrix dA(dev, A);
    DeviceVector dx(dev, x), dy(dev, y.n_rows, y.n_cols);
    check(mbg_spmv(dev.get(), dA.get(), dx.get(), dy.get()));
    dy.download(y);
    if (counter) counter->spmv_bytes += spmv_traffic_bytes(A, x.n_cols);
}

/// y = A^T x, same traffic formula (spmv.hpp:19-21; setup-only in the solvers)
inline void spmv_transpose(const CsrMatrix& A, const MultiVector& x, MultiVector& y,
                           TrafficCounter* counter = nullptr) {
    if (x.n_rows != A.n_rows || y.n_rows != A.n_rows || x.n_cols != y.n_cols)
        throw std::invalid_argument("spmv: dimension mismatch");
    if (x.data.data() == y.data.data()) throw std::invalid_argument("spmv: x and y must be distinct storage");
    Device& dev = Device::default_device();
    DeviceMatrix dA(dev, A);
    DeviceVector dx(dev, x), dy(dev, y.n_rows, y.n_cols);
    check(mbg_spmv_transpose(dev.get(), dA.get(), dx.get(), dy.get()));
    dy.download(y);
    if (counter) counter->spmv_bytes += spmv_traffic_bytes(A, x.n_cols);
}

}  // namespace core

namespace kernels {  // statement.hpp:10-75, execute.hpp:10-30

using VectorId = int;
struct UpdateTerm {
    core::ColumnScalars coeff;
    VectorId vec = -1;
};
struct UpdateStatement {
    VectorId out = -1;
    std::vector<UpdateTerm> terms;
};
struct DotStatement {
    VectorId left = -1;
    VectorId right = -1;
    int slot = -1;
};
using Statement = std::variant<UpdateStatement, DotStatement>;
struct StatementGroup {
    std::vector<Statement> statements;
    bool empty() const { return statements.empty(); }
    int dot_slots() const {
        int mx = -1;
        for (const auto& s : statements)
            if (const auto* d = std::get_if<DotStatement>(&s)) mx = d->slot > mx ? d->slot : mx;
        return mx + 1;
    }
};
struct TrafficSummary {
    int reads = 0;
    int writes = 0;
    int total() const { return reads + writes; }
};
struct ExecOptions {
    int threads = 1;
};

inline std::vector<mbg_statement> to_abi(const StatementGroup& g) {
    std::vector<mbg_statement> out;
    for (const auto& s : g.statements) {
        mbg_statement a{};
        if (const auto* u = std::get_if<UpdateStatement>(&s)) {
            if (u->terms.size() > MBG_MAX_TERMS) throw std::invalid_argument("execute_group: too many terms");
            a.kind = MBG_STMT_UPDATE;
            a.out = u->out;
            a.nterms = static_cast<int>(u->terms.size());
            for (int t = 0; t < a.nterms; ++t) {
                a.term_vec[t] = u->terms[t].vec;
                a.term_coeff[t] = u->terms[t].coeff.values.data();
            }
        } else {
            const auto& d = std::get<DotStatement>(s);
            a.kind = MBG_STMT_DOT;
            a.left = d.left;
            a.right = d.right;
            a.slot = d.slot;
        }
        out.push_back(a);
    }
    return out;
}

inline TrafficSummary analyze_traffic(const StatementGroup& g) {
    auto st = to_abi(g);
    TrafficSummary t;
    check(mbg_analyze_traffic(st.data(), static_cast<int>(st.size()), &t.reads, &t.writes));
    return t;
}

// split_basic (statement.cpp:58-85): singleton groups; updates touching >= 4
// distinct vectors peel their trailing operand pair into a temporary.
inline std::vector<StatementGroup> split_basic(const StatementGroup& group, VectorId first_temp_id) {
    std::vector<StatementGroup> out;
    for (const auto& st : group.statements) {
        if (const auto* up = std::get_if<UpdateStatement>(&st)) {
            UpdateStatement cur = *up;
            VectorId next = first_temp_id;
            for (;;) {
                std::set<VectorId> inv{cur.out};
                for (const auto& t : cur.terms) inv.insert(t.vec);
                if (inv.size() < 4 || cur.terms.size() < 2) break;
                const int m = cur.terms.front().coeff.cols();
                UpdateStatement peeled;
                peeled.out = next++;
                peeled.terms.assign(cur.terms.end() - 2, cur.terms.end());
                out.push_back({{Statement{peeled}}});
                cur.terms.resize(cur.terms.size() - 2);
                cur.terms.push_back({core::ColumnScalars::constant(m, 1.0), peeled.out});
            }
            out.push_back({{Statement{cur}}});
        } else {
            out.push_back({{st}});
        }
    }
    return out;
}

// execute_group (execute.cpp:123-172): single fused pass on the GPU, exact dots.
inline void execute_group(const StatementGroup& group, std::span<core::MultiVector> vectors,
                          std::span<core::ColumnScalars> dot_results, core::TrafficCounter* counter = nullptr,
                          const ExecOptions& opts = {}) {
    (void)opts;
    const TrafficSummary traffic = analyze_traffic(group);
    if (group.empty()) return;
    Device& dev = Device::default_device();
    std::vector<std::unique_ptr<DeviceVector>> dv;
    std::vector<mbg_mv*> handles;
    for (auto& v : vectors) {
        dv.push_back(std::make_unique<DeviceVector>(dev, v));
        handles.push_back(dv.back()->get());
    }
    auto st = to_abi(group);
    const int m = vectors.empty() ? 1 : vectors[0].n_cols;
    const int nslots = static_cast<int>(dot_results.size());
    std::vector<double> dots(static_cast<std::size_t>(nslots > 0 ? nslots : 1) * m, 0.0);
    check(mbg_execute_group(dev.get(), st.data(), static_cast<int>(st.size()), handles.data(),
                            static_cast<int>(handles.size()), dots.data(), nslots));
    std::set<VectorId> written;
    int ndots = 0;
    for (const auto& s : group.statements) {
        if (const auto* u = std::get_if<UpdateStatement>(&s)) written.insert(u->out);
        if (const auto* d = std::get_if<DotStatement>(&s)) {
            dot_results[d->slot].values.assign(dots.begin() + d->slot * m, dots.begin() + (d->slot + 1) * m);
            ++ndots;
        }
    }
    for (VectorId id : written) dv[id]->download(vectors[id]);
    if (counter) {
        counter->vector_reads += traffic.reads;
        counter->vector_writes += traffic.writes;
        if (ndots > 0) counter->reductions.push_back({ndots, m});
    }
}

}  // namespace kernels

namespace solvers {  // SPEC.md:198-278 (missing from the reference tree)

// the six methods; RBiCGStab, PBiCGStab, PPipeBiCGStab are preconditioned
enum class Method {
    BiCGStab = MBG_BICGSTAB, RBiCGStab = MBG_RBICGSTAB, PipeBiCGStab = MBG_PIPEBICGSTAB,
    IBiCGStab = MBG_IBICGSTAB, PBiCGStab = MBG_PBICGSTAB, PPipeBiCGStab = MBG_PPIPEBICGSTAB
};
enum class Formulation { basic = MBG_BASIC, merged = MBG_MERGED, fused = MBG_FUSED };
inline bool is_preconditioned(Method m) {
    return m == Method::RBiCGStab || m == Method::PBiCGStab || m == Method::PPipeBiCGStab;
}

// identity (2 transfers per application) or synthetic(alpha)
// (alpha transfers: alpha/2 scale passes whose factors multiply to exactly 1).
struct Preconditioner {
    enum class Kind { identity, synthetic } kind = Kind::identity;
    int alpha = 2;
    static Preconditioner identity() { return {Kind::identity, 2}; }
    static Preconditioner synthetic(int a) {
        if (a < 2 || a % 2) throw std::invalid_argument("synthetic preconditioner: alpha must be even and >= 2");
        return {Kind::synthetic, a};
    }
};
struct Mode {
    bool fixed = false;
    int iterations = 1000;   // max (converge) or exact (fixed)
    static Mode converge(int max_iters) { return {false, max_iters}; }
    static Mode fixed_count(int n) { return {true, n}; }
};

struct SolveReport {
    int iterations = 0;
    bool converged = false;
    std::vector<core::ColumnScalars> residual_history;   // iterations+1 entries
    core::TrafficCounter traffic;
    double loop_ms = 0.0;
};

struct BreakdownError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Device-resident solve: X holds x0 on entry and the solution on exit.
// precond: required by the preconditioned methods, rejected by the others
// (std::invalid_argument); nullptr = identity for the former.
inline SolveReport solve(Device& dev, const DeviceMatrix& A, const DeviceVector& B, DeviceVector& X, int m,
                         Method method, Formulation form, double tol, Mode mode,
                         const Preconditioner* precond = nullptr) {
    std::vector<double> hist(static_cast<std::size_t>(mode.iterations + 1) * m);
    mbg_report rep{};
    const int pa = precond ? precond->alpha : (is_preconditioned(method) ? 2 : 0);
    const int rc = mbg_solve_pc(dev.get(), A.get(), B.get(), X.get(), static_cast<int>(method),
                                static_cast<int>(form), pa, tol, mode.fixed, mode.iterations, hist.data(), &rep);
    if (rc == MBG_ERR_BREAKDOWN) throw BreakdownError(mbg_last_error());
    check(rc);
    SolveReport r;
    r.iterations = rep.iterations;
    r.converged = rep.converged != 0;
    for (int j = 0; j <= rep.iterations; ++j) {
        core::ColumnScalars h(m);
        for (int c = 0; c < m; ++c) h[c] = hist[static_cast<std::size_t>(j) * m + c];
        r.residual_history.push_back(h);
    }
    r.traffic.vector_reads = rep.vector_reads;
    r.traffic.vector_writes = rep.vector_writes;
    r.traffic.spmv_bytes = rep.spmv_bytes;
    r.loop_ms = rep.loop_ms;
    return r;
}

// Host-container solve: uploads A, B and x0, downloads X.
inline SolveReport solve(const core::CsrMatrix& A, const core::MultiVector& B, core::MultiVector& X, Method method,
                         Formulation form, double tol, Mode mode, const Preconditioner* precond = nullptr) {
    if (!B.same_shape(X) || B.n_rows != A.n_rows) throw std::invalid_argument("solve: shape mismatch");
    Device& dev = Device::default_device();
    DeviceMatrix dA(dev, A);
    DeviceVector dB(dev, B), dX(dev, X);
    SolveReport r = solve(dev, dA, dB, dX, B.n_cols, method, form, tol, mode, precond);
    dX.download(X);
    return r;
}

}  // namespace solvers
}  // namespace mbstab_b200
