// ref_shim.cpp -- C entry points over the REFERENCE's own kernels.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together
// with the reference sources where they lie (/root/reference/proj/src/core/*.cpp,
// proj/src/kernels/{statement,execute}.cpp) into oracle/_ref/libmbstab_ref.so.
// No reference source is copied into this repository.
//
// Used by tests/ to pin the oracle and the product against the reference
// arithmetic, and by bench.py --impl reference as the CPU arm.  The solver
// layer is missing from the reference (proj/CMakeLists.txt:25,28,29,31), so
// ref_solve restates Alg. 2 / 6 / 4 (PAPER.md:1407-1438, 1562-1598,
// 1488-1525) on top of the reference's core::spmv and kernels::execute_group
// with the reference's own (naive, thread-blocked) dot products.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "mbstab/core/csr.hpp"
#include "mbstab/core/generators.hpp"
#include "mbstab/core/spmv.hpp"
#include "mbstab/core/matrix_market.hpp"
#include "mbstab/core/matrix_market.hpp"
#include "mbstab/core/types.hpp"
#include "mbstab/kernels/execute.hpp"
#include "mbstab/kernels/statement.hpp"
#include "mbstab_b200.h"

using namespace mbstab;
using core::ColumnScalars;
using core::CsrMatrix;
using core::MultiVector;
using kernels::DotStatement;
using kernels::Statement;
using kernels::StatementGroup;
using kernels::UpdateStatement;

static thread_local std::string g_err;

extern "C" const char* ref_last_error() { return g_err.c_str(); }

static CsrMatrix make_csr(int64_t n, const int64_t* off, const int32_t* col, const double* val) {
    CsrMatrix A;
    A.n_rows = n;
    A.row_offsets.assign(off, off + n + 1);
    const int64_t nnz = off[n];
    A.col_indices.assign(col, col + nnz);
    A.values.assign(val, val + nnz);
    return A;
}

static MultiVector make_mv(int64_t n, int m, const double* data) {
    MultiVector v(n, m);
    if (data) std::memcpy(v.data.data(), data, sizeof(double) * n * m);
    return v;
}

static StatementGroup make_group(const mbg_statement* st, int ns, int m) {
    StatementGroup g;
    for (int i = 0; i < ns; ++i) {
        if (st[i].kind == MBG_STMT_UPDATE) {
            UpdateStatement u;
            u.out = st[i].out;
            for (int t = 0; t < st[i].nterms; ++t) {
                kernels::UpdateTerm term;
                term.coeff.values.assign(st[i].term_coeff[t], st[i].term_coeff[t] + m);
                term.vec = st[i].term_vec[t];
                u.terms.push_back(term);
            }
            g.statements.push_back(Statement{u});
        } else {
            DotStatement d;
            d.left = st[i].left;
            d.right = st[i].right;
            d.slot = st[i].slot;
            g.statements.push_back(Statement{d});
        }
    }
    return g;
}

extern "C" int ref_gen_poisson_7pt(int nx, int ny, int nz, int64_t* nnz, int64_t* off, int32_t* col,
                                   double* val) {
    try {
        if (!off) { *nnz = core::poisson_7pt_nnz(nx, ny, nz); return 0; }
        CsrMatrix A = core::gen_poisson_7pt(nx, ny, nz);
        *nnz = A.nnz();
        std::copy(A.row_offsets.begin(), A.row_offsets.end(), off);
        std::copy(A.col_indices.begin(), A.col_indices.end(), col);
        std::copy(A.values.begin(), A.values.end(), val);
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_gen_poisson_5pt(int nx, int ny, int64_t* nnz, int64_t* off, int32_t* col, double* val) {
    try {
        if (!off) { *nnz = core::poisson_5pt_nnz(nx, ny); return 0; }
        CsrMatrix A = core::gen_poisson_5pt(nx, ny);
        *nnz = A.nnz();
        std::memcpy(off, A.row_offsets.data(), sizeof(int64_t) * (A.n_rows + 1));
        std::memcpy(col, A.col_indices.data(), sizeof(int32_t) * A.nnz());
        std::memcpy(val, A.values.data(), sizeof(double) * A.nnz());
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_validate(int64_t n, const int64_t* off, const int32_t* col, const double* val) {
    try { make_csr(n, off, col, val).validate(); return 0; }
    catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_spmv(int64_t n, const int64_t* off, const int32_t* col, const double* val, int m,
                        const double* x, double* y, int threads) {
    try {
        CsrMatrix A = make_csr(n, off, col, val);
        MultiVector X = make_mv(n, m, x), Y(n, m);
        core::spmv(A, X, Y, nullptr, threads);
        std::memcpy(y, Y.data.data(), sizeof(double) * n * m);
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_spmv_transpose(int64_t n, const int64_t* off, const int32_t* col, const double* val, int m,
                                  const double* x, double* y) {
    try {
        CsrMatrix A = make_csr(n, off, col, val);
        MultiVector X = make_mv(n, m, x), Y(n, m);
        core::spmv_transpose(A, X, Y, nullptr);
        std::memcpy(y, Y.data.data(), sizeof(double) * n * m);
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

// core::read_matrix_market: two-phase (arrays NULL -> sizes only; the file is re-read).
extern "C" int ref_read_matrix_market(const char* path, int64_t* n, int64_t* nnz, int64_t* off, int32_t* col,
                                      double* val) {
    try {
        CsrMatrix A = core::read_matrix_market(std::string(path));
        *n = A.n_rows;
        *nnz = A.nnz();
        if (off) std::memcpy(off, A.row_offsets.data(), sizeof(int64_t) * (A.n_rows + 1));
        if (col) std::memcpy(col, A.col_indices.data(), sizeof(int32_t) * A.nnz());
        if (val) std::memcpy(val, A.values.data(), sizeof(double) * A.nnz());
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_write_matrix_market(const char* path, int64_t n, const int64_t* off, const int32_t* col,
                                       const double* val) {
    try {
        CsrMatrix A = make_csr(n, off, col, val);
        core::write_matrix_market(A, std::string(path));
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" double ref_spmv_traffic_bytes(int64_t n, int64_t nnz, int m) {
    CsrMatrix A;
    A.n_rows = n;
    A.row_offsets.assign(2, 0);
    A.row_offsets.back() = nnz;  // spmv_traffic_bytes only reads n_rows and nnz()
    return core::spmv_traffic_bytes(A, m);
}

extern "C" int ref_run_group(const mbg_statement* st, int ns, int nvec, int64_t n, int m,
                             double* const* vecs, double* dots, int nslots, int threads) {
    try {
        std::vector<MultiVector> v;
        for (int i = 0; i < nvec; ++i) v.push_back(make_mv(n, m, vecs[i]));
        std::vector<ColumnScalars> d(nslots);
        StatementGroup g = make_group(st, ns, m);
        kernels::ExecOptions o;
        o.threads = threads;
        kernels::execute_group(g, v, d, nullptr, o);
        for (int i = 0; i < nvec; ++i) std::memcpy(vecs[i], v[i].data.data(), sizeof(double) * n * m);
        for (int s = 0; s < nslots; ++s)
            for (int c = 0; c < m; ++c)
                dots[s * m + c] = c < d[s].cols() ? d[s][c] : 0.0;
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_analyze_traffic(const mbg_statement* st, int ns, int m, int* r, int* w) {
    try {
        auto t = kernels::analyze_traffic(make_group(st, ns, m));
        *r = t.reads; *w = t.writes;
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

extern "C" int ref_split_basic_traffic(const mbg_statement* st, int ns, int m, int first_temp, int* r,
                                       int* w, int* ngroups) {
    try {
        auto parts = kernels::split_basic(make_group(st, ns, m), first_temp);
        kernels::TrafficSummary sum;
        for (const auto& g : parts) sum += kernels::analyze_traffic(g);
        *r = sum.reads; *w = sum.writes; *ngroups = static_cast<int>(parts.size());
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}

// ---------------------------------------------------------------------------
// Restated merged solvers on the reference kernels (CPU baseline arm).
// Term expansions follow SURVEY.md Appendix C; dots are the reference's.
// ---------------------------------------------------------------------------
namespace {

struct Ctx {
    std::vector<MultiVector>& v;
    std::vector<ColumnScalars> dots;
    kernels::ExecOptions opts;
    int m;
    void run(const StatementGroup& g) { kernels::execute_group(g, v, dots, nullptr, opts); }
};

kernels::UpdateTerm T(const ColumnScalars& c, int vec) { return kernels::UpdateTerm{c, vec}; }
Statement U(int out, std::vector<kernels::UpdateTerm> terms) { return Statement{UpdateStatement{out, std::move(terms)}}; }
Statement D(int l, int r, int slot) { return Statement{DotStatement{l, r, slot}}; }

ColumnScalars div(const ColumnScalars& a, const ColumnScalars& b) {
    ColumnScalars o(a.cols());
    for (int c = 0; c < a.cols(); ++c) o[c] = a[c] / b[c];
    return o;
}

}  // namespace

// hist (nullable): (maxit+1)*m relative recursive residuals, h_0 = sqrt(rho0/bb),
// h_{j+1} = sqrt(max(res2,0)/bb) -- the same definition as the GPU solver's.
extern "C" int ref_solve_hist(int method, int64_t n, const int64_t* off, const int32_t* col,
                              const double* val, int m, const double* b, double* x, double tol,
                              int fixed, int maxit, int threads, int* iters_out, double* loop_seconds,
                              double* hist);

extern "C" int ref_solve(int method, int64_t n, const int64_t* off, const int32_t* col,
                         const double* val, int m, const double* b, double* x, double tol,
                         int fixed, int maxit, int threads, int* iters_out, double* loop_seconds) {
    return ref_solve_hist(method, n, off, col, val, m, b, x, tol, fixed, maxit, threads, iters_out, loop_seconds,
                          nullptr);
}

extern "C" int ref_solve_hist(int method, int64_t n, const int64_t* off, const int32_t* col,
                              const double* val, int m, const double* b, double* x, double tol,
                              int fixed, int maxit, int threads, int* iters_out, double* loop_seconds,
                              double* hist) {
    try {
        CsrMatrix A = make_csr(n, off, col, val);
        enum { X, B, R, R0, P, V, S, TT, Z, VH, TH, RT, Q, W, Y, NV };
        std::vector<MultiVector> vec;
        for (int i = 0; i < NV; ++i) vec.emplace_back(n, m);
        std::memcpy(vec[X].data.data(), x, sizeof(double) * n * m);
        std::memcpy(vec[B].data.data(), b, sizeof(double) * n * m);
        Ctx cx{vec, std::vector<ColumnScalars>(4), {}, m};
        cx.opts.threads = threads;
        const ColumnScalars one = ColumnScalars::constant(m, 1.0), mone = ColumnScalars::constant(m, -1.0);

        core::spmv(A, vec[X], vec[TT], nullptr, threads);
        cx.run({{U(R, {T(one, B), T(mone, TT)}), U(R0, {T(one, R)}), D(R0, R0, 0), D(B, B, 1)}});
        ColumnScalars rho = cx.dots[0], bb = cx.dots[1], eps2(m);
        for (int c = 0; c < m; ++c) eps2[c] = (tol * tol) * bb[c];
        auto record = [&](int j, const ColumnScalars& r2) {
            if (!hist) return;
            for (int c = 0; c < m; ++c) hist[static_cast<size_t>(j) * m + c] = std::sqrt((r2[c] > 0.0 ? r2[c] : 0.0) / bb[c]);
        };
        record(0, rho);
        auto below = [&](const ColumnScalars& r2) {
            for (int c = 0; c < m; ++c) if (!(r2[c] < eps2[c])) return false;
            return true;
        };
        int it = 0;
        const auto t_loop = std::chrono::steady_clock::now();
        if (method == MBG_BICGSTAB) {
            cx.run({{U(P, {T(one, R)})}});
            for (it = 0; it < maxit; ++it) {
                core::spmv(A, vec[P], vec[V], nullptr, threads);
                cx.run({{D(V, R0, 0)}});
                ColumnScalars alpha = div(rho, cx.dots[0]);
                cx.run({{U(S, {T(one, R), T(-alpha, V)})}});
                core::spmv(A, vec[S], vec[TT], nullptr, threads);
                cx.run({{D(TT, S, 0), D(TT, TT, 1), D(S, S, 2)}});
                ColumnScalars omega = div(cx.dots[0], cx.dots[1]);
                ColumnScalars res2 = cx.dots[2] - omega * cx.dots[0];
                record(it + 1, res2);
                const bool conv = !fixed && below(res2);
                cx.run({{U(X, {T(one, X), T(alpha, P), T(omega, S)}), U(R, {T(one, S), T(-omega, TT)}),
                         D(R, R0, 0)}});
                if (conv) { ++it; break; }
                ColumnScalars beta = div(cx.dots[0], rho) * div(alpha, omega);
                rho = cx.dots[0];
                cx.run({{U(P, {T(one, R), T(beta, P), T(-(beta * omega), V)})}});
            }
        } else if (method == MBG_RBICGSTAB) {
            cx.run({{U(Z, {T(one, R0)}), U(VH, {T(one, R0)})}});
            for (it = 0; it < maxit; ++it) {
                core::spmv(A, vec[VH], vec[V], nullptr, threads);
                cx.run({{D(V, R0, 0)}});
                vec[S].data = vec[V].data;  // identity M^-1
                ColumnScalars alpha = div(rho, cx.dots[0]);
                cx.run({{U(TH, {T(one, Z), T(-alpha, S)})}});
                core::spmv(A, vec[TH], vec[TT], nullptr, threads);
                cx.run({{U(RT, {T(one, R), T(-alpha, V)}), D(TT, RT, 0), D(TT, TT, 1), D(TT, R0, 2),
                         D(RT, RT, 3)}});
                vec[Q].data = vec[TT].data;  // identity M^-1
                ColumnScalars omega = div(cx.dots[0], cx.dots[1]);
                ColumnScalars res2 = cx.dots[3] - omega * cx.dots[0];
                record(it + 1, res2);
                ColumnScalars psi = cx.dots[2];
                cx.run({{U(R, {T(one, RT), T(-omega, TT)})}});
                if (!fixed && below(res2)) {
                    cx.run({{U(X, {T(one, X), T(alpha, VH), T(omega, TH)})}});
                    ++it;
                    break;
                }
                ColumnScalars rhon = -(omega * psi);
                ColumnScalars beta = div(rhon, rho) * div(alpha, omega);
                rho = rhon;
                cx.run({{U(X, {T(one, X), T(alpha, VH), T(omega, TH)}), U(Z, {T(one, TH), T(-omega, Q)}),
                         U(VH, {T(one, Z), T(beta, VH), T(-(beta * omega), S)})}});
            }
        } else if (method == MBG_PIPEBICGSTAB) {
            core::spmv(A, vec[R], vec[W], nullptr, threads);
            core::spmv(A, vec[W], vec[TT], nullptr, threads);
            cx.run({{D(R0, W, 0)}});
            ColumnScalars alpha = div(rho, cx.dots[0]), beta(m, 0.0), omega(m, 0.0);
            for (it = 0; it < maxit; ++it) {
                ColumnScalars nbo = -(beta * omega);
                cx.run({{U(P, {T(one, R), T(beta, P), T(nbo, S)}), U(S, {T(one, W), T(beta, S), T(nbo, Z)}),
                         U(Z, {T(one, TT), T(beta, Z), T(nbo, V)}), U(Q, {T(one, R), T(-alpha, S)}),
                         U(Y, {T(one, W), T(-alpha, Z)}), D(Q, Y, 0), D(Y, Y, 1), D(Q, Q, 2)}});
                core::spmv(A, vec[Z], vec[V], nullptr, threads);
                omega = div(cx.dots[0], cx.dots[1]);
                ColumnScalars res2 = cx.dots[2] - omega * cx.dots[0];
                record(it + 1, res2);
                cx.run({{U(X, {T(one, X), T(alpha, P), T(omega, Q)}), U(R, {T(one, Q), T(-omega, Y)})}});
                if (!fixed && below(res2)) { ++it; break; }
                cx.run({{U(W, {T(one, Y), T(-omega, TT), T(omega * alpha, V)}), D(R0, R, 0), D(R0, Z, 1),
                         D(R0, W, 2), D(R0, S, 3)}});
                core::spmv(A, vec[W], vec[TT], nullptr, threads);
                ColumnScalars rhon = cx.dots[0];
                beta = div(alpha, omega) * div(rhon, rho);
                ColumnScalars den = (cx.dots[2] + beta * cx.dots[3]) - (beta * omega) * cx.dots[1];
                alpha = div(rhon, den);
                rho = rhon;
            }
        } else {
            throw std::invalid_argument("ref_solve: unknown method");
        }
        if (loop_seconds)
            *loop_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
        std::memcpy(x, vec[X].data.data(), sizeof(double) * n * m);
        *iters_out = it;
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return 1; }
}
