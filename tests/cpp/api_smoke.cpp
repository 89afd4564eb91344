// api_smoke.cpp -- exercises the C++ API (include/mbstab_b200.hpp) the way a
// reference user would (core::spmv, kernels::execute_group, solvers::solve)
// and checks it against plain host loops.  Built and run by
// tests/test_gpu_cpp_api.py on the GPU box.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "mbstab_b200.hpp"

using namespace mbstab_b200;

int main() {
    core::CsrMatrix A = core::gen_poisson_7pt(12, 10, 8);
    A.validate();
    const int m = 3;
    core::MultiVector x(A.n_rows, m), y(A.n_rows, m);
    for (std::size_t i = 0; i < x.data.size(); ++i) x.data[i] = std::sin(0.1 * double(i));
    core::TrafficCounter tc;
    core::spmv(A, x, y, &tc);
    for (core::index_t i = 0; i < A.n_rows; ++i)
        for (int c = 0; c < m; ++c) {
            double acc = 0.0;
            for (auto k = A.row_offsets[i]; k < A.row_offsets[i + 1]; ++k) acc += A.values[k] * x(A.col_indices[k], c);
            if (acc != y(i, c)) { std::printf("spmv mismatch at %ld,%d\n", long(i), c); return 1; }
        }
    if (tc.spmv_bytes != core::spmv_traffic_bytes(A, m)) { std::puts("traffic mismatch"); return 1; }

    // execute_group: y2 = 1*x + (-0.5)*y ; dot(y2, x) ; dot(x, x)
    std::vector<core::MultiVector> vecs{x, y, core::MultiVector(A.n_rows, m)};
    std::vector<core::ColumnScalars> dots(2);
    kernels::StatementGroup g;
    g.statements.push_back(kernels::UpdateStatement{2, {{core::ColumnScalars::constant(m, 1.0), 0},
                                                        {core::ColumnScalars::constant(m, -0.5), 1}}});
    g.statements.push_back(kernels::DotStatement{2, 0, 0});
    g.statements.push_back(kernels::DotStatement{0, 0, 1});
    kernels::execute_group(g, vecs, dots, &tc);
    if (tc.vector_reads != 2 || tc.vector_writes != 1 || tc.reductions.size() != 1) { std::puts("counter"); return 1; }
    for (core::index_t i = 0; i < A.n_rows; ++i)
        for (int c = 0; c < m; ++c) {
            double v = 0.0;
            v += 1.0 * x(i, c);
            v += -0.5 * y(i, c);
            if (v != vecs[2](i, c)) { std::puts("update mismatch"); return 1; }
        }
    for (int c = 0; c < m; ++c) {
        double s = 0.0;
        for (core::index_t i = 0; i < A.n_rows; ++i) s += x(i, c) * x(i, c);
        if (std::fabs(s - dots[1][c]) > 1e-12 * std::fabs(s)) { std::puts("dot mismatch"); return 1; }
    }
    auto parts = kernels::split_basic(g, 100);
    if (parts.size() != 3) { std::puts("split_basic"); return 1; }

    // solve from host containers
    core::MultiVector B(A.n_rows, m), X(A.n_rows, m);
    for (std::size_t i = 0; i < B.data.size(); ++i) B.data[i] = std::cos(0.3 * double(i));
    auto rep = solvers::solve(A, B, X, solvers::Method::PipeBiCGStab, solvers::Formulation::merged, 1e-10,
                              solvers::Mode::converge(500));
    if (!rep.converged || rep.residual_history.size() != static_cast<std::size_t>(rep.iterations + 1)) {
        std::puts("solve did not converge");
        return 1;
    }
    core::MultiVector R(A.n_rows, m);
    core::spmv(A, X, R);
    double worst = 0.0;
    for (std::size_t i = 0; i < R.data.size(); ++i) worst = std::fmax(worst, std::fabs(R.data[i] - B.data[i]));
    if (worst > 1e-7) { std::printf("residual %g\n", worst); return 1; }
    // the preconditioned methods with a synthetic preconditioner, and the
    // SPEC.md:205 presence rule
    {
        core::MultiVector X2(A.n_rows, m);
        auto pc = solvers::Preconditioner::synthetic(4);
        auto r2 = solvers::solve(A, B, X2, solvers::Method::PPipeBiCGStab, solvers::Formulation::merged, 1e-10,
                                 solvers::Mode::converge(500), &pc);
        core::MultiVector X3(A.n_rows, m);
        auto r3 = solvers::solve(A, B, X3, solvers::Method::IBiCGStab, solvers::Formulation::merged, 1e-10,
                                 solvers::Mode::converge(500));
        if (!r2.converged || !r3.converged) { std::puts("preconditioned / improved solve"); return 1; }
        try {
            core::MultiVector X4(A.n_rows, m);
            solvers::solve(A, B, X4, solvers::Method::BiCGStab, solvers::Formulation::merged, 1e-10,
                           solvers::Mode::converge(10), &pc);
            std::puts("preconditioner on an unpreconditioned method not rejected");
            return 1;
        } catch (const std::invalid_argument&) {
        }
    }
    // 5-point generator, transpose SpMV and the MatrixMarket round trip
    {
        core::CsrMatrix P5 = core::gen_poisson_5pt(9, 7);
        if (P5.n_rows != 63 || P5.values[0] != 4.0) { std::puts("gen_poisson_5pt"); return 1; }
        core::MultiVector xs(P5.n_rows, 2), y1(P5.n_rows, 2), y2(P5.n_rows, 2);
        for (std::size_t i = 0; i < xs.data.size(); ++i) xs.data[i] = std::sin(0.7 * double(i));
        core::spmv(P5, xs, y1);
        core::spmv_transpose(P5, xs, y2);   // symmetric operator: A^T x == A x elementwise
        for (std::size_t i = 0; i < y1.data.size(); ++i)
            if (std::fabs(y1.data[i] - y2.data[i]) > 1e-14) { std::puts("spmv_transpose"); return 1; }
        const std::string path = "/tmp/mbg_api_smoke.mtx";
        core::write_matrix_market(P5, path);
        core::CsrMatrix R = core::read_matrix_market(path);
        if (R.values != P5.values || R.col_indices != P5.col_indices) { std::puts("matrix market"); return 1; }
    }
    // device-resident solve on the stencil twin -- detected by the upload itself
    // (no grid call, as in the reference) unless MBG_AUTO_GRID=0, then declared
    // with set_grid -- and on the CSR kernels (twin dropped): the same bits
    // (exact dots, same summation order)
    {
        Device dev;
        DeviceMatrix dA(dev, A), dC(dev, A);
        const char* ag = std::getenv("MBG_AUTO_GRID");
        if (!(ag && ag[0] == '0')) {
            if (dA.stencil_kind() != 7) { std::puts("stencil twin not detected at upload"); return 1; }
        } else if (dA.stencil_kind() != 0) {
            std::puts("MBG_AUTO_GRID=0 ignored");
            return 1;
        }
        if (dA.set_grid(12, 10, 8) != 7) { std::puts("stencil twin not built"); return 1; }
        dC.clear_grid();
        if (dC.stencil_kind() != 0) { std::puts("clear_grid"); return 1; }
        const int m8 = 8;
        core::MultiVector B8(A.n_rows, m8), Xs(A.n_rows, m8), Xc(A.n_rows, m8);
        for (std::size_t i = 0; i < B8.data.size(); ++i) B8.data[i] = std::sin(0.1 * double(i));
        DeviceVector dB(dev, B8), dXs(dev, A.n_rows, m8), dXc(dev, A.n_rows, m8);
        auto rs = solvers::solve(dev, dA, dB, dXs, m8, solvers::Method::BiCGStab, solvers::Formulation::fused, 1e-10,
                                 solvers::Mode::converge(500));
        auto rc = solvers::solve(dev, dC, dB, dXc, m8, solvers::Method::BiCGStab, solvers::Formulation::fused, 1e-10,
                                 solvers::Mode::converge(500));
        dXs.download(Xs);
        dXc.download(Xc);
        bool same_hist = rs.residual_history.size() == rc.residual_history.size();
        for (std::size_t i = 0; same_hist && i < rs.residual_history.size(); ++i)
            same_hist = rs.residual_history[i].values == rc.residual_history[i].values;
        if (rs.iterations != rc.iterations || Xs.data != Xc.data || !same_hist) {
            std::puts("stencil twin solve differs from the CSR solve");
            return 1;
        }
    }
    // API misuse throws std::invalid_argument like the reference
    try {
        core::spmv(A, x, x);
        std::puts("aliasing not rejected");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    std::printf("cpp api ok: %d iterations, max |Ax-b| = %.3g\n", rep.iterations, worst);
    return 0;
}
