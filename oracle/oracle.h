/*
 * oracle.h -- CPU restatement of the reference's multi-RHS BiCGStab hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1907_12874_b200/)
 * links, imports or executes this code.  It is used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker.
 *
 * What it restates (paths relative to /root/reference):
 *   - CSR SpMV over an interleaved n x m block:  proj/src/core/spmv.cpp:27-74
 *   - stencil generator gen_poisson_7pt:         proj/src/core/generators.cpp:37-67
 *   - fused update statements (acc from 0.0, terms in order):
 *                                                proj/src/kernels/execute.cpp:97-119
 *   - the solvers (missing from the reference, CMakeLists.txt:25,28,29) from
 *     the paper listings: Alg. 2, Alg. 6
 *     (identity M^-1), Alg. 4, with the per-iteration
 *     schedules and term expansions of SURVEY.md Appendix C and the solve()
 *     contract of SPEC.md:227-235,262-268.
 *
 * One deliberate change: dot products are EXACT
 * (correctly rounded sum of the IEEE-rounded products), not the reference's
 * thread-blocked naive sum (execute.cpp:141-157), so the result does not
 * depend on thread count, GPU count or summation order.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction, as the
 * reference's default -O3 build without -march).
 */
#ifndef MBSTAB_ORACLE_H
#define MBSTAB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t n;        /* rows (square) */
    int64_t nnz;
    int64_t* off;     /* n+1 */
    int32_t* col;     /* nnz, strictly increasing per row */
    double* val;      /* nnz */
} orc_csr;

/* ---- counter-based RNG (pinned in DESIGN.md "Inputs") ---------------- */
uint64_t orc_hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b);
double orc_u01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b);   /* [0,1)  */
double orc_u11(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b);   /* [-1,1) */

/* ---- generators ----------------------------------------------------------
 * kind 0: 7-pt Poisson (diag 6, off -1)            generators.cpp:37-67
 * kind 1: 7-pt convection-diffusion (west -1.3, east -0.7, y/z -1, diag 6)
 * kind 2: 27-pt (diag 26, off -1 + 0.1*u11(seed, matrix stream, row, col))
 * Returns 0 on success. */
/* kind 0 Poisson 7-pt, 1 conv-diff 7-pt, 2 27-pt perturbed, 3 Poisson 5-pt (nz = 1) */
int orc_gen_stencil(int kind, int nx, int ny, int nz, uint64_t seed, orc_csr* out);
/* random banded: n rows, per-row count U{kmin..kmax} incl. diagonal, columns
 * uniform in [i-band, i+band] clipped, off-diag -u01, diag 1.1*sum|off| */
int orc_gen_banded(int64_t n, int64_t band, int kmin, int kmax, uint64_t seed, orc_csr* out);
void orc_csr_free(orc_csr* a);
/* B(i,c) = u11(seed, rhs stream, i, c), interleaved n x m */
void orc_rhs(int64_t n, int m, uint64_t seed, double* b);

/* ---- kernels ------------------------------------------------------------ */
void orc_spmv(const orc_csr* a, int m, const double* x, double* y);
/* y = A^T x: y = 0, then rows i ascending, y(col[k],c) += val[k]*x(i,c)
 * (spmv_transpose, spmv.cpp:76-90) */
void orc_spmv_transpose(const orc_csr* a, int m, const double* x, double* y);
/* out[e] = ((0 + c[0][e%m]*src[0][e]) + c[1][e%m]*src[1][e]) + ... */
void orc_update(int64_t n, int m, int nterms, const double* const* coeff,
                const double* const* src, double* out);
/* exact per-column dot: out[c] = RN( sum_i RN(a(i,c)*b(i,c)) ) */
void orc_dot_exact(int64_t n, int m, const double* a, const double* b, double* out);
/* exact sum of a list of doubles (test hook for the accumulator) */
double orc_sum_exact(int64_t n, const double* v);

/* ---- solver ------------------------------------------------------------- */
enum { ORC_BICGSTAB = 0, ORC_RBICGSTAB = 1, ORC_PIPEBICGSTAB = 2,
       ORC_IBICGSTAB = 3, ORC_PBICGSTAB = 4, ORC_PPIPEBICGSTAB = 5 };
enum { ORC_MERGED = 0, ORC_BASIC = 1 };

typedef struct {
    int iterations;
    int converged;        /* all columns passed the merged test */
    int breakdown;        /* 0 none, else code (1 alpha/delta, 2 omega, 3 beta) */
    int breakdown_iter;
    int breakdown_col;
} orc_report;

/* X: in = x0, out = solution.  hist: (maxit+1)*m doubles, row j = h_j.
 * fixed != 0: run exactly maxit iterations ignoring convergence. */
int orc_solve(const orc_csr* a, int m, const double* b, double* x, int method,
              int formulation, double tol, int fixed, int maxit, double* hist,
              orc_report* rep);
/* Same with an explicit preconditioner: precond_alpha 0 =
 * none (BiCGStab, IBiCGStab, PipeBiCGStab), 2 = identity (one copy), even
 * alpha >= 4 = synthetic(alpha): alpha/2 scale passes by 2.0 / 0.5 whose
 * product is exactly 1.  orc_solve uses 2 for the preconditioned methods. */
int orc_solve_pc(const orc_csr* a, int m, const double* b, double* x, int method,
                 int formulation, int precond_alpha, double tol, int fixed, int maxit,
                 double* hist, orc_report* rep);
int orc_method_preconditioned(int method);

int orc_num_threads(void);
double orc_triad_gbs(long n, int reps);

#ifdef __cplusplus
}
#endif
#endif
