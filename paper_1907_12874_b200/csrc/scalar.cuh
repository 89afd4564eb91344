// scalar.cuh -- per-column scalar recurrences of the three BiCGStab variants
// (ColumnScalars arithmetic, types.hpp:39-83, on the device), convergence,
// breakdown and iteration control, run as a one-block kernel after each
// reduction point (inside the iteration's CUDA graph).
#pragma once

#include <climits>

#include "exact.cuh"

namespace mbg {

// ---- scalar bank / control words ------------------------------------------
enum Scal : int {
    S_ONE, S_MONE, S_BB, S_EPS2, S_RHO, S_ALPHA, S_NALPHA, S_OMEGA, S_NOMEGA,
    S_BETA, S_NBO, S_OA, S_RES2,
    // Improved BiCGStab (Alg. 3) recurrences and group-1 coefficients
    S_PHI, S_PI, S_SIGMA, S_SIGMAP, S_TAU, S_CZ2, S_CZ3, S_NDELTA,
    // synthetic preconditioner scale factors (constant rows)
    S_TWO, S_HALF, NSCAL
};
enum Ctl : int {
    C_STOP, C_CONV, C_ITER, C_ITERS, C_BD, C_BDITER, C_BDCOL, C_CONVERGED, NCTL = 16
};
enum Point : int {
    P_SETUP, P_C_ALPHA, P_C_OMEGA, P_C_BETA, P_R_OMEGA, P_R_END, P_P_OMEGA, P_P_BETA,
    P_I_START, P_I_OMEGA
};

struct ScalArgs {
    int m, point, method, fixed, maxit;
    double tol2;
    double* sc;          // NSCAL * m
    int* ctl;
    double* hist;        // (maxit+1) * m
    int64_t* D[8];       // long accumulators: rounded here (after any cross-GPU allreduce), then cleared
    int nd;
};

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

__device__ __forceinline__ double hist_entry(double res2, double bb) {
    const double r = res2 > 0.0 ? res2 : 0.0;
    return __dsqrt_rn(__ddiv_rn(r, bb));
}

// One block, thread c <-> column c (blockDim >= m).  Expressions follow
// oracle.c operation by operation (separately rounded, no contraction).
// s_dots: shared scratch of nd * m doubles.
static __device__ __forceinline__ void scalar_block(const ScalArgs& a, double* s_dots) {
    __shared__ int s_bad1, s_bad2, s_all;
    int* ctl = a.ctl;
    const int m = a.m;
    const int c = threadIdx.x;
    const bool on = c < m;
    // issue every independent load up front (control words, this column's
    // scalar bank, the slots): one memory round trip instead of three
    const int stop = ctl[C_STOP];
    const int conv_flag = ctl[C_CONV];
    const int j = ctl[C_ITER];
    double* sc = a.sc;
    double scv[NSCAL];
#pragma unroll
    for (int i = 0; i < NSCAL; ++i) scv[i] = on ? sc[i * m + c] : 0.0;
    if (stop) return;
    if (c == 0) { s_bad1 = INT_MAX; s_bad2 = INT_MAX; s_all = 1; }
    // round every (dot, column) long accumulator (one warp each), then clear
    // the (contiguous) slots for their next use
    const int nslot = a.nd * m;
    for (int i = threadIdx.x >> 5; i < nslot; i += blockDim.x >> 5) {
        const double r = warp_round_slot(a.D[i / m] + static_cast<int64_t>(i % m) * NSLOT);
        if ((threadIdx.x & 31) == 0) s_dots[i] = r;
    }
    __syncthreads();
    if (nslot) {
        int64_t* base = a.D[0];
        for (int w = threadIdx.x; w < nslot * NSLOT; w += blockDim.x) base[w] = 0;
    }
#define SCW(i, v) do { const double _v = (v); scv[i] = _v; sc[(i) * m + c] = _v; } while (0)
    double d[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (on)
        for (int i = 0; i < a.nd; ++i) d[i] = s_dots[i * m + c];
    int code1 = 0, code2 = 0;  // breakdown codes for s_bad1 / s_bad2
    switch (a.point) {
        case P_SETUP: {
            // d0 = (r0,r0), d1 = (b,b), d2 = (r0,w) for Pipelined
            if (on) {
                SCW(S_ONE, 1.0); SCW(S_MONE, -1.0);
                SCW(S_RHO, d[0]); SCW(S_BB, d[1]);
                SCW(S_EPS2, __dmul_rn(a.tol2, d[1]));
                a.hist[c] = hist_entry(d[0], d[1]);
                if (!(d[0] < scv[S_EPS2])) s_all = 0;
            }
            __syncthreads();
            if (!a.fixed && s_all) {
                if (c == 0) { ctl[C_STOP] = 1; ctl[C_CONVERGED] = 1; ctl[C_ITERS] = 0; }
                return;
            }
            if (a.method == MBG_IBICGSTAB && on) {
                // Alg. 3 line 2: sigma_-1 = pi_0 = tau_0 = 0, sigma_0 = (r0,u0),
                // rho_0 = alpha_0 = omega_0 = 1, phi_0 = (r0,r0)
                SCW(S_PHI, d[0]); SCW(S_SIGMA, d[2]); SCW(S_SIGMAP, 0.0); SCW(S_PI, 0.0); SCW(S_TAU, 0.0);
                SCW(S_RHO, 1.0); SCW(S_ALPHA, 1.0); SCW(S_OMEGA, 1.0);
            }
            if ((a.method == MBG_PIPEBICGSTAB || a.method == MBG_PPIPEBICGSTAB) && on) {
                const double alpha = __ddiv_rn(d[0], d[2]);
                SCW(S_ALPHA, alpha); SCW(S_NALPHA, -alpha);
                SCW(S_BETA, 0.0); SCW(S_OMEGA, 0.0);
                SCW(S_NBO, -__dmul_rn(0.0, 0.0));
                if (d[2] == 0.0 || !finite_d(alpha)) atomicMin(&s_bad1, c);
            }
            code1 = 1;
            break;
        }
        case P_C_ALPHA: {
            if (on) {
                const double alpha = __ddiv_rn(scv[S_RHO], d[0]);
                SCW(S_ALPHA, alpha); SCW(S_NALPHA, -alpha);
                if (d[0] == 0.0 || !finite_d(alpha)) atomicMin(&s_bad1, c);
            }
            code1 = 1;
            break;
        }
        case P_C_OMEGA:    // d = phi psi theta
        case P_R_OMEGA:    // d = theta phi psi eta
        case P_P_OMEGA: {  // d = theta phi pi
            double num, den, sq;
            if (a.point == P_C_OMEGA) { num = d[0]; den = d[1]; sq = d[2]; }
            else if (a.point == P_R_OMEGA) { num = d[0]; den = d[1]; sq = d[3]; }
            else { num = d[0]; den = d[1]; sq = d[2]; }
            double omega = 0.0, res2 = 0.0;
            if (on) {
                // lucky exact convergence (den == 0 because the residual is exactly 0): omega = 0
                const bool lucky = den == 0.0 && sq == 0.0;
                omega = lucky ? 0.0 : __ddiv_rn(num, den);
                SCW(S_OMEGA, omega); SCW(S_NOMEGA, -omega);
                if (a.point == P_P_OMEGA) SCW(S_OA, __dmul_rn(omega, scv[S_ALPHA]));
                res2 = __dsub_rn(sq, __dmul_rn(omega, num));
                SCW(S_RES2, res2);
                if ((den == 0.0 && !lucky) || !finite_d(omega)) atomicMin(&s_bad2, c);
            }
            __syncthreads();
            if (s_bad2 != INT_MAX) { code2 = 2; break; }
            if (on) {
                a.hist[static_cast<int64_t>(j + 1) * m + c] = hist_entry(res2, scv[S_BB]);
                if (!(res2 < scv[S_EPS2])) s_all = 0;
            }
            __syncthreads();
            const bool conv = !a.fixed && s_all;
            if (c == 0 && conv) ctl[C_CONV] = 1;
            if (a.point == P_R_OMEGA && !conv && on) {
                // rho' = -(omega*psi), beta = (rho'/rho)*(alpha/omega)
                const double rhon = -__dmul_rn(omega, d[2]);
                const double beta = __dmul_rn(__ddiv_rn(rhon, scv[S_RHO]), __ddiv_rn(scv[S_ALPHA], omega));
                SCW(S_BETA, beta); SCW(S_NBO, -__dmul_rn(beta, omega)); SCW(S_RHO, rhon);
                if (!finite_d(beta)) atomicMin(&s_bad1, c);
            }
            code1 = 3;
            break;
        }
        case P_I_START: {
            // Alg. 3 lines 4-7 (expression trees pinned in oracle.c)
            if (on) {
                const double om = scv[S_OMEGA], al = scv[S_ALPHA], pi = scv[S_PI];
                const double rhon = __dadd_rn(__dsub_rn(scv[S_PHI], __dmul_rn(om, scv[S_SIGMAP])),
                                              __dmul_rn(__dmul_rn(om, al), pi));
                const double delta = __dmul_rn(__ddiv_rn(rhon, scv[S_RHO]), al);
                const double beta = __ddiv_rn(delta, om);
                const double tau = __dsub_rn(__dadd_rn(scv[S_SIGMA], __dmul_rn(beta, scv[S_TAU])),
                                             __dmul_rn(delta, pi));
                const double an = __ddiv_rn(rhon, tau);
                if (!finite_d(beta)) atomicMin(&s_bad2, c);
                if (tau == 0.0 || !finite_d(an)) atomicMin(&s_bad1, c);
                SCW(S_CZ2, __dmul_rn(beta, __ddiv_rn(an, al)));
                SCW(S_CZ3, -__dmul_rn(an, delta));
                SCW(S_NDELTA, -delta);
                SCW(S_BETA, beta);
                SCW(S_ALPHA, an); SCW(S_NALPHA, -an);
                SCW(S_RHO, rhon); SCW(S_TAU, tau);
            }
            __syncthreads();
            if (s_bad2 != INT_MAX) { code2 = 3; break; }
            code1 = 1;
            break;
        }
        case P_I_OMEGA: {  // d = phi pi gamma eta theta kappa nu   (Alg. 3 lines 10-12)
            double omega = 0.0, res2 = 0.0;
            if (on) {
                const double theta = d[4], kappa = d[5], nu = d[6];
                const bool lucky = kappa == 0.0 && nu == 0.0;
                omega = lucky ? 0.0 : __ddiv_rn(theta, kappa);
                SCW(S_OMEGA, omega); SCW(S_NOMEGA, -omega);
                res2 = __dsub_rn(nu, __dmul_rn(omega, theta));
                SCW(S_RES2, res2);
                if ((kappa == 0.0 && !lucky) || !finite_d(omega)) atomicMin(&s_bad2, c);
            }
            __syncthreads();
            if (s_bad2 != INT_MAX) { code2 = 2; break; }
            if (on) {
                SCW(S_SIGMAP, scv[S_SIGMA]);
                SCW(S_SIGMA, __dsub_rn(d[2], __dmul_rn(omega, d[3])));
                SCW(S_PHI, d[0]); SCW(S_PI, d[1]);
                a.hist[static_cast<int64_t>(j + 1) * m + c] = hist_entry(res2, scv[S_BB]);
                if (!(res2 < scv[S_EPS2])) s_all = 0;
            }
            __syncthreads();
            if (c == 0 && !a.fixed && s_all) ctl[C_CONV] = 1;
            break;
        }
        case P_C_BETA: {
            if (conv_flag) {
                if (c == 0) { ctl[C_STOP] = 1; ctl[C_CONVERGED] = 1; ctl[C_ITERS] = j + 1; }
                return;
            }
            if (on) {
                const double rhon = d[0];
                const double beta = __dmul_rn(__ddiv_rn(rhon, scv[S_RHO]), __ddiv_rn(scv[S_ALPHA], scv[S_OMEGA]));
                SCW(S_BETA, beta); SCW(S_NBO, -__dmul_rn(beta, scv[S_OMEGA])); SCW(S_RHO, rhon);
                if (!finite_d(beta)) atomicMin(&s_bad1, c);
            }
            code1 = 3;
            break;
        }
        case P_R_END: {
            if (c == 0) {
                if (conv_flag) { ctl[C_STOP] = 1; ctl[C_CONVERGED] = 1; ctl[C_ITERS] = j + 1; }
            }
            break;
        }
        case P_P_BETA: {
            if (conv_flag) {
                if (c == 0) { ctl[C_STOP] = 1; ctl[C_CONVERGED] = 1; ctl[C_ITERS] = j + 1; }
                return;
            }
            if (on) {
                // d = rho' psi sigma delta
                const double omega = scv[S_OMEGA], alpha = scv[S_ALPHA];
                const double beta = __dmul_rn(__ddiv_rn(alpha, omega), __ddiv_rn(d[0], scv[S_RHO]));
                const double den = __dsub_rn(__dadd_rn(d[2], __dmul_rn(beta, d[3])),
                                             __dmul_rn(__dmul_rn(beta, omega), d[1]));
                const double an = __ddiv_rn(d[0], den);
                SCW(S_BETA, beta); SCW(S_ALPHA, an); SCW(S_RHO, d[0]);
                SCW(S_NBO, -__dmul_rn(beta, omega)); SCW(S_NALPHA, -an);
                if (!finite_d(beta)) atomicMin(&s_bad2, c);
                if (den == 0.0 || !finite_d(an)) atomicMin(&s_bad1, c);
            }
            __syncthreads();
            if (s_bad2 != INT_MAX) { code2 = 3; break; }
            code1 = 1;
            break;
        }
    }
#undef SCW
    __syncthreads();
    if (c != 0) return;
    // breakdown bookkeeping (first column)
    if (code2 && s_bad2 != INT_MAX) {
        ctl[C_BD] = code2; ctl[C_BDITER] = j; ctl[C_BDCOL] = s_bad2; ctl[C_ITERS] = j; ctl[C_STOP] = 1;
        return;
    }
    if (code1 && s_bad1 != INT_MAX) {
        // Pipelined's alpha_{j+1} belongs to the next iteration (oracle.c)
        const int it = (a.point == P_P_BETA) ? j + 1 : j;
        ctl[C_BD] = code1; ctl[C_BDITER] = it; ctl[C_BDCOL] = s_bad1; ctl[C_ITERS] = it; ctl[C_STOP] = 1;
        return;
    }
    // end of iteration
    if (a.point == P_C_BETA || a.point == P_R_END || a.point == P_P_BETA) {
        ctl[C_ITER] = j + 1;
        ctl[C_ITERS] = j + 1;
        if (j + 1 >= a.maxit) ctl[C_STOP] = 1;
    }
    if (a.point == P_SETUP && a.maxit <= 0) ctl[C_STOP] = 1;
}


}  // namespace mbg
