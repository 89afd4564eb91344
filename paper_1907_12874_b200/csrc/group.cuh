// group.cuh -- single-pass fused vector-update + exact-dot kernels.
//
// B200 replacement of kernels::execute_group (execute.cpp:123-172): one pass
// over the n x m interleaved elements, every statement of a merged line
// evaluated per element in order with produced values kept in registers
// (the reference's register-reuse rule, statement.hpp:34-38), and all dots of
// the line accumulated exactly in the same pass.
//
// Layout: element e = i*m + c.  The grid is persistent (SM count x resident
// blocks) and walks the elements with a stride that is a multiple of m, so a
// thread always sees the same column c: its coefficients are loaded once and
// its dot accumulators are per-column by construction.  Loads and stores are
// fully coalesced 8-byte accesses (a warp touches 256 contiguous bytes).
//
// Arithmetic: each update is acc = 0.0; acc = acc + coef*v ... in statement
// term order with separately rounded multiply and add (__dmul_rn/__dadd_rn),
// exactly as execute.cpp:104-110 compiled without contraction.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "exact.cuh"
#include "scalar.cuh"

namespace mbg {

constexpr int GMAX_IN = 10, GMAX_OUT = 6, GMAX_CO = 8, GMAX_DOT = 8;

struct GroupArgs {
    int64_t len;                 // n*m
    int m;
    const double* in[GMAX_IN];
    double* out[GMAX_OUT];
    const double* coef[GMAX_CO]; // device arrays of m doubles
    int64_t* slot[GMAX_DOT];     // long accumulators: m * NSLOT words each
    const int* ctl;              // ctl[0] != 0: solve stopped -> no-op
    // 1: every thread walks its trips from the last one down, so the pass sweeps
    // the vectors from their end -- where the pass before it (walking up) left the
    // L2 warm.  Same elements per thread, exact dots: same bits either way.
    int reverse;
};

__device__ __forceinline__ double fmadd_rn(double acc, double c, double v) {
    return __dadd_rn(acc, __dmul_rn(c, v));
}

// ---------------------------------------------------------------------------
// Programs: one struct per merged line of SURVEY.md Appendix C (and the
// singleton statements of the basic formulation).  in/out/co index the
// GroupArgs arrays; prod[] are the dot-product terms of this element.
// ---------------------------------------------------------------------------

// Dot (a, b)                                   e.g. delta = (v, r0)
struct PDot2 {
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 4, MINB = 2;   // 4 packets in flight per trip (C2: dot2 61.6 -> 57.8 us, upd2_sq 71.2 -> 64.2)
    static constexpr const char* NAME = "dot2";
    static constexpr int NIN = 2, NOUT = 0, NCO = 0, NDOT = 1;
    __device__ static void run(const double* in, double*, double* prod, const double*) {
        prod[0] = __dmul_rn(in[0], in[1]);
    }
};
// Dot (a, a)                                   e.g. psi = (t, t)
struct PDot1 {
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 4, MINB = 2;   // 4 packets in flight per trip (C2: dot1 43.1 -> 38.0 us)
    static constexpr const char* NAME = "dot1";
    static constexpr int NIN = 1, NOUT = 0, NCO = 0, NDOT = 1;
    __device__ static void run(const double* in, double*, double* prod, const double*) {
        prod[0] = __dmul_rn(in[0], in[0]);
    }
};
// out = c0*a
struct PUpd1 {
    static constexpr const char* NAME = "upd1";
    static constexpr int NIN = 1, NOUT = 1, NCO = 1, NDOT = 0;
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(0.0, co[0], in[0]);
    }
};
// out = c0*a + c1*b
struct PUpd2 {
    static constexpr const char* NAME = "upd2";
    static constexpr int NIN = 2, NOUT = 1, NCO = 2, NDOT = 0;
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(0.0, co[0], in[0]), co[1], in[1]);
    }
};
// out = c0*a + c1*b + c2*d
struct PUpd3 {
    static constexpr const char* NAME = "upd3";
    static constexpr int NIN = 3, NOUT = 1, NCO = 3, NDOT = 0;
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, co[0], in[0]), co[1], in[1]), co[2], in[2]);
    }
};

// Classical, fused formulation: Alg. 2 line 8 with theta = (s,s) computed where
// s is produced (it is reduced at the same point as phi and psi, so the
// message layout and the traffic are unchanged; the fp64 work of the dots is
// spread over two memory-bound passes instead of one compute-bound one).
//   s = 1*r + (-alpha)*v ; theta = (s, s)
struct PUpd2Sq {
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 4, MINB = 2;   // 4 packets in flight per trip (C2: dot2 61.6 -> 57.8 us, upd2_sq 71.2 -> 64.2)
    static constexpr const char* NAME = "upd2_sq";
    static constexpr int NIN = 2, NOUT = 1, NCO = 2, NDOT = 1;
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double s = fmadd_rn(fmadd_rn(0.0, co[0], in[0]), co[1], in[1]);
        out[0] = s;
        prod[0] = __dmul_rn(s, s);
    }
};
// ... and phi = (t,s), psi = (t,t) in the pass after t = A s
struct PClassicPhiPsi {
    static constexpr bool REDO_SAFE = true;
    static constexpr bool FAST_SUM = true;   // FastTwoSum grows: -6 % (tools/ncu_ab.sh, C2)
    static constexpr const char* NAME = "classic_phipsi";
    static constexpr int NIN = 2, NOUT = 0, NCO = 0, NDOT = 2;   // in: t s
    __device__ static void run(const double* in, double*, double* prod, const double*) {
        prod[0] = __dmul_rn(in[0], in[1]);
        prod[1] = __dmul_rn(in[0], in[0]);
    }
};

// Classical, Alg. 2 line 9: phi=(t,s), psi=(t,t), theta=(s,s)
struct PClassicOmega {
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 1;  // register budget: 3+ dot expansions per column pair
    static constexpr const char* NAME = "classic_omega";
    static constexpr int NIN = 2, NOUT = 0, NCO = 0, NDOT = 3;   // in: t s
    __device__ static void run(const double* in, double*, double* prod, const double*) {
        prod[0] = __dmul_rn(in[0], in[1]);
        prod[1] = __dmul_rn(in[0], in[0]);
        prod[2] = __dmul_rn(in[1], in[1]);
    }
};
// Classical, Alg. 2 line 15:
//   x = 1*x + alpha*p + omega*s ; r = 1*s + (-omega)*t ; rho' = (r, r0)
struct PClassicXR {
    static constexpr bool REDO_SAFE = true;
    static constexpr const char* NAME = "classic_xr";
    static constexpr int NIN = 5, NOUT = 2, NCO = 3, NDOT = 1;   // in: x p s t r0; co: alpha omega -omega
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        const double r = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]);
        out[1] = r;
        prod[0] = __dmul_rn(r, in[4]);
    }
};

// Reordered, Alg. 6 line 11:
//   rt = 1*r + (-alpha)*v ; theta=(t,rt), phi=(t,t), psi=(t,r0), eta=(rt,rt)
struct PReordG7 {
    static constexpr bool REDO_SAFE = true;
    static constexpr bool PREFETCH = true;   // 4 dots: overlap the next packet's loads with the TwoSum chains
    static constexpr int MINB = 2;           // ... with the registers that takes
    static constexpr int UNROLL = 1;  // register budget: 3+ dot expansions per column pair
    static constexpr const char* NAME = "reord_g7";
    static constexpr int NIN = 4, NOUT = 1, NCO = 1, NDOT = 4;   // in: r v t r0; co: -alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double rt = fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]);
        out[0] = rt;
        prod[0] = __dmul_rn(in[2], rt);
        prod[1] = __dmul_rn(in[2], in[2]);
        prod[2] = __dmul_rn(in[2], in[3]);
        prod[3] = __dmul_rn(rt, rt);
    }
};
// ... fused formulation: the same four dots with rt kept in registers only
// (rt is recomputed where r = rt - omega t is formed), one vector write less
struct PReordG7D {
    static constexpr bool REDO_SAFE = true;
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr int UNROLL = 1;
    static constexpr const char* NAME = "reord_g7d";
    static constexpr int NIN = 4, NOUT = 0, NCO = 1, NDOT = 4;   // in: r v t r0; co: -alpha
    __device__ static void run(const double* in, double*, double* prod, const double* co) {
        const double rt = fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]);
        prod[0] = __dmul_rn(in[2], rt);
        prod[1] = __dmul_rn(in[2], in[2]);
        prod[2] = __dmul_rn(in[2], in[3]);
        prod[3] = __dmul_rn(rt, rt);
    }
};
// Reordered, Alg. 6 lines 20-22 (footnote-5 form):
//   x = 1*x + alpha*vh + omega*th ; z = 1*th + (-omega)*q ;
//   vh = 1*z + beta*vh + (-(beta*omega))*s
struct PReordG12 {
    static constexpr const char* NAME = "reord_g12";
    static constexpr int NIN = 5, NOUT = 3, NCO = 5, NDOT = 0;   // in: x vh th q s; co: alpha omega -omega beta -(beta*omega)
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        const double z = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]);
        out[1] = z;
        out[2] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, z), co[3], in[1]), co[4], in[4]);
    }
};

// Reordered, fused formulation with identity M^-1 (q = t, s = v elided): Alg. 6
// line 17's r = 1*rt + (-omega)*t merged into the lines 20-22 pass, which reads
// t (as q) and v (as s) anyway, with rt = 1*r + (-alpha)*v recomputed from r
// (the 4-dot pass keeps it in registers) -- same expressions, same bits
//   x = 1*x + alpha*vh + omega*th ; z = 1*th + (-omega)*q ;
//   vh = 1*z + beta*vh + (-(beta*omega))*s ; r = 1*(1*r + (-alpha)*s) + (-omega)*q
struct PReordG12R {
    static constexpr const char* NAME = "reord_g12r";
    // in: x vh th q s r; co: alpha omega -omega beta -(beta*omega) -alpha
    // (rt = 1*r + (-alpha)*s recomputed as in the dot pass: s = v here)
    static constexpr int NIN = 6, NOUT = 4, NCO = 6, NDOT = 0;
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        const double z = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]);
        out[1] = z;
        out[2] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, z), co[3], in[1]), co[4], in[4]);
        const double rt = fmadd_rn(fmadd_rn(0.0, 1.0, in[5]), co[5], in[4]);
        out[3] = fmadd_rn(fmadd_rn(0.0, 1.0, rt), co[2], in[3]);
    }
};

// ... and with th never stored (formed inside the second SpMM, stencil.cu):
// th = 1*z + (-alpha)*s recomputed here with the expression of its update pass
//   in: x vh z q s r ; out: x z vh r ; co: alpha omega -omega beta -(beta*omega) -alpha
struct PReordG12RZ {
    static constexpr const char* NAME = "reord_g12rz";
    static constexpr int NIN = 6, NOUT = 4, NCO = 6, NDOT = 0;   // in: x vh z q s r
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        const double th = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[5], in[4]);
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], th);
        const double z = fmadd_rn(fmadd_rn(0.0, 1.0, th), co[2], in[3]);
        out[1] = z;
        out[2] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, z), co[3], in[1]), co[4], in[4]);
        const double rt = fmadd_rn(fmadd_rn(0.0, 1.0, in[5]), co[5], in[4]);
        out[3] = fmadd_rn(fmadd_rn(0.0, 1.0, rt), co[2], in[3]);
    }
};

// Pipelined, Alg. 4 line 4:
//   p = 1*r + beta*p + nbo*s ; s = 1*w + beta*s + nbo*z ; z = 1*t + beta*z + nbo*v ;
//   q = 1*r + (-alpha)*s ; y = 1*w + (-alpha)*z ; theta=(q,y), phi=(y,y), pi=(q,q)
struct PPipeG1 {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr int UNROLL = 1;  // register budget: 3+ dot expansions per column pair
    static constexpr const char* NAME = "pipe_g1";
    static constexpr int NIN = 7, NOUT = 5, NCO = 3, NDOT = 3;   // in: r p s w z t v; out: p s z q y; co: beta nbo -alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double r = in[0], p = in[1], s = in[2], w = in[3], z = in[4], t = in[5], v = in[6];
        const double pn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, r), co[0], p), co[1], s);
        const double sn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, w), co[0], s), co[1], z);
        const double zn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, t), co[0], z), co[1], v);
        const double q = fmadd_rn(fmadd_rn(0.0, 1.0, r), co[2], sn);
        const double y = fmadd_rn(fmadd_rn(0.0, 1.0, w), co[2], zn);
        out[0] = pn; out[1] = sn; out[2] = zn; out[3] = q; out[4] = y;
        prod[0] = __dmul_rn(q, y);
        prod[1] = __dmul_rn(y, y);
        prod[2] = __dmul_rn(q, q);
    }
};
// Pipelined, Alg. 4 line 7: x = 1*x + alpha*p + omega*q ; r = 1*q + (-omega)*y
struct PPipeG4 {
    static constexpr const char* NAME = "pipe_g4";
    static constexpr int NIN = 4, NOUT = 2, NCO = 3, NDOT = 0;   // in: x p q y; co: alpha omega -omega
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        out[1] = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]);
    }
};
// Pipelined, Alg. 4 line 12:
//   w = 1*y + (-omega)*t + (omega*alpha)*v ; rho'=(r0,r), psi=(r0,z), sigma=(r0,w), delta=(r0,s)
struct PPipeG5 {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 1;  // register budget: 3+ dot expansions per column pair
    static constexpr const char* NAME = "pipe_g5";
    static constexpr int NIN = 7, NOUT = 1, NCO = 2, NDOT = 4;   // in: y t v r0 r z s; co: -omega omega*alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double w = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        out[0] = w;
        const double r0 = in[3];
        prod[0] = __dmul_rn(r0, in[4]);
        prod[1] = __dmul_rn(r0, in[5]);
        prod[2] = __dmul_rn(r0, w);
        prod[3] = __dmul_rn(r0, in[6]);
    }
};

// Pipelined, fused formulation: q = 1*r + (-alpha)*s and y = 1*w + (-alpha)*z
// live in registers only -- the line-4 pass forms them for its three dots and
// the line-7/12 pass recomputes them from r, w and the new s, z (which it
// reads anyway), with the same expressions, so the bits do not change and q, y
// are never stored (2 vector writes less per iteration, 2 vectors less memory)
//   in: r p s w z t v ; out: p s z ; co: beta nbo -alpha
struct PPipeG1F {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr int UNROLL = 1;
    static constexpr const char* NAME = "pipe_g1f";
    static constexpr int NIN = 7, NOUT = 3, NCO = 3, NDOT = 3;
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double r = in[0], p = in[1], s = in[2], w = in[3], z = in[4], t = in[5], v = in[6];
        const double pn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, r), co[0], p), co[1], s);
        const double sn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, w), co[0], s), co[1], z);
        const double zn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, t), co[0], z), co[1], v);
        const double q = fmadd_rn(fmadd_rn(0.0, 1.0, r), co[2], sn);
        const double y = fmadd_rn(fmadd_rn(0.0, 1.0, w), co[2], zn);
        out[0] = pn; out[1] = sn; out[2] = zn;
        prod[0] = __dmul_rn(q, y);
        prod[1] = __dmul_rn(y, y);
        prod[2] = __dmul_rn(q, q);
    }
};
//   in: x p r w t v r0 z s ; out: x r w ; co: alpha omega -omega omega*alpha -alpha
struct PPipeG45F {
    static constexpr bool REDO_SAFE = true;
    static constexpr bool NO_BATCH = true;
    static constexpr const char* NAME = "pipe_g45f";
    static constexpr int NIN = 9, NOUT = 3, NCO = 5, NDOT = 4, UNROLL = 1;
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double q = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[4], in[8]);
        const double y = fmadd_rn(fmadd_rn(0.0, 1.0, in[3]), co[4], in[7]);
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], q);
        const double r = fmadd_rn(fmadd_rn(0.0, 1.0, q), co[2], y);
        out[1] = r;
        const double w = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, y), co[2], in[4]), co[3], in[5]);
        out[2] = w;
        const double r0 = in[6];
        prod[0] = __dmul_rn(r0, r);
        prod[1] = __dmul_rn(r0, in[7]);
        prod[2] = __dmul_rn(r0, w);
        prod[3] = __dmul_rn(r0, in[8]);
    }
};

// Pipelined, fused formulation: Alg. 4 lines 7 and 12 in ONE pass (the
// convergence break between them only skips w, which the GPU may compute and
// discard): x = 1*x + alpha*p + omega*q ; r = 1*q + (-omega)*y ;
// w = 1*y + (-omega)*t + (omega*alpha)*v ; rho'=(r0,r), psi=(r0,z), sigma=(r0,w), delta=(r0,s)
struct PPipeG45 {
    static constexpr bool REDO_SAFE = true;
    static constexpr bool NO_BATCH = true;   // batched grows +2.6 % here (C4, locked clock)
    static constexpr const char* NAME = "pipe_g45";
    static constexpr int NIN = 9, NOUT = 3, NCO = 4, NDOT = 4, UNROLL = 1;
    // in: x p q y t v r0 z s ; out: x r w ; co: alpha omega -omega omega*alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        const double r = fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]);
        out[1] = r;
        const double w = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[3]), co[2], in[4]), co[3], in[5]);
        out[2] = w;
        const double r0 = in[6];
        prod[0] = __dmul_rn(r0, r);
        prod[1] = __dmul_rn(r0, in[7]);
        prod[2] = __dmul_rn(r0, w);
        prod[3] = __dmul_rn(r0, in[8]);
    }
};

// ---- the other three methods of the paper ----------
// Improved BiCGStab, Alg. 3 line 8:
//   z = alpha'*r + cz2*z + cz3*v ; v = 1*u + beta'*v + (-delta')*q ; s = 1*r + (-alpha')*v
struct PIbcgG1 {
    static constexpr const char* NAME = "ibcg_g1";
    static constexpr int NIN = 5, NOUT = 3, NCO = 6, NDOT = 0;
    // in: r z v u q ; out: z v s ; co: alpha' cz2 cz3 beta' -delta' -alpha'
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        const double r = in[0], z = in[1], v = in[2], u = in[3], q = in[4];
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, co[0], r), co[1], z), co[2], v);
        const double vn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, u), co[3], v), co[4], q);
        out[1] = vn;
        out[2] = fmadd_rn(fmadd_rn(0.0, 1.0, r), co[5], vn);
    }
};
// Alg. 3 line 10: t = 1*u + (-alpha)*q ;
//   phi=(r0,s) pi=(r0,q) gamma=(f0,s) eta=(f0,t) theta=(s,t) kappa=(t,t) nu=(s,s)
// Seven expansions per column: one column per thread (VEC = 1) keeps them in registers.
struct PIbcgG2 {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr bool REDO_SAFE = true;
    static constexpr const char* NAME = "ibcg_g2";
    static constexpr int NIN = 5, NOUT = 1, NCO = 1, NDOT = 7, UNROLL = 1, VEC = 1;
    // in: u q r0 s f0 ; out: t ; co: -alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double u = in[0], q = in[1], r0 = in[2], s = in[3], f0 = in[4];
        const double t = fmadd_rn(fmadd_rn(0.0, 1.0, u), co[0], q);
        out[0] = t;
        prod[0] = __dmul_rn(r0, s);
        prod[1] = __dmul_rn(r0, q);
        prod[2] = __dmul_rn(f0, s);
        prod[3] = __dmul_rn(f0, t);
        prod[4] = __dmul_rn(s, t);
        prod[5] = __dmul_rn(t, t);
        prod[6] = __dmul_rn(s, s);
    }
};
// Alg. 3 line 13: r = 1*s + (-omega)*t ; x = 1*x + 1*z + omega*s
struct PIbcgG3 {
    static constexpr const char* NAME = "ibcg_g3";
    static constexpr int NIN = 4, NOUT = 2, NCO = 2, NDOT = 0;   // in: s t x z ; out: r x ; co: -omega omega
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]);
        out[1] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), 1.0, in[3]), co[1], in[0]);
    }
};
// Preconditioned BiCGStab, Alg. 5: r = 1*s + (-omega)*t ; rho' = (r, r0)
struct PRDot {
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 4, MINB = 2;   // 4 packets in flight per trip (C2: pbcg_r 94.7 -> 86.6 us)
    static constexpr const char* NAME = "pbcg_r";
    static constexpr int NIN = 3, NOUT = 1, NCO = 1, NDOT = 1;   // in: s t r0 ; co: -omega
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double r = fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]);
        out[0] = r;
        prod[0] = __dmul_rn(r, in[2]);
    }
};
// Preconditioned Pipelined BiCGStab, Alg. 7 line 4:
//   ph = 1*rh + beta*ph + nbo*sh ; sh = 1*wh + beta*sh + nbo*zh ; qh = 1*rh + (-alpha)*sh
struct PPpG1 {
    static constexpr const char* NAME = "ppipe_g1";
    static constexpr int NIN = 5, NOUT = 3, NCO = 3, NDOT = 0;   // in: rh ph sh wh zh ; co: beta nbo -alpha
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        const double rh = in[0], ph = in[1], sh = in[2], wh = in[3], zh = in[4];
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, rh), co[0], ph), co[1], sh);
        const double shn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, wh), co[0], sh), co[1], zh);
        out[1] = shn;
        out[2] = fmadd_rn(fmadd_rn(0.0, 1.0, rh), co[2], shn);
    }
};
// Alg. 7 line 5: s, z, q, y as Alg. 4 line 4 (no p) ; theta=(q,y) phi=(y,y) pi=(q,q)
struct PPpG2 {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr int UNROLL = 1;
    static constexpr const char* NAME = "ppipe_g2";
    static constexpr int NIN = 6, NOUT = 4, NCO = 3, NDOT = 3;   // in: r s w z t v ; out: s z q y ; co: beta nbo -alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double r = in[0], s = in[1], w = in[2], z = in[3], t = in[4], v = in[5];
        const double sn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, w), co[0], s), co[1], z);
        const double zn = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, t), co[0], z), co[1], v);
        const double q = fmadd_rn(fmadd_rn(0.0, 1.0, r), co[2], sn);
        const double y = fmadd_rn(fmadd_rn(0.0, 1.0, w), co[2], zn);
        out[0] = sn; out[1] = zn; out[2] = q; out[3] = y;
        prod[0] = __dmul_rn(q, y);
        prod[1] = __dmul_rn(y, y);
        prod[2] = __dmul_rn(q, q);
    }
};
// Alg. 7 line 14: x = 1*x + alpha*ph + omega*qh ;
//   rh = 1*qh + (-omega)*wh + (omega*alpha)*zh
struct PPpG3 {
    static constexpr const char* NAME = "ppipe_g3";
    static constexpr int NIN = 5, NOUT = 2, NCO = 4, NDOT = 0;   // in: x ph qh wh zh ; co: alpha omega -omega omega*alpha
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[0]), co[0], in[1]), co[1], in[2]);
        out[1] = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, in[2]), co[2], in[3]), co[3], in[4]);
    }
};
// Alg. 7 line 15: r = 1*q + (-omega)*y ; w = 1*y + (-omega)*t + (omega*alpha)*v ;
//   rho'=(r0,r) psi=(r0,z) sigma=(r0,w) delta=(r0,s)
struct PPpG4 {
    static constexpr bool PREFETCH = true;
    static constexpr int MINB = 2;
    static constexpr bool REDO_SAFE = true;
    static constexpr int UNROLL = 1;
    static constexpr const char* NAME = "ppipe_g4";
    static constexpr int NIN = 7, NOUT = 2, NCO = 2, NDOT = 4;   // in: q y t v r0 z s ; out: r w ; co: -omega omega*alpha
    __device__ static void run(const double* in, double* out, double* prod, const double* co) {
        const double q = in[0], y = in[1], t = in[2], v = in[3], r0 = in[4];
        const double r = fmadd_rn(fmadd_rn(0.0, 1.0, q), co[0], y);
        const double w = fmadd_rn(fmadd_rn(fmadd_rn(0.0, 1.0, y), co[0], t), co[1], v);
        out[0] = r; out[1] = w;
        prod[0] = __dmul_rn(r0, r);
        prod[1] = __dmul_rn(r0, in[5]);
        prod[2] = __dmul_rn(r0, w);
        prod[3] = __dmul_rn(r0, in[6]);
    }
};

// Programs whose dot products can be recomputed from the pass's inputs after
// the pass (no input overwritten in place feeds a product): their streaming
// loop uses the optimistic grow_lazy and re-walks a thread's elements with the
// careful grow only if that thread met a non-finite value.
template <class P, class = void>
struct redo_safe_of { static constexpr bool value = false; };
template <class P>
struct redo_safe_of<P, decltype(void(P::REDO_SAFE))> { static constexpr bool value = P::REDO_SAFE; };

#ifndef MBG_GROW_BATCH
#define MBG_GROW_BATCH 1
#endif
// Batched lazy grows (exact.cuh grow_lazy_batch) unless a program opts out
// (NO_BATCH): measured at ncu's locked clock, Reordered 4-dot pass -11 %, dot2
// -5 %, phi/psi -3.5 %; the fused Pipelined 4-dot pass +2.6 % (and the careful
// grows of Alg. 4 line 4 spill when batched: +45 %), so those keep per-grow code.
template <class P, class = void>
struct batch_of { static constexpr bool value = true; };
template <class P>
struct batch_of<P, decltype(void(P::NO_BATCH))> { static constexpr bool value = !P::NO_BATCH; };

// FastTwoSum in the streaming grows (exact.cuh two_sum_lazy) where it measured faster.
template <class P, class = void>
struct fast_sum_of { static constexpr bool value = false; };
template <class P>
struct fast_sum_of<P, decltype(void(P::FAST_SUM))> { static constexpr bool value = P::FAST_SUM; };

// Widest packet a program may use (2 unless it declares VEC = 1).
template <class P, class = void>
struct vec_of { static constexpr int value = 2; };
template <class P>
struct vec_of<P, decltype(void(P::VEC))> { static constexpr int value = P::VEC; };

// Register-pipelined loads for dot-heavy programs (the dots' TwoSum chains
// would otherwise serialise with the memory latency): byte-light ones by
// default, multi-dot lines by declaring PREFETCH (+ MINB = 2 for the
// registers).  Measured on B200 (tools/sweep.py, C2/C3): Reordered -3..-5 %,
// Pipelined merged -3.6 %, IBiCGStab -10 %, PPipeBiCGStab -3.5 %; the classical
// x/r line and the fused Pipelined line lose (spills / occupancy) and keep
// the unrolled loads.
template <class P, class = void>
struct prefetch_of {
    static constexpr bool value = P::NDOT >= 1 && P::NIN + P::NOUT <= 3;
};
template <class P>
struct prefetch_of<P, decltype(void(P::PREFETCH))> { static constexpr bool value = P::PREFETCH; };

// Unroll (pairs of packets per trip) unless a program declares UNROLL = 1;
// pipelined programs get their memory parallelism from the prefetch instead.
template <class P, class = void>
struct unroll_of { static constexpr int value = prefetch_of<P>::value ? 1 : 2; };
template <class P>
struct unroll_of<P, decltype(void(P::UNROLL))> { static constexpr int value = P::UNROLL; };

// Resident blocks to budget registers for: pipelined programs are latency
// bound and need 4 blocks of 256 threads (<= 64 registers).
template <class P, class = void>
struct minblocks_of {
    // small pure updates: 3 blocks (<= 85 registers) -- with 2, ptxas spends
    // the budget on a deeper schedule and the 3-term update drops ~5% (B200,
    // C2); wider updates would spill under that cap
    static constexpr int value =
        prefetch_of<P>::value ? (P::NDOT >= 3 ? 3 : 4) : (P::NDOT == 0 && P::NIN + P::NOUT <= 5 ? 3 : 2);
};
template <class P>
struct minblocks_of<P, decltype(void(P::MINB))> { static constexpr int value = P::MINB; };

// ---------------------------------------------------------------------------
// Block-level exact combine.  Threads of a block fall into `classes` column
// classes (thread t is in class t % classes; the block size is classes * 2^q).
// Each thread holds NX expansions; expansion x of class k belongs to the
// long-accumulator slot slot_of(x, k).  The expansions of one class are
// merged exactly (warp shuffles, then a shared-memory tree) and the class
// leader deposits the K terms of each merged expansion into its slot with
// integer atomics -- so no partial buffer and no fold kernel are needed; the
// scalar kernel rounds the slot directly.
// ---------------------------------------------------------------------------
struct SyncBlock {
    __device__ void operator()() const { __syncthreads(); }
};
// nthreads < 0: the whole block; else the first nthreads threads (a power-of-two
// number of warps), synchronised by `sync` (e.g. a named barrier)
template <int NX, class SlotOf, class Sync = SyncBlock>
__device__ __forceinline__ void block_combine(double (&acc)[NX][KEXP], int classes, SlotOf slot_of,
                                              double* sh /* blockDim * KEXP doubles */, Sync sync = Sync(),
                                              int nthreads = -1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = nthreads < 0 ? static_cast<int>(blockDim.x) : nthreads;
    const int k = tid % classes;
#pragma unroll
    for (int x = 0; x < NX; ++x) {
        double (&mine)[KEXP] = acc[x];
        int64_t* slot = slot_of(x, k);
        if (classes <= 32 && (32 % classes) == 0 && (nthr & 31) == 0) {
            for (int off = 16; off >= classes; off >>= 1) {
                double t[KEXP];
#pragma unroll
                for (int i = 0; i < KEXP; ++i) t[i] = __shfl_down_sync(0xffffffffu, mine[i], off);
                if (lane < off) {
                    // the lower terms are almost always exactly zero: skip their grows
#pragma unroll
                    for (int i = 0; i < KEXP; ++i)
                        if (i == 0 || t[i] != 0.0) grow(mine, t[i], slot);
                }
            }
            const int nw = nthr >> 5;
            if (lane < classes) {
#pragma unroll
                for (int i = 0; i < KEXP; ++i) sh[(warp * 32 + lane) * KEXP + i] = mine[i];
            }
            sync();
            for (int s = nw >> 1; s >= 1; s >>= 1) {
                if (warp < s && lane < classes) {
#pragma unroll
                    for (int i = 0; i < KEXP; ++i) {
                        const double v = sh[((warp + s) * 32 + lane) * KEXP + i];
                        if (i == 0 || v != 0.0) grow(mine, v, slot);
                    }
#pragma unroll
                    for (int i = 0; i < KEXP; ++i) sh[(warp * 32 + lane) * KEXP + i] = mine[i];
                }
                sync();
            }
        } else {
#pragma unroll
            for (int i = 0; i < KEXP; ++i) sh[tid * KEXP + i] = mine[i];
            sync();
            for (int s = (nthr / classes) >> 1; s >= 1; s >>= 1) {
                if (tid < s * classes) {
#pragma unroll
                    for (int i = 0; i < KEXP; ++i) {
                        const double v = sh[(tid + s * classes) * KEXP + i];
                        if (i == 0 || v != 0.0) grow(mine, v, slot);
                    }
#pragma unroll
                    for (int i = 0; i < KEXP; ++i) sh[tid * KEXP + i] = mine[i];
                }
                sync();
            }
        }
        if (tid < classes) {
#pragma unroll
            for (int i = 0; i < KEXP; ++i) digits_add_atomic(slot, mine[i]);
        }
        sync();
    }
}

// ---------------------------------------------------------------------------
// The fused group kernel.  VEC = 2: each thread streams 16-byte pairs of
// elements (e, e+1) -- columns c0 = e % m and c0 + 1 (both 0 when m == 1) --
// and keeps one expansion per (dot, column of the pair).  Two pairs per trip
// are loaded before any store (in-place updates such as x = x + ... stay
// correct) for memory-level parallelism.  VEC = 1 covers odd m.
// ---------------------------------------------------------------------------
template <class P, int VEC>
__global__ void __launch_bounds__(256, minblocks_of<P>::value) group_kernel(GroupArgs a) {
    pdl_wait();
    if (a.ctl && a.ctl[0]) return;
    extern __shared__ double sh_dyn[];
    const int m = a.m;
    constexpr int NCO = P::NCO > 0 ? P::NCO : 1;
    constexpr int ND = P::NDOT > 0 ? P::NDOT : 1;
    constexpr int NO = P::NOUT > 0 ? P::NOUT : 1;
    // columns handled by this thread (fixed: the grid stride is a multiple of m)
    const int c0 = (threadIdx.x * VEC) % m;
    const int c1 = VEC == 2 ? (m == 1 ? 0 : c0 + 1) : c0;
    double co0[NCO], co1[NCO];
#pragma unroll
    for (int i = 0; i < P::NCO; ++i) {
        co0[i] = a.coef[i][c0];
        co1[i] = a.coef[i][c1];
    }
    double acc[ND * VEC][KEXP];
#pragma unroll
    for (int d = 0; d < ND * VEC; ++d)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) acc[d][i] = 0.0;
    int64_t* slot0[ND];
    int64_t* slot1[ND];
#pragma unroll
    for (int d = 0; d < P::NDOT; ++d) {
        slot0[d] = a.slot[d] + static_cast<int64_t>(c0) * NSLOT;
        slot1[d] = a.slot[d] + static_cast<int64_t>(c1) * NSLOT;
    }

    const int64_t npk = a.len / VEC;  // packets of VEC elements
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    constexpr int UNR = unroll_of<P>::value;
    using Pk = typename std::conditional<VEC == 2, double2, double>::type;
    // Software pipeline: the next trip's UNR packets are loaded before the
    // current trip's statements and dot expansions run, so the TwoSum chains
    // of the exact dots overlap the memory latency instead of adding to it.
    int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    Pk cur[UNR][P::NIN], nxt[UNR][P::NIN];
    auto load = [&](Pk (&dst)[UNR][P::NIN], int64_t q0) {
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q0 + u * stride < npk)
#pragma unroll
                for (int i = 0; i < P::NIN; ++i) dst[u][i] = reinterpret_cast<const Pk*>(a.in[i])[q0 + u * stride];
    };
    // (only kernels with dots pipeline: the plain updates are memory-bound
    // already and the extra registers would cost occupancy)
    constexpr bool PF = prefetch_of<P>::value;
    constexpr bool RS = redo_safe_of<P>::value && P::NDOT > 0;
    bool bad = false;
    // trips of this thread: T of UNR packets each, walked up or (a.reverse) down
    const int64_t q_first = q, step = UNR * stride;
    const int64_t T = q_first < npk ? (npk - q_first + step - 1) / step : 0;
    const int64_t dq = a.reverse ? -step : step;
    if (a.reverse) q = q_first + (T - 1) * step;
    if constexpr (PF) {
        if (T > 0) load(cur, q);
    }
    for (int64_t trip = 0; trip < T; ++trip, q += dq) {
        if constexpr (PF) {
            if (trip + 1 < T) load(nxt, q + dq);
        } else {
            load(cur, q);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int64_t qu = q + u * stride;
            if (qu >= npk) break;
            double in[P::NIN], o0[NO], p0[ND];
            if constexpr (VEC == 2) {
                double o1[NO], p1[ND];
#pragma unroll
                for (int i = 0; i < P::NIN; ++i) in[i] = cur[u][i].x;
                P::run(in, o0, p0, co0);
#pragma unroll
                for (int i = 0; i < P::NIN; ++i) in[i] = cur[u][i].y;
                P::run(in, o1, p1, co1);
#pragma unroll
                for (int i = 0; i < P::NOUT; ++i) reinterpret_cast<double2*>(a.out[i])[qu] = make_double2(o0[i], o1[i]);
#if MBG_GROW_BATCH
                if constexpr (RS && batch_of<P>::value) {
                    double px[2 * ND];
                    int64_t* sl[2 * ND];
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        px[2 * d] = p0[d];
                        px[2 * d + 1] = p1[d];
                        sl[2 * d] = slot0[d];
                        sl[2 * d + 1] = slot1[d];
                    }
                    grow_lazy_batch<2 * ND, false, fast_sum_of<P>::value>(acc, px, sl);
                } else
#endif
#pragma unroll
                for (int d = 0; d < P::NDOT; ++d) {
                    if constexpr (RS) {
                        grow_lazy<false, fast_sum_of<P>::value>(acc[2 * d], p0[d], slot0[d]);
                        grow_lazy<false, fast_sum_of<P>::value>(acc[2 * d + 1], p1[d], slot1[d]);
                    } else {
                        grow(acc[2 * d], p0[d], slot0[d]);
                        grow(acc[2 * d + 1], p1[d], slot1[d]);
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < P::NIN; ++i) in[i] = cur[u][i];
                P::run(in, o0, p0, co0);
#pragma unroll
                for (int i = 0; i < P::NOUT; ++i) a.out[i][qu] = o0[i];
#pragma unroll
                for (int d = 0; d < P::NDOT; ++d) {
                    if constexpr (RS) grow_lazy<false, fast_sum_of<P>::value>(acc[d], p0[d], slot0[d]);
                    else grow(acc[d], p0[d], slot0[d]);
                }
            }
        }
        if constexpr (PF) {
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int i = 0; i < P::NIN; ++i) cur[u][i] = nxt[u][i];
        }
    }
    pdl_trigger();   // streaming done: the successor may start filling freed SM slots
    if constexpr (RS) {
#pragma unroll
        for (int d = 0; d < P::NDOT * VEC; ++d) bad |= !isfinite(acc[d][0]);
        if (bad) {
            // this thread met a non-finite value: cancel what its fast pass
            // deposited (replay with negated deposits), then recompute its
            // products from the (unchanged) inputs with the careful grow
#pragma unroll
            for (int d = 0; d < ND * VEC; ++d)
#pragma unroll
                for (int i = 0; i < KEXP; ++i) acc[d][i] = 0.0;
            // (the fast pass's order: trips up or down, the packets of a trip ascending)
            int64_t qt = a.reverse ? q_first + (T - 1) * step : q_first;
            for (int64_t trip = 0; trip < T; ++trip, qt += dq)
            for (int u = 0; u < UNR; ++u) {
                const int64_t qr = qt + u * stride;
                if (qr >= npk) break;
                double in[P::NIN], o0[NO], p0[ND];
                if constexpr (VEC == 2) {
                    double o1[NO], p1[ND];
                    Pk v[P::NIN];
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) v[i] = reinterpret_cast<const Pk*>(a.in[i])[qr];
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = v[i].x;
                    P::run(in, o0, p0, co0);
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = v[i].y;
                    P::run(in, o1, p1, co1);
#if MBG_GROW_BATCH
                    if constexpr (batch_of<P>::value) {   // the replay repeats the fast pass's operations exactly
                        double px[2 * ND];
                        int64_t* sl[2 * ND];
#pragma unroll
                        for (int d = 0; d < ND; ++d) {
                            px[2 * d] = p0[d];
                            px[2 * d + 1] = p1[d];
                            sl[2 * d] = slot0[d];
                            sl[2 * d + 1] = slot1[d];
                        }
                        grow_lazy_batch<2 * ND, true, fast_sum_of<P>::value>(acc, px, sl);
                    } else
#endif
#pragma unroll
                    for (int d = 0; d < P::NDOT; ++d) {
                        grow_lazy<true, fast_sum_of<P>::value>(acc[2 * d], p0[d], slot0[d]);
                        grow_lazy<true, fast_sum_of<P>::value>(acc[2 * d + 1], p1[d], slot1[d]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = a.in[i][qr];
                    P::run(in, o0, p0, co0);
#pragma unroll
                    for (int d = 0; d < P::NDOT; ++d) grow_lazy<true, fast_sum_of<P>::value>(acc[d], p0[d], slot0[d]);
                }
            }
#pragma unroll
            for (int d = 0; d < ND * VEC; ++d)
#pragma unroll
                for (int i = 0; i < KEXP; ++i) acc[d][i] = 0.0;
            for (int64_t qr = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; qr < npk; qr += stride) {
                double in[P::NIN], o0[NO], p0[ND];
                if constexpr (VEC == 2) {
                    double o1[NO], p1[ND];
                    Pk v[P::NIN];
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) v[i] = reinterpret_cast<const Pk*>(a.in[i])[qr];
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = v[i].x;
                    P::run(in, o0, p0, co0);
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = v[i].y;
                    P::run(in, o1, p1, co1);
#pragma unroll
                    for (int d = 0; d < P::NDOT; ++d) {
                        grow(acc[2 * d], p0[d], slot0[d]);
                        grow(acc[2 * d + 1], p1[d], slot1[d]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < P::NIN; ++i) in[i] = a.in[i][qr];
                    P::run(in, o0, p0, co0);
#pragma unroll
                    for (int d = 0; d < P::NDOT; ++d) grow(acc[d], p0[d], slot0[d]);
                }
            }
        }
    }
    if constexpr (P::NDOT > 0) {
        int classes;
        if constexpr (VEC == 2) {
            if (m == 1) {
                // both lanes of the pair are column 0: merge the second expansion set
#pragma unroll
                for (int d = 0; d < P::NDOT; ++d)
#pragma unroll
                    for (int i = 0; i < KEXP; ++i) grow(acc[2 * d], acc[2 * d + 1][i], slot0[d]), acc[2 * d + 1][i] = 0.0;
                classes = 1;
            } else {
                classes = m / 2;
            }
        } else {
            classes = m;
        }
        // expansion x = d*VEC + v of class k -> column k*VEC + v (or 0 for m == 1)
        block_combine<ND * VEC>(acc, classes,
                                [&](int x, int k) {
                                    const int d = x / VEC, v = x % VEC;
                                    const int col = m == 1 ? 0 : k * VEC + v;
                                    return a.slot[d] + static_cast<int64_t>(col) * NSLOT;
                                },
                                sh_dyn);
    }
}

// Block size for m columns: m * 2^q <= 256 (m <= 256), else m.
inline int group_block(int m) {   // m <= 256 (checked by the callers)
    if (m > 256) return m;
    int b = m;
    while (b * 2 <= 256) b *= 2;
    return b;
}

}  // namespace mbg
