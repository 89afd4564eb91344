// solver.cu -- device-resident multi-RHS BiCGStab drivers (classical, Reordered,
// Pipelined; merged and basic formulations).
//
// The reference's solver layer is missing (proj/CMakeLists.txt:22-32); the
// recurrences are the paper's merged listings -- Alg. 2 PAPER.md:1407-1438,
// Alg. 6 PAPER.md:1562-1598 (identity M^-1), Alg. 4 PAPER.md:1488-1525 --
// with the schedules and term expansions of SURVEY.md Appendix C and the
// solve() contract of SPEC.md:227-235,262-268.
//
// Everything stays on the device: per-column scalars (ColumnScalars,
// types.hpp:39-83) live in a small scalar bank updated by one-block "scalar"
// kernels after each reduction point; convergence, breakdown and iteration
// count live in a control word array that every kernel checks first, so an
// iteration captured once as a CUDA graph can be replayed blindly and becomes
// a no-op after the solve stops.  The host only polls the control words once
// per chunk of iterations (lagged by one chunk).
#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstdio>
#include <map>
#include <tuple>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "comm.hpp"
#include "kernels.hpp"
#include "scalar.cuh"
#include "solver.hpp"
#include "small.hpp"
#include "stencil.hpp"

namespace mbg {

__global__ void __launch_bounds__(1024) scalar_kernel(ScalArgs a) {
    extern __shared__ double s_dots[];  // nd * m rounded dots
    pdl_wait();
    pdl_trigger();
    scalar_block(a, s_dots);
}

// ===========================================================================
// Solver
// ===========================================================================
// Vector roles (indices into work_); 14 = x0 staging with halo room.
enum {
    V_R, V_R0, V_P, V_V, V_S, V_T, V_Z, V_VH, V_TH, V_RT, V_Q, V_W, V_Y, V_TMP, V_X0,
    V_U, V_F0, V_PH, V_SH, V_QH, V_RH, V_WH, V_ZH, V_BP, V_XP, NWORK
};

// Locality-reordered operator (mbg_csr_set_grid): b, x0 gathered into the
// operator's row order before the solve, x scattered back after it.
__global__ void permute_rows_kernel(const double* __restrict__ in, double* __restrict__ out,
                                    const int32_t* __restrict__ perm, int64_t n, int m, int scatter) {
    const int64_t len = n * m;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / m;
        const int64_t src = static_cast<int64_t>(perm[i]) * m + (e - i * m);
        if (scatter) out[src] = in[e];
        else out[e] = in[src];
    }
}

Solver::Solver(mbg_ctx* ctx, const mbg_csr* a, int m, int method, int formulation, double tol,
               int fixed, int maxit, int precond_alpha)
    : ctx_(ctx), a_(a), m_(m), method_(method), form_(formulation), tol_(tol), fixed_(fixed),
      maxit_(maxit) {
    if (method < 0 || method > 5) throw Invalid("solve: unknown method");
    if (formulation < 0 || formulation > 2) throw Invalid("solve: unknown formulation");
    // a block holds whole column classes (group_block): up to 256 right-hand sides
    if (m < 1 || m > 256) throw Invalid("solve: m must be in [1, 256]");
    if (maxit < 0) throw Invalid("solve: negative iteration count");
    if (!fixed && !(tol > 0.0)) throw Invalid("solve: tol must be > 0 in converge mode");
    // preconditioned ids require a preconditioner, the others reject one
    const bool pre = preconditioned(method);
    if (precond_alpha < 0) precond_alpha = pre ? 2 : 0;
    if (pre && (precond_alpha < 2 || precond_alpha % 2))
        throw Invalid("solve: a preconditioned method needs precond_alpha 2 (identity) or an even synthetic alpha >= 4");
    if (!pre && precond_alpha != 0) throw Invalid("solve: this method takes no preconditioner");
    pa_ = precond_alpha;
    elide_ = formulation == MBG_FUSED && pa_ == 2;
    // a locality-reordered twin of the operator, if the caller provided the grid
    // (not needed when the stencil SpMM handles this m: it stages x planes itself)
    stencil_ = stencil_handles(a, m);
    if (a->reordered && a->peers.empty() && !stencil_) {
        orig_ = a;
        a_ = a = a->reordered.get();
    }
    // delta in the SpMM epilogue pays off for short rows only: with > 12
    // nonzeros per row the gather-bound SpMM loses more to the epilogue's
    // registers than the separate 2-vector dot pass costs (B200: C3 27-point
    // 8.90 vs 8.07 ms/iteration, C5 m=8 5.28 vs 4.97; C2 7-point 0.76 vs 0.84)
    // (stencil SpMM: only with MBG_STENCIL_EPI=1 -- measured slower)
    // (MBG_SPMM_EPI_DELTA=0 / 1 forces the CSR choice for A/B measurements)
    bool csr_delta = a->nnz <= 12 * a->n;
    if (const char* e = std::getenv("MBG_SPMM_EPI_DELTA")) csr_delta = e[0] != '0';
    epi_delta_ = formulation == MBG_FUSED &&
                 (stencil_ ? (stencil_epilogues() || (method == MBG_RBICGSTAB && stencil_delta_epilogue(a, m)))
                           : csr_delta);
    // fused Reordered on a single-GPU 27-point twin (m = 16 / 32): the th update
    // pass is folded into the second SpMM, th is never stored (2 transfers less)
    ax_ = elide_ && method == MBG_RBICGSTAB && !ctx->comm && stencil_ && stencil_axpy_handles(a, m);
    if (method == MBG_IBICGSTAB) {
        if (!a->peers.empty() || a->n_halo) {
            // partitioned: A^T and its own halo plan were built at upload
            if (!a->transposed) throw Invalid("solve: IBiCGStab on a partitioned matrix needs its A^T plan");
            at_ = a->transposed.get();
        } else {
            at_ = orig_ ? csr_transpose_reordered(ctx, orig_) : csr_transpose(ctx, a);
        }
    }
    n_ = a->n;
    len_ = n_ * m;
    // (room for the halo rows of A, and of A^T when f0 = A^T r0 is exchanged)
    rows_alloc_ = a->n + std::max(a->n_halo, at_ ? at_->n_halo : 0);
    // only the vectors the method uses (C4 at m=32 is 8.4 GB per vector)
    std::vector<int> need;
    switch (method) {
        case MBG_BICGSTAB: need = {V_R, V_R0, V_P, V_V, V_S, V_T}; break;
        case MBG_RBICGSTAB:
            need = {V_R, V_R0, V_V, V_T, V_Z, V_VH};
            if (!ax_) need.push_back(V_TH);
            if (!elide_) need.push_back(V_RT);   // fused + identity: rt lives in registers only
            if (!elide_) need.insert(need.end(), {V_S, V_Q});
            break;
        case MBG_PIPEBICGSTAB:
            need = {V_R, V_R0, V_P, V_V, V_S, V_T, V_Z, V_W};
            if (formulation != MBG_FUSED) need.insert(need.end(), {V_Q, V_Y, V_TMP});   // fused: q, y in registers
            break;
        case MBG_IBICGSTAB: need = {V_R, V_R0, V_V, V_S, V_T, V_Z, V_Q, V_U, V_F0}; break;
        case MBG_PBICGSTAB:
            need = {V_R, V_R0, V_P, V_V, V_S, V_T};
            if (!elide_) need.insert(need.end(), {V_PH, V_SH});
            break;
        default:
            need = {V_R, V_R0, V_V, V_S, V_T, V_Z, V_Q, V_W, V_Y, V_TMP, V_PH, V_SH, V_QH, V_RH};
            if (!elide_) need.insert(need.end(), {V_WH, V_ZH});
            break;
    }
    if (orig_) need.insert(need.end(), {V_BP, V_XP});
    work_.resize(NWORK);
    const size_t vlen = static_cast<size_t>(rows_alloc_) * m;
    for (int i : need) work_[i] = pool_take(ctx, vlen);
    if (a->n_halo) work_[V_X0] = pool_take(ctx, vlen);  // x0 staging with halo room
    scal_.alloc(static_cast<size_t>(NSCAL) * m);
    ctl_.alloc(NCTL);
    hist_.alloc(static_cast<size_t>(maxit + 1) * m);
    slots_.alloc(static_cast<size_t>(8) * m * NSLOT);
    MBG_CUDA(cudaMemsetAsync(slots_.p, 0, slots_.n * sizeof(int64_t), ctx->stream));
    MBG_CUDA(cudaMemsetAsync(ctl_.p, 0, ctl_.n * sizeof(int), ctx->stream));
    if (!ctx->ctl_host) MBG_CUDA(cudaMallocHost(&ctx->ctl_host, 64 * sizeof(int)));
    ctl_host_ = ctx->ctl_host;
    for (auto& e : ev_) MBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MBG_CUDA(cudaEventCreate(&t0_));
    MBG_CUDA(cudaEventCreate(&t1_));
}

Solver::~Solver() {
    cudaStreamSynchronize(ctx_->stream);
    for (auto& w : work_) pool_give(ctx_, std::move(w));
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    for (auto& e : ev_) if (e) cudaEventDestroy(e);
    if (t0_) cudaEventDestroy(t0_);
    if (t1_) cudaEventDestroy(t1_);
}

double* Solver::sc(int i) { return scal_.p + static_cast<int64_t>(i) * m_; }
int64_t* Solver::slot(int i) { return slots_.p + static_cast<int64_t>(i) * m_ * NSLOT; }

void Solver::mark_begin(const std::string& label, double bytes) {
    if (!profile_) return;
    Mark mk{label, bytes, nullptr, nullptr};
    MBG_CUDA(cudaEventCreate(&mk.a));
    MBG_CUDA(cudaEventCreate(&mk.b));
    MBG_CUDA(cudaEventRecord(mk.a, ctx_->stream));
    marks_.push_back(mk);
}

void Solver::mark_end() {
    if (!profile_) return;
    MBG_CUDA(cudaEventRecord(marks_.back().b, ctx_->stream));
}

std::string Solver::profile_json() {
    MBG_CUDA(cudaStreamSynchronize(ctx_->stream));
    std::map<std::string, std::tuple<int64_t, double, double>> agg;
    for (auto& mk : marks_) {
        float ms = 0.f;
        MBG_CUDA(cudaEventElapsedTime(&ms, mk.a, mk.b));
        auto& e = agg[mk.label];
        std::get<0>(e) += 1;
        std::get<1>(e) += ms;
        std::get<2>(e) = mk.bytes;
        cudaEventDestroy(mk.a);
        cudaEventDestroy(mk.b);
    }
    marks_.clear();
    std::string out = "{";
    bool first = true;
    for (auto& [k, v] : agg) {
        char buf[256];
        snprintf(buf, sizeof buf, "%s\"%s\": [%lld, %.6f, %.1f]", first ? "" : ", ", k.c_str(),
                 static_cast<long long>(std::get<0>(v)), std::get<1>(v), std::get<2>(v));
        out += buf;
        first = false;
    }
    return out + "}";
}

// Alternating sweep direction of the group passes (solver.hpp rev_next_).
static bool group_reverse_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MBG_GROUP_REVERSE");
        return !(e && e[0] == '0');
    }();
    return on;
}

void Solver::spmm(const double* x, double* y, int epi_kind, const double* aux, int post_point, int post_nd,
                  int first_slot, int reduce) {
    SpmmEpi e;
    e.kind = epi_kind;
    e.aux = aux;
    for (int d = 0; d < 3; ++d) e.slot[d] = slot(first_slot + d);
    const double extra = epi_kind == 1 ? 8.0 * len_ : 0.0;   // aux vector read
    mark_begin(epi_kind ? "spmm+dots" + std::to_string(epi_kind) : std::string("spmm"),
               (stencil_ ? stencil_spmm_bytes(a_->n, a_->nnz, m_) : spmv_compulsory_bytes(a_->n, a_->nnz, m_)) +
                   extra);
    launches_ += apply_operator(ctx_, a_, m_, const_cast<double*>(x), y, ctl_.p, epi_kind ? &e : nullptr);
    mark_end();
    rev_next_ = group_reverse_enabled();
    if (epi_kind) {
        const int nred = reduce < 0 ? (epi_kind == 2 ? 3 : 1) : reduce;
        if (ctx_->comm && nred > 0) {
            comm_allreduce_i64(ctx_, slot(first_slot), static_cast<size_t>(nred) * m_ * NSLOT, ctx_->stream,
                               /*join=*/false);
            pending_join_ = true;
        }
        if (nred > 0) reductions_++;
    }
    if (post_point >= 0) scalars(post_point, post_nd);
}

void Solver::spmm_axpy(const double* z, const double* v, const double* na, double* y) {
    // algorithmic bytes: the stencil SpMM's, plus the second input vector
    mark_begin("spmm+axpy", stencil_spmm_bytes(a_->n, a_->nnz, m_) + 8.0 * len_);
    launches_ += launch_stencil_spmm_axpy(ctx_, a_, m_, z, v, na, y, ctl_.p);
    mark_end();
    rev_next_ = group_reverse_enabled();
}

template <class P>
void Solver::group(std::initializer_list<const double*> in, std::initializer_list<double*> out,
                   std::initializer_list<int> co, int first_slot, int post_point, int post_nd, int reduce) {
    GroupArgs g{};
    g.len = len_;
    g.m = m_;
    int i = 0;
    for (auto p : in) g.in[i++] = p;
    i = 0;
    for (auto p : out) g.out[i++] = p;
    i = 0;
    for (int s : co) g.coef[i++] = sc(s);
    for (int d = 0; d < P::NDOT; ++d) g.slot[d] = slot(first_slot + d);
    g.ctl = ctl_.p;
    g.reverse = rev_next_ ? 1 : 0;
    rev_next_ = group_reverse_enabled() && !rev_next_;
    mark_begin(std::string("group:") + P::NAME, static_cast<double>(P::NIN + P::NOUT) * 8.0 * len_);
    launch_group<P>(ctx_->stream, g, ctx_->num_sms);
    MBG_CUDA(cudaGetLastError());
    mark_end();
    launches_++;
    if (P::NDOT > 0) {
        // multi-GPU: one fused allreduce of all dots of this point (int64 limbs)
        // reduce < 0: this point's own slots; 0: deferred to a later group of
        // the same reduction point; > 0: that many slots from first_slot
        const int nred = reduce < 0 ? P::NDOT : reduce;
        if (ctx_->comm && nred > 0) {
            comm_allreduce_i64(ctx_, slot(first_slot), static_cast<size_t>(nred) * m_ * NSLOT, ctx_->stream,
                               /*join=*/false);
            pending_join_ = true;
        }
        if (nred > 0) reductions_++;
    }
    if (post_point >= 0) scalars(post_point, post_nd);
}

// M^-1: identity = one copy (1R + 1W); synthetic(alpha) =
// alpha/2 in-place scale passes by 2.0, 0.5, ... with a last factor that makes
// the product exactly 1 (oracle.c minv).
void Solver::minv(const double* in, double* out) {
    if (pa_ <= 2) {
        copy(out, in);
        return;
    }
    const int k = pa_ / 2;
    for (int i = 0; i < k; ++i) {
        const int c = i < k - 1 ? ((i & 1) ? S_HALF : S_TWO) : (((k - 1) & 1) ? S_HALF : S_ONE);
        group<PUpd1>({i == 0 ? in : out}, {out}, {c}, 0);
    }
}

void Solver::copy(double* dst, const double* src) {
    mark_begin("copy", 16.0 * len_);
    MBG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(len_) * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx_->stream));
    mark_end();
}

ScalArgs Solver::scal_args(int point, int nd) {
    ScalArgs s{};
    s.m = m_;
    s.point = point;
    s.method = method_;
    s.fixed = fixed_;
    s.maxit = maxit_;
    s.tol2 = tol_ * tol_;
    s.sc = scal_.p;
    s.ctl = ctl_.p;
    s.hist = hist_.p;
    for (int i = 0; i < nd; ++i) s.D[i] = slot(i);
    s.nd = nd;
    return s;
}


void Solver::join() {
    if (pending_join_) comm_join(ctx_);
    pending_join_ = false;
}

void Solver::scalars(int point, int nd) {
    join();   // the dots of this point may still be in an allreduce on the side stream
    ScalArgs s = scal_args(point, nd);
    const int threads = std::min(1024, std::max(((m_ + 31) / 32) * 32, 32 * nd * m_));
    mark_begin("scalar", 0.0);
    launch_pdl(scalar_kernel, dim3(1), dim3(threads), static_cast<size_t>(nd > 0 ? nd : 1) * m_ * sizeof(double),
               ctx_->stream, s);
    MBG_CUDA(cudaGetLastError());
    mark_end();
    launches_++;
}

void Solver::setup(const double* b, double* x) {
    x_user_ = x;
    if (orig_) {   // gather b and x0 into the reordered operator's row order
        const unsigned grid = static_cast<unsigned>(ctx_->num_sms) * 4;
        permute_rows_kernel<<<grid, 256, 0, ctx_->stream>>>(b, w(V_BP), orig_->perm.p, n_, m_, 0);
        permute_rows_kernel<<<grid, 256, 0, ctx_->stream>>>(x, w(V_XP), orig_->perm.p, n_, m_, 0);
        MBG_CUDA(cudaGetLastError());
        launches_ += 2;
        b = w(V_BP);
        x = w(V_XP);
    }
    b_ = b;
    x_ = x;
    double* r = w(V_R);
    double* r0 = w(V_R0);
    double* tmpv = w(V_V);
    if (a_->n_halo) {
        copy(w(V_X0), x);                                // x0 into a buffer with halo room
        spmm(w(V_X0), tmpv);                             // z = A x0
    } else {
        spmm(x, tmpv);                                   // z = A x0
    }
    group<PUpd2>({b, tmpv}, {r}, {S_ONE, S_MONE}, 0);    // r = 1*b + (-1)*z   (needs S_ONE set)
    group<PUpd1>({r}, {r0}, {S_ONE}, 0);                  // r0 = 1*r
    group<PDot1>({r0}, {}, {}, 0);                        // rho = (r0, r0)
    auto zero = [&](int v) {
        if (work_[v].p) MBG_CUDA(cudaMemsetAsync(w(v), 0, static_cast<size_t>(len_) * sizeof(double), ctx_->stream));
    };
    if (method_ == MBG_BICGSTAB || method_ == MBG_PBICGSTAB) {
        group<PUpd1>({r}, {w(V_P)}, {S_ONE}, 2);          // p = 1*r
        group<PDot1>({b}, {}, {}, 1, P_SETUP, 2);         // bb = (b, b)
    } else if (method_ == MBG_RBICGSTAB) {
        minv(r0, w(V_Z));                                 // z0 = M^-1 r0
        copy(w(V_VH), w(V_Z));                            // v^0 = z0
        group<PDot1>({b}, {}, {}, 1, P_SETUP, 2);         // bb = (b, b)
    } else if (method_ == MBG_IBICGSTAB) {
        // Alg. 3 line 1: u0 = A r0, f0 = A^T r0, q0 = v0 = z0 = 0
        spmm(r, w(V_U));
        mark_begin("spmm_t", spmv_compulsory_bytes(at_->n, at_->nnz, m_));
        launches_ += apply_operator(ctx_, at_, m_, r0, w(V_F0), ctl_.p);
        mark_end();
        for (int v : {V_Q, V_V, V_Z}) zero(v);
        group<PDot1>({b}, {}, {}, 1);                     // bb = (b, b)
        group<PDot2>({r0, w(V_U)}, {}, {}, 2, P_SETUP, 3); // sigma0 = (r0, u0)
    } else if (method_ == MBG_PIPEBICGSTAB) {
        group<PDot1>({b}, {}, {}, 1);                     // bb = (b, b)
        for (int v : {V_P, V_S, V_Z}) zero(v);
        spmm(r, w(V_W));                                  // w0 = A r0
        spmm(w(V_W), w(V_T));                             // t0 = A w0
        zero(V_V);                                        // (served as A x0 scratch)
        group<PDot2>({r0, w(V_W)}, {}, {}, 2, P_SETUP, 3); // (r0, w0) ; alpha0
    } else {
        // Alg. 7 line 1: r^0 = M^-1 r0, w0 = A r^0, w^0 = M^-1 w0, t0 = A w^0
        group<PDot1>({b}, {}, {}, 1);                     // bb = (b, b)
        for (int v : {V_PH, V_SH, V_S, V_Z, V_ZH}) zero(v);
        minv(r, w(V_RH));
        spmm(w(V_RH), w(V_W));
        double* wh = elide_ ? w(V_W) : w(V_WH);
        if (!elide_) minv(w(V_W), wh);
        spmm(wh, w(V_T));
        zero(V_V);
        group<PDot2>({r0, w(V_W)}, {}, {}, 2, P_SETUP, 3); // (r0, w0) ; alpha0
    }
}

void Solver::iteration() {
    const bool basic = form_ == MBG_BASIC;
    const bool fused = form_ == MBG_FUSED;
    double *r = w(V_R), *r0 = w(V_R0), *x = x_;
    if (method_ == MBG_BICGSTAB) {
        double *p = w(V_P), *v = w(V_V), *s = w(V_S), *t = w(V_T);
        if (fused && stencil_ && stencil_epilogues()) {
            // stencil SpMM (registers to spare; x of the row staged in shared
            // memory): delta = (v, r0) and phi = (t, s), psi = (t, t) in the SpMM
            // epilogues, theta where s is produced -- 15 vector transfers
            spmm(p, v, 1, r0, P_C_ALPHA, 1, 0, 1);                          // v ; delta -> slot 0 ; alpha
            group<PUpd2Sq>({r, v}, {s}, {S_ONE, S_NALPHA}, 2, -1, 0, 0);   // s ; theta = (s,s) -> slot 2
            spmm(s, t, 4, nullptr, P_C_OMEGA, 3, 0, 3);                    // t ; phi psi -> slots 0,1 ; omega
        } else if (fused) {
            // theta computed where s is produced (spreads the exact-dot work over
            // two passes); delta and phi/psi stay in their own passes: fusing
            // them into the CSR SpMM epilogue costs the SpMM more than it saves
            // (measured on B200)
            spmm(p, v);
            group<PDot2>({v, r0}, {}, {}, 0, P_C_ALPHA, 1);
            group<PUpd2Sq>({r, v}, {s}, {S_ONE, S_NALPHA}, 2, -1, 0, 0);   // s ; theta = (s,s) -> slot 2
            spmm(s, t);
            group<PClassicPhiPsi>({t, s}, {}, {}, 0, P_C_OMEGA, 3, 3);     // phi psi -> slots 0,1 ; omega
        } else {
            spmm(p, v);
            group<PDot2>({v, r0}, {}, {}, 0, P_C_ALPHA, 1);
            group<PUpd2>({r, v}, {s}, {S_ONE, S_NALPHA}, 0);
            spmm(s, t);
            if (basic) {
                group<PDot2>({t, s}, {}, {}, 0);
                group<PDot1>({t}, {}, {}, 1);
                group<PDot1>({s}, {}, {}, 2, P_C_OMEGA, 3);
            } else {
                group<PClassicOmega>({t, s}, {}, {}, 0, P_C_OMEGA, 3);
            }
        }
        if (basic) {
            group<PUpd3>({x, p, s}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
            group<PUpd2>({s, t}, {r}, {S_ONE, S_NOMEGA}, 0);
            group<PDot2>({r, r0}, {}, {}, 0, P_C_BETA, 1);
        } else {
            group<PClassicXR>({x, p, s, t, r0}, {x, r}, {S_ALPHA, S_OMEGA, S_NOMEGA}, 0, P_C_BETA, 1);
        }
        group<PUpd3>({r, p, v}, {p}, {S_ONE, S_BETA, S_NBO}, 0);
    } else if (method_ == MBG_RBICGSTAB) {
        double *z = w(V_Z), *vh = w(V_VH), *v = w(V_V), *th = w(V_TH), *t = w(V_T);
        double* rt = elide_ ? nullptr : w(V_RT);
        // identity M^-1: the fused formulation aliases s = v and q = t instead of copying
        double* s = elide_ ? v : w(V_S);
        double* q = elide_ ? t : w(V_Q);
        if (fused && epi_delta_) {
            spmm(vh, v, 1, r0, P_C_ALPHA, 1);                     // v = A vh ; delta = (v, r0) ; alpha
            if (!elide_) minv(v, s);
        } else {
            spmm(vh, v);
            if (!elide_) minv(v, s);                              // s = M^-1 v
            group<PDot2>({v, r0}, {}, {}, 0, P_C_ALPHA, 1);
        }
        if (ax_) {
            spmm_axpy(z, s, sc(S_NALPHA), t);                    // t = A (z - alpha s), th never stored
        } else {
            group<PUpd2>({z, s}, {th}, {S_ONE, S_NALPHA}, 0);    // th = z - alpha s
            spmm(th, t);
        }
        if (!elide_) minv(t, q);                                  // q = M^-1 t
        if (basic) {
            group<PUpd2>({r, v}, {rt}, {S_ONE, S_NALPHA}, 0);
            group<PDot2>({t, rt}, {}, {}, 0);
            group<PDot1>({t}, {}, {}, 1);
            group<PDot2>({t, r0}, {}, {}, 2);
            group<PDot1>({rt}, {}, {}, 3, P_R_OMEGA, 4);
        } else if (fused && elide_) {
            group<PReordG7D>({r, v, t, r0}, {}, {S_NALPHA}, 0, P_R_OMEGA, 4);   // rt in registers only
        } else {
            group<PReordG7>({r, v, t, r0}, {rt}, {S_NALPHA}, 0, P_R_OMEGA, 4);
        }
        if (ax_) {
            // th and rt recomputed from z, s and r (the expressions of their passes)
            group<PReordG12RZ>({x, vh, z, q, s, r}, {x, z, vh, r},
                               {S_ALPHA, S_OMEGA, S_NOMEGA, S_BETA, S_NBO, S_NALPHA}, 0, P_R_END, 0);
        } else if (fused && elide_) {
            // r = (r - alpha s) - omega t in the x / z / vh pass (t, s are read there as q, s)
            group<PReordG12R>({x, vh, th, q, s, r}, {x, z, vh, r},
                              {S_ALPHA, S_OMEGA, S_NOMEGA, S_BETA, S_NBO, S_NALPHA}, 0, P_R_END, 0);
        } else {
            group<PUpd2>({rt, t}, {r}, {S_ONE, S_NOMEGA}, 0);        // r = rt - omega t
            if (basic) {
                group<PUpd3>({x, vh, th}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
                group<PUpd2>({th, q}, {z}, {S_ONE, S_NOMEGA}, 0);
                group<PUpd3>({z, vh, s}, {vh}, {S_ONE, S_BETA, S_NBO}, 0, P_R_END, 0);
            } else {
                group<PReordG12>({x, vh, th, q, s}, {x, z, vh}, {S_ALPHA, S_OMEGA, S_NOMEGA, S_BETA, S_NBO}, 0,
                                 P_R_END, 0);
            }
        }
    } else if (method_ == MBG_PIPEBICGSTAB) {
        double *p = w(V_P), *s = w(V_S), *wv = w(V_W), *z = w(V_Z), *t = w(V_T), *v = w(V_V);
        double *q = fused ? nullptr : w(V_Q), *y = fused ? nullptr : w(V_Y), *tmp = fused ? nullptr : w(V_TMP);
        // The scalar steps wait for the reductions, which overlap the following
        // SpMM (on the side stream when a communicator allreduces them).
        if (fused) {
            group<PPipeG1F>({r, p, s, wv, z, t, v}, {p, s, z}, {S_BETA, S_NBO, S_NALPHA}, 0, -1, 3);
        } else if (basic) {
            group<PUpd3>({r, p, s}, {p}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd3>({wv, s, z}, {s}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd3>({t, z, v}, {z}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd2>({r, s}, {q}, {S_ONE, S_NALPHA}, 0);
            group<PUpd2>({wv, z}, {y}, {S_ONE, S_NALPHA}, 0);
            group<PDot2>({q, y}, {}, {}, 0);
            group<PDot1>({y}, {}, {}, 1);
            group<PDot1>({q}, {}, {}, 2, -1, 3);
        } else {
            group<PPipeG1>({r, p, s, wv, z, t, v}, {p, s, z, q, y}, {S_BETA, S_NBO, S_NALPHA}, 0,
                           -1, 3);
        }
        spmm(z, v);
        scalars(P_P_OMEGA, 3);
        if (basic) {
            group<PUpd3>({x, p, q}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
            group<PUpd2>({q, y}, {r}, {S_ONE, S_NOMEGA}, 0);
            group<PUpd2>({t, v}, {tmp}, {S_NOMEGA, S_OA}, 0);   // split_basic: trailing pair
            group<PUpd2>({y, tmp}, {wv}, {S_ONE, S_ONE}, 0);
            group<PDot2>({r0, r}, {}, {}, 0);
            group<PDot2>({r0, z}, {}, {}, 1);
            group<PDot2>({r0, wv}, {}, {}, 2);
            group<PDot2>({r0, s}, {}, {}, 3, -1, 4);
        } else if (fused) {
            // q, y recomputed from r, w (read before this pass overwrites them) and the new s, z
            group<PPipeG45F>({x, p, r, wv, t, v, r0, z, s}, {x, r, wv}, {S_ALPHA, S_OMEGA, S_NOMEGA, S_OA, S_NALPHA},
                             0, -1, 4);
        } else {
            group<PPipeG4>({x, p, q, y}, {x, r}, {S_ALPHA, S_OMEGA, S_NOMEGA}, 0);
            group<PPipeG5>({y, t, v, r0, r, z, s}, {wv}, {S_NOMEGA, S_OA}, 0, -1, 4);
        }
        spmm(wv, t);
        scalars(P_P_BETA, 4);
    } else if (method_ == MBG_IBICGSTAB) {
        // Alg. 3: one 7-dot reduction point per iteration
        double *u = w(V_U), *f0 = w(V_F0), *q = w(V_Q), *v = w(V_V), *z = w(V_Z), *s = w(V_S), *t = w(V_T);
        scalars(P_I_START, 0);                                    // rho', delta', beta', tau', alpha'
        if (basic) {
            group<PUpd3>({r, z, v}, {z}, {S_ALPHA, S_CZ2, S_CZ3}, 0);
            group<PUpd3>({u, v, q}, {v}, {S_ONE, S_BETA, S_NDELTA}, 0);
            group<PUpd2>({r, v}, {s}, {S_ONE, S_NALPHA}, 0);
        } else {
            group<PIbcgG1>({r, z, v, u, q}, {z, v, s}, {S_ALPHA, S_CZ2, S_CZ3, S_BETA, S_NDELTA, S_NALPHA}, 0);
        }
        spmm(v, q);
        if (basic) {
            group<PUpd2>({u, q}, {t}, {S_ONE, S_NALPHA}, 0);
            group<PDot2>({r0, s}, {}, {}, 0);
            group<PDot2>({r0, q}, {}, {}, 1);
            group<PDot2>({f0, s}, {}, {}, 2);
            group<PDot2>({f0, t}, {}, {}, 3);
            group<PDot2>({s, t}, {}, {}, 4);
            group<PDot1>({t}, {}, {}, 5);
            group<PDot1>({s}, {}, {}, 6, P_I_OMEGA, 7);
        } else {
            group<PIbcgG2>({u, q, r0, s, f0}, {t}, {S_NALPHA}, 0, P_I_OMEGA, 7);
        }
        if (basic) {
            group<PUpd2>({s, t}, {r}, {S_ONE, S_NOMEGA}, 0);
            group<PUpd3>({x, z, s}, {x}, {S_ONE, S_ONE, S_OMEGA}, 0);
        } else {
            group<PIbcgG3>({s, t, x, z}, {r, x}, {S_NOMEGA, S_OMEGA}, 0);
        }
        scalars(P_R_END, 0);                                      // converged? next iteration
        spmm(r, u);
    } else if (method_ == MBG_PBICGSTAB) {
        // Alg. 5; the x update (independent of beta) runs
        // while the rho' reduction is in flight
        double *p = w(V_P), *v = w(V_V), *s = w(V_S), *t = w(V_T);
        double* ph = elide_ ? p : w(V_PH);
        double* sh = elide_ ? s : w(V_SH);
        if (!elide_) minv(p, ph);
        spmm(ph, v);
        group<PDot2>({v, r0}, {}, {}, 0, P_C_ALPHA, 1);
        group<PUpd2>({r, v}, {s}, {S_ONE, S_NALPHA}, 0);
        if (!elide_) minv(s, sh);
        spmm(sh, t);
        if (basic) {
            group<PDot2>({t, s}, {}, {}, 0);
            group<PDot1>({t}, {}, {}, 1);
            group<PDot1>({s}, {}, {}, 2, P_C_OMEGA, 3);
            group<PUpd2>({s, t}, {r}, {S_ONE, S_NOMEGA}, 0);
            group<PUpd3>({x, ph, sh}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
            group<PDot2>({r, r0}, {}, {}, 0, P_C_BETA, 1);
        } else {
            group<PClassicOmega>({t, s}, {}, {}, 0, P_C_OMEGA, 3);
            group<PRDot>({s, t, r0}, {r}, {S_NOMEGA}, 0);             // r ; rho' (reduction in flight)
            group<PUpd3>({x, ph, sh}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
            scalars(P_C_BETA, 1);
        }
        group<PUpd3>({r, p, v}, {p}, {S_ONE, S_BETA, S_NBO}, 0);
    } else {
        // Alg. 7: both reductions overlap M^-1 + SpMM
        double *rh = w(V_RH), *ph = w(V_PH), *sh = w(V_SH), *qh = w(V_QH), *wv = w(V_W), *t = w(V_T);
        double *s = w(V_S), *z = w(V_Z), *q = w(V_Q), *y = w(V_Y), *v = w(V_V), *tmp = w(V_TMP);
        double* wh = elide_ ? wv : w(V_WH);
        double* zh = elide_ ? z : w(V_ZH);
        if (basic) {
            group<PUpd3>({rh, ph, sh}, {ph}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd3>({wh, sh, zh}, {sh}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd2>({rh, sh}, {qh}, {S_ONE, S_NALPHA}, 0);
            group<PUpd3>({wv, s, z}, {s}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd3>({t, z, v}, {z}, {S_ONE, S_BETA, S_NBO}, 0);
            group<PUpd2>({r, s}, {q}, {S_ONE, S_NALPHA}, 0);
            group<PUpd2>({wv, z}, {y}, {S_ONE, S_NALPHA}, 0);
            group<PDot2>({q, y}, {}, {}, 0);
            group<PDot1>({y}, {}, {}, 1);
            group<PDot1>({q}, {}, {}, 2);
        } else {
            group<PPpG1>({rh, ph, sh, wh, zh}, {ph, sh, qh}, {S_BETA, S_NBO, S_NALPHA}, 0);
            group<PPpG2>({r, s, wv, z, t, v}, {s, z, q, y}, {S_BETA, S_NBO, S_NALPHA}, 0);
        }
        if (!elide_) minv(z, zh);
        spmm(zh, v);
        scalars(P_P_OMEGA, 3);
        if (basic) {
            group<PUpd3>({x, ph, qh}, {x}, {S_ONE, S_ALPHA, S_OMEGA}, 0);
            group<PUpd2>({wh, zh}, {tmp}, {S_NOMEGA, S_OA}, 0);   // split_basic: trailing pair
            group<PUpd2>({qh, tmp}, {rh}, {S_ONE, S_ONE}, 0);
            group<PUpd2>({q, y}, {r}, {S_ONE, S_NOMEGA}, 0);
            group<PUpd2>({t, v}, {tmp}, {S_NOMEGA, S_OA}, 0);
            group<PUpd2>({y, tmp}, {wv}, {S_ONE, S_ONE}, 0);
            group<PDot2>({r0, r}, {}, {}, 0);
            group<PDot2>({r0, z}, {}, {}, 1);
            group<PDot2>({r0, wv}, {}, {}, 2);
            group<PDot2>({r0, s}, {}, {}, 3);
        } else {
            group<PPpG3>({x, ph, qh, wh, zh}, {x, rh}, {S_ALPHA, S_OMEGA, S_NOMEGA, S_OA}, 0);
            group<PPpG4>({q, y, t, v, r0, z, s}, {r, wv}, {S_NOMEGA, S_OA}, 0);
        }
        if (!elide_) minv(wv, wh);
        spmm(wh, t);
        scalars(P_P_BETA, 4);
    }
    join();   // a captured graph must end joined to the origin stream
}

void Solver::run(const double* b, double* x, bool use_graph, int chunk) {
    if (profile_ || comm_is_local(ctx_)) use_graph = false;
    // S_ONE / S_MONE must exist before setup's first group
    std::vector<double> init(static_cast<size_t>(4) * m_);
    for (int c = 0; c < m_; ++c) {
        init[c] = 1.0;
        init[m_ + c] = -1.0;
        init[2 * m_ + c] = 2.0;
        init[3 * m_ + c] = 0.5;
    }
    static_assert(S_MONE == S_ONE + 1 && S_HALF == S_TWO + 1, "constant rows");
    MBG_CUDA(cudaMemcpyAsync(sc(S_ONE), init.data(), 2 * m_ * sizeof(double), cudaMemcpyHostToDevice,
                             ctx_->stream));
    MBG_CUDA(cudaMemcpyAsync(sc(S_TWO), init.data() + 2 * m_, 2 * m_ * sizeof(double), cudaMemcpyHostToDevice,
                             ctx_->stream));
    MBG_CUDA(cudaStreamSynchronize(ctx_->stream));  // init is a stack buffer
    if (ctx_->comm) comm_barrier(ctx_);
    MBG_CUDA(cudaEventRecord(t0_, ctx_->stream));
    setup(b, x);
    join();
    if (profile_) {  // profile the iteration loop only
        MBG_CUDA(cudaStreamSynchronize(ctx_->stream));
        for (auto& mk : marks_) { cudaEventDestroy(mk.a); cudaEventDestroy(mk.b); }
        marks_.clear();
    }
    const int64_t setup_launches = launches_;
    // small systems (cannot fill the GPU): the whole classical loop in one
    // cooperative launch (small.cu), bitwise the same iterations
    const bool small = maxit_ > 0 && method_ == MBG_BICGSTAB && form_ != MBG_BASIC && !ctx_->comm && !orig_ &&
                       !profile_ && ctx_->small_path && small_path_enabled() && len_ <= SMALL_MAX_LEN &&
                       (m_ == 1 || m_ == 2 || m_ == 4 || m_ == 8 || m_ == 16 || m_ == 32);
    if (small) {
        SmallArgs sa{};
        sa.n = n_;
        sa.m = m_;
        sa.off = a_->off.p;
        sa.col = a_->col.p;
        sa.val = a_->val.p;
        sa.x = x_;
        sa.r = w(V_R);
        sa.r0 = w(V_R0);
        sa.p = w(V_P);
        sa.v = w(V_V);
        sa.s = w(V_S);
        sa.t = w(V_T);
        sa.sc = scal_.p;
        sa.ctl = ctl_.p;
        sa.hist = hist_.p;
        sa.slots = slots_.p;
        sa.fused = form_ == MBG_FUSED;
        sa.fixed = fixed_;
        sa.maxit = maxit_;
        sa.tol2 = tol_ * tol_;
        launches_ += launch_small_classical(ctx_->stream, sa, ctx_->num_sms);
    } else if (maxit_ > 0) {
        if (use_graph) {
            cudaGraph_t g;
            MBG_CUDA(cudaStreamBeginCapture(ctx_->stream, cudaStreamCaptureModeThreadLocal));
            iteration();
            MBG_CUDA(cudaStreamEndCapture(ctx_->stream, &g));
            MBG_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
            MBG_CUDA(cudaGraphDestroy(g));
        }
        int64_t per_iter = 0;
        if (use_graph) {
            per_iter = launches_ - setup_launches;
            launches_ = setup_launches;
        }
        int launched = 0, k = 0;
        bool have_prev = false;
        while (launched < maxit_) {
            const int n = std::min(chunk, maxit_ - launched);
            for (int i = 0; i < n; ++i) {
                if (use_graph) {
                    MBG_CUDA(cudaGraphLaunch(graph_exec_, ctx_->stream));
                    launches_ += per_iter;
                } else {
                    iteration();
                }
            }
            launched += n;
            int* snap = ctl_host_ + (k & 1) * NCTL;
            MBG_CUDA(cudaMemcpyAsync(snap, ctl_.p, NCTL * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
            MBG_CUDA(cudaEventRecord(ev_[k & 1], ctx_->stream));
            if (have_prev) {
                int* prev = ctl_host_ + ((k - 1) & 1) * NCTL;
                MBG_CUDA(cudaEventSynchronize(ev_[(k - 1) & 1]));
                if (prev[C_STOP]) break;
            }
            have_prev = true;
            ++k;
        }
    }
    if (orig_) {   // scatter the solution back to the caller's row order
        permute_rows_kernel<<<static_cast<unsigned>(ctx_->num_sms) * 4, 256, 0, ctx_->stream>>>(
            x_, x_user_, orig_->perm.p, n_, m_, 1);
        MBG_CUDA(cudaGetLastError());
        launches_++;
    }
    MBG_CUDA(cudaEventRecord(t1_, ctx_->stream));
    MBG_CUDA(cudaStreamSynchronize(ctx_->stream));
    float ms = 0.f;
    MBG_CUDA(cudaEventElapsedTime(&ms, t0_, t1_));
    loop_ms_ = ms;
    MBG_CUDA(cudaMemcpy(ctl_host_, ctl_.p, NCTL * sizeof(int), cudaMemcpyDeviceToHost));
}

void Solver::report(double* hist_host, mbg_report* rep) {
    const int* c = ctl_host_;
    std::memset(rep, 0, sizeof(*rep));
    rep->iterations = c[C_ITERS];
    rep->converged = c[C_CONVERGED];
    rep->breakdown = c[C_BD];
    rep->breakdown_iter = c[C_BDITER];
    rep->breakdown_col = c[C_BDCOL];
    if (hist_host) {
        const size_t cnt = static_cast<size_t>(rep->iterations + 1) * m_;
        MBG_CUDA(cudaMemcpy(hist_host, hist_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
    int reads = 0, writes = 0, spmvs = 0, apps = 0, nred = 0, dots[8];
    method_schedule_pc(method_, form_, pa_, &reads, &writes, &spmvs, &apps, &nred, dots);
    const int its = rep->iterations;
    // TrafficCounter semantics: the preconditioner's transfers are tallied too
    // (alpha/2 reads + alpha/2 writes per application)
    if (method_ == MBG_RBICGSTAB && form_ == MBG_FUSED && !epi_delta_) reads += 1;   // delta pass: v, r0 vs aux r0
    // fused Reordered merges r = rt - omega t into the x/z/vh pass only when
    // q = t is elided (identity M^-1); otherwise that update is its own pass
    if (method_ == MBG_RBICGSTAB && form_ == MBG_FUSED && !elide_) {
        reads += 1;    // the separate r = rt - omega t pass ...
        writes += 1;   // ... and rt stored by the 4-dot pass
    }
    // th formed inside the second SpMM: its update pass (z, s -> th) is gone and
    // the SpMM reads s beside z (the SpMM-side read is counted as a vector read)
    if (ax_) {
        reads -= 1;
        writes -= 1;
    }
    // classical fused on the stencil SpMM: delta pass (v, r0) -> aux r0 in the
    // SpMM epilogue; phi/psi pass (t, s) -> the second SpMM's epilogue
    const int classic_epi = (method_ == MBG_BICGSTAB && form_ == MBG_FUSED && stencil_ && stencil_epilogues()) ? 3 : 0;
    reads -= classic_epi;
    rep->vector_reads = static_cast<int64_t>(reads + apps * pa_ / 2) * its;
    rep->vector_writes = static_cast<int64_t>(writes + apps * pa_ / 2) * its;
    rep->spmv_bytes = static_cast<double>(spmvs) * its * spmv_traffic_bytes(a_->n, a_->nnz, m_);
    rep->compulsory_bytes =
        (iteration_bytes(method_, form_, pa_, a_->n, a_->nnz, m_) +
         ((method_ == MBG_RBICGSTAB && form_ == MBG_FUSED && !epi_delta_) ? 8.0 * static_cast<double>(len_) : 0.0) +
         ((method_ == MBG_RBICGSTAB && form_ == MBG_FUSED && !elide_) ? 16.0 * static_cast<double>(len_) : 0.0) -
         (ax_ ? 16.0 * static_cast<double>(len_) : 0.0) -
         8.0 * classic_epi * static_cast<double>(len_) -
         // stencil SpMM: no column indices (8 B instead of 12 B per nonzero)
         (stencil_ ? 4.0 * spmvs * static_cast<double>(a_->nnz) : 0.0)) *
        its;
    rep->reductions = static_cast<int64_t>(nred) * its;
    rep->gpu_launches = launches_;
    rep->loop_ms = loop_ms_;
}

}  // namespace mbg
