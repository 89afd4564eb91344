// solver.hpp -- device-resident BiCGStab drivers and the byte model.
#pragma once

#include <initializer_list>
#include <map>
#include <string>
#include <vector>

#include "common.hpp"

namespace mbg {

// Byte model.
double spmv_traffic_bytes(int64_t n, int64_t nnz, int m);      // Eq. (3), spmv.cpp:10-16
double spmv_compulsory_bytes(int64_t n, int64_t nnz, int m);   // x read once
// Per-iteration schedule totals (Table 2 + identity M^-1 copies for the
// preconditioned methods) and the SPEC.md form with the preconditioner apart.
bool preconditioned(int method);
void method_schedule(int method, int formulation, int* reads, int* writes, int* spmvs, int* nred,
                     int* dots_per_reduction);
void method_schedule_pc(int method, int formulation, int precond_alpha, int* reads, int* writes, int* spmvs,
                        int* precond_apps, int* nred, int* dots_per_reduction);
double iteration_bytes(int method, int formulation, int precond_alpha, int64_t n, int64_t nnz, int m);
// A^T of a single-GPU matrix, built once and cached on the matrix (api.cu).
const mbg_csr* csr_transpose(mbg_ctx* ctx, const mbg_csr* a);
// A^T of a reordered operator, terms in the original (reference) order.
const mbg_csr* csr_transpose_reordered(mbg_ctx* ctx, const mbg_csr* orig);

class Solver {
public:
    // precond_alpha < 0: identity (2) for the preconditioned methods, none otherwise
    Solver(mbg_ctx* ctx, const mbg_csr* a, int m, int method, int formulation, double tol, int fixed,
           int maxit, int precond_alpha = -1);
    ~Solver();
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;

    // b, x: device arrays (n*m, owned rows); x holds x0 and receives the solution.
    void run(const double* b, double* x, bool use_graph = true, int chunk = 8);
    void report(double* hist_host, mbg_report* rep);
    // Profiling mode: no graph; every launch bracketed by CUDA events on the
    // main stream.  profile_json() returns {label: [launches, ms, bytes/launch]}.
    void enable_profile() { profile_ = true; }
    std::string profile_json();

private:
    double* w(int i) { return work_[i].p; }
    double* sc(int i);
    int64_t* slot(int i);
    // post_point >= 0: run the scalar step `post_point` over `post_nd` dots
    // after this kernel.  (Running it in the last block of the dot kernel --
    // atomic ticket + fences -- was measured ~1% slower on B200 than the
    // separate one-block kernel inside the CUDA graph, and its register
    // footprint slowed the streaming kernels; removed.)
    void spmm(const double* x, double* y, int epi_kind = 0, const double* aux = nullptr, int post_point = -1,
              int post_nd = 0, int first_slot = 0, int reduce = -1);
    // y = A ((0 + 1*z) + na*v), the input formed per x plane inside the stencil SpMM
    void spmm_axpy(const double* z, const double* v, const double* na, double* y);
    template <class P>
    void group(std::initializer_list<const double*> in, std::initializer_list<double*> out,
               std::initializer_list<int> co, int first_slot, int post_point = -1, int post_nd = 0,
               int reduce = -1);
    struct ScalArgs scal_args(int point, int nd);
    void copy(double* dst, const double* src);
    void minv(const double* in, double* out);   // M^-1 application (identity or synthetic(alpha))
    void scalars(int point, int nd);
    void join();   // main stream waits for an in-flight dot allreduce
    void setup(const double* b, double* x);
    void iteration();

    mbg_ctx* ctx_;
    const mbg_csr* a_;
    int m_, method_, form_;
    int pa_ = 0;            // preconditioner alpha (0 none, 2 identity, >= 4 synthetic)
    bool elide_ = false;    // fused formulation with identity M^-1: applications aliased away
    bool epi_delta_ = false;
    bool ax_ = false;         // fused Reordered: th = z - alpha s formed inside the second SpMM (stencil.cu)
    bool stencil_ = false;    // the operator's SpMM runs on its stencil twin (stencil.cu)  // fused Reordered: delta = (v, r0) in the SpMM epilogue
    const mbg_csr* at_ = nullptr;   // A^T (IBiCGStab setup)
    const mbg_csr* orig_ = nullptr; // caller's operator when a_ is its reordered twin
    double* x_user_ = nullptr;
    double tol_;
    int fixed_, maxit_;
    int64_t n_ = 0, len_ = 0, rows_alloc_ = 0;
    std::vector<DevBuf<double>> work_;
    DevBuf<double> scal_, hist_;
    DevBuf<int> ctl_;
    DevBuf<int64_t> slots_;
    int* ctl_host_ = nullptr;
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    cudaEvent_t t0_ = nullptr, t1_ = nullptr;
    cudaGraphExec_t graph_exec_ = nullptr;
    const double* b_ = nullptr;
    double* x_ = nullptr;
    int64_t launches_ = 0;
    int64_t reductions_ = 0;
    bool pending_join_ = false;
    // direction of the next group pass: after an SpMM (which walks up) the first
    // pass walks down, the next up, ... -- each starts where its predecessor left
    // the L2 warm (group.cuh GroupArgs::reverse; MBG_GROUP_REVERSE=0 off)
    bool rev_next_ = false;
    float loop_ms_ = 0.f;
    // profiling
    bool profile_ = false;
    struct Mark { std::string label; double bytes; cudaEvent_t a, b; };
    std::vector<Mark> marks_;
    void mark_begin(const std::string& label, double bytes);
    void mark_end();
};

}  // namespace mbg
