/*
 * mbstab_b200.h -- C ABI of the B200-native multi-RHS BiCGStab hot path.
 *
 * Plain pointers and sizes only; every function returns an int status
 * (MBG_OK == 0) and never throws.  mbg_last_error() returns the message of
 * the last failure on the calling thread.  The C++ API in mbstab_b200.hpp
 * wraps these calls and rethrows std::invalid_argument / std::runtime_error,
 * matching the reference's error behaviour.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference tree, proj/...):
 *
 *   mbg_csr_upload        core::CsrMatrix + validate()     include/mbstab/core/csr.hpp:13-30,
 *                                                           src/core/csr.cpp:8-32
 *   mbg_mv_*              core::MultiVector                include/mbstab/core/types.hpp:13-35
 *   mbg_spmv              core::spmv                       include/mbstab/core/spmv.hpp:16-17,
 *                                                           src/core/spmv.cpp:54-74
 *   mbg_spmv_traffic_bytes core::spmv_traffic_bytes        src/core/spmv.cpp:10-16
 *   mbg_execute_group     kernels::execute_group           include/mbstab/kernels/execute.hpp:26-30,
 *                                                           src/kernels/execute.cpp:123-172
 *   mbg_analyze_traffic   kernels::analyze_traffic         include/mbstab/kernels/statement.hpp:65
 *   mbg_split_basic_traffic kernels::split_basic (+ analyze) include/mbstab/kernels/statement.hpp:73
 *   mbg_solve             solvers::solve (missing in the reference: proj/CMakeLists.txt:31;
 *                                           contract SPEC.md:227-235)
 *   mbg_method_schedule   solvers::method_schedule (missing: CMakeLists.txt:32)
 *   mbg_gen_*             core::gen_poisson_7pt            src/core/generators.cpp:37-67
 *                         and the BASELINE.json config generators
 *
 * Numerics contract: no FMA contraction anywhere; SpMV
 * sums each (row, column) sequentially in CSR order from 0.0; updates sum
 * terms in statement order from 0.0; dot products are exact (correctly
 * rounded), hence independent of launch shape and GPU count.
 */
#ifndef MBSTAB_B200_H
#define MBSTAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBG_OK 0
#define MBG_ERR_INVALID 1    /* std::invalid_argument in the reference */
#define MBG_ERR_RUNTIME 2    /* std::runtime_error (CUDA / NCCL failure) */
#define MBG_ERR_BREAKDOWN 3  /* solver breakdown */

#define MBG_MAX_TERMS 8

typedef struct mbg_ctx mbg_ctx;
typedef struct mbg_csr mbg_csr;
typedef struct mbg_mv mbg_mv;

/* ---- errors / version ------------------------------------------------- */
const char* mbg_last_error(void);
const char* mbg_version(void);

/* ---- context: one CUDA device, its streams and (optionally) a NCCL comm */
int mbg_ctx_create(int device, mbg_ctx** out);
int mbg_ctx_destroy(mbg_ctx* ctx);
int mbg_ctx_synchronize(mbg_ctx* ctx);
/* Small classical solves (n*m <= 2^20, m a power of two <= 32, one GPU) run
 * their whole iteration loop in one cooperative launch -- bitwise the same
 * iterations as the multi-kernel path.  enable = 0 forces the multi-kernel
 * path on this context (default 1; MBG_SMALL=0 turns it off process-wide). */
int mbg_ctx_set_small_path(mbg_ctx* ctx, int enable);
/* Size the persistent grids for (device SMs - count) SMs, leaving `count` SMs
 * to concurrent kernels (a multi-rank NCCL communicator does this itself with
 * MBG_RESERVE_SMS, default 4, so side-stream collectives overlap the SpMM).
 * Results do not depend on it (bitwise). */
int mbg_ctx_reserve_sms(mbg_ctx* ctx, int count);
/* Checked builds only (make checked -> libmbstab_b200_checked.so): every device
 * allocation has guard zones on both sides; verify all live ones now and
 * return the number of damaged buffers found so far.  Plain builds return an
 * error.  mbg_debug_write_past_end deliberately writes one double past v's
 * allocation (tests of the guard mechanism). */
int mbg_debug_guard_check(int64_t* violations);
int mbg_debug_write_past_end(mbg_mv* v);
/* Multi-GPU: join a communicator of `world` ranks (one process per GPU).
 * nccl_id is the 128-byte ncclUniqueId created by rank 0 (mbg_comm_unique_id)
 * and broadcast by the caller (e.g. torch.distributed). */
int mbg_comm_unique_id(unsigned char out_id[128]);
int mbg_ctx_init_comm(mbg_ctx* ctx, int rank, int world, const unsigned char nccl_id[128]);
/* Validation only: link `world` contexts on ONE device into an emulated
 * communicator (device copies + a sum kernel instead of NCCL, host barriers
 * between rank threads).  Drive each rank from its own host thread. */
int mbg_local_group_create(mbg_ctx** ctxs, int world);

/* ---- CSR matrix ----------------------------------------------------------
 * Square CSR, offsets int64[n+1], cols int32[nnz] strictly increasing per
 * row, vals fp64[nnz].  Validated like CsrMatrix::validate (csr.cpp:8-32). */
int mbg_csr_validate(int64_t n, const int64_t* offsets, const int32_t* cols, int64_t nnz);
int mbg_csr_upload(mbg_ctx* ctx, int64_t n, const int64_t* offsets, const int32_t* cols,
                   const double* vals, mbg_csr** out);
/* Partitioned upload for multi-GPU (one process per GPU): rows are split in
 * nparts contiguous blocks, part p owning global rows [bounds[p], bounds[p+1]);
 * this context's rank owns part my_part.  The full host CSR is given; the halo
 * plan (renumbered local CSR, per-peer send lists and receive windows,
 * interior / boundary row split) is built from its column pattern. */
int mbg_csr_upload_partitioned(mbg_ctx* ctx, int64_t n, const int64_t* offsets, const int32_t* cols,
                               const double* vals, int nparts, const int64_t* bounds, int my_part,
                               mbg_csr** out);
/* Host-only view of the same halo plan (no device): call once with
 * loc_off == NULL for the sizes, then with buffers of n_own+1, nnz_local,
 * n_halo, npeers and sum(peer_send_count) entries. */
int mbg_halo_plan(int64_t n, const int64_t* offsets, const int32_t* cols, const double* vals, int nparts,
                  const int64_t* bounds, int my_part, int64_t* n_own, int64_t* n_halo, int64_t* nnz_local,
                  int32_t* loc_off, int32_t* loc_col, double* loc_val, int64_t* halo_global, int* npeers,
                  int* peer_part, int64_t* peer_send_count, int32_t* peer_send_rows,
                  int64_t* peer_recv_offset, int64_t* peer_recv_count);
/* The same plan for A^T (rows = this part's columns of A, nonzeros in ascending
 * source row -- spmv_transpose's order, src/core/spmv.cpp:76-90): what
 * mbg_csr_upload_partitioned builds for IBiCGStab's f0 = A^T r0 across ranks. */
int mbg_transpose_halo_plan(int64_t n, const int64_t* offsets, const int32_t* cols, const double* vals, int nparts,
                            const int64_t* bounds, int my_part, int64_t* n_own, int64_t* n_halo,
                            int64_t* nnz_local, int32_t* loc_off, int32_t* loc_col, double* loc_val,
                            int64_t* halo_global, int* npeers, int* peer_part, int64_t* peer_send_count,
                            int32_t* peer_send_rows, int64_t* peer_recv_offset, int64_t* peer_recv_count);
/* Same as mbg_csr_upload but a row's column indices may come in any order
 * (each row is still summed in the given order; no duplicates checked
 * beyond range) -- for permuted operators P A P^T that keep every row's
 * original summation order. */
int mbg_csr_upload_any_order(mbg_ctx* ctx, int64_t n, const int64_t* offsets, const int32_t* cols,
                             const double* vals, mbg_csr** out);
/* Structured-grid hint (rows = nx*ny*nz lexicographic points, the GLOBAL
 * grid): an operator whose nonzeros all couple grid neighbours gets a stencil
 * twin (see mbg_csr_stencil_kind); a z-slab partition (whole planes per rank,
 * halo = the two neighbouring planes) gets one for its slab.  On one GPU,
 * long-row stencils (> 12 nonzeros per row) also get a brick-reordered copy
 * P A P^T (8x8x4 bricks; each row keeps its summation order) used for the m
 * the stencil twin does not cover.  Results are bitwise identical (exact dots). */
int mbg_csr_set_grid(mbg_ctx* ctx, mbg_csr* a, int nx, int ny, int nz);
/* mbg_csr_upload and mbg_csr_upload_partitioned detect a lexicographic 7- or
 * 27-point grid operator themselves (the longest row's column offsets give
 * nx, ny, nz; every row is then verified on the device), so the reference's
 * own calls -- CsrMatrix + core::spmv / solve, no grid argument anywhere --
 * reach the stencil twin; MBG_AUTO_GRID=0 turns the detection off and
 * mbg_csr_clear_grid drops a twin (A/B measurements of the CSR path). */
int mbg_csr_clear_grid(mbg_csr* a);
/* Host-only: the grid that detection would try for this matrix (0, 0, 0 = none;
 * no device needed -- the device then verifies every row before the twin is built). */
int mbg_infer_grid(int64_t n, const int64_t* offsets, const int32_t* cols, int* nx, int* ny, int* nz);
int mbg_csr_reordered(const mbg_csr* a);   /* 1 when the solver uses a reordered twin */
/* Stencil twin built at upload or by mbg_csr_set_grid when every nonzero couples a grid
 * point with itself or one of its 26 neighbours: 7 (face neighbours only) or
 * 27; 0 = none.  The SpMM then reads no column indices and stages x as TMA
 * plane boxes (m in {4, 8, 16, 32}; bitwise the CSR result; MBG_STENCIL=0 off). */
int mbg_csr_stencil_kind(const mbg_csr* a);
int mbg_csr_free(mbg_csr* a);
int64_t mbg_csr_rows(const mbg_csr* a);   /* local rows */
int64_t mbg_csr_nnz(const mbg_csr* a);    /* local nnz */
/* SpMM kernel choice made at upload (no reference counterpart; diagnostics):
 * staged = 1 when the gather-once tiling is in use (opt-in, MBG_SPMM_STAGE=1:
 * x rows reused inside tiles, e.g. 27-point stencils; measured slower than the
 * register gathers), reuse = nonzeros per distinct column per tile of that
 * tiling (0 if none). */
int mbg_csr_stage_info(const mbg_csr* a, int* staged, double* reuse);
/* sorted = 1 when the CSR SpMM (m >= 4) walks a length-sorted twin of the rows:
 * rows stored by descending length inside windows of 4096, in groups of 8
 * whose nonzeros lie batch-major (4 per batch, padded), each row's nonzeros in
 * CSR order: spmv.cpp:38-47's per-row sums are unchanged, only which lane
 * computes which row; lane_efficiency = share of the natural order's gather
 * slots that do useful work (the twin is built below 0.92, e.g. the random
 * band of BASELINE config 5; MBG_SPMM_SORT=0/1 forces it off/on). */
int mbg_csr_sort_info(const mbg_csr* a, int* sorted, double* lane_efficiency);
/* Host-only view of that twin's plan (no device).  rowid[nslots] = the row
 * stored in each slot (-1: padding of the last group; nslots <= n + 7: rows
 * of more than 240 nonzeros come last, one slot each, and go to the long-row
 * kernel); group_off[g] = first batch of group g (8 slots), n/8 + 2 entries;
 * tiles[4*ntiles] = (slot0, slot1, batch0, batch1) of whole groups, batch0 = -1
 * for a long row's slot.  Call with the array arguments NULL for the sizes. */
int mbg_sorted_twin_plan(int64_t n, const int64_t* offsets, int window, int64_t* nslots, int32_t* rowid,
                         double* lane_efficiency, int64_t* ntiles, int32_t* tiles, int32_t* group_off);

/* ---- multivector: n x m fp64, row-interleaved (element (i,c) at i*m+c) -- */
int mbg_mv_alloc(mbg_ctx* ctx, int64_t n, int m, mbg_mv** out);
int mbg_mv_free(mbg_mv* v);
int mbg_mv_upload(mbg_mv* v, const double* host);     /* n*m doubles */
int mbg_mv_download(const mbg_mv* v, double* host);   /* n*m doubles */
int mbg_mv_fill(mbg_mv* v, double value);
double* mbg_mv_device_ptr(mbg_mv* v);

/* ---- SpMV / SpMM --------------------------------------------------------
 * y(i,c) = sum_k A(i,k) x(k,c); throws invalid on shape mismatch or x == y
 * (spmv.cpp:20-25).  Enqueued on the context stream. */
int mbg_spmv(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* x, mbg_mv* y);
/* core::spmv_transpose (include/mbstab/core/spmv.hpp:19-21, src/core/spmv.cpp:76-90):
 * y = A^T x, every y(j, c) summed over source rows i in ascending order from
 * 0.0 (the reference's serial loop), bit for bit.  Partitioned matrices use
 * the A^T halo plan built at upload (the rank's rows of y = its columns of A). */
int mbg_spmv_transpose(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* x, mbg_mv* y);
double mbg_spmv_traffic_bytes(int64_t n, int64_t nnz, int m);           /* Eq. (3) */
double mbg_spmv_compulsory_bytes(int64_t n, int64_t nnz, int m);        /* x once */

/* ---- statement groups (statement.hpp:13-45) ------------------------------ */
#define MBG_STMT_UPDATE 0
#define MBG_STMT_DOT 1
typedef struct mbg_statement {
    int kind;                                  /* MBG_STMT_UPDATE / MBG_STMT_DOT */
    int out;                                   /* update: output vector id */
    int nterms;                                /* update: number of terms */
    int term_vec[MBG_MAX_TERMS];               /* update: operand vector ids */
    const double* term_coeff[MBG_MAX_TERMS];   /* update: host arrays of m coeffs */
    int left, right, slot;                     /* dot: operands and result slot */
} mbg_statement;

/* Traffic in whole-vector-transfer units (statement.cpp:25-56). */
int mbg_analyze_traffic(const mbg_statement* stmts, int nstmts, int* reads, int* writes);
/* split_basic(group) followed by analyze_traffic of each piece, summed
 * (statement.cpp:58-85); also returns the number of pieces. */
int mbg_split_basic_traffic(const mbg_statement* stmts, int nstmts, int first_temp_id,
                            int* reads, int* writes, int* ngroups);
/* Single-pass fused execution on the GPU (execute.cpp:123-172).
 * vectors[id] are device multivectors of identical shape; dot_results is a
 * HOST array of nslots*m doubles: slot s, column c at s*m+c (exact dots). */
int mbg_execute_group(mbg_ctx* ctx, const mbg_statement* stmts, int nstmts, mbg_mv* const* vectors,
                      int nvectors, double* dot_results, int nslots);

/* ---- solver --------------------------------------------- */
#define MBG_BICGSTAB 0
#define MBG_RBICGSTAB 1       /* preconditioned (Alg. 6) */
#define MBG_PIPEBICGSTAB 2
#define MBG_IBICGSTAB 3       /* Improved, Alg. 3; f0 = A^T r0 through a local A^T + its halo plan when partitioned */
#define MBG_PBICGSTAB 4       /* preconditioned, Alg. 5 */
#define MBG_PPIPEBICGSTAB 5   /* preconditioned Pipelined, Alg. 7 */
#define MBG_MERGED 0
#define MBG_BASIC 1
/* Merged + beyond-paper fusions: dots fused
 * into the SpMM epilogue, identity-M^-1 copies elided (Reordered), Alg. 4
 * lines 7+12 in one pass (Pipelined).  Bitwise the same results as merged. */
#define MBG_FUSED 2

typedef struct mbg_report {
    int iterations;
    int converged;
    int breakdown;          /* 0 none; 1 alpha (delta), 2 omega, 3 beta */
    int breakdown_iter;
    int breakdown_col;
    /* traffic counted like TrafficCounter (types.hpp:95-109) */
    int64_t vector_reads;
    int64_t vector_writes;
    double spmv_bytes;          /* Eq. (3) */
    double compulsory_bytes;    /* roofline byte model */
    int64_t reductions;         /* reduction points executed */
    int64_t gpu_launches;       /* kernels launched by the solve loop */
    double loop_ms;             /* device time of the iteration loop */
} mbg_report;

/* X holds x0 on entry and the solution on exit.  hist: host array of
 * (max_iters+1)*m doubles or NULL; row j = relative recursive residual h_j.
 * fixed != 0: run exactly max_iters iterations (benchmark mode). */
int mbg_solve(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method,
              int formulation, double tol, int fixed, int max_iters, double* hist,
              mbg_report* report);
/* True relative residual per column, out[c] = ||b - A x||_2 / ||b||_2 (the
 * SolveReport's recomputed residual), exact dots. */
int mbg_true_residual(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, const mbg_mv* x, double* out);

/* Explicit preconditioner: precond_alpha 0 = none (required
 * by BiCGStab, IBiCGStab, PipeBiCGStab), 2 = identity M^-1 (one copy per
 * application), even alpha >= 4 = synthetic(alpha): alpha/2 scale passes by
 * 2.0 / 0.5 whose product is exactly 1 (alpha transfers per application).
 * The preconditioned methods (RBiCGStab, PBiCGStab, PPipeBiCGStab) require
 * alpha >= 2; mbg_solve passes 2 for them and 0 otherwise. */
int mbg_solve_pc(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method,
                 int formulation, int precond_alpha, double tol, int fixed, int max_iters,
                 double* hist, mbg_report* report);
/* Same solve with HOST b/x buffers (n*m doubles): uploads b and x0, solves,
 * downloads x.  The reference-facing end-to-end entry point. */
int mbg_solve_host(mbg_ctx* ctx, const mbg_csr* a, int m, const double* b_host, double* x_host,
                   int method, int formulation, double tol, int fixed, int max_iters,
                   double* hist, mbg_report* report);

/* Page-locked host buffers for mbg_solve_host / mbg_mv_upload-style traffic:
 * pinned b / x are DMA'd directly at link rate (55 GB/s on the GPU box);
 * pageable ones go through an internal pinned staging pipeline. */
int mbg_host_alloc(size_t bytes, void** out);
int mbg_host_free(void* p);

/* Profiling solve (bench.py roofline): identical numerics, launched without a
 * graph with CUDA events around every kernel of the iteration loop; writes
 * {"label": [launches, total_ms, algorithmic_bytes_per_launch], ...} to json. */
int mbg_solve_profile(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method,
                      int formulation, double tol, int fixed, int max_iters, char* json, int cap,
                      mbg_report* report);

/* Per-iteration schedule totals: vector reads/writes,
 * SpMVs, reduction points and dots per reduction (up to 8 entries). */
int mbg_method_schedule(int method, int formulation, int* reads, int* writes, int* spmvs,
                        int* nreductions, int* dots_per_reduction);
/* SPEC.md:236-244 form: vector transfers WITHOUT preconditioner traffic (e.g.
 * PPipeBiCGStab merged 34) plus the M^-1 applications per iteration (each
 * costs precond_alpha transfers; 0 when the fused formulation elides identity
 * copies).  mbg_method_schedule above = this + 2 transfers per identity copy. */
int mbg_method_schedule_pc(int method, int formulation, int precond_alpha, int* reads, int* writes,
                           int* spmvs, int* precond_applications, int* nreductions,
                           int* dots_per_reduction);

/* ---- MatrixMarket ingest (host; core::read_matrix_market / write_matrix_market,
 * proj/src/core/matrix_market.cpp:38-113,121-133) ------------
 * mbg_mm_read parses a coordinate real/integer, general/symmetric file (all
 * host threads) into a host CSR held by *handle: n, nnz returned; errors are
 * the reference's "<name>:<line>: message" (MBG_ERR_RUNTIME).  Symmetric
 * files are expanded, duplicates summed (file order), rows sorted by column.
 * mbg_mm_copy fills caller arrays (offsets n+1, cols/vals nnz; any may be
 * NULL); mbg_mm_free releases the handle.  The arrays feed mbg_csr_upload or
 * mbg_csr_upload_partitioned (general halo plan) unchanged. */
int mbg_mm_read(const char* path, void** handle, int64_t* n, int64_t* nnz);
int mbg_mm_copy(const void* handle, int64_t* offsets, int32_t* cols, double* vals);
void mbg_mm_free(void* handle);
/* "matrix coordinate real general", 1-based, values printed with %.17g. */
int mbg_mm_write(const char* path, int64_t n, const int64_t* offsets, const int32_t* cols,
                 const double* vals);

/* ---- fusion micro-benchmark (Fig. 2 / Table 1)
 * Runs #1 (three passes, 9N transfers), #2 (two updates merged, 5N) and #3
 * (three updates merged, 5N) over n doubles, each timed over reps launches with
 * CUDA events.  ms_per_run[3], gbs_per_run[3] (may be NULL); identical = 1 when
 * run #3 reproduced run #1's y and z bit for bit. */
int mbg_fusion_bench(mbg_ctx* ctx, int64_t n, int reps, double* ms_per_run, double* gbs_per_run,
                     int* identical);

/* ---- config generators (host) --------------------------------------------
 * kind 0 Poisson 7-pt (gen_poisson_7pt), 1 conv-diff 7-pt, 2 27-pt perturbed,
 * 3 Poisson 5-pt (gen_poisson_5pt, generators.cpp:69-91; nz must be 1).
 * Two-phase: call with NULL cols/vals to get nnz (offsets may be NULL too). */
int mbg_gen_stencil(int kind, int nx, int ny, int nz, uint64_t seed, int64_t* nnz,
                    int64_t* offsets, int32_t* cols, double* vals);
int mbg_gen_banded(int64_t n, int64_t band, int kmin, int kmax, uint64_t seed, int64_t* nnz,
                   int64_t* offsets, int32_t* cols, double* vals);
int mbg_gen_rhs(int64_t n, int m, uint64_t seed, double* b);

/* ---- exact-dot limb format (host hooks for partition tests) ----------------
 * A slot is mbg_exact_slot_words() int64 words per column.  accumulate adds
 * RN(a(i,c)*b(i,c)) exactly into D[c]; slots from different row ranges or
 * ranks combine by int64 addition; round gives the correctly rounded sum. */
int mbg_exact_slot_words(void);
int mbg_exact_accumulate_host(int64_t n, int m, const double* a, const double* b, int64_t* D);
int mbg_exact_round_host(const int64_t* D, int count, double* out);

/* number of kernels this context has launched (telemetry) */
int64_t mbg_ctx_launches(const mbg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
