// comm.hpp -- multi-GPU plumbing: NCCL communicator, fused dot allreduce and
// the halo-exchanging distributed SpMM (row partition).
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace mbg {

// y = A x on this rank's rows.  x must have room for the halo rows after the
// owned rows.  Single GPU: one SpMM launch.  Partitioned: pack + NCCL
// send/recv of the boundary rows on the side stream while the interior rows
// are multiplied on the main stream, then the boundary rows.  Returns the
// number of kernels launched.
struct SpmmEpi;
int apply_operator(mbg_ctx* ctx, const mbg_csr* a, int m, double* x, double* y, const int* ctl,
                   const SpmmEpi* epi = nullptr);

// Sum int64 limbs over all ranks (exact, order-independent).  join=false
// leaves the allreduce in flight on the side stream so the main stream's next
// kernels (the Pipelined SpMM, the Reordered copy) overlap it; comm_join()
// makes the main stream wait for it before the slots are read.
void comm_allreduce_i64(mbg_ctx* ctx, int64_t* buf, size_t count, cudaStream_t st, bool join = true);
void comm_join(mbg_ctx* ctx);
void comm_barrier(mbg_ctx* ctx);
void comm_destroy(mbg_ctx* ctx);
bool comm_is_local(const mbg_ctx* ctx);   // single-GPU emulation (no graph capture)

// Host-side partition / halo plan (plan.cpp).  Rows [begin[p], begin[p+1])
// belong to part p.  Local numbering: owned rows 0..n_own-1, then halo rows
// grouped by owner part (ascending), ascending global index inside a group.
struct HaloPlan {
    int64_t n_own = 0, n_halo = 0, nnz = 0;
    std::vector<int32_t> off;            // n_own+1 (local CSR, int32)
    std::vector<int32_t> col;            // nnz (local numbering)
    std::vector<double> val;
    std::vector<int64_t> halo_global;    // n_halo global ids
    std::vector<int32_t> interior, boundary;
    struct Peer {
        int part;
        std::vector<int32_t> send_rows;  // local owned rows to send (ascending global)
        int64_t recv_offset = 0, recv_count = 0;
    };
    std::vector<Peer> peers;             // parts we exchange with (ascending)
};
HaloPlan build_halo_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val,
                         int nparts, const int64_t* begin, int my_part);
// The same for A^T (rows = owned columns of A, nonzeros in ascending source row).
HaloPlan build_transpose_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val,
                              int nparts, const int64_t* begin, int my_part);

}  // namespace mbg
