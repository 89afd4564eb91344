// common.hpp -- shared host-side plumbing of the B200 library: error
// handling across the C ABI, CUDA checks and the context / container structs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

#include "mbstab_b200.h"

namespace mbg {

// The reference throws std::invalid_argument for API misuse (spmv.cpp:20-25,
// execute.cpp:42-82, csr.cpp:8-32) and the C ABI maps it to MBG_ERR_INVALID.
struct Invalid : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct Breakdown : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);

#define MBG_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess)                                                                \
            (void)cudaGetLastError(), /* do not leak the error into later launches */         \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(_e) +    \
                                     " at " __FILE__ ":" + std::to_string(__LINE__) + ": " #call); \
    } while (0)

// Device buffer with RAII.
template <class T>
struct DevBuf;

#ifdef MBG_CHECKED
// Checked builds (make checked -> libmbstab_b200_checked.so; MBG_CHECKED=1
// selects it in the Python binding): every device allocation carries guard
// zones of GUARD_BYTES filled with GUARD_BYTE on both sides; they are verified
// when the buffer is freed and on demand (mbg_debug_guard_check), so an
// out-of-bounds write by any kernel is caught -- the substitute for
// compute-sanitizer memcheck, which this GPU pool does not allow.
constexpr size_t GUARD_BYTES = 64u << 10;
constexpr unsigned char GUARD_BYTE = 0xA5;
void* guarded_alloc(size_t bytes);     // returns the user pointer
void guarded_free(void* user);         // verifies, then frees
#endif

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
#ifdef MBG_CHECKED
        if (count) p = static_cast<T*>(guarded_alloc(count * sizeof(T)));
#else
        if (count) MBG_CUDA(cudaMalloc(&p, count * sizeof(T)));
#endif
        n = count;
    }
    void ensure(size_t count) { if (count > n) alloc(count); }
    void release() {
#ifdef MBG_CHECKED
        if (p) guarded_free(p);
#else
        if (p) cudaFree(p);
#endif
        p = nullptr;
        n = 0;
    }
};

struct Comm;        // comm.cu
struct StencilOp;   // stencil.hpp

}  // namespace mbg

// ---- ABI objects ------------------------------------------------------------
struct mbg_ctx {
    int device = 0;
    int num_sms = 0;                 // SMs the persistent grids are sized for
    int num_sms_device = 0;          // SMs of the device (num_sms + those reserved for NCCL)
    cudaStream_t stream = nullptr;   // main stream: all hot-path kernels
    cudaStream_t side = nullptr;     // side stream: overlapped reductions / halo
    mbg::Comm* comm = nullptr;       // multi-GPU communicator (nullptr: single GPU)
    // scratch for the API-level execute_group (reduction buffers)
    mbg::DevBuf<int64_t> scratch_i64;
    mbg::DevBuf<double> scratch_f64;
    mbg::DevBuf<int> scratch_ctl;
    int64_t launches = 0;            // kernels launched by this context
    bool small_path = true;          // one-launch loop for small classical solves (small.cu)
    // pool of large work vectors reused across solves (no cudaMalloc per solve)
    std::vector<mbg::DevBuf<double>> pool;
    // pinned host memory reused across calls: control-word snapshots and the
    // staging buffer of the host-buffer entry points
    int* ctl_host = nullptr;        // 64 ints
    unsigned char* stage = nullptr;
    size_t stage_bytes = 0;
};

namespace mbg {
inline DevBuf<double> pool_take(mbg_ctx* ctx, size_t n) {
    for (size_t i = 0; i < ctx->pool.size(); ++i) {
        if (ctx->pool[i].n >= n && ctx->pool[i].n <= 2 * n + (1u << 20)) {
            DevBuf<double> b = std::move(ctx->pool[i]);
            ctx->pool.erase(ctx->pool.begin() + static_cast<long>(i));
            return b;
        }
    }
    return DevBuf<double>(n);
}
inline void pool_give(mbg_ctx* ctx, DevBuf<double>&& b) {
    if (b.p) ctx->pool.push_back(std::move(b));
}
}  // namespace mbg

// Device CSR.  Offsets are stored int32 when nnz < 2^31 (the byte model's
// 4-byte offsets, Eq. (3)); cols int32, vals fp64.  For a row partition the
// local matrix has n_local rows and its columns are renumbered into the local
// x layout [owned rows | halo rows] (see halo.cu).
struct mbg_csr {
    mbg_ctx* ctx = nullptr;
    int device = 0;           // owning device (freeing must not touch ctx)
    int64_t n_global = 0;
    int64_t n = 0;            // local rows
    int64_t nnz = 0;          // local nnz
    int64_t row_begin = 0;    // first owned global row
    mbg::DevBuf<int32_t> off;
    mbg::DevBuf<int32_t> col;
    mbg::DevBuf<double> val;
    // multi-GPU halo plan (empty for a single GPU)
    int64_t n_halo = 0;                       // halo rows appended after the owned rows
    mbg::DevBuf<int32_t> interior_rows;       // rows whose columns are all owned
    mbg::DevBuf<int32_t> boundary_rows;       // rows touching halo columns
    int64_t n_interior = 0, n_boundary = 0;
    // SpMM tile plans (spmm.cu): all rows, interior rows, boundary rows
    mbg::DevBuf<int4> tiles_all, tiles_interior, tiles_boundary;
    mbg::DevBuf<int32_t> long_all, long_interior, long_boundary;   // rows beyond a tile's capacity
    // gather-once tilings (stencil-like matrices; empty when not worth it)
    mbg::DevBuf<int4> stiles_all, stiles_interior, stiles_boundary;
    mbg::DevBuf<int2> umeta_all, umeta_interior, umeta_boundary;
    mbg::DevBuf<int32_t> ucols_all, ucols_interior, ucols_boundary;
    mbg::DevBuf<uint16_t> lcol_all, lcol_split;    // per nonzero, for the all / interior+boundary tilings
    double stage_reuse = 0.0;
    // length-sorted twins of the row classes (spmm.cu build_sorted_twin): built
    // when the natural row order leaves warps waiting on their longest row
    struct SortedDev {
        mbg::DevBuf<int32_t> off, col, rowid, long_rows;
        mbg::DevBuf<double> val;
        mbg::DevBuf<int4> tiles;
        mbg::DevBuf<int> sched;               // {next tile, finished blocks}, self-rewinding
    };
    SortedDev sorted_all, sorted_interior, sorted_boundary;
    double lane_efficiency = 1.0;             // spmm_lane_efficiency of the natural order
    struct Peer {
        int rank;
        int64_t send_count, recv_count;
        int64_t recv_offset;                  // first halo slot for this peer
        mbg::DevBuf<int32_t> send_rows;       // local rows packed for this peer
    };
    std::vector<Peer> peers;
    std::unique_ptr<mbg_csr> transposed;      // A^T, built on first use (IBiCGStab f0 = A^T r0)
    // locality reordering (mbg_csr_set_grid): P A P^T with every row's
    // nonzeros in their original order, and perm[new] = old row
    std::unique_ptr<mbg_csr> reordered;
    mbg::DevBuf<int32_t> perm;
    std::vector<int32_t> perm_host;
    // structured-grid twin (mbg_csr_set_grid; stencil.cu): implicit columns
    std::shared_ptr<mbg::StencilOp> stencil;
};

struct mbg_mv {
    mbg_ctx* ctx = nullptr;
    int device = 0;
    int64_t n = 0;        // rows (owned)
    int64_t n_alloc = 0;  // rows allocated (owned + halo capacity)
    int m = 0;
    mbg::DevBuf<double> data;
};
