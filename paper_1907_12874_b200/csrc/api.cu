// api.cpp -- the C ABI (include/mbstab_b200.h): context, containers, SpMV,
// execute_group and solve.  No exception crosses the boundary; invalid usage
// maps to MBG_ERR_INVALID with the reference's message text.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "comm.hpp"
#include "common.hpp"
#include "kernels.hpp"
#include "solver.hpp"
#include "stencil.hpp"

namespace mbg {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return MBG_OK;
    } catch (const Invalid& e) {
        set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const Breakdown& e) {
        set_error(e.what());
        return MBG_ERR_BREAKDOWN;
    } catch (const std::exception& e) {
        set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

static void use(mbg_ctx* ctx) {
    if (!ctx) throw Invalid("null context");
    MBG_CUDA(cudaSetDevice(ctx->device));
}

// CsrMatrix::validate (csr.cpp:8-32), same messages.
static void validate_csr(int64_t n, const int64_t* off, const int32_t* col, int64_t nnz, bool sorted = true) {
    if (n < 0) throw Invalid("csr: negative row count");
    if (!off) throw Invalid("csr: row_offsets length must be n_rows+1");
    if (off[0] != 0) throw Invalid("csr: row_offsets[0] must be 0");
    if (off[n] != nnz) throw Invalid("csr: row_offsets back must equal nnz");
    for (int64_t i = 0; i < n; ++i) {
        if (off[i] > off[i + 1])
            throw Invalid("csr: row_offsets not non-decreasing at row " + std::to_string(i));
        for (int64_t k = off[i]; k < off[i + 1]; ++k) {
            const int32_t c = col[k];
            if (c < 0 || c >= n) throw Invalid("csr: column index out of range in row " + std::to_string(i));
            if (sorted && k > off[i] && col[k - 1] >= c)
                throw Invalid("csr: column indices not strictly increasing in row " + std::to_string(i));
        }
    }
}

template <class T>
static void upload(DevBuf<T>& d, const T* h, size_t n, cudaStream_t st) {
    d.alloc(n);
    if (n) MBG_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

}  // namespace mbg

using namespace mbg;

extern "C" const char* mbg_last_error(void) { return g_error.c_str(); }
extern "C" const char* mbg_version(void) { return "mbstab_b200 0.1 (sm_100a)"; }

extern "C" int mbg_ctx_create(int device, mbg_ctx** out) {
    return guarded([&] {
        if (!out) throw Invalid("null output");
        int ndev = 0;
        MBG_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw Invalid("ctx_create: no such CUDA device");
        MBG_CUDA(cudaSetDevice(device));
        auto* c = new mbg_ctx();
        c->device = device;
        MBG_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        c->num_sms_device = c->num_sms;
        MBG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        MBG_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        *out = c;
    });
}

extern "C" int mbg_ctx_destroy(mbg_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->side);
        comm_destroy(ctx);
        ctx->scratch_i64.release();
        ctx->scratch_f64.release();
        ctx->scratch_ctl.release();
        ctx->pool.clear();
        if (ctx->ctl_host) cudaFreeHost(ctx->ctl_host);
        if (ctx->stage) cudaFreeHost(ctx->stage);
        cudaStreamDestroy(ctx->stream);
        cudaStreamDestroy(ctx->side);
        delete ctx;
    });
}

extern "C" int mbg_ctx_synchronize(mbg_ctx* ctx) {
    return guarded([&] {
        use(ctx);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        MBG_CUDA(cudaStreamSynchronize(ctx->side));
    });
}

extern "C" int mbg_csr_validate(int64_t n, const int64_t* off, const int32_t* col, int64_t nnz) {
    return guarded([&] { validate_csr(n, off, col, nnz); });
}

// Gather-once SpMM tilings (spmm.cu spmm_stage_kernel), for tiles that reuse
// x rows (>= 2 nonzeros per distinct column, e.g. 27-point stencils): opt-in
// with MBG_SPMM_STAGE=1 (tests, A/B measurements; measured slower).
static int stage_mode() {
    const char* e = std::getenv("MBG_SPMM_STAGE");
    return e ? std::atoi(e) : -1;
}

static void stage_tilings(mbg_ctx* ctx, mbg_csr* a, const std::vector<int32_t>& off32, const int32_t* col,
                          const std::vector<int32_t>* all, const std::vector<int32_t>* interior,
                          const std::vector<int32_t>* boundary) {
    const int mode = stage_mode();
    if (mode != 1) return;   // opt-in (measured slower): no O(nnz) host pass at every upload
    const int64_t ncols = a->n + a->n_halo;
    std::vector<uint16_t> lcol(static_cast<size_t>(a->nnz) + 16, 0);
    if (all) {
        StageTiling st;
        if (!build_stage_tiles(off32, col, *all, ncols, lcol, st)) return;
        a->stage_reuse = st.reuse;
        if (mode != 1) return;
        upload(a->stiles_all, st.tiles.data(), st.tiles.size(), ctx->stream);
        upload(a->umeta_all, st.umeta.data(), st.umeta.size(), ctx->stream);
        upload(a->ucols_all, st.ucols.data(), st.ucols.size(), ctx->stream);
        upload(a->lcol_all, lcol.data(), lcol.size(), ctx->stream);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
        StageTiling si, sb;
        if (!build_stage_tiles(off32, col, *interior, ncols, lcol, si)) return;
        if (!build_stage_tiles(off32, col, *boundary, ncols, lcol, sb)) return;
        a->stage_reuse = si.reuse;
        if (mode != 1) return;
        upload(a->stiles_interior, si.tiles.data(), si.tiles.size(), ctx->stream);
        upload(a->umeta_interior, si.umeta.data(), si.umeta.size(), ctx->stream);
        upload(a->ucols_interior, si.ucols.data(), si.ucols.size(), ctx->stream);
        upload(a->stiles_boundary, sb.tiles.data(), sb.tiles.size(), ctx->stream);
        upload(a->umeta_boundary, sb.umeta.data(), sb.umeta.size(), ctx->stream);
        upload(a->ucols_boundary, sb.ucols.data(), sb.ucols.size(), ctx->stream);
        upload(a->lcol_split, lcol.data(), lcol.size(), ctx->stream);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
}

// Length-sorted twin of one row class (spmm.cu): built when fewer than 92 % of
// the natural order's gather slots do useful work (rows of widely different
// lengths side by side, e.g. the random band of BASELINE config 5; stencil
// operators stay above 0.97).  MBG_SPMM_SORT=0 / 1 forces it off / on,
// MBG_SPMM_SORT_WINDOW sets the sorting window (rows; default 4096).
static int sort_mode() {
    const char* e = std::getenv("MBG_SPMM_SORT");
    return e ? std::atoi(e) : -1;
}

static void sorted_twin_to_device(mbg_ctx* ctx, mbg_csr* a, mbg_csr::SortedDev& d, const std::vector<int32_t>& off32,
                                  const int32_t* col, const double* val, const std::vector<int32_t>& rows) {
    const int mode = sort_mode();
    if (mode == 0 || rows.empty()) return;
    const double eff = spmm_lane_efficiency(off32, rows);
    a->lane_efficiency = std::min(a->lane_efficiency, eff);
    if (mode != 1 && eff >= 0.92) return;
    int window = 4096;
    if (const char* e = std::getenv("MBG_SPMM_SORT_WINDOW")) window = std::max(64, std::atoi(e));
    SortedTwin t;
    build_sorted_twin(off32, col, val, rows, window, t);
    constexpr int PAD = 8;   // the tile kernel's bulk copies round ranges up
    t.off.resize(t.off.size() + PAD, t.off.back());
    t.col.resize(t.col.size() + PAD, 0);
    t.val.resize(t.val.size() + PAD, 0.0);
    upload(d.off, t.off.data(), t.off.size(), ctx->stream);
    upload(d.col, t.col.data(), t.col.size(), ctx->stream);
    upload(d.val, t.val.data(), t.val.size(), ctx->stream);
    upload(d.rowid, t.rowid.data(), t.rowid.size(), ctx->stream);
    upload(d.tiles, t.tiles.data(), t.tiles.size(), ctx->stream);
    upload(d.long_rows, t.long_rows.data(), t.long_rows.size(), ctx->stream);
    d.sched.alloc(2);
    MBG_CUDA(cudaMemsetAsync(d.sched.p, 0, 2 * sizeof(int), ctx->stream));
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));   // t's vectors are the copy sources
}

// Upload a (local) CSR with int32 offsets.  Arrays are padded by 8 entries so
// the SpMM's 16-byte-aligned TMA bulk copies may round a tile's range up.
static void csr_arrays_to_device(mbg_ctx* ctx, mbg_csr* a, int64_t n, const std::vector<int32_t>& off32,
                                 const int32_t* col, const double* val, int64_t nnz) {
    constexpr int PAD = 8;
    std::vector<int32_t> o(off32);
    o.resize(off32.size() + PAD, off32.back());
    upload(a->off, o.data(), o.size(), ctx->stream);
    a->col.alloc(static_cast<size_t>(nnz) + PAD);
    a->val.alloc(static_cast<size_t>(nnz) + PAD);
    MBG_CUDA(cudaMemsetAsync(a->col.p, 0, (nnz + PAD) * sizeof(int32_t), ctx->stream));
    MBG_CUDA(cudaMemsetAsync(a->val.p, 0, (nnz + PAD) * sizeof(double), ctx->stream));
    if (nnz) {
        MBG_CUDA(cudaMemcpyAsync(a->col.p, col, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        MBG_CUDA(cudaMemcpyAsync(a->val.p, val, nnz * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    a->n = n;
    a->nnz = nnz;
    std::vector<int32_t> all(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) all[i] = static_cast<int32_t>(i);
    auto t = build_spmm_tiles(off32, all);
    upload(a->tiles_all, t.data(), t.size(), ctx->stream);
    auto lr = long_rows_of(t);
    upload(a->long_all, lr.data(), lr.size(), ctx->stream);
    stage_tilings(ctx, a, off32, col, &all, nullptr, nullptr);
    sorted_twin_to_device(ctx, a, a->sorted_all, off32, col, val, all);
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));
}

namespace mbg {
struct HostCsr {
    std::vector<int32_t> off, col;
    std::vector<double> val;
};

static HostCsr download_csr(mbg_ctx* ctx, const mbg_csr* a) {
    HostCsr h;
    h.off.resize(static_cast<size_t>(a->n) + 1);
    h.col.resize(static_cast<size_t>(a->nnz));
    h.val.resize(static_cast<size_t>(a->nnz));
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    MBG_CUDA(cudaMemcpy(h.off.data(), a->off.p, h.off.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (a->nnz) {
        MBG_CUDA(cudaMemcpy(h.col.data(), a->col.p, h.col.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
        MBG_CUDA(cudaMemcpy(h.val.data(), a->val.p, h.val.size() * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return h;
}

static std::unique_ptr<mbg_csr> make_device_csr(mbg_ctx* ctx, int64_t n, const HostCsr& h) {
    auto t = std::make_unique<mbg_csr>();
    t->ctx = ctx;
    t->device = ctx->device;
    t->n_global = n;
    csr_arrays_to_device(ctx, t.get(), n, h.off, h.col.data(), h.val.data(), static_cast<int64_t>(h.col.size()));
    return t;
}

// Transpose by a stable counting sort over rows in ascending order: row j of
// A^T lists its source rows in the order they are visited.
static HostCsr transpose_host(int64_t n, const HostCsr& a) {
    HostCsr t;
    const int64_t nnz = static_cast<int64_t>(a.col.size());
    t.off.assign(static_cast<size_t>(n) + 1, 0);
    t.col.resize(static_cast<size_t>(nnz));
    t.val.resize(static_cast<size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) ++t.off[static_cast<size_t>(a.col[k]) + 1];
    for (int64_t j = 0; j < n; ++j) t.off[j + 1] += t.off[j];
    std::vector<int32_t> pos(t.off.begin(), t.off.end() - 1);
    for (int64_t i = 0; i < n; ++i)
        for (int32_t k = a.off[i]; k < a.off[i + 1]; ++k) {
            const int32_t q = pos[a.col[k]]++;
            t.col[q] = static_cast<int32_t>(i);
            t.val[q] = a.val[k];
        }
    return t;
}

// P A P^T: row `nw` of the result is row order[nw] of A with its nonzeros in
// their original order and columns renumbered by pos (= order^-1).
static HostCsr permute_host(int64_t n, const HostCsr& a, const std::vector<int32_t>& order,
                            const std::vector<int32_t>& pos) {
    HostCsr p;
    p.off.assign(static_cast<size_t>(n) + 1, 0);
    for (int64_t nw = 0; nw < n; ++nw) {
        const int32_t o = order[nw];
        p.off[nw + 1] = p.off[nw] + (a.off[o + 1] - a.off[o]);
    }
    p.col.resize(a.col.size());
    p.val.resize(a.val.size());
    for (int64_t nw = 0; nw < n; ++nw) {
        const int32_t o = order[nw];
        int32_t q = p.off[nw];
        for (int32_t k = a.off[o]; k < a.off[o + 1]; ++k, ++q) {
            p.col[q] = pos[a.col[k]];
            p.val[q] = a.val[k];
        }
    }
    return p;
}

// A^T for IBiCGStab's f0 = A^T r0 (core::spmv_transpose, spmv.cpp:76-90): the
// stable counting sort keeps the reference's ascending-row summation order,
// so the ordinary SpMM on A^T adds the terms of y_j in exactly the reference's
// serial order.  For a reordered operator the transpose is built from the
// ORIGINAL matrix (same order of terms) and then permuted.  Cached on A.
const mbg_csr* csr_transpose(mbg_ctx* ctx, const mbg_csr* a) {
    auto* am = const_cast<mbg_csr*>(a);
    if (am->transposed) return am->transposed.get();
    HostCsr t = transpose_host(a->n, download_csr(ctx, a));
    am->transposed = make_device_csr(ctx, a->n, t);
    return am->transposed.get();
}

const mbg_csr* csr_transpose_reordered(mbg_ctx* ctx, const mbg_csr* orig) {
    auto* r = orig->reordered.get();
    if (r->transposed) return r->transposed.get();
    HostCsr t = transpose_host(orig->n, download_csr(ctx, orig));
    std::vector<int32_t> pos(orig->perm_host.size());
    for (size_t nw = 0; nw < pos.size(); ++nw) pos[orig->perm_host[nw]] = static_cast<int32_t>(nw);
    r->transposed = make_device_csr(ctx, orig->n, permute_host(orig->n, t, orig->perm_host, pos));
    return r->transposed.get();
}
}  // namespace mbg

static void csr_to_device(mbg_ctx* ctx, mbg_csr* a, int64_t n, const int64_t* off, const int32_t* col,
                          const double* val) {
    const int64_t nnz = off[n];
    if (nnz > INT32_MAX - 64) throw Invalid("csr: nnz >= 2^31 needs 64-bit offsets (not supported)");
    std::vector<int32_t> off32(n + 1);
    for (int64_t i = 0; i <= n; ++i) off32[i] = static_cast<int32_t>(off[i]);
    csr_arrays_to_device(ctx, a, n, off32, col, val, nnz);
}

// Structured-grid detection at upload (the reference's operator API has no
// grid call: a maintainer who swaps core::spmv / solve gets the stencil twin
// without one).  The longest row of a lexicographic 7- or 27-point operator
// is an interior point whose column offsets spell the grid: {+-1, +-nx,
// +-nx*ny} or dz*nx*ny + dy*nx + dx.  The guess is then verified against
// every row on the device (build_stencil); anything else keeps the CSR path.
// MBG_AUTO_GRID=0 turns the detection off.
static bool infer_grid(int64_t n, const int64_t* off, const int32_t* col, int& nx, int& ny, int& nz) {
    if (const char* e = std::getenv("MBG_AUTO_GRID"))
        if (e[0] == '0') return false;
    if (n < 27) return false;
    int64_t best = 0, len = 0;
    for (int64_t i = 0; i < n; ++i)
        if (off[i + 1] - off[i] > len) {
            len = off[i + 1] - off[i];
            best = i;
        }
    if (len != 7 && len != 27) return false;
    std::vector<int64_t> pos;   // the positive offsets, ascending (columns are sorted)
    for (int64_t k = off[best]; k < off[best + 1]; ++k) {
        const int64_t d = col[k] - best;
        if (d > 0) pos.push_back(d);
    }
    const size_t half = static_cast<size_t>(len / 2);
    if (pos.size() != half || col[off[best] + static_cast<int64_t>(half)] != best) return false;
    for (size_t i = 0; i < half; ++i)   // symmetric pattern
        if (col[off[best] + static_cast<int64_t>(half) - 1 - static_cast<int64_t>(i)] - best != -pos[i]) return false;
    const int64_t gx = len == 7 ? pos[1] : pos[2], gxy = len == 7 ? pos[2] : pos[8];
    if (pos[0] != 1 || gx < 3 || gxy % gx || n % gxy || gxy / gx < 3 || n / gxy < 3 || gx > INT32_MAX) return false;
    if (len == 27) {
        const int64_t want[13] = {1, gx - 1, gx, gx + 1, gxy - gx - 1, gxy - gx, gxy - gx + 1, gxy - 1, gxy, gxy + 1,
                                  gxy + gx - 1, gxy + gx, gxy + gx + 1};
        for (int i = 0; i < 13; ++i)
            if (pos[static_cast<size_t>(i)] != want[i]) return false;
    }
    nx = static_cast<int>(gx);
    ny = static_cast<int>(gxy / gx);
    nz = static_cast<int>(n / gxy);
    return true;
}

// Host-only: the grid the upload would try for this matrix (0 = none).  The
// guess is verified on the device before the stencil twin is built.
extern "C" int mbg_infer_grid(int64_t n, const int64_t* off, const int32_t* col, int* nx, int* ny, int* nz) {
    return guarded([&] {
        if (n < 0 || !off || !nx || !ny || !nz) throw Invalid("infer_grid: null argument");
        if (n > 0 && !col) throw Invalid("infer_grid: null columns");
        *nx = *ny = *nz = 0;
        int x = 0, y = 0, z = 0;
        if (infer_grid(n, off, col, x, y, z)) {
            *nx = x;
            *ny = y;
            *nz = z;
        }
    });
}

static void detect_grid(mbg_ctx* ctx, mbg_csr* a, int64_t n, const int64_t* off, const int32_t* col) {
    int nx = 0, ny = 0, nz = 0;
    if (a->stencil || !infer_grid(n, off, col, nx, ny, nz)) return;
    a->stencil = build_stencil(ctx, a, nx, ny, nz);   // nullptr unless every row fits the grid
}

extern "C" int mbg_csr_clear_grid(mbg_csr* a) {
    return guarded([&] {
        if (!a) throw Invalid("clear_grid: null matrix");
        a->stencil.reset();
    });
}

extern "C" int mbg_csr_upload(mbg_ctx* ctx, int64_t n, const int64_t* off, const int32_t* col,
                              const double* val, mbg_csr** out) {
    return guarded([&] {
        use(ctx);
        if (!out) throw Invalid("null output");
        validate_csr(n, off, col, off ? off[n] : 0);
        auto* a = new mbg_csr();
        try {
            a->ctx = ctx;
            a->device = ctx->device;
            a->n_global = n;
            csr_to_device(ctx, a, n, off, col, val);
            detect_grid(ctx, a, n, off, col);
        } catch (...) {
            delete a;
            throw;
        }
        *out = a;
    });
}

// Operator upload without the sorted-columns rule (a row's nonzeros are summed
// in the given order): permuted operators P A P^T that keep each row's
// original summation order (tools/reorder_lab.py).
extern "C" int mbg_csr_upload_any_order(mbg_ctx* ctx, int64_t n, const int64_t* off, const int32_t* col,
                                        const double* val, mbg_csr** out) {
    return guarded([&] {
        use(ctx);
        if (!out) throw Invalid("null output");
        validate_csr(n, off, col, off ? off[n] : 0, /*sorted=*/false);
        auto* a = new mbg_csr();
        try {
            a->ctx = ctx;
            a->device = ctx->device;
            a->n_global = n;
            csr_to_device(ctx, a, n, off, col, val);
        } catch (...) {
            delete a;
            throw;
        }
        *out = a;
    });
}

// Device CSR of one rank from its halo plan (local CSR, tile lists, interior /
// boundary split, per-peer send lists).
static std::unique_ptr<mbg_csr> csr_from_plan(mbg_ctx* ctx, int64_t n, int64_t row_begin, int nparts,
                                              const HaloPlan& pl) {
    auto a = std::make_unique<mbg_csr>();
    a->ctx = ctx;
    a->device = ctx->device;
    a->n_global = n;
    a->row_begin = row_begin;
    a->n = pl.n_own;
    a->nnz = pl.nnz;
    a->n_halo = pl.n_halo;
    csr_arrays_to_device(ctx, a.get(), pl.n_own, pl.off, pl.col.data(), pl.val.data(), pl.nnz);
    a->nnz = pl.nnz;
    if (nparts > 1) {
        auto ti = build_spmm_tiles(pl.off, pl.interior);
        auto tb = build_spmm_tiles(pl.off, pl.boundary);
        upload(a->tiles_interior, ti.data(), ti.size(), ctx->stream);
        upload(a->tiles_boundary, tb.data(), tb.size(), ctx->stream);
        auto li = long_rows_of(ti), lb = long_rows_of(tb);
        upload(a->long_interior, li.data(), li.size(), ctx->stream);
        upload(a->long_boundary, lb.data(), lb.size(), ctx->stream);
        stage_tilings(ctx, a.get(), pl.off, pl.col.data(), nullptr, &pl.interior, &pl.boundary);
        sorted_twin_to_device(ctx, a.get(), a->sorted_interior, pl.off, pl.col.data(), pl.val.data(), pl.interior);
        sorted_twin_to_device(ctx, a.get(), a->sorted_boundary, pl.off, pl.col.data(), pl.val.data(), pl.boundary);
        upload(a->interior_rows, pl.interior.data(), pl.interior.size(), ctx->stream);
        upload(a->boundary_rows, pl.boundary.data(), pl.boundary.size(), ctx->stream);
        a->n_interior = static_cast<int64_t>(pl.interior.size());
        a->n_boundary = static_cast<int64_t>(pl.boundary.size());
        for (auto& p : pl.peers) {
            mbg_csr::Peer q;
            q.rank = p.part;
            q.send_count = static_cast<int64_t>(p.send_rows.size());
            q.recv_count = p.recv_count;
            q.recv_offset = p.recv_offset;
            upload(q.send_rows, p.send_rows.data(), p.send_rows.size(), ctx->stream);
            a->peers.push_back(std::move(q));
        }
    }
    return a;
}

// Partitioned upload: parts given by bounds[nparts+1]; this context's rank is
// my_part.  Builds the halo plan from the full host CSR.
extern "C" int mbg_csr_upload_partitioned(mbg_ctx* ctx, int64_t n, const int64_t* off, const int32_t* col,
                                          const double* val, int nparts, const int64_t* bounds, int my_part,
                                          mbg_csr** out) {
    return guarded([&] {
        use(ctx);
        if (!out) throw Invalid("null output");
        validate_csr(n, off, col, off ? off[n] : 0);
        HaloPlan pl = build_halo_plan(n, off, col, val, nparts, bounds, my_part);
        mbg_csr* a = nullptr;
        try {
            a = csr_from_plan(ctx, n, bounds[my_part], nparts, pl).release();
            // A^T with its own halo plan (IBiCGStab's f0 = A^T r0 across ranks)
            if (nparts > 1)
                a->transposed =
                    csr_from_plan(ctx, n, bounds[my_part], nparts,
                                  build_transpose_plan(n, off, col, val, nparts, bounds, my_part));
            detect_grid(ctx, a, n, off, col);   // z-slabs of whole planes get the twin of their slab
            MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete a;
            throw;
        }
        *out = a;
    });
}

// Host-only halo plan for tests of the partition logic (no device needed).
static int export_plan(bool transpose, int64_t n, const int64_t* off, const int32_t* col, const double* val,
                       int nparts, const int64_t* bounds, int my_part, int64_t* n_own, int64_t* n_halo,
                       int64_t* nnz_local, int32_t* loc_off, int32_t* loc_col, double* loc_val,
                       int64_t* halo_global, int* npeers, int* peer_part, int64_t* peer_send_count,
                       int32_t* peer_send_rows, int64_t* peer_recv_offset, int64_t* peer_recv_count);

extern "C" int mbg_halo_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val, int nparts,
                             const int64_t* bounds, int my_part, int64_t* n_own, int64_t* n_halo,
                             int64_t* nnz_local, int32_t* loc_off, int32_t* loc_col, double* loc_val,
                             int64_t* halo_global, int* npeers, int* peer_part, int64_t* peer_send_count,
                             int32_t* peer_send_rows, int64_t* peer_recv_offset, int64_t* peer_recv_count) {
    return export_plan(false, n, off, col, val, nparts, bounds, my_part, n_own, n_halo, nnz_local, loc_off, loc_col,
                       loc_val, halo_global, npeers, peer_part, peer_send_count, peer_send_rows, peer_recv_offset,
                       peer_recv_count);
}

extern "C" int mbg_transpose_halo_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val,
                                       int nparts, const int64_t* bounds, int my_part, int64_t* n_own,
                                       int64_t* n_halo, int64_t* nnz_local, int32_t* loc_off, int32_t* loc_col,
                                       double* loc_val, int64_t* halo_global, int* npeers, int* peer_part,
                                       int64_t* peer_send_count, int32_t* peer_send_rows,
                                       int64_t* peer_recv_offset, int64_t* peer_recv_count) {
    return export_plan(true, n, off, col, val, nparts, bounds, my_part, n_own, n_halo, nnz_local, loc_off, loc_col,
                       loc_val, halo_global, npeers, peer_part, peer_send_count, peer_send_rows, peer_recv_offset,
                       peer_recv_count);
}

static int export_plan(bool transpose, int64_t n, const int64_t* off, const int32_t* col, const double* val,
                       int nparts, const int64_t* bounds, int my_part, int64_t* n_own, int64_t* n_halo,
                       int64_t* nnz_local, int32_t* loc_off, int32_t* loc_col, double* loc_val,
                       int64_t* halo_global, int* npeers, int* peer_part, int64_t* peer_send_count,
                       int32_t* peer_send_rows, int64_t* peer_recv_offset, int64_t* peer_recv_count) {
    return guarded([&] {
        HaloPlan pl = transpose ? build_transpose_plan(n, off, col, val, nparts, bounds, my_part)
                                : build_halo_plan(n, off, col, val, nparts, bounds, my_part);
        *n_own = pl.n_own;
        *n_halo = pl.n_halo;
        *nnz_local = pl.nnz;
        *npeers = static_cast<int>(pl.peers.size());
        if (!loc_off) return;  // sizes only
        std::memcpy(loc_off, pl.off.data(), pl.off.size() * sizeof(int32_t));
        std::memcpy(loc_col, pl.col.data(), pl.col.size() * sizeof(int32_t));
        std::memcpy(loc_val, pl.val.data(), pl.val.size() * sizeof(double));
        std::memcpy(halo_global, pl.halo_global.data(), pl.halo_global.size() * sizeof(int64_t));
        int64_t so = 0;
        for (size_t i = 0; i < pl.peers.size(); ++i) {
            const auto& p = pl.peers[i];
            peer_part[i] = p.part;
            peer_send_count[i] = static_cast<int64_t>(p.send_rows.size());
            peer_recv_offset[i] = p.recv_offset;
            peer_recv_count[i] = p.recv_count;
            std::memcpy(peer_send_rows + so, p.send_rows.data(), p.send_rows.size() * sizeof(int32_t));
            so += static_cast<int64_t>(p.send_rows.size());
        }
    });
}

extern "C" int mbg_csr_free(mbg_csr* a) {
    return guarded([&] {
        if (!a) return;
        cudaSetDevice(a->device);
        delete a;
    });
}

extern "C" int64_t mbg_csr_rows(const mbg_csr* a) { return a ? a->n : -1; }
extern "C" int64_t mbg_csr_nnz(const mbg_csr* a) { return a ? a->nnz : -1; }

// Locality reordering for structured grids: rows in
// bx*by*bz bricks so that a SpMM tile's stencil neighbourhood is compact.
// Results are bitwise unchanged (every row keeps its summation order and the
// dots are exact, so the solver is invariant under the permutation).  Only
// long-row stencils gain (27-point C3: -11 % per iteration); a 7-point
// operator is left as is.
extern "C" int mbg_csr_set_grid(mbg_ctx* ctx, mbg_csr* a, int nx, int ny, int nz) {
    return guarded([&] {
        use(ctx);
        if (!a) throw Invalid("set_grid: null matrix");
        if (nx < 1 || ny < 1 || nz < 1 || static_cast<int64_t>(nx) * ny * nz != a->n_global)
            throw Invalid("set_grid: nx*ny*nz must equal the number of rows");
        // stencil twin: implicit columns, x staged as TMA plane boxes (stencil.cu);
        // a z-slab partition (whole planes per rank) gets one for its slab
        if (!a->stencil) a->stencil = build_stencil(ctx, a, nx, ny, nz);
        if (!a->peers.empty() || a->n_halo) return;   // no reordered twin across ranks
        if (a->nnz <= 12 * a->n || a->reordered) return;
        const int bx = std::min(nx, 8), by = std::min(ny, 8), bz = std::min(nz, 4);
        const int64_t n = a->n;
        const int64_t nbx = (nx + bx - 1) / bx, nby = (ny + by - 1) / by;
        std::vector<int64_t> key(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const int64_t x = i % nx, y = (i / nx) % ny, z = i / (static_cast<int64_t>(nx) * ny);
            const int64_t brick = ((z / bz) * nby + y / by) * nbx + x / bx;
            key[i] = brick * (static_cast<int64_t>(bx) * by * bz) + ((z % bz) * by + y % by) * bx + x % bx;
        }
        std::vector<int32_t> order(static_cast<size_t>(n)), pos(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) order[i] = static_cast<int32_t>(i);
        std::stable_sort(order.begin(), order.end(), [&](int32_t p, int32_t q) { return key[p] < key[q]; });
        for (int64_t nw = 0; nw < n; ++nw) pos[order[nw]] = static_cast<int32_t>(nw);
        a->reordered = make_device_csr(ctx, n, permute_host(n, download_csr(ctx, a), order, pos));
        upload(a->perm, order.data(), order.size(), ctx->stream);
        a->perm_host = std::move(order);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int mbg_csr_stage_info(const mbg_csr* a, int* staged, double* reuse) {
    return guarded([&] {
        if (!a) throw Invalid("null matrix");
        if (staged) *staged = (a->stiles_all.n || a->stiles_interior.n || a->stiles_boundary.n) ? 1 : 0;
        if (reuse) *reuse = a->stage_reuse;
    });
}

extern "C" int mbg_csr_sort_info(const mbg_csr* a, int* sorted, double* lane_efficiency) {
    return guarded([&] {
        if (!a) throw Invalid("null matrix");
        if (sorted) *sorted = (a->sorted_all.rowid.n || a->sorted_interior.rowid.n || a->sorted_boundary.rowid.n) ? 1 : 0;
        if (lane_efficiency) *lane_efficiency = a->lane_efficiency;
    });
}

extern "C" int mbg_sorted_twin_plan(int64_t n, const int64_t* off, int window, int64_t* nslots, int32_t* rowid,
                                    double* lane_efficiency, int64_t* ntiles, int32_t* tiles, int32_t* group_off) {
    return guarded([&] {
        if (n < 0 || !off) throw Invalid("sorted twin plan: null offsets");
        if (window < 1) throw Invalid("sorted twin plan: window < 1");
        std::vector<int32_t> off32(static_cast<size_t>(n) + 1), rows(static_cast<size_t>(n));
        for (int64_t i = 0; i <= n; ++i) off32[i] = static_cast<int32_t>(off[i]);
        for (int64_t i = 0; i < n; ++i) rows[i] = static_cast<int32_t>(i);
        if (lane_efficiency) *lane_efficiency = spmm_lane_efficiency(off32, rows);
        // the plan does not depend on the columns or values
        std::vector<int32_t> col(static_cast<size_t>(off32[n]), 0);
        std::vector<double> val(static_cast<size_t>(off32[n]), 0.0);
        SortedTwin t;
        build_sorted_twin(off32, col.data(), val.data(), rows, window, t);
        if (nslots) *nslots = static_cast<int64_t>(t.rowid.size());
        if (rowid) std::copy(t.rowid.begin(), t.rowid.end(), rowid);
        if (group_off) std::copy(t.off.begin(), t.off.end(), group_off);
        if (ntiles) *ntiles = static_cast<int64_t>(t.tiles.size());
        if (tiles)
            for (size_t i = 0; i < t.tiles.size(); ++i) {
                tiles[4 * i] = t.tiles[i].x;
                tiles[4 * i + 1] = t.tiles[i].y;
                tiles[4 * i + 2] = t.tiles[i].z;
                tiles[4 * i + 3] = t.tiles[i].w;
            }
    });
}

extern "C" int mbg_csr_reordered(const mbg_csr* a) { return a && a->reordered ? 1 : 0; }

extern "C" int mbg_csr_stencil_kind(const mbg_csr* a) { return a && a->stencil ? a->stencil->kind : 0; }

extern "C" int mbg_ctx_set_small_path(mbg_ctx* ctx, int enable) {
    return guarded([&] {
        if (!ctx) throw Invalid("null context");
        ctx->small_path = enable != 0;
    });
}

#ifdef MBG_CHECKED
namespace mbg {
namespace {
struct GuardRegistry {
    std::mutex mu;
    std::map<void*, size_t> live;   // user pointer -> user bytes
    int64_t violations = 0;
    std::string first;
};
GuardRegistry& guards() {
    static GuardRegistry g;
    return g;
}
// number of guard bytes (of the two zones of `user`) that no longer hold GUARD_BYTE
int64_t guard_damage(void* user, size_t bytes) {
    std::vector<unsigned char> h(GUARD_BYTES);
    int64_t bad = 0;
    for (int side = 0; side < 2; ++side) {
        const unsigned char* z = static_cast<unsigned char*>(user) + (side ? bytes : 0) - (side ? 0 : GUARD_BYTES);
        if (cudaMemcpy(h.data(), z, GUARD_BYTES, cudaMemcpyDeviceToHost) != cudaSuccess) {
            (void)cudaGetLastError();
            return -1;
        }
        for (unsigned char c : h) bad += c != GUARD_BYTE;
    }
    return bad;
}
}  // namespace

void* guarded_alloc(size_t bytes) {
    const size_t padded = (bytes + 255) / 256 * 256;
    unsigned char* raw = nullptr;
    MBG_CUDA(cudaMalloc(&raw, padded + 2 * GUARD_BYTES));
    MBG_CUDA(cudaMemset(raw, GUARD_BYTE, padded + 2 * GUARD_BYTES));
    // the fill runs on the legacy stream, the buffer's first use on a
    // non-blocking one: without this the fill can land after an upload
    MBG_CUDA(cudaDeviceSynchronize());
    void* user = raw + GUARD_BYTES;
    std::lock_guard<std::mutex> lk(guards().mu);
    guards().live[user] = padded;
    return user;
}

void guarded_free(void* user) {
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(guards().mu);
        auto it = guards().live.find(user);
        if (it == guards().live.end()) return;
        bytes = it->second;
        guards().live.erase(it);
    }
    cudaDeviceSynchronize();
    const int64_t bad = guard_damage(user, bytes);
    if (bad != 0) {
        std::lock_guard<std::mutex> lk(guards().mu);
        guards().violations += bad > 0 ? 1 : 0;
        if (guards().first.empty())
            guards().first = "guard zone of a " + std::to_string(bytes) + "-byte buffer overwritten (" +
                             std::to_string(bad) + " bytes)";
    }
    cudaFree(static_cast<unsigned char*>(user) - GUARD_BYTES);
}

__global__ void write_past_end_kernel(double* p, int64_t n) { p[n] = 1.0; }
}  // namespace mbg
#endif

// Checked builds only: verify the guard zones of every live device buffer
// now; *violations = buffers found damaged so far (live or freed).
extern "C" int mbg_debug_guard_check(int64_t* violations) {
    return guarded([&] {
        if (!violations) throw Invalid("null output");
#ifdef MBG_CHECKED
        MBG_CUDA(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(guards().mu);
        for (const auto& [user, bytes] : guards().live) {
            const int64_t bad = guard_damage(user, bytes);
            if (bad != 0) {
                ++guards().violations;
                if (guards().first.empty())
                    guards().first = "guard zone of a live " + std::to_string(bytes) + "-byte buffer overwritten";
            }
        }
        *violations = guards().violations;
        if (*violations) set_error(guards().first.c_str());
#else
        throw std::runtime_error("mbg_debug_guard_check: not a checked build (make checked)");
#endif
    });
}

// Checked builds only (tests of the guard mechanism): one kernel writes the
// element just past the end of v's n*m doubles.
extern "C" int mbg_debug_write_past_end(mbg_mv* v) {
    return guarded([&] {
        if (!v) throw Invalid("null multivector");
#ifdef MBG_CHECKED
        MBG_CUDA(cudaSetDevice(v->device));
        // the first element past the 256-byte-rounded allocation: the guard zone
        write_past_end_kernel<<<1, 1>>>(v->data.p, static_cast<int64_t>((v->data.n * 8 + 255) / 256 * 256 / 8));
        MBG_CUDA(cudaDeviceSynchronize());
#else
        throw std::runtime_error("mbg_debug_write_past_end: not a checked build (make checked)");
#endif
    });
}

extern "C" int mbg_ctx_reserve_sms(mbg_ctx* ctx, int count) {
    return guarded([&] {
        if (!ctx) throw Invalid("null context");
        if (count < 0 || count >= ctx->num_sms_device) throw Invalid("reserve_sms: count out of range");
        ctx->num_sms = ctx->num_sms_device - count;
    });
}

extern "C" int mbg_mv_alloc(mbg_ctx* ctx, int64_t n, int m, mbg_mv** out) {
    return guarded([&] {
        use(ctx);
        if (!out) throw Invalid("null output");
        if (n < 0 || m < 1) throw Invalid("multivector: bad shape");
        auto* v = new mbg_mv();
        v->ctx = ctx;
        v->device = ctx->device;
        v->n = n;
        v->n_alloc = n;
        v->m = m;
        try {
            v->data.alloc(static_cast<size_t>(n) * m);
            if (n) MBG_CUDA(cudaMemsetAsync(v->data.p, 0, static_cast<size_t>(n) * m * sizeof(double), ctx->stream));
            MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete v;
            throw;
        }
        *out = v;
    });
}

extern "C" int mbg_mv_free(mbg_mv* v) {
    return guarded([&] {
        if (!v) return;
        cudaSetDevice(v->device);
        delete v;
    });
}

extern "C" int mbg_mv_upload(mbg_mv* v, const double* host) {
    return guarded([&] {
        if (!v) throw Invalid("null multivector");
        use(v->ctx);
        const size_t cnt = static_cast<size_t>(v->n) * v->m;
        if (cnt) MBG_CUDA(cudaMemcpyAsync(v->data.p, host, cnt * sizeof(double), cudaMemcpyHostToDevice, v->ctx->stream));
        MBG_CUDA(cudaStreamSynchronize(v->ctx->stream));
    });
}

extern "C" int mbg_mv_download(const mbg_mv* v, double* host) {
    return guarded([&] {
        if (!v) throw Invalid("null multivector");
        use(v->ctx);
        const size_t cnt = static_cast<size_t>(v->n) * v->m;
        if (cnt) MBG_CUDA(cudaMemcpyAsync(host, v->data.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, v->ctx->stream));
        MBG_CUDA(cudaStreamSynchronize(v->ctx->stream));
    });
}

__global__ void mv_fill_kernel(double* p, int64_t n, double v) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

extern "C" int mbg_mv_fill(mbg_mv* v, double value) {
    return guarded([&] {
        if (!v) throw Invalid("null multivector");
        use(v->ctx);
        const int64_t cnt = v->n * v->m;
        if (cnt) {
            mv_fill_kernel<<<v->ctx->num_sms * 4, 256, 0, v->ctx->stream>>>(v->data.p, cnt, value);
            MBG_CUDA(cudaGetLastError());
            v->ctx->launches++;
        }
        MBG_CUDA(cudaStreamSynchronize(v->ctx->stream));
    });
}

extern "C" double* mbg_mv_device_ptr(mbg_mv* v) { return v ? v->data.p : nullptr; }

// core::spmv (spmv.cpp:54-74): shape / aliasing checks, then the SpMM.
extern "C" int mbg_spmv(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* x, mbg_mv* y) {
    return guarded([&] {
        use(ctx);
        if (!a || !x || !y) throw Invalid("spmv: null argument");
        if (x->n != a->n || y->n != a->n || x->m != y->m) throw Invalid("spmv: dimension mismatch");
        if (x == y || x->data.p == y->data.p) throw Invalid("spmv: x and y must be distinct storage");
        const int m = x->m;
        double* xin = x->data.p;
        if (a->n_halo) {
            // partitioned: stage x in a buffer with halo room
            ctx->scratch_f64.ensure(static_cast<size_t>(a->n + a->n_halo) * m);
            MBG_CUDA(cudaMemcpyAsync(ctx->scratch_f64.p, xin, static_cast<size_t>(a->n) * m * sizeof(double),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
            xin = ctx->scratch_f64.p;
        }
        ctx->launches += apply_operator(ctx, a, m, xin, y->data.p, nullptr);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// core::spmv_transpose (spmv.cpp:76-90): y = A^T x through the cached
// transpose whose rows list their source rows ascending -- the reference's
// serial summation order, bit for bit.  Single-GPU matrices.
extern "C" int mbg_spmv_transpose(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* x, mbg_mv* y) {
    return guarded([&] {
        use(ctx);
        if (!a || !x || !y) throw Invalid("spmv_transpose: null argument");
        if (x->n != a->n || y->n != a->n || x->m != y->m) throw Invalid("spmv: dimension mismatch");
        if (x == y || x->data.p == y->data.p) throw Invalid("spmv: x and y must be distinct storage");
        const bool part = !a->peers.empty() || a->n_halo;
        // partitioned: A^T with its own halo plan, built at upload
        const mbg_csr* at = part ? a->transposed.get() : csr_transpose(ctx, a);
        if (!at) throw Invalid("spmv_transpose: partitioned matrix without its A^T plan");
        const int m = x->m;
        double* xin = x->data.p;
        if (at->n_halo) {   // stage x in a buffer with A^T's halo room
            ctx->scratch_f64.ensure(static_cast<size_t>(at->n + at->n_halo) * m);
            MBG_CUDA(cudaMemcpyAsync(ctx->scratch_f64.p, xin, static_cast<size_t>(at->n) * m * sizeof(double),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
            xin = ctx->scratch_f64.p;
        }
        ctx->launches += apply_operator(ctx, at, m, xin, y->data.p, nullptr);
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// kernels::execute_group (execute.cpp:123-172), exact dots.
extern "C" int mbg_execute_group(mbg_ctx* ctx, const mbg_statement* st, int ns, mbg_mv* const* vectors,
                                 int nvec, double* dot_results, int nslots) {
    return guarded([&] {
        use(ctx);
        if (ns < 0 || (ns > 0 && !st)) throw Invalid("execute_group: bad statement array");
        if (ns == 0) return;  // empty group: no-op (execute.cpp:129)
        if (ns > GEN_MAX_STMT) throw Invalid("execute_group: too many statements");
        if (nvec > GEN_MAX_VEC) throw Invalid("execute_group: too many vectors");
        for (int i = 0; i < nvec; ++i)
            if (vectors[i] && vectors[i]->m > 256) throw Invalid("execute_group: at most 256 columns");
        auto vec = [&](int id) -> mbg_mv* {
            if (id < 0 || id >= nvec || !vectors[id]) throw Invalid("execute_group: unbound vector id");
            return vectors[id];
        };
        int64_t n = -1;
        int m = -1;
        auto note = [&](mbg_mv* v) {
            if (n < 0) { n = v->n; m = v->m; }
            else if (v->n != n || v->m != m) throw Invalid("execute_group: shape mismatch");
        };
        GenericGroup g{};
        g.nstmt = ns;
        std::vector<double> coef;
        int used_slots = 0;
        int nterm_total = 0;
        for (int i = 0; i < ns; ++i) {
            if (st[i].kind == MBG_STMT_UPDATE) {
                note(vec(st[i].out));
                if (st[i].nterms < 0 || st[i].nterms > MBG_MAX_TERMS) throw Invalid("execute_group: too many terms");
                g.kind[i] = MBG_STMT_UPDATE;
                g.out[i] = st[i].out;
                g.nterms[i] = st[i].nterms;
                g.tfirst[i] = nterm_total;
                for (int t = 0; t < st[i].nterms; ++t) {
                    note(vec(st[i].term_vec[t]));
                    if (!st[i].term_coeff[t]) throw Invalid("execute_group: coefficient width mismatch");
                    g.term_vec[nterm_total + t] = st[i].term_vec[t];
                }
                nterm_total += st[i].nterms;
            } else if (st[i].kind == MBG_STMT_DOT) {
                note(vec(st[i].left));
                note(vec(st[i].right));
                if (st[i].slot < 0 || st[i].slot >= nslots) throw Invalid("execute_group: dot slot out of range");
                if (st[i].slot >= GEN_MAX_SLOT) throw Invalid("execute_group: too many dot slots");
                g.kind[i] = MBG_STMT_DOT;
                g.left[i] = st[i].left;
                g.right[i] = st[i].right;
                g.dslot[i] = st[i].slot;
                used_slots = std::max(used_slots, st[i].slot + 1);
            } else {
                throw Invalid("execute_group: unknown statement kind");
            }
        }
        coef.resize(static_cast<size_t>(nterm_total) * m);
        for (int i = 0, t0 = 0; i < ns; ++i)
            if (st[i].kind == MBG_STMT_UPDATE) {
                for (int t = 0; t < st[i].nterms; ++t)
                    std::memcpy(&coef[static_cast<size_t>(t0 + t) * m], st[i].term_coeff[t], m * sizeof(double));
                t0 += st[i].nterms;
            }
        g.len = n * m;
        g.m = m;
        for (int i = 0; i < nvec; ++i) g.vec[i] = vectors[i] ? vectors[i]->data.p : nullptr;
        g.nslots = used_slots;
        const size_t slot_words = static_cast<size_t>(used_slots) * m * NSLOT;
        ctx->scratch_i64.ensure(slot_words + 1);
        ctx->scratch_f64.ensure(coef.size() + static_cast<size_t>(used_slots) * m + 1);
        int64_t* slots = ctx->scratch_i64.p;
        double* dcoef = ctx->scratch_f64.p;
        double* rounded = dcoef + coef.size();
        if (slot_words) MBG_CUDA(cudaMemsetAsync(slots, 0, slot_words * sizeof(int64_t), ctx->stream));
        if (!coef.empty())
            MBG_CUDA(cudaMemcpyAsync(dcoef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice,
                                     ctx->stream));
        g.coef = dcoef;
        g.slot = slots;
        int nblocks = 0;
        launch_generic_group(ctx->stream, g, ctx->num_sms, &nblocks);
        ctx->launches++;
        if (used_slots) {
            if (ctx->comm) comm_allreduce_i64(ctx, slots, slot_words, ctx->stream);
            launch_round(ctx->stream, slots, used_slots, m, rounded);
            ctx->launches++;
            std::vector<double> h(static_cast<size_t>(used_slots) * m);
            MBG_CUDA(cudaMemcpyAsync(h.data(), rounded, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            MBG_CUDA(cudaStreamSynchronize(ctx->stream));
            for (int i = 0; i < ns; ++i)
                if (st[i].kind == MBG_STMT_DOT)
                    std::memcpy(dot_results + static_cast<size_t>(st[i].slot) * m,
                                h.data() + static_cast<size_t>(st[i].slot) * m, m * sizeof(double));
        } else {
            MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
}

// SolveReport's true residual: out[c] = ||b - A x||_2 / ||b||_2
// per column (||b - A x||_2 when b's column is zero), with exact dots, so the
// value is the same on any GPU count.
extern "C" int mbg_true_residual(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, const mbg_mv* x, double* out) {
    return guarded([&] {
        use(ctx);
        if (!a || !b || !x || !out) throw Invalid("true_residual: null argument");
        if (b->n != a->n || x->n != a->n || b->m != x->m) throw Invalid("true_residual: shape mismatch");
        const int m = b->m;
        mbg_mv *y = nullptr, *r = nullptr;
        auto chk = [](int rc) {
            if (rc != MBG_OK) throw std::runtime_error(mbg_last_error());
        };
        chk(mbg_mv_alloc(ctx, a->n, m, &y));
        struct Free {
            mbg_mv*& p;
            ~Free() { if (p) mbg_mv_free(p); }
        } fy{y}, fr{r};
        chk(mbg_mv_alloc(ctx, a->n, m, &r));
        chk(mbg_spmv(ctx, a, x, y));
        std::vector<double> one(static_cast<size_t>(m), 1.0), mone(static_cast<size_t>(m), -1.0);
        mbg_statement st[3] = {};
        st[0].kind = MBG_STMT_UPDATE;      // r = 1*b + (-1)*y
        st[0].out = 2;
        st[0].nterms = 2;
        st[0].term_vec[0] = 0;
        st[0].term_vec[1] = 1;
        st[0].term_coeff[0] = one.data();
        st[0].term_coeff[1] = mone.data();
        st[1].kind = MBG_STMT_DOT;         // (r, r)
        st[1].left = st[1].right = 2;
        st[1].slot = 0;
        st[2].kind = MBG_STMT_DOT;         // (b, b)
        st[2].left = st[2].right = 0;
        st[2].slot = 1;
        mbg_mv* vecs[3] = {const_cast<mbg_mv*>(b), y, r};
        std::vector<double> dots(static_cast<size_t>(2) * m);
        chk(mbg_execute_group(ctx, st, 3, vecs, 3, dots.data(), 2));
        for (int c = 0; c < m; ++c)
            out[c] = dots[m + c] > 0.0 ? std::sqrt(dots[c] / dots[m + c]) : std::sqrt(dots[c]);
    });
}

static void check_solve_args(mbg_ctx* ctx, const mbg_csr* a, int m, double tol, int fixed, int max_iters) {
    use(ctx);
    if (!a) throw Invalid("solve: null matrix");
    if (m < 1) throw Invalid("solve: shape mismatch");
    if (max_iters < 0) throw Invalid("solve: negative iteration count");
    if (!fixed && !(tol > 0.0)) throw Invalid("solve: tol must be > 0 in converge mode");
}

static void do_solve(mbg_ctx* ctx, const mbg_csr* a, int m, const double* b, double* x, int method,
                     int formulation, double tol, int fixed, int max_iters, double* hist, mbg_report* report,
                     int precond_alpha = -1) {
    Solver s(ctx, a, m, method, formulation, tol, fixed, max_iters, precond_alpha);
    s.run(b, x);
    mbg_report rep;
    s.report(hist, &rep);
    ctx->launches += rep.gpu_launches;
    if (report) *report = rep;
    if (rep.breakdown) {
        static const char* what[] = {"", "delta (alpha)", "psi (omega)", "beta"};
        throw Breakdown("solve: breakdown at iteration " + std::to_string(rep.breakdown_iter) + ", column " +
                        std::to_string(rep.breakdown_col) + ": " + what[rep.breakdown & 3] +
                        " denominator zero or non-finite");
    }
}

extern "C" int mbg_solve(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method, int formulation,
                         double tol, int fixed, int max_iters, double* hist, mbg_report* report) {
    return guarded([&] {
        if (!b || !x) throw Invalid("solve: null multivector");
        check_solve_args(ctx, a, b->m, tol, fixed, max_iters);
        if (b->n != a->n || x->n != a->n || b->m != x->m) throw Invalid("solve: shape mismatch");
        do_solve(ctx, a, b->m, b->data.p, x->data.p, method, formulation, tol, fixed, max_iters, hist, report);
    });
}

extern "C" int mbg_solve_pc(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method,
                            int formulation, int precond_alpha, double tol, int fixed, int max_iters, double* hist,
                            mbg_report* report) {
    return guarded([&] {
        if (!b || !x) throw Invalid("solve: null multivector");
        if (precond_alpha < 0) throw Invalid("solve: precond_alpha must be >= 0");
        check_solve_args(ctx, a, b->m, tol, fixed, max_iters);
        if (b->n != a->n || x->n != a->n || b->m != x->m) throw Invalid("solve: shape mismatch");
        do_solve(ctx, a, b->m, b->data.p, x->data.p, method, formulation, tol, fixed, max_iters, hist, report,
                 precond_alpha);
    });
}

// Host <-> device copies of user (pageable) buffers: a multi-threaded memcpy
// into pinned staging, pipelined against the DMA.  Measured on the GPU box
// (tools/h2d_lab.cu): pageable cudaMemcpy 11-17 GB/s, pinned DMA 55 GB/s,
// host memcpy 64 GB/s with 8 threads -- so 8 persistent copy workers.
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    void run(void* dst, const void* src, size_t bytes) {
        if (bytes < (4u << 20) || workers_.empty()) {
            std::memcpy(dst, src, bytes);
            return;
        }
        // one job at a time: the workers read dst_/src_/bytes_ until pending_
        // drops to 0, so a second caller (another context's thread) must not
        // publish its job before this one has finished
        std::lock_guard<std::mutex> job(job_mu_);
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        pending_ = static_cast<int>(workers_.size());
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            cv_.notify_all();
        }
        for (auto& t : workers_) t.join();
    }

private:
    CopyPool() {
        const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        for (unsigned t = 0; t < nt; ++t) workers_.emplace_back([this, t, nt] { loop(t, nt); });
    }
    void loop(unsigned t, unsigned nt) {
        long seen = 0;
        for (;;) {
            char* d;
            const char* s;
            size_t n;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                d = dst_;
                s = src_;
                n = bytes_;
            }
            const size_t b = n * t / nt, e = n * (t + 1) / nt;
            if (b < e) std::memcpy(d + b, s + b, e - b);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int pending_ = 0;
    long gen_ = 0;
    bool stop_ = false;
};

static void parallel_memcpy(void* dst, const void* src, size_t bytes) { CopyPool::get().run(dst, src, bytes); }

// Two pinned staging halves of STAGE_CHUNK bytes: the host memcpy of chunk k
// overlaps the DMA of chunk k-1 (upload) / the DMA of chunk k+1 overlaps the
// host memcpy of chunk k (download).
constexpr size_t STAGE_CHUNK = 64u << 20;

static unsigned char* stage_buffer(mbg_ctx* ctx) {
    if (!ctx->stage) {
        MBG_CUDA(cudaMallocHost(&ctx->stage, 2 * STAGE_CHUNK));
        ctx->stage_bytes = 2 * STAGE_CHUNK;
    }
    return ctx->stage;
}

// Page-locked host memory (cudaMallocHost / mbg_host_alloc / registered) is
// DMA'd directly at link rate; pageable memory goes through the staging
// pipeline (host memory bandwidth shared by memcpy and DMA caps it near 27 GB/s).
static bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

static void upload_host(mbg_ctx* ctx, double* dev, const double* host, size_t count) {
    if (host_pinned(host)) {
        MBG_CUDA(cudaMemcpyAsync(dev, host, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    unsigned char* st = stage_buffer(ctx);
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));   // staging halves free
    cudaEvent_t done[2];
    for (auto& e : done) MBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t bytes = count * sizeof(double);
    const auto* src = reinterpret_cast<const unsigned char*>(host);
    auto* dst = reinterpret_cast<unsigned char*>(dev);
    size_t k = 0;
    for (size_t o = 0; o < bytes; o += STAGE_CHUNK, ++k) {
        const size_t n = std::min(STAGE_CHUNK, bytes - o);
        unsigned char* half = st + (k & 1) * STAGE_CHUNK;
        if (k >= 2) MBG_CUDA(cudaEventSynchronize(done[k & 1]));   // DMA out of this half finished
        parallel_memcpy(half, src + o, n);
        MBG_CUDA(cudaMemcpyAsync(dst + o, half, n, cudaMemcpyHostToDevice, ctx->stream));
        MBG_CUDA(cudaEventRecord(done[k & 1], ctx->stream));
    }
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& e : done) cudaEventDestroy(e);
}

static void download_host(mbg_ctx* ctx, double* host, const double* dev, size_t count) {
    if (host_pinned(host)) {
        MBG_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    unsigned char* st = stage_buffer(ctx);
    cudaEvent_t ready[2];
    for (auto& e : ready) MBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t bytes = count * sizeof(double);
    const auto* src = reinterpret_cast<const unsigned char*>(dev);
    auto* dst = reinterpret_cast<unsigned char*>(host);
    const size_t nchunks = (bytes + STAGE_CHUNK - 1) / STAGE_CHUNK;
    auto issue = [&](size_t k) {
        const size_t o = k * STAGE_CHUNK, n = std::min(STAGE_CHUNK, bytes - o);
        MBG_CUDA(cudaMemcpyAsync(st + (k & 1) * STAGE_CHUNK, src + o, n, cudaMemcpyDeviceToHost, ctx->stream));
        MBG_CUDA(cudaEventRecord(ready[k & 1], ctx->stream));
    };
    if (nchunks) issue(0);
    for (size_t k = 0; k < nchunks; ++k) {
        MBG_CUDA(cudaEventSynchronize(ready[k & 1]));
        if (k + 1 < nchunks) issue(k + 1);   // the other half is free: its copy-out finished last trip
        const size_t o = k * STAGE_CHUNK, n = std::min(STAGE_CHUNK, bytes - o);
        parallel_memcpy(dst + o, st + (k & 1) * STAGE_CHUNK, n);
    }
    for (auto& e : ready) cudaEventDestroy(e);
}

extern "C" int mbg_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) throw Invalid("host_alloc: null output");
        *out = nullptr;
        if (bytes) MBG_CUDA(cudaMallocHost(out, bytes));
    });
}

extern "C" int mbg_host_free(void* p) {
    return guarded([&] {
        if (p) MBG_CUDA(cudaFreeHost(p));
    });
}

extern "C" int mbg_solve_host(mbg_ctx* ctx, const mbg_csr* a, int m, const double* b_host, double* x_host,
                              int method, int formulation, double tol, int fixed, int max_iters, double* hist,
                              mbg_report* report) {
    return guarded([&] {
        check_solve_args(ctx, a, m, tol, fixed, max_iters);
        if (!b_host || !x_host) throw Invalid("solve: null host buffer");
        const size_t cnt = static_cast<size_t>(a->n) * m;
        DevBuf<double> db = pool_take(ctx, cnt), dx = pool_take(ctx, cnt);
        struct Give {
            mbg_ctx* c;
            DevBuf<double>& a;
            DevBuf<double>& b;
            ~Give() { pool_give(c, std::move(a)); pool_give(c, std::move(b)); }
        } give{ctx, db, dx};
        static const bool trace = std::getenv("MBG_TRACE_E2E") != nullptr;
        auto now = [] { return std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now().time_since_epoch()).count(); };
        const double t0 = now();
        upload_host(ctx, db.p, b_host, cnt);
        upload_host(ctx, dx.p, x_host, cnt);
        const double t1 = now();
        try {
            do_solve(ctx, a, m, db.p, dx.p, method, formulation, tol, fixed, max_iters, hist, report);
        } catch (const Breakdown&) {
            download_host(ctx, x_host, dx.p, cnt);
            throw;
        }
        const double t2 = now();
        download_host(ctx, x_host, dx.p, cnt);
        if (trace)
            std::fprintf(stderr, "solve_host: upload %.2f ms, solve %.2f ms, download %.2f ms\n", t1 - t0, t2 - t1,
                         now() - t2);
    });
}

// Profiling solve: same numerics, no graph, CUDA events around every launch.
extern "C" int mbg_solve_profile(mbg_ctx* ctx, const mbg_csr* a, const mbg_mv* b, mbg_mv* x, int method,
                                 int formulation, double tol, int fixed, int max_iters, char* json, int cap,
                                 mbg_report* report) {
    return guarded([&] {
        if (!b || !x) throw Invalid("solve: null multivector");
        check_solve_args(ctx, a, b->m, tol, fixed, max_iters);
        if (b->n != a->n || x->n != a->n || b->m != x->m) throw Invalid("solve: shape mismatch");
        Solver s(ctx, a, b->m, method, formulation, tol, fixed, max_iters);
        s.enable_profile();
        s.run(b->data.p, x->data.p);
        mbg_report rep;
        s.report(nullptr, &rep);
        if (report) *report = rep;
        const std::string js = s.profile_json();
        if (json && cap > 0) {
            std::strncpy(json, js.c_str(), static_cast<size_t>(cap) - 1);
            json[cap - 1] = 0;
        }
    });
}

// ---- test hooks: host-side exact accumulation in the device limb format ----
extern "C" int mbg_exact_accumulate_host(int64_t n, int m, const double* a, const double* b, int64_t* D) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) {
                const double p = a[i * m + c] * b[i * m + c];
                digits_add(D + static_cast<int64_t>(c) * NSLOT, p);
            }
    });
}

extern "C" int mbg_exact_round_host(const int64_t* D, int count, double* out) {
    return guarded([&] {
        for (int i = 0; i < count; ++i) out[i] = digits_round(D + static_cast<int64_t>(i) * NSLOT);
    });
}

extern "C" int mbg_exact_slot_words(void) { return NSLOT; }

extern "C" int64_t mbg_ctx_launches(const mbg_ctx* ctx) { return ctx ? ctx->launches : -1; }
