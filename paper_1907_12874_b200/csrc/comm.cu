// comm.cu -- NCCL communicator, exact-dot allreduce and the halo-exchanging
// distributed SpMM.  One process per GPU; rank 0 creates the ncclUniqueId,
// the caller broadcasts it (torch.distributed in bench.py), every rank joins.
//
// Collectives replace the paper's MPI_Allreduce / non-blocking halo p2p
// (PAPER.md:580-706).  All NCCL calls are issued on the context's side stream,
// in the same order on every rank, ordered against the main stream by events,
// so they can overlap the interior SpMM (halo) or the next SpMM (Pipelined
// dot allreduce).
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "comm.hpp"
#include "kernels.hpp"
#include "stencil.hpp"

namespace mbg {

#define MBG_NCCL(call)                                                                         \
    do {                                                                                       \
        ncclResult_t _r = (call);                                                              \
        if (_r != ncclSuccess)                                                                 \
            throw std::runtime_error(std::string("NCCL error ") + ncclGetErrorString(_r) +     \
                                     " at " __FILE__ ":" + std::to_string(__LINE__));          \
    } while (0)

// Single-GPU emulation of a multi-rank communicator (validation only): P
// contexts on one device, one host thread per rank.  Collectives do the same
// data movement as the NCCL path with device copies / a sum kernel ordered by
// cross-stream events; host barriers only publish pointers and events, no
// kernel ever waits on another (B200_PROFILING.md).
struct LocalGroup {
    int P = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<const void*> ptr;          // published buffer per rank
    std::vector<cudaEvent_t> ev;           // published event per rank
    std::vector<std::vector<int64_t>> seg; // halo: seg[q][r] = offset (rows) of q's segment for r
    std::vector<cudaEvent_t> consumed;     // halo: rank r finished copying from its peers
    explicit LocalGroup(int p) : P(p), ptr(p), ev(p), seg(p), consumed(p, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = generation;
        if (++arrived == P) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != g; }))
            throw std::runtime_error("local communicator: barrier timeout (a rank failed)");
    }
};

struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    cudaEvent_t ev_main = nullptr, ev_side = nullptr;
    DevBuf<double> sendbuf;
    DevBuf<int> one;
    // local (single-GPU) emulation
    std::shared_ptr<LocalGroup> local;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_consumed = nullptr;
    DevBuf<int64_t> tmp;
};

__global__ void local_sum_kernel(const int64_t* const* srcs, int P, int64_t count, int64_t* dst) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t s = 0;
        for (int q = 0; q < P; ++q) s += srcs[q][i];
        dst[i] = s;
    }
}

__global__ void halo_pack_kernel(const double* __restrict__ x, const int32_t* __restrict__ rows, int64_t count,
                                 int m, double* __restrict__ out) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= count * m) return;
    const int64_t i = e / m;
    const int c = static_cast<int>(e - i * m);
    out[e] = x[static_cast<int64_t>(rows[i]) * m + c];
}

static void main_to_side(mbg_ctx* ctx) {
    MBG_CUDA(cudaEventRecord(ctx->comm->ev_main, ctx->stream));
    MBG_CUDA(cudaStreamWaitEvent(ctx->side, ctx->comm->ev_main, 0));
}

static void side_to_main(mbg_ctx* ctx) {
    MBG_CUDA(cudaEventRecord(ctx->comm->ev_side, ctx->side));
    MBG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->comm->ev_side, 0));
}

int apply_operator(mbg_ctx* ctx, const mbg_csr* a, int m, double* x, double* y, const int* ctl,
                   const SpmmEpi* epi) {
    const bool hint = a->n > 0 && a->nnz > 12 * a->n;
    // the length-sorted twin pays off from m = 4 (B200, config 5's random band,
    // per SpMM: m = 4 -3 %, 8 -9 %, 16 -8 %, 32 -17 % free-running, -29 / -38 / -50 % at
    // m = 8 / 16 / 32 at locked clocks; m <= 2 is bound by 8- and 16-byte gather
    // wavefronts either way and loses 1-8 % to the scattered y rows)
    const bool tile_m = m == 4 || m == 8 || m == 16 || m == 32;
    auto tiles = [hint, tile_m](const mbg::DevBuf<int4>& t, const mbg::DevBuf<int32_t>& l, const mbg::DevBuf<int4>& st,
                                const mbg::DevBuf<int2>& um, const mbg::DevBuf<int32_t>& uc,
                                const mbg::DevBuf<uint16_t>& lc, const mbg_csr::SortedDev& sd) {
        SpmmTiles r{t.p, static_cast<int64_t>(t.n), l.p, static_cast<int64_t>(l.n), hint};
        if (sd.rowid.p && tile_m) {   // length-sorted twin of this row class
            r.tiles = sd.tiles.p;
            r.count = static_cast<int64_t>(sd.tiles.n);
            r.long_rows = sd.long_rows.p;
            r.nlong = static_cast<int64_t>(sd.long_rows.n);
            r.rowid = sd.rowid.p;
            r.s_off = sd.off.p;
            r.s_col = sd.col.p;
            r.s_val = sd.val.p;
            r.sched = sd.sched.p;
        }
        if (st.n && lc.p) {
            r.stiles = st.p;
            r.umeta = um.p;
            r.ucols = uc.p;
            r.lcol = lc.p;
            r.scount = static_cast<int64_t>(st.n);
        }
        return r;
    };
    if (a->peers.empty()) {
        if (stencil_handles(a, m)) return launch_stencil_spmm(ctx, a, m, x, y, ctl, epi);
        return launch_spmm(ctx->stream, tiles(a->tiles_all, a->long_all, a->stiles_all, a->umeta_all, a->ucols_all, a->lcol_all, a->sorted_all), a->n, nullptr, a->off.p, a->col.p, a->val.p, m, x,
                           y, ctl, ctx->num_sms, epi);
    }
    Comm* cm = ctx->comm;
    if (!cm) throw Invalid("spmv: partitioned matrix needs a communicator (mbg_ctx_init_comm)");
    int64_t total = 0;
    for (const auto& p : a->peers) total += p.send_count;
    cm->sendbuf.ensure(static_cast<size_t>(total) * m);
    int launches = 0;
    main_to_side(ctx);
    int64_t so = 0;
    for (const auto& p : a->peers) {
        if (p.send_count) {
            const int64_t cnt = p.send_count * m;
            halo_pack_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, ctx->side>>>(
                x, p.send_rows.p, p.send_count, m, cm->sendbuf.p + so * m);
            MBG_CUDA(cudaGetLastError());
            ++launches;
        }
        so += p.send_count;
    }
    if (cm->local) {
        LocalGroup& g = *cm->local;
        // my send segments, by destination rank
        std::vector<int64_t> seg(g.P, -1);
        int64_t o = 0;
        for (const auto& p : a->peers) {
            seg[p.rank] = o;
            o += p.send_count;
        }
        MBG_CUDA(cudaEventRecord(cm->ev_a, ctx->side));
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.ptr[cm->rank] = cm->sendbuf.p;
            g.ev[cm->rank] = cm->ev_a;
            g.seg[cm->rank] = seg;
        }
        g.barrier();
        for (const auto& p : a->peers) {
            if (!p.recv_count) continue;
            MBG_CUDA(cudaStreamWaitEvent(ctx->side, g.ev[p.rank], 0));
            const double* src = static_cast<const double*>(g.ptr[p.rank]) + g.seg[p.rank][cm->rank] * m;
            MBG_CUDA(cudaMemcpyAsync(x + (a->n + p.recv_offset) * m, src, static_cast<size_t>(p.recv_count) * m * 8,
                                     cudaMemcpyDeviceToDevice, ctx->side));
        }
        MBG_CUDA(cudaEventRecord(cm->ev_consumed, ctx->side));
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.consumed[cm->rank] = cm->ev_consumed;
        }
        g.barrier();
        // my send buffer may be repacked only after every peer copied from it
        for (const auto& p : a->peers) MBG_CUDA(cudaStreamWaitEvent(ctx->side, g.consumed[p.rank], 0));
        g.barrier();
    } else {
    MBG_NCCL(ncclGroupStart());
    so = 0;
    for (const auto& p : a->peers) {
        if (p.send_count)
            MBG_NCCL(ncclSend(cm->sendbuf.p + so * m, static_cast<size_t>(p.send_count) * m, ncclDouble, p.rank,
                              cm->comm, ctx->side));
        if (p.recv_count)
            MBG_NCCL(ncclRecv(x + (a->n + p.recv_offset) * m, static_cast<size_t>(p.recv_count) * m, ncclDouble,
                              p.rank, cm->comm, ctx->side));
        so += p.send_count;
    }
    MBG_NCCL(ncclGroupEnd());
    }
    if (stencil_handles(a, m)) {
        // z-slab on the stencil twin: the interior planes overlap the
        // exchange, the two face planes wait for the halo planes
        const int nzl = a->stencil->nz;
        launches += launch_stencil_spmm(ctx, a, m, x, y, ctl, epi, 1, nzl - 1);
        side_to_main(ctx);
        launches += launch_stencil_spmm(ctx, a, m, x, y, ctl, epi, 0, 1);
        if (nzl > 1) launches += launch_stencil_spmm(ctx, a, m, x, y, ctl, epi, nzl - 1, nzl);
        return launches;
    }
    // interior rows overlap the exchange; boundary rows wait for the halo
    launches += launch_spmm(ctx->stream, tiles(a->tiles_interior, a->long_interior, a->stiles_interior, a->umeta_interior,
                                                      a->ucols_interior, a->lcol_split, a->sorted_interior), a->n_interior, a->interior_rows.p, a->off.p,
                            a->col.p, a->val.p, m, x, y, ctl, ctx->num_sms, epi);
    side_to_main(ctx);
    launches += launch_spmm(ctx->stream, tiles(a->tiles_boundary, a->long_boundary, a->stiles_boundary, a->umeta_boundary,
                                                      a->ucols_boundary, a->lcol_split, a->sorted_boundary), a->n_boundary, a->boundary_rows.p, a->off.p,
                            a->col.p, a->val.p, m, x, y, ctl, ctx->num_sms, epi);
    return launches;
}

void comm_allreduce_i64(mbg_ctx* ctx, int64_t* buf, size_t count, cudaStream_t st, bool join) {
    Comm* cm = ctx->comm;
    if (!cm || cm->world == 1) return;
    (void)st;
    main_to_side(ctx);
    if (cm->local) {
        LocalGroup& g = *cm->local;
        cm->tmp.ensure(count);
        MBG_CUDA(cudaEventRecord(cm->ev_a, ctx->side));
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.ptr[cm->rank] = buf;
            g.ev[cm->rank] = cm->ev_a;
        }
        g.barrier();
        std::vector<const int64_t*> srcs(g.P);
        for (int q = 0; q < g.P; ++q) {
            MBG_CUDA(cudaStreamWaitEvent(ctx->side, g.ev[q], 0));
            srcs[q] = static_cast<const int64_t*>(g.ptr[q]);
        }
        DevBuf<const int64_t*> dsrc(g.P);
        MBG_CUDA(cudaMemcpyAsync(dsrc.p, srcs.data(), g.P * sizeof(void*), cudaMemcpyHostToDevice, ctx->side));
        local_sum_kernel<<<64, 256, 0, ctx->side>>>(dsrc.p, g.P, static_cast<int64_t>(count), cm->tmp.p);
        MBG_CUDA(cudaGetLastError());
        MBG_CUDA(cudaEventRecord(cm->ev_b, ctx->side));
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.ev[cm->rank] = cm->ev_b;
        }
        g.barrier();
        for (int q = 0; q < g.P; ++q) MBG_CUDA(cudaStreamWaitEvent(ctx->side, g.ev[q], 0));
        MBG_CUDA(cudaMemcpyAsync(buf, cm->tmp.p, count * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->side));
        MBG_CUDA(cudaStreamSynchronize(ctx->side));   // dsrc / tmp lifetime; validation path only
        g.barrier();
    } else {
        MBG_NCCL(ncclAllReduce(buf, buf, count, ncclInt64, ncclSum, cm->comm, ctx->side));
    }
    if (join) side_to_main(ctx);
}

void comm_join(mbg_ctx* ctx) {
    if (ctx->comm && ctx->comm->world > 1) side_to_main(ctx);
}

void comm_barrier(mbg_ctx* ctx) {
    Comm* cm = ctx->comm;
    if (!cm) return;
    if (cm->local) {
        MBG_CUDA(cudaStreamSynchronize(ctx->stream));
        cm->local->barrier();
        return;
    }
    cm->one.ensure(1);
    MBG_NCCL(ncclAllReduce(cm->one.p, cm->one.p, 1, ncclInt32, ncclSum, cm->comm, ctx->side));
    MBG_CUDA(cudaStreamSynchronize(ctx->side));
}

bool comm_is_local(const mbg_ctx* ctx) { return ctx->comm && ctx->comm->local; }

void comm_destroy(mbg_ctx* ctx) {
    if (!ctx->comm) return;
    Comm* cm = ctx->comm;
    if (cm->comm) ncclCommDestroy(cm->comm);
    if (cm->ev_a) cudaEventDestroy(cm->ev_a);
    if (cm->ev_b) cudaEventDestroy(cm->ev_b);
    if (cm->ev_consumed) cudaEventDestroy(cm->ev_consumed);
    if (cm->ev_main) cudaEventDestroy(cm->ev_main);
    if (cm->ev_side) cudaEventDestroy(cm->ev_side);
    delete cm;
    ctx->comm = nullptr;
    ctx->num_sms = ctx->num_sms_device;
}

// SMs kept free of the persistent grids while a multi-rank NCCL communicator
// is active (MBG_RESERVE_SMS, default 4): the SpMM / group / stencil kernels
// size their grids to fill every SM they are given, so a side-stream NCCL
// kernel (halo sendrecv under the interior SpMM, the Pipelined dot allreduce
// under the next SpMM) would otherwise get no SM until they drain and the
// overlap would serialise.  NCCL is capped at the same number of CTAs.
int reserved_sms() {
    const char* e = std::getenv("MBG_RESERVE_SMS");
    const int v = e && *e ? std::atoi(e) : 4;
    return std::max(0, std::min(v, 32));
}

}  // namespace mbg

extern "C" int mbg_comm_unique_id(unsigned char out_id[128]) {
    try {
        ncclUniqueId id;
        MBG_NCCL(ncclGetUniqueId(&id));
        static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
        std::memcpy(out_id, id.internal, 128);
        return MBG_OK;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

extern "C" int mbg_ctx_init_comm(mbg_ctx* ctx, int rank, int world, const unsigned char nccl_id[128]) {
    try {
        if (!ctx) throw mbg::Invalid("null context");
        if (world < 1 || rank < 0 || rank >= world) throw mbg::Invalid("init_comm: bad rank/world");
        MBG_CUDA(cudaSetDevice(ctx->device));
        mbg::comm_destroy(ctx);
        auto* cm = new mbg::Comm();
        cm->rank = rank;
        cm->world = world;
        ncclUniqueId id;
        std::memcpy(id.internal, nccl_id, 128);
        const int reserve = world > 1 ? mbg::reserved_sms() : 0;
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        if (reserve > 0) {
            cfg.minCTAs = 1;
            cfg.maxCTAs = reserve;
        }
        ncclResult_t r = ncclCommInitRankConfig(&cm->comm, world, id, rank, &cfg);
        if (r != ncclSuccess) {
            delete cm;
            throw std::runtime_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        MBG_CUDA(cudaEventCreateWithFlags(&cm->ev_main, cudaEventDisableTiming));
        MBG_CUDA(cudaEventCreateWithFlags(&cm->ev_side, cudaEventDisableTiming));
        ctx->comm = cm;
        ctx->num_sms = std::max(1, ctx->num_sms_device - reserve);
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

// Link `world` contexts on one device into an emulated communicator (tests).
extern "C" int mbg_local_group_create(mbg_ctx** ctxs, int world) {
    try {
        if (!ctxs || world < 1) throw mbg::Invalid("local group: bad arguments");
        auto grp = std::make_shared<mbg::LocalGroup>(world);
        for (int r = 0; r < world; ++r) {
            mbg_ctx* ctx = ctxs[r];
            if (!ctx) throw mbg::Invalid("local group: null context");
            MBG_CUDA(cudaSetDevice(ctx->device));
            mbg::comm_destroy(ctx);
            auto* cm = new mbg::Comm();
            cm->rank = r;
            cm->world = world;
            cm->local = grp;
            for (cudaEvent_t* e : {&cm->ev_main, &cm->ev_side, &cm->ev_a, &cm->ev_b, &cm->ev_consumed})
                MBG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            ctx->comm = cm;
        }
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}
