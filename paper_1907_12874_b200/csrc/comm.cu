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

#include <cstring>

#include "comm.hpp"
#include "kernels.hpp"

namespace mbg {

#define MBG_NCCL(call)                                                                         \
    do {                                                                                       \
        ncclResult_t _r = (call);                                                              \
        if (_r != ncclSuccess)                                                                 \
            throw std::runtime_error(std::string("NCCL error ") + ncclGetErrorString(_r) +     \
                                     " at " __FILE__ ":" + std::to_string(__LINE__));          \
    } while (0)

struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    cudaEvent_t ev_main = nullptr, ev_side = nullptr;
    DevBuf<double> sendbuf;
    DevBuf<int> one;
};

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
    auto tiles = [](const mbg::DevBuf<int4>& t, const mbg::DevBuf<int32_t>& l) {
        return SpmmTiles{t.p, static_cast<int64_t>(t.n), l.p, static_cast<int64_t>(l.n)};
    };
    if (a->peers.empty()) {
        return launch_spmm(ctx->stream, tiles(a->tiles_all, a->long_all), a->n, nullptr, a->off.p, a->col.p, a->val.p, m, x,
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
    // interior rows overlap the exchange; boundary rows wait for the halo
    launches += launch_spmm(ctx->stream, tiles(a->tiles_interior, a->long_interior), a->n_interior, a->interior_rows.p, a->off.p,
                            a->col.p, a->val.p, m, x, y, ctl, ctx->num_sms, epi);
    side_to_main(ctx);
    launches += launch_spmm(ctx->stream, tiles(a->tiles_boundary, a->long_boundary), a->n_boundary, a->boundary_rows.p, a->off.p,
                            a->col.p, a->val.p, m, x, y, ctl, ctx->num_sms, epi);
    return launches;
}

void comm_allreduce_i64(mbg_ctx* ctx, int64_t* buf, size_t count, cudaStream_t st) {
    Comm* cm = ctx->comm;
    if (!cm || cm->world == 1) return;
    (void)st;
    main_to_side(ctx);
    MBG_NCCL(ncclAllReduce(buf, buf, count, ncclInt64, ncclSum, cm->comm, ctx->side));
    side_to_main(ctx);
}

void comm_barrier(mbg_ctx* ctx) {
    Comm* cm = ctx->comm;
    if (!cm) return;
    cm->one.ensure(1);
    MBG_NCCL(ncclAllReduce(cm->one.p, cm->one.p, 1, ncclInt32, ncclSum, cm->comm, ctx->side));
    MBG_CUDA(cudaStreamSynchronize(ctx->side));
}

void comm_destroy(mbg_ctx* ctx) {
    if (!ctx->comm) return;
    Comm* cm = ctx->comm;
    if (cm->comm) ncclCommDestroy(cm->comm);
    if (cm->ev_main) cudaEventDestroy(cm->ev_main);
    if (cm->ev_side) cudaEventDestroy(cm->ev_side);
    delete cm;
    ctx->comm = nullptr;
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
        ncclResult_t r = ncclCommInitRank(&cm->comm, world, id, rank);
        if (r != ncclSuccess) {
            delete cm;
            throw std::runtime_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        MBG_CUDA(cudaEventCreateWithFlags(&cm->ev_main, cudaEventDisableTiming));
        MBG_CUDA(cudaEventCreateWithFlags(&cm->ev_side, cudaEventDisableTiming));
        ctx->comm = cm;
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}
