// spmm.cu -- CSR SpMM  Y = A X  over the row-interleaved n x m fp64 block.
//
// Restates spmv_rows (spmv.cpp:27-50): for every (row, column) the products
// val[k]*x(col[k], c) are added to acc = 0.0 sequentially in CSR order with
// separately rounded multiply and add -- bitwise the reference's arithmetic.
//
// B200 design (m in {1,2,4,8,16,32}):
//   * the matrix is cut at upload into row tiles of <= 192 rows and <= 1920
//     nonzeros (tile list in HBM, see build_spmm_tiles);
//   * a persistent grid walks the tiles; per block a single thread streams the
//     next tile's row offsets, column indices and values into shared memory
//     with TMA bulk copies (cp.async.bulk, mbarrier complete_tx), double
//     buffered, so the CSR stream (12 B/nnz + 4 B/row) is fetched
//     asynchronously while the current tile computes;
//   * each lane owns one row and two adjacent columns: the x gather of one
//     nonzero is a 16-byte read-only load (x rows are reused across
//     neighbouring rows from L1/L2) and a warp's y store is contiguous;
//   * gathers are issued in batches of 4 nonzeros before the ordered adds.
//   Sizing (tools/spmm_lab.cu sweep on B200, C2 shape): 4 resident blocks of
//   256 threads (<= 64 registers, 2 x 24 KB stages) beat deeper pipelines,
//   larger tiles, wider gather batches and two rows per lane, all of which
//   trade occupancy for in-flight bytes and lose.  (A stage of 2048 nonzeros
//   instead of 1920 pushes the block's shared memory past the 196 KB carve-out
//   step, leaves L1 28 KB instead of 60 and nearly doubles the SpMM's time.)
//   * ragged matrices (m >= 4): the same kernel walks a length-sorted twin of
//     the rows (build_sorted_twin: rows by descending length, groups of 8 stored
//     batch-major, tiles claimed from a counter) -- see the SORTED template
//     parameter below and DESIGN.md section 8.
// Any other m uses a thread-per-(row, column) kernel with the same arithmetic.
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <thread>
#include <type_traits>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"
#include "tma.cuh"

namespace mbg {


// smem layout per stage: offsets | cols | vals (each 16-byte aligned)
constexpr int STAGES = 2;
constexpr int OFF_CAP = SPMM_TILE_ROWS + 8;
constexpr int NNZ_PAD = SPMM_TILE_NNZ + 8;
constexpr int BUF_BYTES = OFF_CAP * 4 + NNZ_PAD * 4 + NNZ_PAD * 8;
constexpr int SMEM_HEAD = 128;  // STAGES mbarriers + STAGES tile metas
constexpr int SPMM_SMEM = SMEM_HEAD + STAGES * BUF_BYTES;
static_assert(BUF_BYTES % 16 == 0, "buffer alignment");
static_assert((OFF_CAP * 4) % 16 == 0 && (NNZ_PAD * 4) % 16 == 0, "region alignment");
static_assert(STAGES * BUF_BYTES >= 256 * KEXP * 8, "combine scratch aliases the stages");
static_assert(8 * STAGES <= 32 && 32 + 16 * STAGES <= SMEM_HEAD, "head layout");

// Fused SpMM epilogue (SpmmEpi kinds 1-3): the exact dot terms of one
// finished row; lane columns cp, cp+1.
template <int M, int EPI, int VW, int ND>
__device__ __forceinline__ void spmm_epi_row(double (&ex)[ND * VW][KEXP], const SpmmEpi& epi, int cp, int row,
                                             double t0, double t1, const double* __restrict__ x) {
    if constexpr (EPI == 3) {
        grow(ex[0], __dmul_rn(t0, t0), epi.slot[0] + static_cast<int64_t>(cp) * NSLOT);
        if constexpr (VW == 2) grow(ex[1], __dmul_rn(t1, t1), epi.slot[0] + static_cast<int64_t>(cp + 1) * NSLOT);
    } else if constexpr (EPI == 1) {
        const double* au = epi.aux + static_cast<int64_t>(row) * M + cp;
        grow(ex[0], __dmul_rn(t0, au[0]), epi.slot[0] + static_cast<int64_t>(cp) * NSLOT);
        if constexpr (VW == 2) grow(ex[1], __dmul_rn(t1, au[1]), epi.slot[0] + static_cast<int64_t>(cp + 1) * NSLOT);
    } else if constexpr (EPI == 2) {
        double s0, s1 = 0.0;
        if constexpr (VW == 2) {
            const double2 sv = __ldg(reinterpret_cast<const double2*>(x + static_cast<int64_t>(row) * M + cp));
            s0 = sv.x;
            s1 = sv.y;
        } else {
            s0 = __ldg(x + row);
        }
#pragma unroll
        for (int v = 0; v < VW; ++v) {
            const double t = v ? t1 : t0, sv = v ? s1 : s0;
            const int64_t so = static_cast<int64_t>(cp + v) * NSLOT;
            grow(ex[0 * VW + v], __dmul_rn(t, sv), epi.slot[0] + so);
            grow(ex[1 * VW + v], __dmul_rn(t, t), epi.slot[1] + so);
            grow(ex[2 * VW + v], __dmul_rn(sv, sv), epi.slot[2] + so);
        }
    }
}

// EPI: 0 plain; 1/2/3 fused dot epilogues (kernels.hpp SpmmEpi kinds); 4 plain
// for long rows (> 12 nonzeros on average) at m = 32: 6 gathers in flight per
// lane, 3-block register budget.
// SORTED: the length-sorted twin (build_sorted_twin) -- slots instead of rows,
// in groups of 8 slots whose nonzeros are stored batch-major (batch = 4
// nonzeros; column -1 = padding): for batch b the 8 rows' column quadruples
// are 128 contiguous bytes and their value pairs 2 x 128, so a lane reads 4
// columns and 4 values with three 16-byte shared-memory loads and the 8 rows a
// warp walks hit 8 different bank groups -- one wavefront per load, not the 2-8
// of rows stored one after the other (the load/store pipe, shared by the x
// gathers and these reads, is what bounds the kernel at m = 8).  `off` holds
// the groups' cumulative batch counts; tiles are claimed from a counter.
template <int M, int EPI, bool SORTED = false>
__global__ void __launch_bounds__(256, EPI == 0 ? 4 : (EPI == 2 ? 2 : 3)) spmm_tma_kernel(const int4* __restrict__ tiles, int ntiles,
                                                       const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       const int* __restrict__ ctl, SpmmEpi epi,
                                                       const int32_t* __restrict__ rowid, int* sched) {
    pdl_wait();
    if (ctl && ctl[0]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    int4* meta = reinterpret_cast<int4*>(smem + 32);
    unsigned char* bufs = smem + SMEM_HEAD;
    const int tid = threadIdx.x;

    if (tid == 0) {
        for (int b = 0; b < STAGES; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // sched == nullptr: block b walks tiles b, b + grid, ...; else (length-sorted
    // twin: tiles of unequal work) the next unclaimed tile, a tile row of -1
    // telling the block that none is left
    auto issue = [&](int i, int b) {
        const int t = SORTED ? atomicAdd(&sched[0], 1) : static_cast<int>(blockIdx.x + i * gridDim.x);
        if (t >= ntiles) {
            if constexpr (SORTED) {
                meta[b] = make_int4(-1, 0, 0, 0);
                mbar_arrive(&bars[b]);
            }
            return;
        }
        const int4 tl = tiles[t];
        if constexpr (SORTED) {
            // (slot0, slot1, first batch, end batch) of whole groups; a negative
            // batch marks a row beyond a stage (long-row kernel; epilogue only)
            meta[b] = tl;
            if (tl.z < 0) {
                mbar_arrive(&bars[b]);
                return;
            }
            unsigned char* buf = bufs + b * BUF_BYTES;
            const uint32_t cnt = static_cast<uint32_t>(tl.w - tl.z) * 32u;   // entries (8 rows x 4 per batch)
            mbar_expect_tx(&bars[b], cnt * 12u);
            if (cnt) {
                bulk_g2s(buf + OFF_CAP * 4, col + static_cast<int64_t>(tl.z) * 32, cnt * 4u, &bars[b]);
                bulk_g2s(buf + OFF_CAP * 4 + NNZ_PAD * 4, val + static_cast<int64_t>(tl.z) * 32, cnt * 8u, &bars[b]);
            }
            return;
        }
        const int r0a = tl.x & ~3, r1a = (tl.y + 1 + 3) & ~3;
        const int k0a = tl.z & ~3, k1a = (tl.w + 3) & ~3;
        const bool lng = tl.w - tl.z > SPMM_TILE_NNZ;
        meta[b] = make_int4(tl.x, tl.y, r0a, k0a);
        unsigned char* buf = bufs + b * BUF_BYTES;
        const uint32_t boff = static_cast<uint32_t>(r1a - r0a) * 4u;
        const uint32_t bnnz = lng ? 0u : static_cast<uint32_t>(k1a - k0a);
        mbar_expect_tx(&bars[b], boff + bnnz * 12u);
        bulk_g2s(buf, off + r0a, boff, &bars[b]);
        if (bnnz) {
            bulk_g2s(buf + OFF_CAP * 4, col + k0a, bnnz * 4u, &bars[b]);
            bulk_g2s(buf + OFF_CAP * 4 + NNZ_PAD * 4, val + k0a, bnnz * 8u, &bars[b]);
        }
    };
    if (tid == 0)
        for (int b = 0; b < STAGES; ++b) issue(b, b);

    constexpr int VW = M >= 2 ? 2 : 1;        // columns per lane
    // gathers in flight per lane: 4 (4 blocks/SM); EPI 4 = the long-row m = 32
    // variant, 6 per lane with a 3-block register budget.  In the solver
    // (tools/sweep.py) it is faster only at m = 32 (C5 15.6 -> 13.9 ms/it);
    // at m = 8/16 (C5) and on the 27-point C3 it loses 4-12 % although the
    // isolated SpMM (tools/spmm_lab.cu) prefers it there too.
    constexpr int BATCH = EPI == 4 ? 6 : 4;
    constexpr int LPR = M / VW;               // lanes per row
    constexpr int RPP = 256 / LPR;            // rows per pass of the block
    constexpr int ND = EPI == 2 ? 3 : 1;      // dots of the fused epilogue
    const int cp = (tid % LPR) * VW;
    double ex[ND * VW][KEXP];
#pragma unroll
    for (int q = 0; q < ND * VW; ++q)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) ex[q][i] = 0.0;

    // fused epilogue: exact dot terms of one finished row
    auto epilogue = [&](int row, double t0, double t1) { spmm_epi_row<M, EPI, VW, ND>(ex, epi, cp, row, t0, t1, x); };

    for (int i = 0;; ++i) {
        if (!SORTED && static_cast<int>(blockIdx.x + i * gridDim.x) >= ntiles) break;
        const int b = i % STAGES;
        while (!mbar_try_wait(&bars[b], static_cast<uint32_t>((i / STAGES) & 1))) {
        }
        const int4 mt = meta[b];
        if (SORTED && mt.x < 0) break;   // claimed past the last tile
        const int r0 = mt.x, r1 = mt.y, r0a = mt.z, k0a = mt.w;
        const unsigned char* buf = bufs + b * BUF_BYTES;
        const int32_t* s_off = reinterpret_cast<const int32_t*>(buf);
        const int32_t* s_col = reinterpret_cast<const int32_t*>(buf + OFF_CAP * 4);
        const double* s_val = reinterpret_cast<const double*>(buf + OFF_CAP * 4 + NNZ_PAD * 4);
        const bool lng = SORTED ? mt.z < 0 : s_off[r1 - r0a] - s_off[r0 - r0a] > SPMM_TILE_NNZ;
        if (lng) {
            // a row longer than the stage capacity was multiplied beforehand by
            // spmm_long_rows_kernel; only its fused epilogue runs here
            if constexpr (EPI >= 1 && EPI <= 3) {
                if (tid < LPR) {
                    const int row = SORTED ? rowid[r0] : r0;
                    double a0, a1 = 0.0;
                    if constexpr (VW == 2) {
                        const double2 yv = *reinterpret_cast<const double2*>(y + static_cast<int64_t>(row) * M + cp);
                        a0 = yv.x;
                        a1 = yv.y;
                    } else {
                        a0 = y[row];
                    }
                    epilogue(row, a0, a1);
                }
            }
        } else {
            const int32_t* cs = s_col - k0a;   // index with the global k
            const double* vs = s_val - k0a;
            for (int rr = tid / LPR; rr < r1 - r0; rr += RPP) {
                // slot = position in the (possibly length-sorted) row storage;
                // row = where its result goes (sorted twin: rowid[slot], -1 = no row)
                const int slot = r0 + rr;
                const int row = SORTED ? __ldg(rowid + slot) : slot;
                int k0, k1;
                const int4* c4 = nullptr;
                const double2* v2 = nullptr;
                if constexpr (SORTED) {
                    // batches of this slot's group: [k0, k1) counts batches, not nonzeros
                    const int g = slot >> 3;
                    k0 = __ldg(off + g) - r0a;        // r0a = the tile's first batch
                    k1 = __ldg(off + g + 1) - r0a;
                    c4 = reinterpret_cast<const int4*>(s_col) + k0 * 8 + (slot & 7);
                    v2 = reinterpret_cast<const double2*>(s_val) + k0 * 16 + (slot & 7);
                } else {
                    k0 = s_off[slot - r0a];
                    k1 = s_off[slot + 1 - r0a];
                }
                double a0 = 0.0, a1 = 0.0;
                // batches of BATCH nonzeros: index/value loads, then the gathers, then
                // the ordered adds (BATCH gathers in flight per lane)
                for (int k = k0; k < k1; k += SORTED ? 1 : BATCH) {
                    int j[BATCH];
                    double va[BATCH];
                    bool ok[BATCH];
                    if constexpr (SORTED) {
                        static_assert(!SORTED || BATCH == 4, "the twin stores batches of 4");
                        const int4 jj = c4[(k - k0) * 8];
                        const double2 v01 = v2[(k - k0) * 16];
                        const double2 v23 = v2[(k - k0) * 16 + 8];
                        j[0] = jj.x; j[1] = jj.y; j[2] = jj.z; j[3] = jj.w;
                        va[0] = v01.x; va[1] = v01.y; va[2] = v23.x; va[3] = v23.y;
#pragma unroll
                        for (int q = 0; q < BATCH; ++q) ok[q] = j[q] >= 0;
                    } else {
#pragma unroll
                        for (int q = 0; q < BATCH; ++q) {
                            ok[q] = k + q < k1;
                            if (ok[q]) { j[q] = cs[k + q]; va[q] = vs[k + q]; }
                        }
                    }
                    if constexpr (VW == 2) {
                        double2 xa[BATCH];
#pragma unroll
                        for (int q = 0; q < BATCH; ++q)
                            if (ok[q])
                                xa[q] = __ldg(reinterpret_cast<const double2*>(x + static_cast<int64_t>(j[q]) * M + cp));
#pragma unroll
                        for (int q = 0; q < BATCH; ++q)
                            if (ok[q]) {
                                a0 = __dadd_rn(a0, __dmul_rn(va[q], xa[q].x));
                                a1 = __dadd_rn(a1, __dmul_rn(va[q], xa[q].y));
                            }
                    } else {
                        double xa[BATCH];
#pragma unroll
                        for (int q = 0; q < BATCH; ++q)
                            if (ok[q]) xa[q] = __ldg(x + j[q]);
#pragma unroll
                        for (int q = 0; q < BATCH; ++q)
                            if (ok[q]) a0 = __dadd_rn(a0, __dmul_rn(va[q], xa[q]));
                    }
                }
                if (SORTED && row < 0) continue;   // a padding slot of the last group
                if constexpr (VW == 2)
                    *reinterpret_cast<double2*>(y + static_cast<int64_t>(row) * M + cp) = make_double2(a0, a1);
                else
                    y[row] = a0;
                if constexpr (EPI >= 1 && EPI <= 3) epilogue(row, a0, a1);
            }
        }
        // (a warp-asynchronous release of the stage -- last warp out refills --
        // measured 6% slower on C3: warps drifting onto different tiles split
        // the L1 working set that the 27-point gathers depend on; on the
        // length-sorted twin of config 5's band it changes nothing at m = 8 / 16
        // and loses 1-6 % at m = 32)
        __syncthreads();  // every thread is done with stage b
        if (tid == 0) issue(i + STAGES, b);
    }
    pdl_trigger();
    if (SORTED && tid == 0) {
        // the last block out rewinds the tile counter for the next launch (the
        // fences order every block's claims before its count and the rewind
        // after the last count)
        __threadfence();
        const unsigned last = gridDim.x - 1;
        if (atomicInc(reinterpret_cast<unsigned*>(&sched[1]), last) == last) {
            __threadfence();
            atomicExch(&sched[0], 0);
        }
    }
    if constexpr (EPI >= 1 && EPI <= 3) {
        // no bulk copy is in flight any more: the stage memory is free scratch
        double* sh = reinterpret_cast<double*>(bufs);
        block_combine<ND * VW>(ex, M >= 2 ? LPR : 1,
                               [&](int q, int k) {
                                   const int c_ = M >= 2 ? k * VW + q % VW : 0;
                                   return epi.slot[q / VW] + static_cast<int64_t>(c_) * NSLOT;
                               },
                               sh);
    }
}

// ---------------------------------------------------------------------------
// Gather-ahead SpMM ("staged" tiling).  Per tile the distinct columns
// (<= STAGE_UCOLS) are gathered ONCE into shared memory with 16-byte cp.async
// and every nonzero reads its x row from there through a 16-bit local index
// (2 B/nnz instead of the 4 B column).  The gathers of tile i+1 are issued
// before tile i is computed (two x buffers, three CSR stages), so the L2
// latency of the gathers -- what bounds the register-gather kernel (a lane
// waits ~2 L2 round trips per row) -- overlaps the arithmetic of the previous
// tile.  Same arithmetic as spmm_tma_kernel: per (row, column) sequential
// CSR-order adds from 0.0.
// ---------------------------------------------------------------------------
constexpr int S_STAGES = 3;
constexpr int S_OFF_CAP = STAGE_ROWS + 8;     // int32
constexpr int S_LCOL_CAP = STAGE_NNZ + 16;    // uint16 (k0 rounded down to 8)
constexpr int S_VAL_CAP = STAGE_NNZ + 4;      // double (k0 rounded down to 2)
constexpr int S_UCOL_CAP = STAGE_UCOLS + 8;   // int32 (u0 rounded down to 4)
constexpr int S_BUF = S_OFF_CAP * 4 + S_LCOL_CAP * 2 + S_VAL_CAP * 8 + S_UCOL_CAP * 4;
constexpr int S_HEAD = 128;                   // 3 mbarriers + 3 x 2 int4 metas
static_assert(S_BUF % 16 == 0 && (S_OFF_CAP * 4) % 16 == 0 && (S_LCOL_CAP * 2) % 16 == 0 &&
                  (S_VAL_CAP * 8) % 16 == 0, "stage alignment");
static_assert(S_STAGES * S_BUF >= 256 * KEXP * 8, "combine scratch aliases the stages");
static_assert(8 * S_STAGES <= 32 && 32 + 32 * S_STAGES <= S_HEAD, "head layout");
constexpr int stage_smem(int m) { return S_HEAD + S_STAGES * S_BUF + 2 * STAGE_UCOLS * m * 8; }
constexpr int stage_minb(int m, int epi) {
    return (m >= 32 || epi == 2) ? 1 : (m >= 16 ? 2 : (epi == 0 ? 3 : 2));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int M, int EPI>
__global__ void __launch_bounds__(256, stage_minb(M, EPI))
    spmm_stage_kernel(const int4* __restrict__ tiles, const int2* __restrict__ umeta, int ntiles,
                      const int32_t* __restrict__ off, const uint16_t* __restrict__ lcol,
                      const double* __restrict__ val, const int32_t* __restrict__ ucols,
                      const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ ctl,
                      SpmmEpi epi) {
    static_assert(M >= 4, "x rows of >= 32 bytes");
    pdl_wait();
    if (ctl && ctl[0]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    int4* meta = reinterpret_cast<int4*>(smem + 32);   // [stage][2]
    unsigned char* bufs = smem + S_HEAD;
    double* xsb = reinterpret_cast<double*>(smem + S_HEAD + S_STAGES * S_BUF);   // [2][STAGE_UCOLS * M]
    const int tid = threadIdx.x;

    if (tid == 0) {
        for (int b = 0; b < S_STAGES; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int i, int b) {
        const int t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) return;
        const int4 tl = tiles[t];
        const int2 um = umeta[t];
        const int r0a = tl.x & ~3, r1a = (tl.y + 1 + 3) & ~3;
        const int k0l = tl.z & ~7, k1l = (tl.w + 7) & ~7;
        const int k0v = tl.z & ~1, k1v = (tl.w + 1) & ~1;
        const int u0a = um.x & ~3, u1a = (um.x + um.y + 3) & ~3;
        meta[2 * b] = make_int4(tl.x, tl.y, r0a, k0l);
        meta[2 * b + 1] = make_int4(k0v, um.x - u0a, um.y, 0);
        unsigned char* buf = bufs + b * S_BUF;
        const uint32_t boff = static_cast<uint32_t>(r1a - r0a) * 4u;
        const uint32_t blc = static_cast<uint32_t>(k1l - k0l) * 2u;
        const uint32_t bval = static_cast<uint32_t>(k1v - k0v) * 8u;
        const uint32_t buc = static_cast<uint32_t>(u1a - u0a) * 4u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[b], boff + blc + bval + buc);
        bulk_g2s(buf, off + r0a, boff, &bars[b]);
        if (blc) bulk_g2s(buf + S_OFF_CAP * 4, lcol + k0l, blc, &bars[b]);
        if (bval) bulk_g2s(buf + S_OFF_CAP * 4 + S_LCOL_CAP * 2, val + k0v, bval, &bars[b]);
        if (buc) bulk_g2s(buf + S_OFF_CAP * 4 + S_LCOL_CAP * 2 + S_VAL_CAP * 8, ucols + u0a, buc, &bars[b]);
    };
    if (tid == 0)
        for (int b = 0; b < S_STAGES; ++b) issue(b, b);

    constexpr int VW = 2;
    constexpr int LPR = M / VW;
    constexpr int RPP = 256 / LPR;
    constexpr int ND = EPI == 2 ? 3 : 1;
    constexpr int CPR = M / 2;               // 16-byte chunks per x row
    const int cp = (tid % LPR) * VW;
    double ex[ND * VW][KEXP];
#pragma unroll
    for (int q = 0; q < ND * VW; ++q)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) ex[q][i] = 0.0;

    auto wait_stage = [&](int i) {
        const int b = i % S_STAGES;
        while (!mbar_try_wait(&bars[b], static_cast<uint32_t>((i / S_STAGES) & 1))) {
        }
    };
    // issue the cp.async gathers of tile i's distinct x rows into x buffer i & 1
    auto gather = [&](int i) {
        const int b = i % S_STAGES;
        const int4 mu = meta[2 * b + 1];
        const int32_t* s_uc =
            reinterpret_cast<const int32_t*>(bufs + b * S_BUF + S_OFF_CAP * 4 + S_LCOL_CAP * 2 + S_VAL_CAP * 8) + mu.y;
        double* xs = xsb + (i & 1) * (STAGE_UCOLS * M);
        const int U = mu.z;
        for (int c = tid; c < U * CPR; c += 256) {
            const int u = c / CPR, part = c - u * CPR;
            cp_async16(xs + u * M + part * 2, x + static_cast<int64_t>(s_uc[u]) * M + part * 2);
        }
    };
    if (static_cast<int>(blockIdx.x) < ntiles) {
        wait_stage(0);
        gather(0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");

    for (int i = 0;; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        if (t >= ntiles) break;
        if (t + static_cast<int>(gridDim.x) < ntiles) {   // the next tile's gathers fly during this tile
            wait_stage(i + 1);
            gather(i + 1);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 1;" ::: "memory");
        __syncthreads();   // tile i's x rows (every thread's cp.async) are in shared memory
        const int b = i % S_STAGES;
        const int4 mt = meta[2 * b];
        const int4 mu = meta[2 * b + 1];
        const int r0 = mt.x, r1 = mt.y, r0a = mt.z, k0l = mt.w, k0v = mu.x;
        const unsigned char* buf = bufs + b * S_BUF;
        const int32_t* s_off = reinterpret_cast<const int32_t*>(buf);
        const uint16_t* s_lc = reinterpret_cast<const uint16_t*>(buf + S_OFF_CAP * 4) - k0l;   // global k
        const double* s_val = reinterpret_cast<const double*>(buf + S_OFF_CAP * 4 + S_LCOL_CAP * 2) - k0v;
        const double* xs = xsb + (i & 1) * (STAGE_UCOLS * M);
        for (int rr = tid / LPR; rr < r1 - r0; rr += RPP) {
            const int row = r0 + rr;
            const int k0 = s_off[row - r0a], k1 = s_off[row + 1 - r0a];
            double a0 = 0.0, a1 = 0.0;
            for (int k = k0; k < k1; k += 4) {
                int j[4];
                double va[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (k + q < k1) { j[q] = s_lc[k + q]; va[q] = s_val[k + q]; }
                double2 xa[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (k + q < k1) xa[q] = *reinterpret_cast<const double2*>(xs + j[q] * M + cp);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (k + q < k1) {
                        a0 = __dadd_rn(a0, __dmul_rn(va[q], xa[q].x));
                        a1 = __dadd_rn(a1, __dmul_rn(va[q], xa[q].y));
                    }
            }
            *reinterpret_cast<double2*>(y + static_cast<int64_t>(row) * M + cp) = make_double2(a0, a1);
            if constexpr (EPI >= 1 && EPI <= 3) spmm_epi_row<M, EPI, VW, ND>(ex, epi, cp, row, a0, a1, x);
        }
        __syncthreads();  // stage b and x buffer i & 1 are free
        if (tid == 0) issue(i + S_STAGES, b);
    }
    pdl_trigger();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if constexpr (EPI >= 1 && EPI <= 3) {
        double* sh = reinterpret_cast<double*>(bufs);
        block_combine<ND * VW>(ex, LPR,
                               [&](int q, int k) {
                                   return epi.slot[q / VW] + static_cast<int64_t>(k * VW + q % VW) * NSLOT;
                               },
                               sh);
    }
}

// Rows longer than a tile's shared-memory capacity: one thread per (row,
// column), nonzeros read from global memory in CSR order (rare; runs before
// the tile kernel, which then only applies the fused epilogue to them).
__global__ void spmm_long_rows_kernel(int nlong, const int32_t* __restrict__ rows, const int32_t* __restrict__ off,
                                      const int32_t* __restrict__ col, const double* __restrict__ val, int m,
                                      const double* __restrict__ x, double* __restrict__ y,
                                      const int* __restrict__ ctl) {
    pdl_wait();
    pdl_trigger();
    if (ctl && ctl[0]) return;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<int64_t>(nlong) * m) return;
    const int row = rows[e / m];
    const int c = static_cast<int>(e % m);
    double acc = 0.0;
    for (int k = off[row]; k < off[row + 1]; ++k)
        acc = __dadd_rn(acc, __dmul_rn(val[k], x[static_cast<int64_t>(col[k]) * m + c]));
    y[static_cast<int64_t>(row) * m + c] = acc;
}

// Any m: one thread per (row, column) element over an explicit row list.
__global__ void __launch_bounds__(256) spmm_generic_kernel(int64_t nrows, const int32_t* __restrict__ rows,
                                                           const int32_t* __restrict__ off,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ val, int m,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y,
                                                           const int* __restrict__ ctl) {
    pdl_wait();
    pdl_trigger();
    if (ctl && ctl[0]) return;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= nrows * m) return;
    const int64_t ri = e / m;
    const int c = static_cast<int>(e - ri * m);
    const int64_t row = rows ? rows[ri] : ri;
    const int k0 = off[row], k1 = off[row + 1];
    double acc = 0.0;
    for (int k = k0; k < k1; ++k)
        acc = __dadd_rn(acc, __dmul_rn(val[k], x[static_cast<int64_t>(col[k]) * m + c]));
    y[row * m + c] = acc;
}

template <int M, int EPI, bool SORTED>
static void launch_tma_s(cudaStream_t st, const SpmmTiles& tl, const int32_t* off, const int32_t* col,
                         const double* val, const double* x, double* y, const int* ctl, int num_sms,
                         const SpmmEpi& epi) {
    const int occ =
        kernel_occupancy(reinterpret_cast<const void*>(&spmm_tma_kernel<M, EPI, SORTED>), 256, SPMM_SMEM);
    const int grid = static_cast<int>(std::min<int64_t>(tl.count, static_cast<int64_t>(num_sms) * occ));
    launch_pdl(spmm_tma_kernel<M, EPI, SORTED>, dim3(grid), dim3(256), SPMM_SMEM, st, tl.tiles,
               static_cast<int>(tl.count), off, col, val, x, y, ctl, epi, tl.rowid, tl.sched);
}

template <int M, int EPI>
static void launch_tma(cudaStream_t st, const SpmmTiles& tl, const int32_t* off, const int32_t* col,
                       const double* val, const double* x, double* y, const int* ctl, int num_sms,
                       const SpmmEpi& epi) {
    if constexpr (EPI != 4 && M >= 4) {   // apply_operator offers the twin from m = 4
        if (tl.rowid) return launch_tma_s<M, EPI, true>(st, tl, off, col, val, x, y, ctl, num_sms, epi);
    }
    if (tl.rowid) throw Invalid("spmv: internal: length-sorted twin below m = 4");
    launch_tma_s<M, EPI, false>(st, tl, off, col, val, x, y, ctl, num_sms, epi);
}

template <int M>
static void launch_tma_epi(cudaStream_t st, const SpmmTiles& tl, const int32_t* off, const int32_t* col,
                           const double* val, const double* x, double* y, const int* ctl, int num_sms,
                           const SpmmEpi* epi) {
    if ((!epi || epi->kind == 0) && tl.long_rows_hint && M >= 32 && !tl.rowid)
        launch_tma<M, 4>(st, tl, off, col, val, x, y, ctl, num_sms, SpmmEpi{});
    else if (!epi || epi->kind == 0)
        launch_tma<M, 0>(st, tl, off, col, val, x, y, ctl, num_sms, SpmmEpi{});
    else if (epi->kind == 1)
        launch_tma<M, 1>(st, tl, off, col, val, x, y, ctl, num_sms, *epi);
    else if (epi->kind == 3)
        launch_tma<M, 3>(st, tl, off, col, val, x, y, ctl, num_sms, *epi);
    else
        launch_tma<M, 2>(st, tl, off, col, val, x, y, ctl, num_sms, *epi);
}

template <int M, int EPI>
static void launch_stage(cudaStream_t st, const SpmmTiles& tl, const int32_t* off, const double* val,
                         const double* x, double* y, const int* ctl, int num_sms, const SpmmEpi& epi) {
    constexpr int smem = stage_smem(M);
    const int occ = kernel_occupancy(reinterpret_cast<const void*>(&spmm_stage_kernel<M, EPI>), 256, smem);
    const int grid = static_cast<int>(std::min<int64_t>(tl.scount, static_cast<int64_t>(num_sms) * occ));
    launch_pdl(spmm_stage_kernel<M, EPI>, dim3(grid), dim3(256), static_cast<size_t>(smem), st, tl.stiles, tl.umeta,
               static_cast<int>(tl.scount), off,
                                                       tl.lcol, val, tl.ucols, x, y, ctl, epi);
}

template <int M>
static void launch_stage_epi(cudaStream_t st, const SpmmTiles& tl, const int32_t* off, const double* val,
                             const double* x, double* y, const int* ctl, int num_sms, const SpmmEpi* epi) {
    if (!epi || epi->kind == 0)
        launch_stage<M, 0>(st, tl, off, val, x, y, ctl, num_sms, SpmmEpi{});
    else if (epi->kind == 1)
        launch_stage<M, 1>(st, tl, off, val, x, y, ctl, num_sms, *epi);
    else if (epi->kind == 3)
        launch_stage<M, 3>(st, tl, off, val, x, y, ctl, num_sms, *epi);
    else
        launch_stage<M, 2>(st, tl, off, val, x, y, ctl, num_sms, *epi);
}

int launch_spmm(cudaStream_t st, const SpmmTiles& tl, int64_t nrows, const int32_t* rows, const int32_t* off,
                const int32_t* col, const double* val, int m, const double* x, double* y, const int* ctl,
                int num_sms, const SpmmEpi* epi) {
    if (nrows <= 0) return 0;
    if (tl.stiles && tl.scount > 0 && (m == 4 || m == 8 || m == 16 || m == 32)) {
        switch (m) {
            case 4: launch_stage_epi<4>(st, tl, off, val, x, y, ctl, num_sms, epi); break;
            case 8: launch_stage_epi<8>(st, tl, off, val, x, y, ctl, num_sms, epi); break;
            case 16: launch_stage_epi<16>(st, tl, off, val, x, y, ctl, num_sms, epi); break;
            default: launch_stage_epi<32>(st, tl, off, val, x, y, ctl, num_sms, epi); break;
        }
        MBG_CUDA(cudaGetLastError());
        return 1;
    }
    int launched = 0;
    if (tl.nlong > 0 && (m == 1 || m == 2 || m == 4 || m == 8 || m == 16 || m == 32)) {
        const int64_t tot = tl.nlong * m;
        spmm_long_rows_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            static_cast<int>(tl.nlong), tl.long_rows, off, col, val, m, x, y, ctl);
        ++launched;
    }
    if (tl.rowid) {   // the tile kernel walks the length-sorted twin
        off = tl.s_off;
        col = tl.s_col;
        val = tl.s_val;
    }
    switch (m) {
        case 1: launch_tma_epi<1>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        case 2: launch_tma_epi<2>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        case 4: launch_tma_epi<4>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        case 8: launch_tma_epi<8>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        case 16: launch_tma_epi<16>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        case 32: launch_tma_epi<32>(st, tl, off, col, val, x, y, ctl, num_sms, epi); break;
        default: {
            if (epi && epi->kind != 0) throw Invalid("spmv: fused epilogue needs m in {1,2,4,8,16,32}");
            if (tl.rowid) throw Invalid("spmv: internal: sorted twin with a generic m");
            const int64_t total = nrows * m;
            spmm_generic_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(nrows, rows, off, col,
                                                                                            val, m, x, y, ctl);
        }
    }
    MBG_CUDA(cudaGetLastError());
    return launched + 1;
}

// Host: cut row segments into tiles of <= SPMM_TILE_ROWS rows and
// <= SPMM_TILE_NNZ nonzeros; a longer row gets a tile of its own (read from
// global memory by the kernel).  rows: sorted local row ids of one class
// (all rows, interior or boundary); tiles never span a gap.
std::vector<int32_t> long_rows_of(const std::vector<int4>& tiles) {
    std::vector<int32_t> out;
    for (const auto& t : tiles)
        if (t.w - t.z > SPMM_TILE_NNZ) out.push_back(t.x);
    return out;
}

bool build_stage_tiles(const std::vector<int32_t>& off, const int32_t* col, const std::vector<int32_t>& rows,
                       int64_t ncols, std::vector<uint16_t>& lcol, StageTiling& out) {
    out = StageTiling{};
    std::vector<int32_t> stamp(static_cast<size_t>(ncols), -1), pos(static_cast<size_t>(ncols), 0);
    std::vector<int32_t> cur;
    cur.reserve(STAGE_UCOLS);
    int64_t nnz_total = 0, u_total = 0;
    int32_t tid = 0;
    size_t i = 0;
    while (i < rows.size()) {
        const int r0 = rows[i];
        int r1 = r0;
        size_t j = i;
        cur.clear();
        while (j < rows.size() && rows[j] == r1 && r1 - r0 < STAGE_ROWS) {
            const int k0 = off[r1], k1 = off[r1 + 1];
            if (k1 - off[r0] > STAGE_NNZ) break;
            int fresh = 0;
            for (int k = k0; k < k1; ++k) fresh += stamp[col[k]] != tid;
            if (static_cast<int>(cur.size()) + fresh > STAGE_UCOLS) break;
            for (int k = k0; k < k1; ++k)
                if (stamp[col[k]] != tid) {
                    stamp[col[k]] = tid;
                    cur.push_back(col[k]);
                }
            ++r1;
            ++j;
        }
        if (r1 == r0) return false;   // one row beyond the limits: keep the plain kernel
        std::sort(cur.begin(), cur.end());
        for (size_t u = 0; u < cur.size(); ++u) pos[cur[u]] = static_cast<int32_t>(u);
        for (int k = off[r0]; k < off[r1]; ++k) lcol[k] = static_cast<uint16_t>(pos[col[k]]);
        out.tiles.push_back(make_int4(r0, r1, off[r0], off[r1]));
        out.umeta.push_back(make_int2(static_cast<int>(out.ucols.size()), static_cast<int>(cur.size())));
        out.ucols.insert(out.ucols.end(), cur.begin(), cur.end());
        nnz_total += off[r1] - off[r0];
        u_total += static_cast<int64_t>(cur.size());
        ++tid;
        i = j;
    }
    out.ucols.resize(out.ucols.size() + 8, 0);   // bulk copies round the last range up
    out.reuse = u_total ? static_cast<double>(nnz_total) / static_cast<double>(u_total) : 0.0;
    return true;
}

static bool tile_align() {
    static const bool on = [] {
        const char* e = std::getenv("MBG_TILE_ALIGN");
        return !(e && e[0] == '0');
    }();
    return on;
}

double spmm_lane_efficiency(const std::vector<int32_t>& off, const std::vector<int32_t>& rows) {
    int64_t useful = 0, slots = 0;
    for (size_t i = 0; i < rows.size(); i += 8) {
        int mx = 0;
        const size_t e = std::min(rows.size(), i + 8);
        for (size_t j = i; j < e; ++j) {
            const int b = (off[rows[j] + 1] - off[rows[j]] + 3) / 4;
            useful += b;
            mx = std::max(mx, b);
        }
        slots += static_cast<int64_t>(mx) * static_cast<int64_t>(e - i);
    }
    return slots ? static_cast<double>(useful) / static_cast<double>(slots) : 1.0;
}

// Host helper: fn(begin, end) over [0, n) in chunks that are multiples of
// `grain`, on up to 16 threads (the twin of an 8M-row matrix is built at upload).
template <class F>
static void host_parallel(size_t n, size_t grain, F fn) {
    const size_t units = (n + grain - 1) / grain;
    const unsigned nt = static_cast<unsigned>(
        std::min<size_t>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())), std::max<size_t>(1, units / 64)));
    if (nt <= 1) {
        fn(size_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (units + nt - 1) / nt * grain;
    for (unsigned t = 0; t < nt; ++t) {
        const size_t b = std::min(n, t * per), e = std::min(n, (t + 1) * per);
        if (b < e) th.emplace_back([=] { fn(b, e); });
    }
    for (auto& x : th) x.join();
}

void build_sorted_twin(const std::vector<int32_t>& off, const int32_t* col, const double* val,
                       const std::vector<int32_t>& rows, int window, SortedTwin& out) {
    out = SortedTwin{};
    // rows beyond a stage (a group's batches must fit one) go to the long-row kernel
    constexpr int MAX_BATCHES = SPMM_TILE_NNZ / 32;
    std::vector<int32_t> reg;
    reg.reserve(rows.size());
    for (int32_t r : rows) {
        if ((off[r + 1] - off[r] + 3) / 4 > MAX_BATCHES) out.long_rows.push_back(r);
        else reg.push_back(r);
    }
    const size_t n = reg.size();
    const size_t nslots = (n + 7) & ~size_t(7);
    out.rowid.assign(nslots + out.long_rows.size(), -1);
    host_parallel(n, static_cast<size_t>(window), [&](size_t begin, size_t end) {
        std::vector<int32_t> idx;
        for (size_t w0 = begin; w0 < end; w0 += static_cast<size_t>(window)) {
            const size_t w1 = std::min(n, w0 + static_cast<size_t>(window));
            idx.assign(reg.begin() + static_cast<std::ptrdiff_t>(w0), reg.begin() + static_cast<std::ptrdiff_t>(w1));
            std::stable_sort(idx.begin(), idx.end(),
                             [&](int32_t a, int32_t b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
            std::copy(idx.begin(), idx.end(), out.rowid.begin() + static_cast<std::ptrdiff_t>(w0));
        }
    });
    // groups of 8 slots, each with the batches of its longest row
    const size_t G = nslots / 8;
    out.off.assign(G + 1, 0);
    for (size_t g = 0; g < G; ++g) {
        int nb = 0;
        for (int r8 = 0; r8 < 8; ++r8) {
            const int32_t r = out.rowid[g * 8 + r8];
            if (r >= 0) nb = std::max(nb, (off[r + 1] - off[r] + 3) / 4);
        }
        const int64_t next = static_cast<int64_t>(out.off[g]) + nb;
        if (next * 32 > INT32_MAX - 64) throw Invalid("csr: the length-sorted copy needs 64-bit offsets");
        out.off[g + 1] = static_cast<int32_t>(next);
    }
    // batch-major inside a group: columns [batch][row][4], values [batch][half][row][2]
    const size_t entries = static_cast<size_t>(out.off[G]) * 32;
    out.col.resize(entries);
    out.val.resize(entries);
    host_parallel(G, 1, [&](size_t gb, size_t ge) {   // groups own disjoint ranges of col / val
        std::fill(out.col.begin() + static_cast<std::ptrdiff_t>(out.off[gb]) * 32,
                  out.col.begin() + static_cast<std::ptrdiff_t>(out.off[ge]) * 32, -1);
        std::fill(out.val.begin() + static_cast<std::ptrdiff_t>(out.off[gb]) * 32,
                  out.val.begin() + static_cast<std::ptrdiff_t>(out.off[ge]) * 32, 0.0);
        for (size_t g = gb; g < ge; ++g)
            for (int r8 = 0; r8 < 8; ++r8) {
                const int32_t r = out.rowid[g * 8 + static_cast<size_t>(r8)];
                if (r < 0) continue;
                const int len = off[r + 1] - off[r];
                for (int e = 0; e < len; ++e) {
                    const size_t b = static_cast<size_t>(out.off[g]) + static_cast<size_t>(e / 4);
                    const int q = e & 3;
                    out.col[(b * 8 + static_cast<size_t>(r8)) * 4 + static_cast<size_t>(q)] = col[off[r] + e];
                    out.val[((b * 2 + static_cast<size_t>(q >> 1)) * 8 + static_cast<size_t>(r8)) * 2 +
                            static_cast<size_t>(q & 1)] = val[off[r] + e];
                }
            }
    });
    // tiles of whole groups: <= SPMM_TILE_ROWS slots, <= MAX_BATCHES batches; one cut by
    // the batch cap keeps a multiple of 64 slots (whole block passes at m = 8)
    size_t g = 0;
    while (g < G) {
        size_t h = g;
        while (h < G && (h - g) * 8 < static_cast<size_t>(SPMM_TILE_ROWS) && out.off[h + 1] - out.off[g] <= MAX_BATCHES) ++h;
        if ((h - g) * 8 < static_cast<size_t>(SPMM_TILE_ROWS) && h < G && h - g >= 8) h = g + ((h - g) & ~size_t(7));
        out.tiles.push_back(make_int4(static_cast<int>(g * 8), static_cast<int>(h * 8), out.off[g], out.off[h]));
        g = h;
    }
    // one epilogue-only tile per long row (slot after the groups, batch -1)
    for (size_t i = 0; i < out.long_rows.size(); ++i) {
        out.rowid[nslots + i] = out.long_rows[i];
        out.tiles.push_back(make_int4(static_cast<int>(nslots + i), static_cast<int>(nslots + i + 1), -1, -1));
    }
}

std::vector<int4> build_spmm_tiles(const std::vector<int32_t>& off, const std::vector<int32_t>& rows, bool sorted) {
    std::vector<int4> out;
    size_t i = 0;
    while (i < rows.size()) {
        const int r0 = rows[i];
        int r1 = r0;
        size_t j = i;
        while (j < rows.size() && rows[j] == r1 && r1 - r0 < SPMM_TILE_ROWS &&
               (off[r1 + 1] - off[r0] <= SPMM_TILE_NNZ || r1 == r0)) {
            ++r1;
            ++j;
        }
        // a block pass covers 256 / (m/2) rows (64 at m = 8, 32 at m = 16, 16
        // at m = 32): a tile cut by the nonzero cap is trimmed to a multiple of
        // 64 (else 16) rows so that no pass runs half empty (B200, C5 random
        // band: m=8 1244 -> 1159 us, m=16 1851 -> 1737 us per SpMM; a 27-point
        // CSR operator loses L1 reuse with the smaller tiles, but declared on
        // its grid it runs on the stencil twin anyway; MBG_TILE_ALIGN=0: off)
        if (tile_align() && r1 - r0 < SPMM_TILE_ROWS) {
            const int len = r1 - r0;
            // (length-sorted twin: a tile's rows have one length, the longest
            // ones -- 60 rows of 32 -- keep their single nearly full pass)
            const int al = len >= 64 ? (len & ~63) : (len >= 16 && !sorted ? (len & ~15) : len);
            j -= static_cast<size_t>(len - al);
            r1 = r0 + al;
        }
        out.push_back(make_int4(r0, r1, off[r0], off[r1]));
        i = j;
    }
    return out;
}

}  // namespace mbg
