// kernels.hpp -- host-side launchers of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "group.cuh"

namespace mbg {

// CSR SpMM over the interleaved block (spmm.cu).  The row set to compute is
// given twice: as a tile list (TMA-pipelined kernels, m in {1,2,4,8,16,32})
// and as an explicit row list (nullptr = rows [0, nrows)) for other m.
constexpr int SPMM_TILE_ROWS = 192;
constexpr int SPMM_TILE_NNZ = 1920;
struct SpmmTiles {
    const int4* tiles = nullptr;   // (r0, r1, k0, k1) per tile
    int64_t count = 0;
    const int32_t* long_rows = nullptr;  // rows of the single-row tiles beyond SPMM_TILE_NNZ
    int64_t nlong = 0;
    bool long_rows_hint = false;         // average row length > 12: use the 3-block variant
    // gather-once ("staged") tiling, set when the matrix reuses x rows inside
    // a tile (stencils): per tile the unique columns, and per nonzero its
    // 16-bit index into them (spmm.cu spmm_stage_kernel)
    const int4* stiles = nullptr;        // (r0, r1, k0, k1) per staged tile
    const int2* umeta = nullptr;         // (u0, U): the tile's columns are ucols[u0 .. u0+U)
    const int32_t* ucols = nullptr;
    const uint16_t* lcol = nullptr;      // indexed by the global nonzero k
    int64_t scount = 0;
    // length-sorted twin (build_sorted_twin): `tiles` then index slots of the
    // row-permuted copy (s_off / s_col / s_val) and rowid[slot] is the row the
    // slot's result belongs to; long_rows stay original row ids
    const int32_t* rowid = nullptr;
    const int32_t* s_off = nullptr;
    const int32_t* s_col = nullptr;
    const double* s_val = nullptr;
    // {next tile, finished blocks}: the twin's tiles differ in work (rows of one
    // length per tile), so blocks claim them from a counter instead of striding
    int* sched = nullptr;
};
// Optional fused epilogue of the SpMM y = A x (beyond-paper merge):
//   kind 1: slot[0] += exact (y, aux)                    e.g. delta = (v, r0)
//   kind 2: slot[0..2] += exact (y, x), (y, y), (x, x)    phi, psi, theta of Alg. 2
//   kind 3: slot[0] += exact (y, y)                       e.g. psi = (t, t)
//   kind 4: slot[0..1] += exact (y, x), (y, y)            phi, psi of Alg. 2 (stencil SpMM only)
struct SpmmEpi {
    int kind = 0;
    const double* aux = nullptr;
    int64_t* slot[3] = {nullptr, nullptr, nullptr};
};
int launch_spmm(cudaStream_t st, const SpmmTiles& tl, int64_t nrows, const int32_t* rows, const int32_t* off,
                const int32_t* col, const double* val, int m, const double* x, double* y, const int* ctl,
                int num_sms, const SpmmEpi* epi = nullptr);
std::vector<int4> build_spmm_tiles(const std::vector<int32_t>& off, const std::vector<int32_t>& rows,
                                   bool sorted = false);
std::vector<int32_t> long_rows_of(const std::vector<int4>& tiles);

// Length-sorted twin of one row class (SELL-C-sigma's sigma step without the
// padding): inside windows of `window` consecutive rows of the class the rows
// are stored by descending length, every row's nonzeros in their CSR order, so
// the lanes of a warp and the warps of a tile walk rows of (nearly) one length
// and finish together.  Only the storage order of the rows changes: each
// (row, column) sum is the same sequence of operations.
// std::vector without value-initialisation on resize (the twin's 2.4 GB of
// columns / values are first touched by the threads that fill them)
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind { using other = DefaultInitAlloc<U>; };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U>&) {}
    template <class U>
    void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
    template <class U, class... A>
    void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
};
template <class T>
using RawVec = std::vector<T, DefaultInitAlloc<T>>;

struct SortedTwin {
    std::vector<int32_t> off, rowid;
    RawVec<int32_t> col;
    RawVec<double> val;
    std::vector<int4> tiles;          // over slots
    std::vector<int32_t> long_rows;   // original row ids of the one-row tiles beyond SPMM_TILE_NNZ
};
// Share of the gather slots of 8-row warps (batches of 4 nonzeros) that do
// useful work in the natural row order; the twin is built below ~0.92.
double spmm_lane_efficiency(const std::vector<int32_t>& off, const std::vector<int32_t>& rows);
void build_sorted_twin(const std::vector<int32_t>& off, const int32_t* col, const double* val,
                       const std::vector<int32_t>& rows, int window, SortedTwin& out);

// Gather-once tiling: tiles of <= STAGE_ROWS rows, <= STAGE_NNZ nonzeros and
// <= STAGE_UCOLS distinct columns.  lcol (size >= nnz, shared by disjoint row
// classes) receives each nonzero's index into its tile's column list.
// Returns false (and builds nothing) when a single row exceeds the limits.
constexpr int STAGE_ROWS = 128, STAGE_NNZ = 1024, STAGE_UCOLS = 256;
struct StageTiling {
    std::vector<int4> tiles;
    std::vector<int2> umeta;
    std::vector<int32_t> ucols;
    double reuse = 0.0;   // nonzeros per staged x row
};
bool build_stage_tiles(const std::vector<int32_t>& off, const int32_t* col, const std::vector<int32_t>& rows,
                       int64_t ncols, std::vector<uint16_t>& lcol, StageTiling& out);

// Generic statement-group interpreter (API-level execute_group).
constexpr int GEN_MAX_VEC = 16, GEN_MAX_STMT = 16, GEN_MAX_SLOT = 8;
struct GenericGroup {
    int64_t len;
    int m;
    int nstmt;
    double* vec[GEN_MAX_VEC];
    // statement s: kind, out, nterms, first term index; dot: left, right, slot
    int kind[GEN_MAX_STMT], out[GEN_MAX_STMT], nterms[GEN_MAX_STMT], tfirst[GEN_MAX_STMT];
    int left[GEN_MAX_STMT], right[GEN_MAX_STMT], dslot[GEN_MAX_STMT];
    int term_vec[GEN_MAX_STMT * MBG_MAX_TERMS];
    const double* coef;   // device: term t, column c at coef[t*m + c]
    int nslots;
    int64_t* slot;        // nslots * m * NSLOT
};
void launch_generic_group(cudaStream_t st, const GenericGroup& g, int num_sms, int* nblocks_out);

// Round long accumulators into doubles out[s*m + c] and clear them (kernels.cu).
void launch_round(cudaStream_t st, int64_t* D, int nslots, int m, double* out);

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its stream predecessor drains (it calls pdl_wait() first).  MBG_PDL=0
// turns it off (A/B measurements).
bool pdl_enabled();
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MBG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Occupancy-sized persistent grid for a group kernel instantiation.
// blocks/SM of `kernel` on the current device (sets its dynamic shared-memory
// attribute there first); cached per device, thread-safe
int kernel_occupancy(const void* kernel, int threads, size_t smem);
int group_grid(const void* kernel, int block, size_t smem, int num_sms, int64_t len);

template <class P>
inline int launch_group(cudaStream_t st, const GroupArgs& a, int num_sms) {
    const int block = group_block(a.m);
    size_t smem = P::NDOT > 0 ? static_cast<size_t>(block) * KEXP * sizeof(double) : 0;
    if constexpr (vec_of<P>::value == 2) {
        if ((a.m % 2 == 0 || a.m == 1) && a.len % 2 == 0) {
            const int grid =
                group_grid(reinterpret_cast<const void*>(&group_kernel<P, 2>), block, smem, num_sms, a.len / 2);
            launch_pdl(group_kernel<P, 2>, dim3(grid), dim3(block), smem, st, a);
            return grid;
        }
    }
    const int grid = group_grid(reinterpret_cast<const void*>(&group_kernel<P, 1>), block, smem, num_sms, a.len);
    launch_pdl(group_kernel<P, 1>, dim3(grid), dim3(block), smem, st, a);
    return grid;
}

}  // namespace mbg
