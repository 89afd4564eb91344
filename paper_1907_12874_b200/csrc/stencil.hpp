// stencil.hpp -- structured-grid SpMM (stencil.cu).
//
// When the caller declares the grid (mbg_csr_set_grid) and every nonzero of
// the CSR couples a point with one of its 26 grid neighbours (or itself), the
// operator gets a stencil twin: per xy-tile plane a chunk of values laid out
// slot-major plus a per-row slot mask.  Column indices are then implicit, so
// the SpMM streams 8 B per nonzero instead of 12 (+4 B/row mask instead of
// the 4 B/row offsets) and stages x as TMA tensor boxes of grid planes in
// shared memory.  Each (row, column) is still summed in CSR order from 0.0
// (ascending column == ascending slot on a grid), so results are bitwise
// those of the CSR SpMM (spmv.cpp:40-46).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"

namespace mbg {

constexpr int STENCIL_BX = 32;   // tile width along x (grid points)

struct StencilLayout {
    int by = 0;                     // tile height along y
    int zpart = 0;                  // 1: 27-point z-part chunks (stencil27z_kernel) -- see stencil.cu
    int64_t chunk_bytes = 0;        // S * 32*by * 8 (values) + 32*by * 4 (masks)
    DevBuf<unsigned char> chunks;   // [(tile * nz + z)] chunks
};

// Local numbering of a (possibly z-slab partitioned) operator: owned rows are
// the global rows [row_begin, row_begin + n_own) = whole planes z0 .. z0+nzl-1;
// halo columns (plan.cpp: ascending global ids after the owned rows) are the
// plane z0-1 (when `lower`) followed by the plane z0+nzl (when the op's `upper`).
struct GridMap {
    int nx, ny;
    int64_t row_begin, n_own;
    int z0, nzl;
    int lower;
#ifdef __CUDACC__
    __device__ int64_t global_col(int64_t j) const {
        if (j < n_own) return row_begin + j;
        const int64_t nxy = static_cast<int64_t>(nx) * ny;
        int64_t h = j - n_own;
        if (lower) {
            if (h < nxy) return static_cast<int64_t>(z0 - 1) * nxy + h;
            h -= nxy;
        }
        return static_cast<int64_t>(z0 + nzl) * nxy + h;
    }
#endif
};

struct StencilOp {
    int nx = 0, ny = 0;
    int nz = 0;            // local planes (the whole grid on one GPU)
    int nzg = 0;           // global planes
    GridMap map{};         // local -> global numbering
    int upper = 0;         // halo plane above the slab
    int kind = 0;          // 7 (face neighbours only) or 27
    int64_t nnz = 0;
    std::vector<std::unique_ptr<StencilLayout>> layouts;   // built lazily per tile height
};

// Analyse the device CSR of `a` on the grid; returns nullptr when some
// nonzero is not a grid neighbour (the CSR SpMM stays in use).
std::shared_ptr<StencilOp> build_stencil(mbg_ctx* ctx, const mbg_csr* a, int nx, int ny, int nz);
// True when the stencil SpMM handles m (4, 8, 16, 32; not disabled by MBG_STENCIL=0).
bool stencil_handles(const mbg_csr* a, int m);
// MBG_STENCIL_EPI=1: the solver moves exact dots into the stencil SpMM's
// epilogue (classical delta, phi/psi; Reordered delta).  Measured slower on
// B200 (the TwoSum chains of the epilogue are latency-bound at the stencil
// kernel's 8-10 warps per SM), hence off by default.
bool stencil_epilogues();
// y = A x through the stencil twin; returns the number of kernel launches.
// epi: optional fused exact-dot epilogue (kernels.hpp SpmmEpi, kinds 1-4).
struct SpmmEpi;
// [zbeg, zend): local planes to compute (default: all); a z-slab partition
// runs its interior planes while the halo planes travel, then the two faces.
int launch_stencil_spmm(mbg_ctx* ctx, const mbg_csr* a, int m, const double* x, double* y, const int* ctl,
                        const SpmmEpi* epi = nullptr, int zbeg = 0, int zend = -1);
// y = A xin with xin = (0 + 1*z) + na*v (na: m per-column coefficients),
// formed per x plane in shared memory -- the Reordered th = z - alpha s update
// fused into its SpMM (same expression, same bits).  Single-GPU 27-point
// operators at m = 16 / 32 (stencil_axpy_handles); returns kernel launches.
bool stencil_axpy_handles(const mbg_csr* a, int m);
// The z-marching 27-point kernel (m = 16 / 32) carries the delta = (y, aux)
// epilogue (SpmmEpi kind 1) -- the fused Reordered delta pass folded into the
// first SpMM.  Opt-in (MBG_Z27_EPI=1): measured slower on B200.
bool stencil_delta_epilogue(const mbg_csr* a, int m);
int launch_stencil_spmm_axpy(mbg_ctx* ctx, const mbg_csr* a, int m, const double* z, const double* v,
                             const double* na, double* y, const int* ctl);
// Algorithmic bytes of one stencil SpMM: x read once, y written once, 8 B per
// nonzero value, 4 B per row mask.
double stencil_spmm_bytes(int64_t n, int64_t nnz, int m);

}  // namespace mbg
