// stencil.cu -- SpMM  Y = A X  for operators declared on a structured grid.
//
// Same arithmetic as spmv_rows (spmv.cpp:40-46) and spmm.cu: each (row,
// column) is the sequential sum, in CSR order from 0.0, of separately rounded
// products val[k]*x(col[k], c).  On an nx*ny*nz grid (lexicographic rows) a
// nonzero that couples a point with a neighbour (dz, dy, dx) in {-1,0,1}^3
// has a "slot"; ascending columns are ascending slots, so summing a row's
// present slots in slot order IS the CSR order.  The twin built at
// mbg_csr_set_grid therefore drops the column indices:
//
//   chunk (tile t, plane z) = values[S][32*BY] (slot-major; -0.0 where a slot
//                             is absent) | mask[32*BY] (bit s: slot s present;
//                             bit 31: the row misses an in-grid neighbour)
//
// for xy-tiles of 32 x BY points (rows of odd lines swap 4-point blocks: bank
// spread).  An absent slot's x operand is the TMA zero fill of an out-of-grid
// point, and (-0.0)*(+0.0) = -0.0 is the exact identity of IEEE addition, so
// only bit-31 rows need a predicate.
//
// Kernel: persistent and warp-specialised.  Block ranges of whole tiles (or
// z-segments) start at the same z and march through the planes, so an x plane
// is fetched from HBM about once and its halo lines hit L2 for the
// neighbouring tiles.  A producer warp streams the x planes as TMA tensor
// boxes (m, 34|35, BY+2, 1) of x viewed as (planes, ny, nx, m) -- a second
// tensor map addresses the halo planes of a z-slab partition -- into a 5-deep
// ring and the value chunks (cp.async.bulk) into a 3-deep ring, gated by
// full / empty mbarriers.  A compute lane owns 4 consecutive points along x
// and 2 columns: the 6 x points of a stencil line are loaded once from shared
// memory and reused by the 3 dx slots of the 4 rows.
//
// Bytes per SpMM (the roofline's algorithmic count): 16*N*m (x once, y once)
// + 8*nnz (values) + 4*N (masks); versus 16*N*m + 12*nnz + 4*N for CSR.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "comm.hpp"
#include "common.hpp"
#include "exact.cuh"
#include "group.cuh"
#include "kernels.hpp"
#include "stencil.hpp"
#include "tma.cuh"

namespace mbg {

// ---- analysis and layout (device kernels over the uploaded CSR) -----------

// Row slot swizzle inside a chunk: odd lines (BY = 4 layout) or lines 1-3 of
// each 4 (BY = 8 layout, m = 4) swap 4-point blocks, so the value / mask loads
// of the groups that share a quarter warp fall on different banks.
__host__ __device__ constexpr int stencil_swz(int by, int ly) { return by == 8 ? ((ly & 3) << 2) : ((ly & 1) << 2); }


__device__ __forceinline__ void grid_coords(int64_t i, int nx, int ny, int& x, int& y, int& z) {
    x = static_cast<int>(i % nx);
    const int64_t t = i / nx;
    y = static_cast<int>(t % ny);
    z = static_cast<int>(t / ny);
}

// 7-point slot order = ascending column order: -z, -y, -x, centre, +x, +y, +z
__device__ __forceinline__ int face_slot(int dz, int dy, int dx) {
    if (dz) return dz < 0 ? 0 : 6;
    if (dy) return dy < 0 ? 1 : 5;
    return 3 + dx;
}

// flags: 1 = a nonzero outside the 3x3x3 neighbourhood; 2 = a non-face
// neighbour (27-point); 4 = slots not strictly ascending within a row
__global__ void stencil_scan_kernel(GridMap gm, const int32_t* __restrict__ off, const int32_t* __restrict__ col,
                                    unsigned* flags) {
    unsigned f = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < gm.n_own;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int xi, yi, zi;
        grid_coords(gm.row_begin + i, gm.nx, gm.ny, xi, yi, zi);
        int prev = -1;
        for (int k = off[i]; k < off[i + 1]; ++k) {
            int xj, yj, zj;
            grid_coords(gm.global_col(col[k]), gm.nx, gm.ny, xj, yj, zj);
            const int dx = xj - xi, dy = yj - yi, dz = zj - zi;
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) {
                f |= 1u;
                continue;
            }
            const int s = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
            if (s <= prev) f |= 4u;
            prev = s;
            if ((dx != 0) + (dy != 0) + (dz != 0) > 1) f |= 2u;
        }
    }
    if (f) atomicOr(flags, f);
}

// Absent slots hold -0.0: their x operand is either the TMA zero fill of an
// out-of-grid point (+0.0), making the term exactly -0.0, the identity of
// IEEE addition (acc + -0.0 == acc for every acc, signed zeros and NaNs
// included), or -- for an in-grid neighbour the CSR leaves out -- the row is
// flagged (mask bit 31) and takes the predicated path.
__global__ void stencil_clear_kernel(int64_t nchunks, int S, int RT, int64_t chunk_bytes, unsigned char* chunks) {
    const int64_t per = chunk_bytes / 8;   // 8-byte words per chunk
    const int64_t nval = static_cast<int64_t>(S) * RT;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nchunks * per;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t w = e % per;
        reinterpret_cast<unsigned long long*>(chunks)[e] = w < nval ? 0x8000000000000000ull : 0ull;
    }
}

__global__ void stencil_fill_kernel(GridMap gm, int nzg, int by, int S, int ntx, int64_t chunk_bytes,
                                    const int32_t* __restrict__ off, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, unsigned char* __restrict__ chunks) {
    const int RT = STENCIL_BX * by;
    const int nx = gm.nx, ny = gm.ny;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < gm.n_own;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int xi, yi, zi;
        grid_coords(gm.row_begin + i, nx, ny, xi, yi, zi);
        const int64_t t = static_cast<int64_t>(yi / by) * ntx + xi / STENCIL_BX;
        // row slot inside the chunk: odd lines swap 4-point blocks pairwise
        // (bank spread for the m = 8 lane layout; 4-aligned blocks stay contiguous)
        const int ly = yi % by;
        const int r = ly * STENCIL_BX + ((xi % STENCIL_BX) ^ stencil_swz(by, ly));
        unsigned char* c = chunks + (t * gm.nzl + (zi - gm.z0)) * chunk_bytes;
        double* V = reinterpret_cast<double*>(c);
        uint32_t* MK = reinterpret_cast<uint32_t*>(c + static_cast<int64_t>(S) * RT * 8);
        uint32_t mask = 0;
        for (int k = off[i]; k < off[i + 1]; ++k) {
            int xj, yj, zj;
            grid_coords(gm.global_col(col[k]), nx, ny, xj, yj, zj);
            const int dx = xj - xi, dy = yj - yi, dz = zj - zi;
            const int s = S == 27 ? (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1) : face_slot(dz, dy, dx);
            V[static_cast<int64_t>(s) * RT + r] = val[k];
            mask |= 1u << s;
        }
        // an absent slot whose neighbour lies inside the grid needs the predicated path
        bool check = false;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (S == 7 && (dx != 0) + (dy != 0) + (dz != 0) > 1) continue;
                    const int s = S == 27 ? (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1) : face_slot(dz, dy, dx);
                    const bool inside = xi + dx >= 0 && xi + dx < nx && yi + dy >= 0 && yi + dy < ny &&
                                        zi + dz >= 0 && zi + dz < nzg;
                    if (inside && !((mask >> s) & 1u)) check = true;
                }
        MK[r] = mask | (check ? 0x80000000u : 0u);
    }
}

// z-part layout of a 27-point chunk (stencil27z_kernel): the 27 slots split
// by dz into three parts of 9, each [9][RT] doubles, with the row masks after
// part 0:  part0 (dz=-1) | mask[RT] | part1 (dz=0) | part2 (dz=+1).  Rows are
// not swizzled (r = ly * 32 + lx).  The kernel streams, for x plane p, part 0
// of row plane p+1, part 1 of p and part 2 of p-1.
__host__ __device__ constexpr int64_t zpart_off(int d, int RT) {
    return d == 0 ? 0 : (static_cast<int64_t>(9 * d) * RT * 8 + static_cast<int64_t>(RT) * 4);
}

__global__ void stencil_fill_zpart_kernel(GridMap gm, int nzg, int by, int ntx, int64_t chunk_bytes,
                                          const int32_t* __restrict__ off, const int32_t* __restrict__ col,
                                          const double* __restrict__ val, unsigned char* __restrict__ chunks) {
    const int RT = STENCIL_BX * by;
    const int nx = gm.nx, ny = gm.ny;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < gm.n_own;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int xi, yi, zi;
        grid_coords(gm.row_begin + i, nx, ny, xi, yi, zi);
        const int64_t t = static_cast<int64_t>(yi / by) * ntx + xi / STENCIL_BX;
        const int r = (yi % by) * STENCIL_BX + xi % STENCIL_BX;
        unsigned char* c = chunks + (t * gm.nzl + (zi - gm.z0)) * chunk_bytes;
        auto slot = [&](int s) -> double* {
            return reinterpret_cast<double*>(c + zpart_off(s / 9, RT)) + static_cast<int64_t>(s % 9) * RT + r;
        };
        for (int s = 0; s < 27; ++s) *slot(s) = -0.0;
        uint32_t mask = 0;
        for (int k = off[i]; k < off[i + 1]; ++k) {
            int xj, yj, zj;
            grid_coords(gm.global_col(col[k]), nx, ny, xj, yj, zj);
            const int s = (zj - zi + 1) * 9 + (yj - yi + 1) * 3 + (xj - xi + 1);
            *slot(s) = val[k];
            mask |= 1u << s;
        }
        bool check = false;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int s = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
                    const bool inside = xi + dx >= 0 && xi + dx < nx && yi + dy >= 0 && yi + dy < ny &&
                                        zi + dz >= 0 && zi + dz < nzg;
                    if (inside && !((mask >> s) & 1u)) check = true;
                }
        reinterpret_cast<uint32_t*>(c + 9 * static_cast<int64_t>(RT) * 8)[r] = mask | (check ? 0x80000000u : 0u);
    }
}

// ---- the SpMM kernel --------------------------------------------------------

struct StencilGeom {
    int nx, ny;
    int nz;               // planes of this launch's range [zbeg, zbeg + nz)
    int zbeg;             // first local plane of the range
    int nzl;              // local planes (chunk layout); planes -1 / nzl come from the halo map
    int lower, upper;     // halo planes present below / above (z-slab partition)
    int ntx;              // tiles along x
    int64_t steps;        // tile-planes per column half: ntiles * nz
    int nranges;          // step ranges (blocks per column half)
    int kt;               // whole tiles per range (kt >= 1, zseg == nz) ...
    int zseg;             // ... or one z-segment of zseg planes of one tile per range (kt == 0)
    int mode;             // lab switch (MBG_STENCIL_MODE): 0 normal, 1 no arithmetic, 2 no data movement
    const unsigned char* chunks;
    int64_t chunk_bytes;
};

template <int MC, int BY>
struct StencilShape {
    static constexpr int LPR = MC / 2;                       // lanes per 4-point group (2 columns each)
    static constexpr int THREADS = 8 * BY * LPR;             // compute threads: 8 groups along x, BY along y
    static constexpr int NCW = THREADS / 32;                 // compute warps (+1 producer warp)
    static constexpr int LW = MC <= 8 ? 35 : 34;             // x-plane line width (35: bank spread at m <= 8)
    static constexpr int RT = STENCIL_BX * BY;               // rows per tile plane
    static constexpr int PLANE = LW * (BY + 2) * MC;         // doubles per x plane (the TMA box)
    static constexpr int PSTRIDE = (PLANE + 15) / 16 * 16;   // ring slot stride: 128-byte aligned boxes
};

template <int ST, int BY>
__host__ __device__ constexpr int stencil_chunk_bytes() { return ST * STENCIL_BX * BY * 8 + STENCIL_BX * BY * 4; }

#ifndef MBG_STENCIL_XR8
#define MBG_STENCIL_XR8 5
#define MBG_STENCIL_VR8 3
#endif
// ring depths (x planes, value chunks); m = 8 blocks may trade depth for occupancy
template <int MC>
struct StencilRings {
    static constexpr int XR = MC == 8 ? MBG_STENCIL_XR8 : 5;
    static constexpr int VR = MC == 8 ? MBG_STENCIL_VR8 : 3;
};
constexpr int STENCIL_HEAD = 256;               // mbarriers

template <int MC, int ST, int BY>
__host__ __device__ constexpr int stencil_smem() {
    return STENCIL_HEAD + StencilRings<MC>::XR * StencilShape<MC, BY>::PSTRIDE * 8 +
           StencilRings<MC>::VR * stencil_chunk_bytes<ST, BY>();
}

// acc[r][c] += v * x: the reference's  acc = acc + val*x  (no FMA)
#define MBG_ACC(r, v, xv)                                        \
    do {                                                         \
        acc[r][0] = __dadd_rn(acc[r][0], __dmul_rn((v), (xv).x)); \
        acc[r][1] = __dadd_rn(acc[r][1], __dmul_rn((v), (xv).y)); \
    } while (0)

template <int MC, int ST, int BY, bool CHECK>
__device__ __forceinline__ void stencil_rows(double (&acc)[4][2], const double* __restrict__ P0,
                                             const double* __restrict__ P1, const double* __restrict__ P2,
                                             const double* __restrict__ V, const uint32_t (&mk)[4], int gy, int lx0,
                                             int cp, int r0) {
    using SH = StencilShape<MC, BY>;
    constexpr int LW = SH::LW, RT = SH::RT;
    auto ld2 = [](const double* p) { return *reinterpret_cast<const double2*>(p); };
    auto vals = [&](int s, double (&v)[4]) {
        const double2 a = ld2(V + s * RT + r0), b = ld2(V + s * RT + r0 + 2);
        v[0] = a.x;
        v[1] = a.y;
        v[2] = b.x;
        v[3] = b.y;
    };
    // point (line ly, x offset j from lx0 - 1) of a plane
    auto pt = [&](const double* P, int ly, int j) { return ld2(P + ((gy + ly) * LW + lx0 + j) * MC + cp); };
    if constexpr (ST == 27) {
#pragma unroll
        for (int dz = 0; dz < 3; ++dz) {
            const double* P = dz == 0 ? P0 : (dz == 1 ? P1 : P2);
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
                double2 xp[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) xp[j] = pt(P, dy, j);
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    const int s = dz * 9 + dy * 3 + dx;
                    double v[4];
                    vals(s, v);
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (!CHECK || ((mk[r] >> s) & 1u)) MBG_ACC(r, v[r], xp[r + dx]);
                }
            }
        }
    } else {
        // slots: 0 (-z), 1 (-y), 2 3 4 (-x, centre, +x), 5 (+y), 6 (+z)
        auto line1 = [&](const double* P, int ly, int s) {
            double2 xp[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) xp[r] = pt(P, ly, r + 1);
            double v[4];
            vals(s, v);
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (!CHECK || ((mk[r] >> s) & 1u)) MBG_ACC(r, v[r], xp[r]);
        };
        line1(P0, 1, 0);
        line1(P1, 0, 1);
        {
            double2 xp[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) xp[j] = pt(P1, 1, j);
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                double v[4];
                vals(2 + dx, v);
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (!CHECK || ((mk[r] >> (2 + dx)) & 1u)) MBG_ACC(r, v[r], xp[r + dx]);
            }
        }
        line1(P1, 2, 5);
        line1(P2, 1, 6);
    }
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// Persistent, warp-specialised: block b owns an equal range of the step
// sequence s = tile * nz + z (z fastest) of one column half; the range is
// cut into z-segments at tile boundaries.  The producer warp streams, per
// segment, the x planes za-1 .. zb (TMA tensor boxes) and the value chunks
// za .. zb-1 (bulk copies) through the rings, gated by "empty" barriers that
// the compute warps arrive on when they are done with a slot; compute warps
// never wait on each other.  MT: columns of the block vector; MC: columns of
// one block (MT / MC column halves run as adjacent blocks over the same
// range, so the second read of a value chunk hits L2).
// EPI (kernels.hpp SpmmEpi kinds): 0 none; 1 (y, aux); 2 (y, x), (y, y),
// (x, x); 3 (y, y); 4 (y, x), (y, y) -- exact dots of the finished rows, x
// being the SpMM input at the row itself (the centre point of the staged plane).
template <int EPI>
struct StencilEpiDots {
    static constexpr int value = EPI == 2 ? 3 : (EPI == 4 ? 2 : 1);
};

template <int MT, int MC, int ST, int BY, int EPI>
__global__ void __launch_bounds__(StencilShape<MC, BY>::THREADS + 32)
    stencil_spmm_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
                        StencilGeom g, double* __restrict__ y, const int* __restrict__ ctl, SpmmEpi epi) {
    using SH = StencilShape<MC, BY>;
    constexpr int CS = MT / MC;
    constexpr int XR = StencilRings<MC>::XR, VR = StencilRings<MC>::VR;
    constexpr int CB = stencil_chunk_bytes<ST, BY>();
    static_assert(CB % 16 == 0 && (SH::PSTRIDE * 8) % 128 == 0, "ring slot alignment");
    pdl_wait();
    if (ctl && ctl[0]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* xfull = reinterpret_cast<uint64_t*>(smem);
    uint64_t* xempty = xfull + XR;
    uint64_t* vfull = xempty + XR;
    uint64_t* vempty = vfull + VR;
    double* xr = reinterpret_cast<double*>(smem + STENCIL_HEAD);
    unsigned char* vr = smem + STENCIL_HEAD + XR * SH::PSTRIDE * 8;

    const int h = blockIdx.x % CS;
    const int rb = blockIdx.x / CS;
    // ranges move through z in lockstep (every range starts at the same z), so
    // a plane of x is read by all its neighbouring tiles at about the same time
    // the block's segments (tile, first plane, planes): with whole tiles per
    // block the tiles are strided by the number of ranges, so at any moment all
    // blocks work on one contiguous band of tiles at about the same plane --
    // a tile's y neighbours (t +- ntx) are in the band and their shared halo
    // lines hit L2 (C4 320^3 m=32: DRAM reads 15.0 -> 11.0 GB, 3.67 -> 3.38 ms
    // per SpMM, against contiguous tile ranges); else one z-segment of a tile
    const int ntiles = static_cast<int>(g.steps / g.nz);
    const int nsegs_b = g.kt > 0 ? g.kt : 1;
    auto segment = [&](int si, int& t, int& za, int& steps) {
        if (g.kt > 0) {
            t = rb + si * g.nranges;
            za = 0;
            steps = t < ntiles ? g.nz : 0;
        } else {
            const int nseg = (g.nz + g.zseg - 1) / g.zseg;
            t = rb / nseg;
            const int sg = rb % nseg;
            za = sg * g.zseg;
            steps = t < ntiles ? min(g.nz, za + g.zseg) - za : 0;
        }
    };
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < XR; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&xempty[b], SH::NCW);
        }
        for (int b = 0; b < VR; ++b) {
            mbar_init(&vfull[b], 1);
            mbar_init(&vempty[b], SH::NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= SH::THREADS) {   // ---- producer warp
        if (tid == SH::THREADS && g.mode != 2) {
            int64_t Q = 0, j = 0;   // plane loads / chunk loads issued so far
            auto plane = [&](int t, int p) {   // p: plane within the range
                const int b = static_cast<int>(Q % XR);
                if (Q >= XR) mbar_wait(&xempty[b], static_cast<uint32_t>((Q / XR - 1) & 1));
                mbar_expect_tx(&xfull[b], static_cast<uint32_t>(SH::PLANE * 8));
                const int pl = g.zbeg + p;   // local plane; -1 / nzl: halo (or zero fill)
                const void* map = &xmap;
                int pz = pl;
                if (pl < 0 && g.lower) {
                    map = &hmap;
                    pz = 0;
                } else if (pl >= g.nzl && g.upper) {
                    map = &hmap;
                    pz = g.lower;
                }
                tensor4d_g2s(xr + b * SH::PSTRIDE, map, h * MC, (t % g.ntx) * STENCIL_BX - 1, (t / g.ntx) * BY - 1, pz,
                             &xfull[b]);
                ++Q;
            };
            auto chunk = [&](int t, int z) {
                const int b = static_cast<int>(j % VR);
                if (j >= VR) mbar_wait(&vempty[b], static_cast<uint32_t>((j / VR - 1) & 1));
                mbar_expect_tx(&vfull[b], static_cast<uint32_t>(CB));
                bulk_g2s(vr + b * CB, g.chunks + (static_cast<int64_t>(t) * g.nzl + g.zbeg + z) * g.chunk_bytes,
                         static_cast<uint32_t>(CB), &vfull[b]);
                ++j;
            };
            for (int si = 0; si < nsegs_b; ++si) {
                int t, za, steps;
                segment(si, t, za, steps);
                if (steps <= 0) break;
                plane(t, za - 1);
                plane(t, za);
                for (int i = 0; i < steps; ++i) {
                    plane(t, za + i + 1);
                    chunk(t, za + i);
                }
            }
        }
        // no griddepcontrol.launch_dependents here: the producer finishes long
        // before the compute warps, and an early trigger let the next kernel's
        // blocks in early (C3 Reordered: +0.55 ms per iteration on B200); the
        // dependents launch when the blocks exit
        return;
    }

    // ---- compute warps: lane -> (4-point group gx along x, line gy, column pair cl)
    const int lane = tid & 31, warp = tid >> 5;
    const int cl = lane % SH::LPR, gl = lane / SH::LPR;
    int gx, gy;
    if constexpr (SH::LPR == 8) {   // 4 groups per warp, one line
        gx = (warp & 1) * 4 + gl;
        gy = warp >> 1;
    } else if constexpr (SH::LPR == 2) {   // m = 4: 16 groups per warp, four lines
        // a quarter warp = 4 groups at the same x on four consecutive lines:
        // line width 35 = 3 (mod 4) puts their 32-byte points on distinct banks
        gx = (warp & 1) * 4 + (gl >> 2);
        gy = (warp >> 1) * 4 + (gl & 3);
    } else {                        // 8 groups per warp, two lines
        // an LDS.128 is served 8 lanes (128 B) at a time: the two groups of a
        // quarter warp take the same x on two lines (odd line width 35 ->
        // opposite bank halves), conflict-free
        gx = (warp & 1) * 4 + (gl >> 1);
        gy = (warp >> 1) * 2 + (gl & 1);
    }
    const int lx0 = gx * 4, cp = cl * 2, r0 = gy * STENCIL_BX + (lx0 ^ stencil_swz(BY, gy));
    // one expansion per (dot, column); (one per row of the lane's 4 as well
    // -- independent chains -- was measured slower: 226 registers, 1 block/SM)
    constexpr int ND = StencilEpiDots<EPI>::value;
    constexpr int NEX = EPI ? ND * 2 : 1;
    double ex[NEX][KEXP];
#pragma unroll
    for (int q = 0; q < NEX; ++q)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) ex[q][i] = 0.0;
    const int col0 = h * MC + cp;   // this lane's first column
    int64_t Q = 0, j = 0;
    for (int si = 0; si < nsegs_b; ++si) {
        int t, za, steps;
        segment(si, t, za, steps);
        if (steps <= 0) break;
        const int xg0 = (t % g.ntx) * STENCIL_BX + lx0, yg = (t / g.ntx) * BY + gy;
        const bool yok = yg < g.ny;
        for (int i = 0; i < steps; ++i, ++j) {
            if (g.mode != 2) {
                for (int64_t q = (i == 0 ? Q : Q + i + 2); q <= Q + i + 2; ++q)
                    mbar_wait(&xfull[q % XR], static_cast<uint32_t>((q / XR) & 1));
                mbar_wait(&vfull[j % VR], static_cast<uint32_t>((j / VR) & 1));
            }
            const double* P0 = xr + ((Q + i) % XR) * SH::PSTRIDE;
            const double* P1 = xr + ((Q + i + 1) % XR) * SH::PSTRIDE;
            const double* P2 = xr + ((Q + i + 2) % XR) * SH::PSTRIDE;
            // epilogue operand (y, aux): issued before the arithmetic so its
            // latency hides behind it
            double2 axs[4];
            if constexpr (EPI == 1) {
                const int64_t rowz = (static_cast<int64_t>(g.zbeg + za + i) * g.ny + yg) * g.nx;
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    axs[r] = (yok && xg0 + r < g.nx)
                                 ? __ldg(reinterpret_cast<const double2*>(epi.aux + (rowz + xg0 + r) * MT + col0))
                                 : make_double2(0.0, 0.0);
            }
            const unsigned char* ch = vr + (j % VR) * CB;
            const double* V = reinterpret_cast<const double*>(ch);
            const uint4 m4 = *reinterpret_cast<const uint4*>(ch + ST * SH::RT * 8 + r0 * 4);
            const uint32_t mk[4] = {m4.x, m4.y, m4.z, m4.w};
            double acc[4][2];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r][0] = acc[r][1] = 0.0;
            if (g.mode == 1) {
            } else if (!((m4.x | m4.y | m4.z | m4.w) & 0x80000000u) || g.mode == 2)
                stencil_rows<MC, ST, BY, false>(acc, P0, P1, P2, V, mk, gy, lx0, cp, r0);
            else
                stencil_rows<MC, ST, BY, true>(acc, P0, P1, P2, V, mk, gy, lx0, cp, r0);
            __syncwarp();
            if (lane == 0 && g.mode != 2) {   // this warp is done with plane Q+i (as z-1) and chunk j
                mbar_arrive(&xempty[(Q + i) % XR]);
                mbar_arrive(&vempty[j % VR]);
            }
            if (yok) {
                const int64_t rowz = (static_cast<int64_t>(g.zbeg + za + i) * g.ny + yg) * g.nx;
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (xg0 + r < g.nx) {
                        const int64_t e = (rowz + xg0 + r) * MT + col0;
                        *reinterpret_cast<double2*>(y + e) = make_double2(acc[r][0], acc[r][1]);
                        if constexpr (EPI != 0) {
                            double2 xs = make_double2(0.0, 0.0);
                            if constexpr (EPI == 1)
                                xs = axs[r];
                            else if constexpr (EPI == 2 || EPI == 4)
                                xs = *reinterpret_cast<const double2*>(P1 + ((gy + 1) * SH::LW + lx0 + r + 1) * MC + cp);
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                const double yv = acc[r][c], xv = c ? xs.y : xs.x;
                                int64_t* s0p = epi.slot[0] + static_cast<int64_t>(col0 + c) * NSLOT;
                                // expansion index: dot * 2 + column
                                if constexpr (EPI == 1 || EPI == 2 || EPI == 4)
                                    grow(ex[c], __dmul_rn(yv, xv), s0p);
                                if constexpr (EPI == 3) grow(ex[c], __dmul_rn(yv, yv), s0p);
                                if constexpr (EPI == 2 || EPI == 4)
                                    grow(ex[2 + c], __dmul_rn(yv, yv),
                                         epi.slot[1] + static_cast<int64_t>(col0 + c) * NSLOT);
                                if constexpr (EPI == 2)
                                    grow(ex[4 + c], __dmul_rn(xv, xv),
                                         epi.slot[2] + static_cast<int64_t>(col0 + c) * NSLOT);
                            }
                        }
                    }
            }
        }
        if (lane == 0 && g.mode != 2) {   // the segment's last two planes
            mbar_arrive(&xempty[(Q + steps) % XR]);
            mbar_arrive(&xempty[(Q + steps + 1) % XR]);
        }
        Q += steps + 2;
    }
    if constexpr (EPI != 0) {
        // every load was consumed: the x ring is free scratch for the combine
        // (compute warps only: named barrier 1 over SH::THREADS threads)
        struct SyncCompute {
            __device__ void operator()() const {
                asm volatile("bar.sync 1, %0;" ::"n"(SH::THREADS) : "memory");
            }
        };
        SyncCompute{}();   // every compute warp is done reading the rings
        block_combine<ND * 2>(ex, SH::LPR,
                              [&](int q, int k) {
                                  return epi.slot[q / 2] + static_cast<int64_t>(h * MC + k * 2 + q % 2) * NSLOT;
                              },
                              xr, SyncCompute{}, SH::THREADS);
    }
}

// ---- 27-point z-marching SpMM (m = 16 per block) ---------------------------
//
// The 27-point kernel above keeps three x planes resident per output plane and
// re-reads every x line from shared memory for each of the three row planes it
// feeds; with the per-row value broadcasts the shared-memory pipe, not HBM, set
// its time (C3: 0.69 ms against 0.52 ms of compulsory bytes).  Here each x
// plane p is read from shared memory ONCE and feeds all three row planes it
// touches: row plane p-1 (its slots 18-26, dz = +1: the row is then complete
// and stored), row plane p (slots 9-17) and row plane p+1 (slots 0-8, a fresh
// accumulator).  A row therefore still adds its 27 slots in ascending order
// (dz, dy, dx) -- the CSR order -- bit for bit.  A lane owns 2 consecutive
// points x 4 columns (registers: 3 row planes x 2 points x 4 columns of
// accumulators); a quarter warp is two point pairs of one line, whose x loads
// fall on complementary bank quads (even groups load column pair 2q first,
// odd groups 2q+1 first) and whose value loads are two 16-byte broadcasts:
// every shared-memory wavefront is fully used.  Per x plane the producer warp
// issues one TMA tensor box (the plane) and three bulk copies (part 0 of row
// plane p+1 with its masks, part 1 of p, part 2 of p-1) into XR / VR rings.
template <int MC>
struct Z27Shape {
    static constexpr int LPG = MC / 4;                      // lanes per point pair (4 columns each)
    static constexpr int THREADS = 16 * 4 * LPG;            // 16 point pairs x 4 lines
    static constexpr int NCW = THREADS / 32;
    static constexpr int LW = 34;
    static constexpr int RT = STENCIL_BX * 4;
    static constexpr int PLANE = LW * 6 * MC;               // doubles per x-plane box
    static constexpr int PSTRIDE = (PLANE + 15) / 16 * 16;
    static constexpr int CB = 27 * RT * 8 + RT * 4;         // one chunk (= one value-ring slot)
};

// VS > 0 (the fused-input variant): the SpMM input is xin = (0 + 1*z) + na*v
// with na a per-column coefficient (Reordered: th = z - alpha s, Alg. 6 line 6
// in the same expression and rounding as the separate update pass).  The x
// ring then holds z boxes, converted in place to xin boxes once their v box
// (a VS-deep staging ring) has landed, before the step reads them.
template <int MC, int XR, int VR, int VS = 0>
__host__ __device__ constexpr int z27_smem() {
    return STENCIL_HEAD + (XR + VS) * Z27Shape<MC>::PSTRIDE * 8 + VR * Z27Shape<MC>::CB;
}

// converter warps of the fused-input variant (they form xin one plane ahead of
// the compute warps, so the conversion never stalls them)
constexpr int Z27_CONV = 64;

// EPI = 1: delta = (y, aux) of the finished rows accumulated exactly in the
// epilogue (the Reordered delta = (v, r0), SpmmEpi kind 1), one expansion per
// (lane, column), combined per block at the end.
template <int MT, int MC, int XR, int VR, int VS = 0, int EPI = 0>
__global__ void __launch_bounds__(Z27Shape<MC>::THREADS + (VS > 0 ? Z27_CONV : 0) + 32, XR == 2 ? 2 : 1)
    stencil27z_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
                      StencilGeom g, double* __restrict__ y, const int* __restrict__ ctl,
                      const __grid_constant__ CUtensorMap vmap, const double* __restrict__ na, SpmmEpi epi) {
    static_assert(EPI == 0 || (EPI == 1 && VS == 0), "z-marching epilogue: kind 1 on the plain input only");
    using SH = Z27Shape<MC>;
    constexpr int CS = MT / MC, RT = SH::RT, CB = SH::CB;
    constexpr int P0B = 9 * RT * 8 + RT * 4;   // part 0 + masks
    constexpr int PB = 9 * RT * 8;             // part 1 / part 2
    static_assert(MC == 16, "z-marching lane map is written for 16 columns per block");
    static_assert(CB % 16 == 0 && (SH::PSTRIDE * 8) % 128 == 0 && P0B % 16 == 0, "ring slot alignment");
    pdl_wait();
    if (ctl && ctl[0]) return;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* xfull = reinterpret_cast<uint64_t*>(smem);
    uint64_t* xempty = xfull + XR;
    uint64_t* vfull = xempty + XR;
    uint64_t* vempty = vfull + VR;
    uint64_t* sempty = vempty + VR;   // v staging ring (VS > 0)
    uint64_t* ready = sempty + VS;    // xin box formed (VS > 0)
    double* xr = reinterpret_cast<double*>(smem + STENCIL_HEAD);
    double* vs = xr + XR * SH::PSTRIDE;
    unsigned char* vr = smem + STENCIL_HEAD + (XR + VS) * SH::PSTRIDE * 8;
    static_assert(3 * XR + 2 * VR + VS <= STENCIL_HEAD / 8, "barrier header");
    constexpr int NCONV = VS > 0 ? Z27_CONV : 0;
    constexpr int PROD = SH::THREADS + NCONV;   // first thread of the producer warp

    const int h = blockIdx.x % CS;
    const int rb = blockIdx.x / CS;
    const int ntiles = static_cast<int>(g.steps / g.nz);
    const int nsegs_b = g.kt > 0 ? g.kt : 1;
    auto segment = [&](int si, int& t, int& za, int& steps) {
        if (g.kt > 0) {
            t = rb + si * g.nranges;
            za = 0;
            steps = t < ntiles ? g.nz : 0;
        } else {
            const int nseg = (g.nz + g.zseg - 1) / g.zseg;
            t = rb / nseg;
            const int sg = rb % nseg;
            za = sg * g.zseg;
            steps = t < ntiles ? min(g.nz, za + g.zseg) - za : 0;
        }
    };
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < XR; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&xempty[b], SH::NCW);
        }
        for (int b = 0; b < VR; ++b) {
            mbar_init(&vfull[b], 1);
            mbar_init(&vempty[b], SH::NCW);
        }
        for (int b = 0; b < VS; ++b) mbar_init(&sempty[b], NCONV);
        for (int b = 0; b < (VS > 0 ? XR : 0); ++b) mbar_init(&ready[b], NCONV);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if constexpr (VS > 0) {
        if (tid >= SH::THREADS && tid < PROD) {   // ---- converter warps: xin = (0 + 1*z) + na*v, in place
            const int ct = tid - SH::THREADS;
            // the thread's column pair is fixed (NCONV pairs per sweep, MC columns)
            const double2 nc = make_double2(na[h * MC + (2 * ct) % MC], na[h * MC + (2 * ct) % MC + 1]);
            int64_t q = 0;
            for (int si = 0; si < nsegs_b; ++si) {
                int t, za, steps;
                segment(si, t, za, steps);
                if (steps <= 0) break;
                for (int i = 0; i < steps + 2; ++i, ++q) {
                    mbar_wait(&xfull[q % XR], static_cast<uint32_t>((q / XR) & 1));
                    double2* zb = reinterpret_cast<double2*>(xr + (q % XR) * SH::PSTRIDE);
                    const double2* vb = reinterpret_cast<const double2*>(vs + (q % VS) * SH::PSTRIDE);
#pragma unroll 4
                    for (int e = ct; e < SH::PLANE / 2; e += NCONV) {
                        const double2 zz = zb[e], vv = vb[e];
                        zb[e] = make_double2(__dadd_rn(__dadd_rn(0.0, __dmul_rn(1.0, zz.x)), __dmul_rn(nc.x, vv.x)),
                                             __dadd_rn(__dadd_rn(0.0, __dmul_rn(1.0, zz.y)), __dmul_rn(nc.y, vv.y)));
                    }
                    mbar_arrive(&sempty[q % VS]);   // v box consumed
                    mbar_arrive(&ready[q % XR]);    // (release: this thread's xin stores)
                }
            }
            return;
        }
    }
    if (tid >= PROD) {   // ---- producer warp: one slot of each ring per x plane
        if (tid == PROD) {
            int64_t q = 0;   // x planes (= steps) issued so far
            for (int si = 0; si < nsegs_b; ++si) {
                int t, za, steps;
                segment(si, t, za, steps);
                if (steps <= 0) break;
                const unsigned char* cbase = g.chunks + static_cast<int64_t>(t) * g.nzl * g.chunk_bytes;
                for (int i = 0; i < steps + 2; ++i, ++q) {
                    const int p = za - 1 + i;   // x plane within the range
                    const int bx = static_cast<int>(q % XR), bv = static_cast<int>(q % VR);
                    if (q >= XR) mbar_wait(&xempty[bx], static_cast<uint32_t>((q / XR - 1) & 1));
                    if (q >= VR) mbar_wait(&vempty[bv], static_cast<uint32_t>((q / VR - 1) & 1));
                    if constexpr (VS > 0) {
                        const int bs = static_cast<int>(q % VS);
                        if (q >= VS) mbar_wait(&sempty[bs], static_cast<uint32_t>((q / VS - 1) & 1));
                        // z box into the x ring, v box into the staging ring, one barrier
                        mbar_expect_tx(&xfull[bx], static_cast<uint32_t>(2 * SH::PLANE * 8));
                        tensor4d_g2s(vs + bs * SH::PSTRIDE, &vmap, h * MC, (t % g.ntx) * STENCIL_BX - 1,
                                     (t / g.ntx) * 4 - 1, g.zbeg + p, &xfull[bx]);
                    } else {
                        mbar_expect_tx(&xfull[bx], static_cast<uint32_t>(SH::PLANE * 8));
                    }
                    const int pl = g.zbeg + p;
                    const void* map = &xmap;
                    int pz = pl;
                    if (pl < 0 && g.lower) {
                        map = &hmap;
                        pz = 0;
                    } else if (pl >= g.nzl && g.upper) {
                        map = &hmap;
                        pz = g.lower;
                    }
                    tensor4d_g2s(xr + bx * SH::PSTRIDE, map, h * MC, (t % g.ntx) * STENCIL_BX - 1,
                                 (t / g.ntx) * 4 - 1, pz, &xfull[bx]);
                    const bool n0 = i < steps;                             // row plane p+1 in [za, zb)
                    const bool n1 = i >= 1 && i <= steps;                  // row plane p
                    const bool n2 = i >= 2;                                // row plane p-1
                    const uint32_t bytes = (n0 ? P0B : 0) + (n1 ? PB : 0) + (n2 ? PB : 0);
                    mbar_expect_tx(&vfull[bv], bytes);
                    unsigned char* dst = vr + bv * CB;
                    const int64_t zl = g.zbeg + p;   // local plane of the x plane
                    if (n0) bulk_g2s(dst, cbase + (zl + 1) * g.chunk_bytes, P0B, &vfull[bv]);
                    if (n1) bulk_g2s(dst + P0B, cbase + zl * g.chunk_bytes + P0B, PB, &vfull[bv]);
                    if (n2) bulk_g2s(dst + P0B + PB, cbase + (zl - 1) * g.chunk_bytes + P0B + PB, PB, &vfull[bv]);
                }
            }
        }
        return;
    }

    // ---- compute warps: lane -> (point pair px, line gy, column quad cq)
    const int lane = tid & 31, warp = tid >> 5;
    const int cq = lane % SH::LPG, gl = lane / SH::LPG;
    const int gy = warp >> 1, px = (warp & 1) * 8 + gl;
    const int lx0 = px * 2, r0 = gy * STENCIL_BX + lx0;
    const int odd = gl & 1;
    const int cpa = (2 * cq + odd) * 2, cpb = (2 * cq + 1 - odd) * 2;   // column pairs in load order
    // three accumulator sets (and row masks) whose roles rotate every x plane:
    // old = row plane p-1, mid = p, new = p+1 (the step body is instantiated
    // for the three rotations, so no register moves)
    double A0[2][4], A1[2][4], A2[2][4];
    uint32_t M0[2] = {0, 0}, M1[2] = {0, 0}, M2[2] = {0, 0};
    // EPI: one expansion per accumulator column (cpa, cpa + 1, cpb, cpb + 1)
    constexpr int NEX = EPI ? 4 : 1;
    double ex[NEX][KEXP];
#pragma unroll
    for (int c = 0; c < NEX; ++c)
#pragma unroll
        for (int k = 0; k < KEXP; ++k) ex[c][k] = 0.0;
    int64_t q = 0;
    for (int si = 0; si < nsegs_b; ++si) {
        int t, za, steps;
        segment(si, t, za, steps);
        if (steps <= 0) break;
        const int xg0 = (t % g.ntx) * STENCIL_BX + lx0, yg = (t / g.ntx) * 4 + gy;
        const bool yok = yg < g.ny;
        // one x plane: all three targets computed unconditionally (a target
        // outside [za, zb) accumulates stale ring data and is never stored),
        // so the chains of the three row planes interleave without branches
        auto body = [&](int i, double (&ao)[2][4], double (&am)[2][4], double (&an)[2][4], uint32_t (&mo)[2],
                        uint32_t (&mm)[2], uint32_t (&mn)[2]) {
            if constexpr (VS > 0) mbar_wait(&ready[q % XR], static_cast<uint32_t>((q / XR) & 1));
            else mbar_wait(&xfull[q % XR], static_cast<uint32_t>((q / XR) & 1));
            mbar_wait(&vfull[q % VR], static_cast<uint32_t>((q / VR) & 1));
            const double* P = xr + (q % XR) * SH::PSTRIDE;
            const unsigned char* ch = vr + (q % VR) * CB;
            const double* V0 = reinterpret_cast<const double*>(ch);
            const double* V1 = reinterpret_cast<const double*>(ch + P0B);
            const double* V2 = reinterpret_cast<const double*>(ch + P0B + PB);
            if (i < steps) {
                const uint2 mk = *reinterpret_cast<const uint2*>(ch + 9 * RT * 8 + r0 * 4);
                mn[0] = mk.x;
                mn[1] = mk.y;
            } else {
                mn[0] = mn[1] = 0;
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) an[r][c] = 0.0;
            const bool ck = ((mn[0] | mn[1] | mm[0] | mm[1] | mo[0] | mo[1]) & 0x80000000u) != 0;
            // epilogue operand of the rows finished this step, issued before the
            // arithmetic so its latency hides behind it
            double2 axa[2], axb[2];
            if constexpr (EPI == 1) {
                const int64_t rowz = (static_cast<int64_t>(g.zbeg + za + i - 2) * g.ny + yg) * g.nx;
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const bool ok = i >= 2 && yok && xg0 + r < g.nx;
                    const double* src = epi.aux + (rowz + xg0 + r) * MT + h * MC;
                    axa[r] = ok ? __ldg(reinterpret_cast<const double2*>(src + cpa)) : make_double2(0.0, 0.0);
                    axb[r] = ok ? __ldg(reinterpret_cast<const double2*>(src + cpb)) : make_double2(0.0, 0.0);
                }
            }
            auto lines = [&](auto check) {
                constexpr bool CK = decltype(check)::value;
#pragma unroll
                for (int dy = 0; dy < 3; ++dy) {
                    double2 xa[4], xb[4];
                    const double* L = P + ((gy + dy) * SH::LW + lx0) * MC;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        xa[j] = *reinterpret_cast<const double2*>(L + j * MC + cpa);
                        xb[j] = *reinterpret_cast<const double2*>(L + j * MC + cpb);
                    }
                    // accumulator columns 0,1 <-> pair cpa, 2,3 <-> pair cpb (odd lanes
                    // hold their pairs swapped; the store puts them back)
                    auto term = [&](double (&acc)[2][4], const double* V, const uint32_t (&mk)[2], int shift) {
#pragma unroll
                        for (int dx = 0; dx < 3; ++dx) {
                            const double2 v = *reinterpret_cast<const double2*>(V + (dy * 3 + dx) * RT + r0);
#pragma unroll
                            for (int r = 0; r < 2; ++r) {
                                if (CK && !((mk[r] >> (shift + dy * 3 + dx)) & 1u)) continue;
                                const double vv = r ? v.y : v.x;
                                acc[r][0] = __dadd_rn(acc[r][0], __dmul_rn(vv, xa[r + dx].x));
                                acc[r][1] = __dadd_rn(acc[r][1], __dmul_rn(vv, xa[r + dx].y));
                                acc[r][2] = __dadd_rn(acc[r][2], __dmul_rn(vv, xb[r + dx].x));
                                acc[r][3] = __dadd_rn(acc[r][3], __dmul_rn(vv, xb[r + dx].y));
                            }
                        }
                    };
                    term(ao, V2, mo, 18);
                    term(am, V1, mm, 9);
                    term(an, V0, mn, 0);
                }
            };
            if (__any_sync(0xffffffffu, ck)) lines(std::true_type{});
            else lines(std::false_type{});
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&xempty[q % XR]);
                mbar_arrive(&vempty[q % VR]);
            }
            if (i >= 2 && yok) {   // row plane p-1 = za + i - 2 is complete
                const int64_t rowz = (static_cast<int64_t>(g.zbeg + za + i - 2) * g.ny + yg) * g.nx;
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (xg0 + r < g.nx) {
                        double* dst = y + (rowz + xg0 + r) * MT + h * MC;
                        *reinterpret_cast<double2*>(dst + cpa) = make_double2(ao[r][0], ao[r][1]);
                        *reinterpret_cast<double2*>(dst + cpb) = make_double2(ao[r][2], ao[r][3]);
                        if constexpr (EPI == 1) {   // PDot2 order: v * r0
                            int64_t* s0 = epi.slot[0] + static_cast<int64_t>(h * MC) * NSLOT;
                            int64_t* const sl[4] = {s0 + static_cast<int64_t>(cpa) * NSLOT,
                                                    s0 + static_cast<int64_t>(cpa + 1) * NSLOT,
                                                    s0 + static_cast<int64_t>(cpb) * NSLOT,
                                                    s0 + static_cast<int64_t>(cpb + 1) * NSLOT};
                            const double pr[4] = {__dmul_rn(ao[r][0], axa[r].x), __dmul_rn(ao[r][1], axa[r].y),
                                                  __dmul_rn(ao[r][2], axb[r].x), __dmul_rn(ao[r][3], axb[r].y)};
                            grow_batch<4>(ex, pr, sl);
                        }
                    }
            }
            ++q;
        };
        const int n = steps + 2;
        for (int i = 0; i < n;) {
            body(i, A0, A1, A2, M0, M1, M2);
            if (++i == n) break;
            body(i, A1, A2, A0, M1, M2, M0);
            if (++i == n) break;
            body(i, A2, A0, A1, M2, M0, M1);
            ++i;
        }
    }
    if constexpr (EPI == 1) {
        // every load was consumed: the x ring is scratch for the block combine
        // (compute warps only: named barrier 1); class = lane % 8 fixes (cq, odd)
        struct SyncCompute {
            __device__ void operator()() const { asm volatile("bar.sync 1, %0;" ::"n"(SH::THREADS) : "memory"); }
        };
        SyncCompute{}();
        block_combine<4>(ex, 8,
                         [&](int xi, int k) {
                             const int kq = k % 4, ko = (k / 4) & 1;
                             const int ca = (2 * kq + ko) * 2, cb = (2 * kq + 1 - ko) * 2;
                             const int col = xi < 2 ? ca + xi : cb + xi - 2;
                             return epi.slot[0] + static_cast<int64_t>(h * MC + col) * NSLOT;
                         },
                         xr, SyncCompute{}, SH::THREADS);
    }
}

#undef MBG_ACC

// ---- host side ----------------------------------------------------------------

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        MBG_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool stencil_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MBG_STENCIL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

StencilLayout& layout_for(mbg_ctx* ctx, const mbg_csr* a, int by, int zpart = 0) {
    StencilOp& op = *a->stencil;
    for (auto& l : op.layouts)
        if (l->by == by && l->zpart == zpart) return *l;
    auto l = std::make_unique<StencilLayout>();
    l->by = by;
    l->zpart = zpart;
    const int S = op.kind;
    const int RT = STENCIL_BX * by;
    l->chunk_bytes = static_cast<int64_t>(S) * RT * 8 + RT * 4;
    const int64_t ntx = (op.nx + STENCIL_BX - 1) / STENCIL_BX, nty = (op.ny + by - 1) / by;
    const size_t bytes = static_cast<size_t>(ntx * nty * op.nz * l->chunk_bytes);
    l->chunks.alloc(bytes);
    const int grid = ctx->num_sms * 8;
    if (zpart) {
        // tile rows outside the grid stay zero (never stored)
        MBG_CUDA(cudaMemsetAsync(l->chunks.p, 0, bytes, ctx->stream));
        stencil_fill_zpart_kernel<<<grid, 256, 0, ctx->stream>>>(op.map, op.nzg, by, static_cast<int>(ntx),
                                                                 l->chunk_bytes, a->off.p, a->col.p, a->val.p,
                                                                 l->chunks.p);
    } else {
        stencil_clear_kernel<<<grid, 256, 0, ctx->stream>>>(ntx * nty * op.nz, S, RT, l->chunk_bytes, l->chunks.p);
        stencil_fill_kernel<<<grid, 256, 0, ctx->stream>>>(op.map, op.nzg, by, S, static_cast<int>(ntx),
                                                           l->chunk_bytes, a->off.p, a->col.p, a->val.p, l->chunks.p);
    }
    MBG_CUDA(cudaGetLastError());
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    op.layouts.push_back(std::move(l));
    return *op.layouts.back();
}

struct ZRange {
    int zbeg, zend;   // local planes [zbeg, zend)
};

template <int MT, int MC, int ST, int BY, int EPI>
void launch_one(mbg_ctx* ctx, const mbg_csr* a, const StencilLayout& L, const double* x, double* y,
                const int* ctl, const SpmmEpi& epi, ZRange zr) {
    const StencilOp& op = *a->stencil;
    if (zr.zend <= zr.zbeg) return;
    constexpr int smem = stencil_smem<MC, ST, BY>();
    constexpr int threads = StencilShape<MC, BY>::THREADS + 32;   // + producer warp
    constexpr int CS = MT / MC;
    const int occ =
        kernel_occupancy(reinterpret_cast<const void*>(&stencil_spmm_kernel<MT, MC, ST, BY, EPI>), threads, smem);
    // x viewed as a (planes, ny, nx, MT) fp64 tensor; box (MC, LW, BY + 2, 1):
    // the owned planes, and the halo planes appended after them (z-slabs)
    auto encode = [&](CUtensorMap& tm, const double* base, int planes) {
        const cuuint64_t dims[4] = {static_cast<cuuint64_t>(MT), static_cast<cuuint64_t>(op.nx),
                                    static_cast<cuuint64_t>(op.ny), static_cast<cuuint64_t>(planes)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(MT) * 8, static_cast<cuuint64_t>(op.nx) * MT * 8,
                                       static_cast<cuuint64_t>(op.nx) * op.ny * MT * 8};
        const cuuint32_t box[4] = {static_cast<cuuint32_t>(MC), static_cast<cuuint32_t>(StencilShape<MC, BY>::LW),
                                   static_cast<cuuint32_t>(BY + 2), 1u};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            throw std::runtime_error("stencil SpMM: cuTensorMapEncodeTiled failed (" +
                                     std::to_string(static_cast<int>(r)) + ")");
    };
    CUtensorMap tm, hm;
    encode(tm, x, op.nz);
    const int nhp = op.map.lower + op.upper;
    if (nhp) encode(hm, x + a->n * MT, nhp);
    else hm = tm;
    StencilGeom gm{};
    gm.nx = op.nx;
    gm.ny = op.ny;
    gm.nz = zr.zend - zr.zbeg;
    gm.zbeg = zr.zbeg;
    gm.nzl = op.nz;
    gm.lower = op.map.lower;
    gm.upper = op.upper;
    gm.ntx = (op.nx + STENCIL_BX - 1) / STENCIL_BX;
    gm.steps = static_cast<int64_t>(gm.ntx) * ((op.ny + BY - 1) / BY) * gm.nz;
    gm.chunks = L.chunks.p;
    gm.chunk_bytes = L.chunk_bytes;
    static const int mode = env_int("MBG_STENCIL_MODE", 0);
    gm.mode = mode;
    // persistent grid: every resident slot gets an equal share of the steps
    const int64_t slots = static_cast<int64_t>(occ) * ctx->num_sms / CS;
    // work split: whole tiles per block when there are at least as many tiles
    // as block slots, else every tile cut into equal z-segments
    const int64_t ntiles = gm.steps / gm.nz;
    if (ntiles >= slots) {
        gm.kt = static_cast<int>((ntiles + slots - 1) / slots);
        gm.zseg = gm.nz;
        gm.nranges = static_cast<int>((ntiles + gm.kt - 1) / gm.kt);
    } else {
        const int k = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(slots / ntiles, gm.nz)));
        gm.kt = 0;
        gm.zseg = (gm.nz + k - 1) / k;
        gm.nranges = static_cast<int>(ntiles * ((gm.nz + gm.zseg - 1) / gm.zseg));
    }
    const int grid = gm.nranges * CS;
    launch_pdl(stencil_spmm_kernel<MT, MC, ST, BY, EPI>, dim3(grid), dim3(threads), static_cast<size_t>(smem),
               ctx->stream, tm, hm, gm, y, ctl, epi);
}

// work split of a persistent stencil grid (shared by both kernels)
void split_work(StencilGeom& gm, int64_t slots) {
    const int64_t ntiles = gm.steps / gm.nz;
    if (ntiles >= slots) {
        gm.kt = static_cast<int>((ntiles + slots - 1) / slots);
        gm.zseg = gm.nz;
        gm.nranges = static_cast<int>((ntiles + gm.kt - 1) / gm.kt);
    } else {
        const int k = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(slots / ntiles, gm.nz)));
        gm.kt = 0;
        gm.zseg = (gm.nz + k - 1) / k;
        gm.nranges = static_cast<int>(ntiles * ((gm.nz + gm.zseg - 1) / gm.zseg));
    }
}

// VS > 0: the fused-input variant, x = z, v / na as stencil27z_kernel describes;
// EPI = 1: the delta epilogue (epi kind 1)
template <int MT, int MC, int XR, int VR, int VS = 0, int EPI = 0>
void launch_z27(mbg_ctx* ctx, const mbg_csr* a, const StencilLayout& L, const double* x, double* y, const int* ctl,
                ZRange zr, const double* v = nullptr, const double* na = nullptr, const SpmmEpi& epi = SpmmEpi{}) {
    using SH = Z27Shape<MC>;
    const StencilOp& op = *a->stencil;
    if (zr.zend <= zr.zbeg) return;
    constexpr int smem = z27_smem<MC, XR, VR, VS>();
    constexpr int threads = SH::THREADS + (VS > 0 ? Z27_CONV : 0) + 32;
    constexpr int CS = MT / MC;
    const int occ =
        kernel_occupancy(reinterpret_cast<const void*>(&stencil27z_kernel<MT, MC, XR, VR, VS, EPI>), threads, smem);
    auto encode = [&](CUtensorMap& tm, const double* base, int planes) {
        const cuuint64_t dims[4] = {static_cast<cuuint64_t>(MT), static_cast<cuuint64_t>(op.nx),
                                    static_cast<cuuint64_t>(op.ny), static_cast<cuuint64_t>(planes)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(MT) * 8, static_cast<cuuint64_t>(op.nx) * MT * 8,
                                       static_cast<cuuint64_t>(op.nx) * op.ny * MT * 8};
        const cuuint32_t box[4] = {static_cast<cuuint32_t>(MC), static_cast<cuuint32_t>(SH::LW), 6u, 1u};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            throw std::runtime_error("stencil SpMM: cuTensorMapEncodeTiled failed (" +
                                     std::to_string(static_cast<int>(r)) + ")");
    };
    CUtensorMap tm, hm;
    encode(tm, x, op.nz);
    const int nhp = op.map.lower + op.upper;
    if (nhp) encode(hm, x + a->n * MT, nhp);
    else hm = tm;
    StencilGeom gm{};
    gm.nx = op.nx;
    gm.ny = op.ny;
    gm.nz = zr.zend - zr.zbeg;
    gm.zbeg = zr.zbeg;
    gm.nzl = op.nz;
    gm.lower = op.map.lower;
    gm.upper = op.upper;
    gm.ntx = (op.nx + STENCIL_BX - 1) / STENCIL_BX;
    gm.steps = static_cast<int64_t>(gm.ntx) * ((op.ny + 3) / 4) * gm.nz;
    gm.chunks = L.chunks.p;
    gm.chunk_bytes = L.chunk_bytes;
    split_work(gm, static_cast<int64_t>(occ) * ctx->num_sms / CS);
    CUtensorMap vm = tm;
    if constexpr (VS > 0) encode(vm, v, op.nz);
    launch_pdl(stencil27z_kernel<MT, MC, XR, VR, VS, EPI>, dim3(gm.nranges * CS), dim3(threads),
               static_cast<size_t>(smem), ctx->stream, tm, hm, gm, y, ctl, vm, na, epi);
}

// MBG_STENCIL_Z: 0 = the three-plane kernel for 27-point m = 16 / 32 too;
// else the z-marching kernel with the ring depths listed at the dispatch
// (default 3: x ring 4, value ring 3; C3 SpMM 676 -> 507 us on B200)
int z27_mode() {
    static const int v = env_int("MBG_STENCIL_Z", 3);
    return v;
}

}  // namespace

std::shared_ptr<StencilOp> build_stencil(mbg_ctx* ctx, const mbg_csr* a, int nx, int ny, int nz) {
    const int64_t nxy = static_cast<int64_t>(nx) * ny;
    if (nx < 1 || ny < 1 || nz < 1 || nxy * nz != a->n_global || a->n == 0) return nullptr;
    // a partition must own whole planes; its halo must be exactly the planes
    // next to the slab (plan.cpp orders them by ascending global id)
    if (a->row_begin % nxy || a->n % nxy) return nullptr;
    GridMap gm{};
    gm.nx = nx;
    gm.ny = ny;
    gm.row_begin = a->row_begin;
    gm.n_own = a->n;
    gm.z0 = static_cast<int>(a->row_begin / nxy);
    gm.nzl = static_cast<int>(a->n / nxy);
    const bool partitioned = !a->peers.empty() || a->n_halo;
    gm.lower = partitioned && gm.z0 > 0;
    const bool upper = partitioned && gm.z0 + gm.nzl < nz;
    if (a->n_halo != nxy * (gm.lower + upper)) return nullptr;
    DevBuf<unsigned> flags(1);
    MBG_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(unsigned), ctx->stream));
    stencil_scan_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(gm, a->off.p, a->col.p, flags.p);
    MBG_CUDA(cudaGetLastError());
    unsigned f = 0;
    MBG_CUDA(cudaMemcpyAsync(&f, flags.p, sizeof f, cudaMemcpyDeviceToHost, ctx->stream));
    MBG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (f & 5u) return nullptr;
    auto op = std::make_shared<StencilOp>();
    op->nx = nx;
    op->ny = ny;
    op->nz = gm.nzl;
    op->nzg = nz;
    op->map = gm;
    op->upper = upper;
    op->kind = (f & 2u) ? 27 : 7;
    op->nnz = a->nnz;
    return op;
}

bool stencil_epilogues() {
    static const bool on = env_int("MBG_STENCIL_EPI", 0) != 0;
    return on;
}

bool stencil_handles(const mbg_csr* a, int m) {
    return a && a->stencil && stencil_enabled() && (m == 4 || m == 8 || m == 16 || m == 32);
}

double stencil_spmm_bytes(int64_t n, int64_t nnz, int m) {
    return 16.0 * static_cast<double>(n) * m + 8.0 * static_cast<double>(nnz) + 4.0 * static_cast<double>(n);
}

template <int MT, int MC, int ST, int BY>
void launch_epi(mbg_ctx* ctx, const mbg_csr* a, const StencilLayout& L, const double* x, double* y, const int* ctl,
                const SpmmEpi* epi, ZRange zr) {
    const SpmmEpi none{};
    switch (epi ? epi->kind : 0) {
        case 0: launch_one<MT, MC, ST, BY, 0>(ctx, a, L, x, y, ctl, none, zr); break;
        case 1: launch_one<MT, MC, ST, BY, 1>(ctx, a, L, x, y, ctl, *epi, zr); break;
        case 2: launch_one<MT, MC, ST, BY, 2>(ctx, a, L, x, y, ctl, *epi, zr); break;
        case 3: launch_one<MT, MC, ST, BY, 3>(ctx, a, L, x, y, ctl, *epi, zr); break;
        case 4: launch_one<MT, MC, ST, BY, 4>(ctx, a, L, x, y, ctl, *epi, zr); break;
        default: throw Invalid("stencil SpMM: unknown epilogue kind");
    }
}

template <int BY>
void launch_by(mbg_ctx* ctx, const mbg_csr* a, int m, const double* x, double* y, const int* ctl,
               const SpmmEpi* epi, ZRange zr) {
    const int kind = a->stencil->kind;
    if constexpr (BY == 4) {
        if (kind == 27 && (m == 16 || m == 32) && epi && epi->kind == 1 && z27_mode() != 0) {
            const StencilLayout& Z = layout_for(ctx, a, 4, 1);
            if (m == 16) launch_z27<16, 16, 4, 3, 0, 1>(ctx, a, Z, x, y, ctl, zr, nullptr, nullptr, *epi);
            else launch_z27<32, 16, 4, 3, 0, 1>(ctx, a, Z, x, y, ctl, zr, nullptr, nullptr, *epi);
            return;
        }
        if (kind == 27 && (m == 16 || m == 32) && (!epi || epi->kind == 0) && z27_mode() != 0) {
            const StencilLayout& Z = layout_for(ctx, a, 4, 1);
            // ring depths (x planes, value slots): 1 (3,2)  2 (2,2; 2 blocks/SM)
            // 3 (4,3, default)  4 (3,3)  5 (4,4)  6 (5,3)  7 (4,2)
            auto go = [&](auto mt) {
                constexpr int MT = decltype(mt)::value;
                switch (z27_mode()) {
                    case 2: launch_z27<MT, 16, 2, 2>(ctx, a, Z, x, y, ctl, zr); break;
                    case 3: launch_z27<MT, 16, 4, 3>(ctx, a, Z, x, y, ctl, zr); break;
                    case 4: launch_z27<MT, 16, 3, 3>(ctx, a, Z, x, y, ctl, zr); break;
                    case 5: launch_z27<MT, 16, 4, 4>(ctx, a, Z, x, y, ctl, zr); break;
                    case 6: launch_z27<MT, 16, 5, 3>(ctx, a, Z, x, y, ctl, zr); break;
                    case 7: launch_z27<MT, 16, 4, 2>(ctx, a, Z, x, y, ctl, zr); break;
                    default: launch_z27<MT, 16, 3, 2>(ctx, a, Z, x, y, ctl, zr); break;
                }
            };
            if (m == 16) go(std::integral_constant<int, 16>{});
            else go(std::integral_constant<int, 32>{});
            return;
        }
    }
    const StencilLayout& L = layout_for(ctx, a, BY);
    switch (m) {
        case 4:
            if constexpr (BY == 8) {
                if (kind == 27) launch_epi<4, 4, 27, BY>(ctx, a, L, x, y, ctl, epi, zr);
                else launch_epi<4, 4, 7, BY>(ctx, a, L, x, y, ctl, epi, zr);
            }
            break;
        case 8:
            if (kind == 27) launch_epi<8, 8, 27, BY>(ctx, a, L, x, y, ctl, epi, zr);
            else launch_epi<8, 8, 7, BY>(ctx, a, L, x, y, ctl, epi, zr);
            break;
        case 16:
            if (kind == 27) launch_epi<16, 16, 27, BY>(ctx, a, L, x, y, ctl, epi, zr);
            else launch_epi<16, 16, 7, BY>(ctx, a, L, x, y, ctl, epi, zr);
            break;
        case 32:
            if (kind == 27) launch_epi<32, 16, 27, BY>(ctx, a, L, x, y, ctl, epi, zr);
            else launch_epi<32, 16, 7, BY>(ctx, a, L, x, y, ctl, epi, zr);
            break;
        default:
            throw Invalid("stencil SpMM: m must be 4, 8, 16 or 32");
    }
}

bool stencil_delta_epilogue(const mbg_csr* a, int m) {
    static const bool on = env_int("MBG_Z27_EPI", 0) != 0;
    return on && stencil_handles(a, m) && a->stencil->kind == 27 && (m == 16 || m == 32) && z27_mode() != 0;
}

bool stencil_axpy_handles(const mbg_csr* a, int m) {
    static const bool on = env_int("MBG_STENCIL_AX", 1) != 0;
    return on && stencil_handles(a, m) && a->stencil->kind == 27 && (m == 16 || m == 32) && z27_mode() != 0 &&
           a->stencil->map.lower == 0 && a->stencil->upper == 0 && a->peers.empty() && a->n_halo == 0;
}

int launch_stencil_spmm_axpy(mbg_ctx* ctx, const mbg_csr* a, int m, const double* z, const double* v,
                             const double* na, double* y, const int* ctl) {
    if (!stencil_axpy_handles(a, m)) throw Invalid("stencil SpMM: fused input needs a 27-point m = 16 / 32 twin");
    const StencilLayout& Z = layout_for(ctx, a, 4, 1);
    const ZRange zr{0, a->stencil->nz};
    // rings: x (z boxes) 3, v staging 2, values 3 (the 227 KB budget; value
    // depth 3 is what matters, tools/spmm_time.py sweep in DESIGN.md)
    // MBG_STENCIL_AXR (lab): ring depths x / values / v staging  1: 3/3/2  2: 4/3/1  3: 4/2/2
    static const int rings = env_int("MBG_STENCIL_AXR", 1);
    auto go = [&](auto mt) {
        constexpr int MT = decltype(mt)::value;
        if (rings == 2) launch_z27<MT, 16, 4, 3, 1>(ctx, a, Z, z, y, ctl, zr, v, na);
        else if (rings == 3) launch_z27<MT, 16, 4, 2, 2>(ctx, a, Z, z, y, ctl, zr, v, na);
        else launch_z27<MT, 16, 3, 3, 2>(ctx, a, Z, z, y, ctl, zr, v, na);
    };
    if (m == 16) go(std::integral_constant<int, 16>{});
    else go(std::integral_constant<int, 32>{});
    return 1;
}

int launch_stencil_spmm(mbg_ctx* ctx, const mbg_csr* a, int m, const double* x, double* y, const int* ctl,
                        const SpmmEpi* epi, int zbeg, int zend) {
    const int nz = a->stencil->nz;
    if (zend < 0) zend = nz;
    zbeg = std::max(0, zbeg);
    zend = std::min(nz, zend);
    if (zend <= zbeg) return 0;
    // m = 4: 32 x 8 tiles (128 compute threads per block, four lines per warp)
    if (m == 4) launch_by<8>(ctx, a, m, x, y, ctl, epi, ZRange{zbeg, zend});
    else launch_by<4>(ctx, a, m, x, y, ctl, epi, ZRange{zbeg, zend});
    return 1;
}

}  // namespace mbg
