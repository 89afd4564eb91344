// small.cu -- the whole classical BiCGStab iteration loop in ONE cooperative
// kernel, for systems too small to fill the GPU (BASELINE config C1: a 32^3
// Poisson matrix, m = 1, 32K rows; latency-bound at ~10 launches/iteration).
//
// Same arithmetic as the multi-kernel path, statement for statement: the
// group programs' run() functions (group.cuh), the CSR row sums of spmv_rows
// (spmv.cpp:40-46), exact dots (grow + block_combine into the long
// accumulators -- order-independent, so the different thread mapping changes
// no bit) and the scalar recurrences of scalar_block() (scalar.cuh), run by
// block 0 between grid-wide barriers.  Results are bitwise those of the
// multi-kernel solver (tests/test_gpu_small.py).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "group.cuh"
#include "kernels.hpp"
#include "scalar.cuh"
#include "small.hpp"

namespace cg = cooperative_groups;

namespace mbg {

namespace {

// y = A x and, for the element just computed, the exact dots of program P on
// (y, w) -- the thread owns its element, so no barrier separates the SpMM from
// the dot pass (PDot2: (y, w); PClassicOmega: (y, w), (y, y), (w, w);
// PClassicPhiPsi: (y, w), (y, y))
template <class P>
__device__ void small_spmm_dots(const SmallArgs& a, const double* __restrict__ x, double* __restrict__ y,
                                const double* __restrict__ w, double* sh) {
    constexpr int ND = P::NDOT;
    const int m = a.m;
    const int c0 = threadIdx.x % m;
    double acc[ND][KEXP];
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
        for (int k = 0; k < KEXP; ++k) acc[d][k] = 0.0;
    const int64_t len = a.n * m;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = e / m;
        double yv = 0.0;
        for (int k = a.off[row]; k < a.off[row + 1]; ++k)
            yv = __dadd_rn(yv, __dmul_rn(a.val[k], x[static_cast<int64_t>(a.col[k]) * m + c0]));
        y[e] = yv;
        const double v[2] = {yv, w[e]};
        double pr[ND];
        P::run(v, nullptr, pr, nullptr);
#pragma unroll
        for (int d = 0; d < ND; ++d) grow(acc[d], pr[d], a.slots + (static_cast<int64_t>(d) * m + c0) * NSLOT);
    }
    block_combine<ND>(acc, m, [&](int q, int k) { return a.slots + (static_cast<int64_t>(q) * m + k) * NSLOT; },
                      sh);
}

// One merged line over all elements (group_kernel's VEC = 1 path with the
// careful grow); the block size and the grid stride are multiples of m, so a
// thread keeps one column.
struct Line {   // operands of one merged line (vector pointers, scalar-bank rows)
    const double* in[5];
    double* out[2];
    int co[3];
};

template <class P>
__device__ void small_group(const SmallArgs& a, const Line& ln, int first_slot, double* sh) {
    constexpr int NCO = P::NCO > 0 ? P::NCO : 1;
    constexpr int ND = P::NDOT > 0 ? P::NDOT : 1;
    constexpr int NO = P::NOUT > 0 ? P::NOUT : 1;
    const int m = a.m;
    const int c0 = threadIdx.x % m;
    double cof[NCO];
#pragma unroll
    for (int q = 0; q < P::NCO; ++q) cof[q] = a.sc[static_cast<int64_t>(ln.co[q]) * m + c0];
    double acc[ND][KEXP];
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
        for (int k = 0; k < KEXP; ++k) acc[d][k] = 0.0;
    const int64_t len = a.n * m;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < len;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v[P::NIN > 0 ? P::NIN : 1], o[NO], pr[ND];
#pragma unroll
        for (int q = 0; q < P::NIN; ++q) v[q] = ln.in[q][e];
        P::run(v, o, pr, cof);
#pragma unroll
        for (int q = 0; q < P::NOUT; ++q) ln.out[q][e] = o[q];
#pragma unroll
        for (int d = 0; d < P::NDOT; ++d)
            grow(acc[d], pr[d], a.slots + (static_cast<int64_t>(first_slot + d) * m + c0) * NSLOT);
    }
    if constexpr (P::NDOT > 0) {
        block_combine<ND>(acc, m,
                          [&](int x, int k) {
                              return a.slots + (static_cast<int64_t>(first_slot + x) * m + k) * NSLOT;
                          },
                          sh);
    }
}

__device__ ScalArgs small_scal(const SmallArgs& a, int point, int nd) {
    ScalArgs s{};
    s.m = a.m;
    s.point = point;
    s.method = MBG_BICGSTAB;
    s.fixed = a.fixed;
    s.maxit = a.maxit;
    s.tol2 = a.tol2;
    s.sc = a.sc;
    s.ctl = a.ctl;
    s.hist = a.hist;
    for (int i = 0; i < nd; ++i) s.D[i] = a.slots + static_cast<int64_t>(i) * a.m * NSLOT;
    s.nd = nd;
    return s;
}

__global__ void __launch_bounds__(256) small_classical_kernel(SmallArgs a) {
    extern __shared__ double sh[];   // max(256 * KEXP, 3 * m) doubles
    cg::grid_group grid = cg::this_grid();
    volatile const int* stop = a.ctl + C_STOP;
    auto scalars = [&](int point, int nd) {
        grid.sync();   // every block's dot deposits are in the long accumulators
        if (blockIdx.x == 0) scalar_block(small_scal(a, point, nd), sh);
        grid.sync();   // the new scalars (and the stop word) are visible to every block
    };
    for (int it = 0; it < a.maxit && !*stop; ++it) {
        small_spmm_dots<PDot2>(a, a.p, a.v, a.r0, sh);                            // v = A p ; delta = (v, r0)
        scalars(P_C_ALPHA, 1);
        if (*stop) break;
        if (a.fused)
            small_group<PUpd2Sq>(a, Line{{a.r, a.v}, {a.s}, {S_ONE, S_NALPHA}}, 2, sh);   // s ; theta -> slot 2
        else
            small_group<PUpd2>(a, Line{{a.r, a.v}, {a.s}, {S_ONE, S_NALPHA}}, 0, sh);     // s = r - alpha v
        grid.sync();
        if (a.fused)
            small_spmm_dots<PClassicPhiPsi>(a, a.s, a.t, a.s, sh);                 // t = A s ; phi psi -> slots 0,1
        else
            small_spmm_dots<PClassicOmega>(a, a.s, a.t, a.s, sh);                  // t = A s ; phi psi theta
        scalars(P_C_OMEGA, 3);
        if (*stop) break;
        small_group<PClassicXR>(a, Line{{a.x, a.p, a.s, a.t, a.r0}, {a.x, a.r}, {S_ALPHA, S_OMEGA, S_NOMEGA}}, 0, sh);
        scalars(P_C_BETA, 1);
        if (*stop) break;
        small_group<PUpd3>(a, Line{{a.r, a.p, a.v}, {a.p}, {S_ONE, S_BETA, S_NBO}}, 0, sh);   // p update
        grid.sync();
    }
}

}  // namespace

bool small_path_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MBG_SMALL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int launch_small_classical(cudaStream_t st, const SmallArgs& a, int num_sms) {
    const size_t smem = static_cast<size_t>(256) * KEXP * sizeof(double);
    const int occ = kernel_occupancy(reinterpret_cast<const void*>(&small_classical_kernel), 256, smem);
    // one element per thread as far as co-residency allows: the phases are
    // latency-bound, so more blocks win (C1: 128 blocks 0.049 ms/it, 32 blocks 0.062)
    const int64_t need = (a.n * a.m + 255) / 256;
    const int grid =
        static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, static_cast<int64_t>(num_sms) * occ)));
    SmallArgs args = a;
    void* params[] = {&args};
    MBG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(small_classical_kernel), dim3(grid), dim3(256),
                                         params, smem, st));
    return 1;
}

}  // namespace mbg
