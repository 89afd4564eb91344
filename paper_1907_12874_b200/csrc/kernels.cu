// kernels.cu -- SpMM, exact-dot fold/round and the generic group interpreter
// for sm_100a.
#include <mutex>
#include <unordered_map>

#include "common.hpp"
#include "kernels.hpp"

namespace mbg {

// ===========================================================================
// SpMM  y = A x  over the row-interleaved n x m block.
//
// Restates spmv_rows (spmv.cpp:27-50): for each (row, column) the products
// val[k]*x(col[k], c) are added to acc = 0.0 sequentially in CSR order, with
// separately rounded multiply and add.  Mapping (m | 32): a warp covers
// 32/m consecutive rows, lane = column, so the x-gather of one nonzero is m*8
// contiguous bytes and the y store of a warp is 256 contiguous bytes.  col/val
// are read with the no-allocate streaming hint (used once) and x through the
// read-only path (reused across neighbouring rows from L1/L2).  Nonzeros are
// processed in batches of 8: all index/value loads, then all gathers, then the
// ordered adds, to keep 16+ loads in flight per thread.
// ===========================================================================
template <int M>
__global__ void __launch_bounds__(256) spmm_kernel(int64_t nrows, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ off,
                                                   const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   const int* __restrict__ ctl) {
    if (ctl && ctl[0]) return;
    constexpr int RPW = 32 / M;
    const int lane = threadIdx.x & 31;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t ri = w * RPW + lane / M;
    const int c = lane % M;
    if (ri >= nrows) return;
    const int64_t row = rows ? rows[ri] : ri;
    const int k0 = __ldg(off + row), k1 = __ldg(off + row + 1);
    double acc = 0.0;
    for (int k = k0; k < k1; k += 8) {
        const int cnt = min(8, k1 - k);
        int j[8];
        double a[8], xv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < cnt) {
                j[i] = __ldcs(col + k + i);
                a[i] = __ldcs(val + k + i);
            }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < cnt) xv[i] = __ldg(x + static_cast<int64_t>(j[i]) * M + c);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < cnt) acc = __dadd_rn(acc, __dmul_rn(a[i], xv[i]));
    }
    y[row * M + c] = acc;
}

// Any m: one thread per (row, column) element.
__global__ void __launch_bounds__(256) spmm_generic_kernel(int64_t nrows, const int32_t* __restrict__ rows,
                                                           const int32_t* __restrict__ off,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ val, int m,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y,
                                                           const int* __restrict__ ctl) {
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

void launch_spmm(cudaStream_t st, int64_t nrows, const int32_t* rows, const int32_t* off,
                 const int32_t* col, const double* val, int m, const double* x, double* y,
                 const int* ctl) {
    if (nrows <= 0) return;
    const int block = 256;
    auto grid_for = [&](int M) {
        const int64_t warps = (nrows + (32 / M) - 1) / (32 / M);
        return static_cast<unsigned>((warps * 32 + block - 1) / block);
    };
    switch (m) {
        case 1: spmm_kernel<1><<<grid_for(1), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        case 2: spmm_kernel<2><<<grid_for(2), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        case 4: spmm_kernel<4><<<grid_for(4), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        case 8: spmm_kernel<8><<<grid_for(8), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        case 16: spmm_kernel<16><<<grid_for(16), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        case 32: spmm_kernel<32><<<grid_for(32), block, 0, st>>>(nrows, rows, off, col, val, x, y, ctl); break;
        default: {
            const int64_t total = nrows * m;
            spmm_generic_kernel<<<static_cast<unsigned>((total + block - 1) / block), block, 0, st>>>(
                nrows, rows, off, col, val, m, x, y, ctl);
        }
    }
    MBG_CUDA(cudaGetLastError());
}

// ===========================================================================
// Fold: block partials + long accumulator -> D, then clear the slot.
// ===========================================================================
__global__ void fold_kernel(FoldArgs f) {
    if (f.ctl && f.ctl[0]) return;
    const int c = blockIdx.x, s = blockIdx.y, lane = threadIdx.x;
    int64_t* slot = f.slot[s] + static_cast<int64_t>(c) * NSLOT;
    int64_t* D = f.D[s] + static_cast<int64_t>(c) * NSLOT;
    const double* part = f.part[s] + static_cast<int64_t>(c) * f.nblocks * KEXP;
    double acc[KEXP] = {0.0, 0.0, 0.0};
    for (int b = lane; b < f.nblocks; b += 32)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) grow(acc, part[b * KEXP + i], slot);
    for (int o = 16; o >= 1; o >>= 1) {
        double t[KEXP];
#pragma unroll
        for (int i = 0; i < KEXP; ++i) t[i] = __shfl_down_sync(0xffffffffu, acc[i], o);
        if (lane < o)
#pragma unroll
            for (int i = 0; i < KEXP; ++i) grow(acc, t[i], slot);
    }
    __shared__ int64_t sd[NSLOT];
    __syncwarp();
    __threadfence_block();
    for (int j = lane; j < NSLOT; j += 32) {
        sd[j] = atomicExch(reinterpret_cast<unsigned long long*>(slot + j), 0ull);
    }
    __syncwarp();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) digits_add(sd, acc[i]);
    __syncwarp();
    // one parallel carry step: words stay below 2^33 in magnitude
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int j = lane + 32 * q;
        if (j < NDIG) {
            const int64_t v = sd[j];
            const int64_t low = (j < NDIG - 1) ? (v & 0xffffffffll) : v;
            const int64_t cin = j > 0 ? (sd[j - 1] >> 32) : 0;
            D[j] = low + cin;
        } else if (j < NSLOT) {
            D[j] = sd[j];
        }
    }
}

void launch_fold(cudaStream_t st, const FoldArgs& f, int nslots) {
    fold_kernel<<<dim3(f.m, nslots), 32, 0, st>>>(f);
    MBG_CUDA(cudaGetLastError());
}

__global__ void round_kernel(const int64_t* D, int nslots, int m, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nslots * m) out[i] = digits_round(D + static_cast<int64_t>(i) * NSLOT);
}

void launch_round(cudaStream_t st, const int64_t* D, int nslots, int m, double* out) {
    const int n = nslots * m;
    round_kernel<<<(n + 127) / 128, 128, 0, st>>>(D, nslots, m, out);
    MBG_CUDA(cudaGetLastError());
}

int group_grid(const void* kernel, int block, size_t smem, int num_sms, int64_t len) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    int occ;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(kernel);
        if (it == cache.end()) {
            MBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem));
            if (occ < 1) occ = 1;
            if (occ > 8) occ = 8;
            cache[kernel] = occ;
        } else {
            occ = it->second;
        }
    }
    const int64_t need = (len + block - 1) / block;
    const int64_t cap = static_cast<int64_t>(num_sms) * occ;
    return static_cast<int>(need < cap ? (need < 1 ? 1 : need) : cap);
}

// ===========================================================================
// Generic group interpreter: runtime statement list, reference semantics
// (statements in order per element, each output written through to memory
// and re-read by later statements -- execute.cpp:97-119).  Exact dots.
// ===========================================================================
__global__ void __launch_bounds__(256) generic_group_kernel(GenericGroup g) {
    extern __shared__ double sh_dyn[];
    const int m = g.m;
    const int c = threadIdx.x % m;
    double acc[GEN_MAX_SLOT][KEXP];
#pragma unroll
    for (int s = 0; s < GEN_MAX_SLOT; ++s)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) acc[s][i] = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < g.len; e += stride) {
        for (int st = 0; st < g.nstmt; ++st) {
            if (g.kind[st] == MBG_STMT_UPDATE) {
                double a = 0.0;
                for (int t = 0; t < g.nterms[st]; ++t) {
                    const int ti = g.tfirst[st] + t;
                    a = __dadd_rn(a, __dmul_rn(g.coef[ti * m + c], g.vec[g.term_vec[ti]][e]));
                }
                g.vec[g.out[st]][e] = a;
            } else {
                const double p = __dmul_rn(g.vec[g.left[st]][e], g.vec[g.right[st]][e]);
                const int sl = g.dslot[st];
#pragma unroll
                for (int s = 0; s < GEN_MAX_SLOT; ++s)
                    if (s == sl) grow(acc[s], p, g.slot + (static_cast<int64_t>(s) * m + c) * NSLOT);
            }
        }
    }
    if (g.nslots == 0) return;
    // block combine through the same path as the fused kernels, slot by slot
    for (int s = 0; s < g.nslots; ++s) {
        double one[1][KEXP];
#pragma unroll
        for (int i = 0; i < KEXP; ++i) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < GEN_MAX_SLOT; ++q)
                if (q == s) v = acc[q][i];
            one[0][i] = v;
        }
        GroupArgs a{};
        a.m = m;
        a.slot[0] = g.slot + static_cast<int64_t>(s) * m * NSLOT;
        a.part[0] = g.part + static_cast<int64_t>(s) * m * gridDim.x * KEXP;
        block_combine<1>(one, a, c, sh_dyn);
    }
}

void launch_generic_group(cudaStream_t st, const GenericGroup& g, int num_sms, int* nblocks_out) {
    const int block = group_block(g.m);
    const size_t smem = static_cast<size_t>(block) * KEXP * sizeof(double);
    const int grid = group_grid(reinterpret_cast<const void*>(&generic_group_kernel), block, smem, num_sms, g.len);
    generic_group_kernel<<<grid, block, smem, st>>>(g);
    MBG_CUDA(cudaGetLastError());
    *nblocks_out = grid;
}

}  // namespace mbg
