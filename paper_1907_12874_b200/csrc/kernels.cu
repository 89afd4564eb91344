#include <cstdlib>
// kernels.cu -- SpMM, exact-dot fold/round and the generic group interpreter
// for sm_100a.
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include "common.hpp"
#include "kernels.hpp"

namespace mbg {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MBG_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

__global__ void round_kernel(int64_t* D, int nslots, int m, double* out) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // one warp per slot
    if (i < nslots * m) {
        const double r = warp_round_slot(D + static_cast<int64_t>(i) * NSLOT);
        if ((threadIdx.x & 31) == 0) out[i] = r;
    }
}

void launch_round(cudaStream_t st, int64_t* D, int nslots, int m, double* out) {
    const int n = nslots * m;
    round_kernel<<<(n + 3) / 4, 128, 0, st>>>(D, nslots, m, out);
    MBG_CUDA(cudaGetLastError());
}

int kernel_occupancy(const void* kernel, int threads, size_t smem) {
    // keyed by (device, kernel, threads, smem): the dynamic shared-memory
    // attribute is per device, so a second context on another device sets it
    // again before its first launch (function-static caches did not)
    struct Key {
        int dev;
        const void* k;
        int threads;
        size_t smem;
        bool operator<(const Key& o) const {
            return std::tie(dev, k, threads, smem) < std::tie(o.dev, o.k, o.threads, o.smem);
        }
    };
    static std::mutex mu;
    static std::map<Key, int> cache;
    int dev = 0;
    MBG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const Key key{dev, kernel, threads, smem};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (smem > (48u << 10))
        MBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    MBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    if (occ < 1) occ = 1;
    cache[key] = occ;
    return occ;
}

int group_grid(const void* kernel, int block, size_t smem, int num_sms, int64_t len) {
    const int occ = std::min(8, kernel_occupancy(kernel, block, smem));
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
    (void)c;
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
        block_combine<1>(one, m,
                         [&](int, int k) { return g.slot + (static_cast<int64_t>(s) * m + k) * NSLOT; }, sh_dyn);
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
