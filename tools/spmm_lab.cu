// spmm_lab.cu -- standalone SpMM variant benchmark (config C2 shape by default).
// Builds a conv-diff 7-pt matrix, runs several kernel designs, checks every
// output bitwise against a simple reference kernel and prints us / GB/s.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 tools/spmm_lab.cu -o build/spmm_lab
// ./build/spmm_lab [grid=128] [m=8]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- reference
__global__ void k_ref(int n, const int* off, const int* col, const double* val, int m, const double* x, double* y) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * m) return;
    int r = e / m, c = e % m;
    double a = 0.0;
    for (int k = off[r]; k < off[r + 1]; ++k) a = __dadd_rn(a, __dmul_rn(val[k], x[(int64_t)col[k] * m + c]));
    y[e] = a;
}

// ---------------------------------------------------------------- V1: direct, lanes=(row, 2 cols)
template <int M, int B, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_direct(int n, const int* __restrict__ off, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ x,
                                                double* __restrict__ y) {
    constexpr int LPR = M / 2, RPB = 256 / LPR;
    const int row = blockIdx.x * RPB + threadIdx.x / LPR;
    const int cp = (threadIdx.x % LPR) * 2;
    if (row >= n) return;
    const int k0 = __ldg(off + row), k1 = __ldg(off + row + 1);
    double a0 = 0.0, a1 = 0.0;
    for (int k = k0; k < k1; k += B) {
        int j[B];
        double v[B];
        double2 xv[B];
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (k + q < k1) { j[q] = __ldg(col + k + q); v[q] = __ldg(val + k + q); }
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (k + q < k1) xv[q] = __ldg((const double2*)(x + (int64_t)j[q] * M + cp));
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (k + q < k1) { a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q].x)); a1 = __dadd_rn(a1, __dmul_rn(v[q], xv[q].y)); }
    }
    *(double2*)(y + (int64_t)row * M + cp) = make_double2(a0, a1);
}

__device__ __forceinline__ int ld_na_i(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_na_d(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
template <int M, int B, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_direct_na(int n, const int* __restrict__ off, const int* __restrict__ col,
                                                   const double* __restrict__ val, const double* __restrict__ x,
                                                   double* __restrict__ y) {
    constexpr int VW = M >= 2 ? 2 : 1;
    constexpr int LPR = M / VW, RPB = 256 / LPR;
    const int row = blockIdx.x * RPB + threadIdx.x / LPR;
    const int cp = (threadIdx.x % LPR) * VW;
    if (row >= n) return;
    const int k0 = ld_na_i(off + row), k1 = ld_na_i(off + row + 1);
    double a0 = 0.0, a1 = 0.0;
    for (int k = k0; k < k1; k += B) {
        int j[B];
        double v[B];
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (k + q < k1) { j[q] = ld_na_i(col + k + q); v[q] = ld_na_d(val + k + q); }
        if constexpr (VW == 2) {
            double2 xv[B];
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (k + q < k1) xv[q] = __ldg((const double2*)(x + (int64_t)j[q] * M + cp));
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (k + q < k1) { a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q].x)); a1 = __dadd_rn(a1, __dmul_rn(v[q], xv[q].y)); }
        } else {
            double xv[B];
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (k + q < k1) xv[q] = __ldg(x + j[q]);
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (k + q < k1) a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q]));
        }
    }
    if constexpr (VW == 2) *(double2*)(y + (int64_t)row * M + cp) = make_double2(a0, a1);
    else y[row] = a0;
}

// ---------------------------------------------------------------- V4: warp-cooperative coalesced CSR loads + shuffles
// warp covers R = 32/LPR rows; lanes load the warp's nnz range coalesced, rows fetch their entries by shuffle.
template <int M>
__global__ void __launch_bounds__(256) k_warpshfl(int n, const int* __restrict__ off, const int* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ x,
                                                  double* __restrict__ y) {
    constexpr int LPR = M / 2, R = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int wrow0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * R;
    if (wrow0 >= n) return;
    const int myr = lane / LPR, cp = (lane % LPR) * 2;
    const int row = wrow0 + myr;
    // offsets of the warp's rows: lane i < R+1 loads off[wrow0 + i]
    int o = 0;
    if (lane <= R) o = __ldg(off + min(wrow0 + lane, n));
    const int base = __shfl_sync(0xffffffffu, o, 0);
    const int k0 = __shfl_sync(0xffffffffu, o, myr) - base;
    const int k1 = __shfl_sync(0xffffffffu, o, myr + 1) - base;
    const int total = __shfl_sync(0xffffffffu, o, R) - base;
    double a0 = 0.0, a1 = 0.0;
    for (int cb = 0; cb < total; cb += 32) {
        // chunk [cb, cb+32) of the warp's nonzeros in registers
        int cj = 0;
        double cv = 0.0;
        if (cb + lane < total) { cj = __ldg(col + base + cb + lane); cv = __ldg(val + base + cb + lane); }
        const int lo = max(k0, cb), hi = min(k1, cb + 32);
        // all lanes iterate the max count in lockstep for the shuffles
        int cnt = hi - lo;
        int mx = cnt;
        for (int s = 16; s; s >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, s));
        for (int t = 0; t < mx; t += 4) {
            int jj[4];
            double vv[4];
            double2 xv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int src = (lo + t + q - cb) & 31;
                jj[q] = __shfl_sync(0xffffffffu, cj, src);
                vv[q] = __shfl_sync(0xffffffffu, cv, src);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (t + q < cnt) xv[q] = __ldg((const double2*)(x + (int64_t)jj[q] * M + cp));
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (t + q < cnt) { a0 = __dadd_rn(a0, __dmul_rn(vv[q], xv[q].x)); a1 = __dadd_rn(a1, __dmul_rn(vv[q], xv[q].y)); }
        }
    }
    if (row < n) *(double2*)(y + (int64_t)row * M + cp) = make_double2(a0, a1);
}

// ---------------------------------------------------------------- TMA tiled (parametrised)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int M, int TR, int TN, int ST, int RPT, int B, int MINB, int NT = 256, bool CONTIG = false, int PFD = 0,
          int VWP = 0>
__global__ void __launch_bounds__(NT, MINB) k_tma(const int4* __restrict__ tiles, int ntiles, const int* __restrict__ off,
                                                   const int* __restrict__ col, const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y) {
    constexpr int OFFC = TR + 8, NNZP = TN + 8, BUF = OFFC * 4 + NNZP * 12;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = (uint64_t*)smem;
    int4* meta = (int4*)(smem + 64);
    unsigned char* bufs = smem + 192;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int b = 0; b < ST; ++b) mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int per = (ntiles + gridDim.x - 1) / gridDim.x;
    auto tile_of = [&](int i) { return CONTIG ? (i < per ? blockIdx.x * per + i : ntiles) : blockIdx.x + i * gridDim.x; };
    auto issue = [&](int i, int b) {
        const int t = tile_of(i);
        if (t >= ntiles) return;
        const int4 tl = tiles[t];
        const int r0a = tl.x & ~3, r1a = (tl.y + 1 + 3) & ~3, k0a = tl.z & ~3, k1a = (tl.w + 3) & ~3;
        meta[b] = make_int4(tl.x, tl.y, r0a, k0a);
        unsigned char* buf = bufs + b * BUF;
        const uint32_t bo = (r1a - r0a) * 4u, bn = (k1a - k0a);
        mbar_expect_tx(&bars[b], bo + bn * 12u);
        bulk_g2s(buf, off + r0a, bo, &bars[b]);
        bulk_g2s(buf + OFFC * 4, col + k0a, bn * 4u, &bars[b]);
        bulk_g2s(buf + OFFC * 4 + NNZP * 4, val + k0a, bn * 8u, &bars[b]);
        if constexpr (PFD > 0) {   // warm L2 with the tile PFD trips ahead
            const int tp = tile_of(i + PFD);
            if (tp < ntiles) {
                const int4 tq = tiles[tp];
                const int q0 = tq.z & ~3, q1 = (tq.w + 3) & ~3;
                l2_prefetch(col + q0, (q1 - q0) * 4u);
                l2_prefetch(val + q0, (q1 - q0) * 8u);
            }
        }
    };
    if (tid == 0)
        for (int b = 0; b < ST; ++b) issue(b, b);
    constexpr int VW = VWP ? VWP : (M >= 2 ? 2 : 1);
    constexpr int LPR = M / VW, RPP = NT / LPR;
    const int cp = (tid % LPR) * VW;
    for (int i = 0;; ++i) {
        const int t = tile_of(i);
        if (t >= ntiles) break;
        const int b = i % ST;
        while (!mbar_try_wait(&bars[b], (i / ST) & 1)) {
        }
        const int4 mt = meta[b];
        const int r0 = mt.x, r1 = mt.y, r0a = mt.z, k0a = mt.w;
        const unsigned char* buf = bufs + b * BUF;
        const int* s_off = (const int*)buf;
        const int* s_col = (const int*)(buf + OFFC * 4) - k0a;
        const double* s_val = (const double*)(buf + OFFC * 4 + NNZP * 4) - k0a;
        for (int rr = tid / LPR; rr < r1 - r0; rr += RPP) {
            const int row = r0 + rr;
            const int k0 = s_off[row - r0a], k1 = s_off[row + 1 - r0a];
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            for (int k = k0; k < k1; k += B) {
                int j[B];
                double v[B];
#pragma unroll
                for (int q = 0; q < B; ++q)
                    if (k + q < k1) { j[q] = s_col[k + q]; v[q] = s_val[k + q]; }
                if constexpr (VW == 4) {
                    double2 xv[B], xw[B];
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) {
                            xv[q] = __ldg((const double2*)(x + (int64_t)j[q] * M + cp));
                            xw[q] = __ldg((const double2*)(x + (int64_t)j[q] * M + cp + 2));
                        }
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) {
                            a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q].x)); a1 = __dadd_rn(a1, __dmul_rn(v[q], xv[q].y));
                            a2 = __dadd_rn(a2, __dmul_rn(v[q], xw[q].x)); a3 = __dadd_rn(a3, __dmul_rn(v[q], xw[q].y));
                        }
                } else if constexpr (VW == 2) {
                    double2 xv[B];
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) xv[q] = __ldg((const double2*)(x + (int64_t)j[q] * M + cp));
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) { a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q].x)); a1 = __dadd_rn(a1, __dmul_rn(v[q], xv[q].y)); }
                } else {
                    double xv[B];
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) xv[q] = __ldg(x + j[q]);
#pragma unroll
                    for (int q = 0; q < B; ++q)
                        if (k + q < k1) a0 = __dadd_rn(a0, __dmul_rn(v[q], xv[q]));
                }
            }
            if constexpr (VW == 4) {
                *(double2*)(y + (int64_t)row * M + cp) = make_double2(a0, a1);
                *(double2*)(y + (int64_t)row * M + cp + 2) = make_double2(a2, a3);
            } else if constexpr (VW == 2) *(double2*)(y + (int64_t)row * M + cp) = make_double2(a0, a1);
            else y[row] = a0;
        }
        __syncthreads();
        if (tid == 0) issue(i + ST, b);
    }
}

std::vector<int4> make_tiles(const std::vector<int>& off, int n, int TR, int TN) {
    std::vector<int4> t;
    int r = 0;
    while (r < n) {
        int r1 = r;
        while (r1 < n && r1 - r < TR && off[r1 + 1] - off[r] <= TN) ++r1;
        if (r1 == r) { printf("row too long\n"); exit(1); }
        t.push_back(make_int4(r, r1, off[r], off[r1]));
        r = r1;
    }
    return t;
}

struct Ctx {
    int n, m, nnz;
    int *off, *col;
    double *val, *x, *y, *yref;
    std::vector<int> hoff;
    double bytes;
};

template <class F>
void timeit(const char* name, Ctx& c, F launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaMemset(c.y, 0, (size_t)c.n * c.m * 8));
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> h1((size_t)c.n * c.m), h2((size_t)c.n * c.m);
    CK(cudaMemcpy(h1.data(), c.y, h1.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), c.yref, h2.size() * 8, cudaMemcpyDeviceToHost));
    const bool ok = memcmp(h1.data(), h2.data(), h1.size() * 8) == 0;
    for (int w = 0; w < 3; ++w) launch();
    const int reps = 20;
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double us = 1000.0 * ms / reps;
    printf("%-34s %8.1f us  %7.1f GB/s  %s\n", name, us, c.bytes / us / 1e3, ok ? "bitwise-ok" : "MISMATCH");
}

template <int M, int TR, int TN, int ST, int RPT, int B, int MINB, int NT = 256, bool CONTIG = false, int PFD = 0,
          int VWP = 0>
void run_tma(Ctx& c, const char* name) {
    auto tiles = make_tiles(c.hoff, c.n, TR, TN);
    int4* dt;
    CK(cudaMalloc(&dt, tiles.size() * sizeof(int4)));
    CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice));
    constexpr int BUF = (TR + 8) * 4 + (TN + 8) * 12;
    const int smem = 192 + ST * BUF;
    auto kern = k_tma<M, TR, TN, ST, RPT, B, MINB, NT, CONTIG, PFD, VWP>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = std::min<int>((int)tiles.size(), sms * occ);
    char nm[128];
    snprintf(nm, sizeof nm, "%s occ=%d", name, occ);
    timeit(nm, c, [&] { kern<<<grid, NT, smem>>>(dt, (int)tiles.size(), c.off, c.col, c.val, c.x, c.y); });
    CK(cudaFree(dt));
}

static int g_kind = 0;  // 0 conv-diff 7pt, 1 27pt, 2 banded random (n = g^3)

template <int M>
int run_all(int g) {
    const int n = g * g * g, plane = g * g;
    std::vector<int> off(n + 1 + 8), col;
    std::vector<double> val;
    off[0] = 0;
    uint64_t st = 12345;
    auto rnd = [&]() { st = st * 6364136223846793005ull + 1442695040888963407ull; return st >> 33; };
    for (int r = 0; r < n; ++r) {
        int x = r % g, y = (r / g) % g, z = r / plane;
        auto put = [&](int c, double v) { col.push_back(c); val.push_back(v); };
        if (g_kind == 0) {
            if (z > 0) put(r - plane, -1.0);
            if (y > 0) put(r - g, -1.0);
            if (x > 0) put(r - 1, -1.3);
            put(r, 6.0);
            if (x < g - 1) put(r + 1, -0.7);
            if (y < g - 1) put(r + g, -1.0);
            if (z < g - 1) put(r + plane, -1.0);
        } else if (g_kind == 1) {
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (z + dz < 0 || z + dz >= g || y + dy < 0 || y + dy >= g || x + dx < 0 || x + dx >= g) continue;
                        put(r + dz * plane + dy * g + dx, (dx | dy | dz) ? -1.0 : 26.0);
                    }
        } else {
            const int k = 16 + rnd() % 17;
            std::vector<int> cs{r};
            const int lo = std::max(0, r - 65536), hi = std::min(n - 1, r + 65536);
            while ((int)cs.size() < k) {
                int c = lo + (int)(rnd() % (uint64_t)(hi - lo + 1));
                bool dup = false;
                for (int q : cs) dup |= q == c;
                if (!dup) cs.push_back(c);
            }
            std::sort(cs.begin(), cs.end());
            for (int c : cs) put(c, c == r ? 20.0 : -0.5);
        }
        off[r + 1] = (int)col.size();
    }
    for (int i = n + 1; i < n + 9; ++i) off[i] = off[n];
    const int nnz = (int)col.size();
    col.resize(nnz + 8, 0);
    val.resize(nnz + 8, 0.0);
    Ctx c;
    c.n = n;
    c.m = M;
    c.nnz = nnz;
    c.hoff = off;
    c.bytes = 16.0 * M * n + 12.0 * nnz + 4.0 * (n + 1);
    CK(cudaMalloc(&c.off, off.size() * 4));
    CK(cudaMalloc(&c.col, col.size() * 4));
    CK(cudaMalloc(&c.val, val.size() * 8));
    CK(cudaMalloc(&c.x, (size_t)n * M * 8));
    CK(cudaMalloc(&c.y, (size_t)n * M * 8));
    CK(cudaMalloc(&c.yref, (size_t)n * M * 8));
    CK(cudaMemcpy(c.off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.col, col.data(), col.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.val, val.data(), val.size() * 8, cudaMemcpyHostToDevice));
    std::vector<double> hx((size_t)n * M);
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = ((i * 2654435761u) % 1000003) / 1000003.0 - 0.5;
    CK(cudaMemcpy(c.x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
    k_ref<<<(unsigned)(((int64_t)n * M + 255) / 256), 256>>>(n, c.off, c.col, c.val, M, c.x, c.yref);
    CK(cudaDeviceSynchronize());
    printf("n=%d nnz=%d m=%d compulsory %.1f MB\n", n, nnz, M, c.bytes / 1e6);

    // copy roofline for reference
    {
        double *a, *b;
        size_t N = (size_t)1 << 28;
        CK(cudaMalloc(&a, N));
        CK(cudaMalloc(&b, N));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CK(cudaMemcpy(b, a, N, cudaMemcpyDeviceToDevice));
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) CK(cudaMemcpy(b, a, N, cudaMemcpyDeviceToDevice));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s %8.1f us  %7.1f GB/s\n", "cudaMemcpy D2D 256MB", 100 * ms, 2.0 * N * 10 / (ms / 1000) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    timeit("ref thread/(row,col)", c, [&] {
        k_ref<<<(unsigned)(((int64_t)n * M + 255) / 256), 256>>>(n, c.off, c.col, c.val, M, c.x, c.y);
    });
    run_tma<M, 192, 1920, 2, 1, 4, 4>(c, "tma 192r 2st B4 minb4");
    run_tma<M, 192, 1920, 2, 1, 8, 3>(c, "tma 192r 2st B8 minb3");
    run_tma<M, 192, 1920, 2, 1, 8, 2>(c, "tma 192r 2st B8 minb2");
    run_tma<M, 192, 1920, 2, 1, 6, 3>(c, "tma 192r 2st B6 minb3");
    if constexpr (M >= 8) {
        run_tma<M, 256, 1920, 2, 1, 4, 3, 256, false, 0, 4>(c, "tma 256r 2st B4 minb3 VW4");
        run_tma<M, 256, 1920, 2, 1, 2, 4, 256, false, 0, 4>(c, "tma 256r 2st B2 minb4 VW4");
        run_tma<M, 256, 1920, 2, 1, 8, 2, 256, false, 0, 4>(c, "tma 256r 2st B8 minb2 VW4");
    }
    return 0;
}

int main(int argc, char** argv) {
    const int g = argc > 1 ? atoi(argv[1]) : 128;
    const int m = argc > 2 ? atoi(argv[2]) : 8;
    g_kind = argc > 3 ? atoi(argv[3]) : 0;
    if (m == 1) return run_all<1>(g);
    if (m == 8) return run_all<8>(g);
    if (m == 32) return run_all<32>(g);
    if (m == 16) return run_all<16>(g);
    return run_all<4>(g);
}
