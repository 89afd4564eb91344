// group_lab.cu -- how should a dot-heavy group pass (two input streams, one
// or two exact dots, m = 8 columns) feed its TwoSum chains on B200?
//   reg1 : register prefetch one trip ahead (the shipped scheme)
//   reg2 : register prefetch two trips ahead
//   tma  : cp.async.bulk into an S-stage shared-memory ring (mbarrier
//          complete_tx), consumers read their packets from smem
//   naive: plain (inexact) sum, the memory-bound floor
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_1907_12874_b200/csrc \
//      tools/group_lab.cu -o build/group_lab
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "exact.cuh"

using namespace mbg;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

constexpr int M = 8;
constexpr int BS = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Batched grow of NG independent expansions: one finiteness branch and one
// level-3 branch per batch instead of two per expansion, so the NG TwoSum
// chains are straight-line code the scheduler can interleave.
__device__ __forceinline__ bool nonfinite(double s) {
    return (static_cast<uint32_t>(__double2hiint(s)) & 0x7ff00000u) == 0x7ff00000u;
}
template <int NG>
__device__ __forceinline__ void grow_batch(double (&a)[NG][KEXP], const double (&x)[NG], int64_t* const (&sl)[NG]) {
    double s0[NG];
    bool bad = false;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        s0[g] = __dadd_rn(a[g][0], x[g]);
        bad |= nonfinite(s0[g]);
    }
    if (bad) {
#pragma unroll
        for (int g = 0; g < NG; ++g) grow(a[g], x[g], sl[g]);
        return;
    }
    double e1[NG];
    bool any = false;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        const double b0 = __dsub_rn(s0[g], a[g][0]);
        const double e0 = __dadd_rn(__dsub_rn(a[g][0], __dsub_rn(s0[g], b0)), __dsub_rn(x[g], b0));
        const double s1 = __dadd_rn(a[g][1], e0);
        const double b1 = __dsub_rn(s1, a[g][1]);
        e1[g] = __dadd_rn(__dsub_rn(a[g][1], __dsub_rn(s1, b1)), __dsub_rn(e0, b1));
        a[g][0] = s0[g];
        a[g][1] = s1;
        any |= e1[g] != 0.0;
    }
    if (any) {
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            if (e1[g] != 0.0) {
                const double s2 = __dadd_rn(a[g][2], e1[g]);
                const double b2 = __dsub_rn(s2, a[g][2]);
                const double e2 = __dadd_rn(__dsub_rn(a[g][2], __dsub_rn(s2, b2)), __dsub_rn(e1[g], b2));
                a[g][2] = s2;
                if (e2 != 0.0) digits_add_atomic(sl[g], e2);
            }
        }
    }
}

// Anchored two-level accumulator ("bins"): level sums live in doubles pinned
// to a binade, S1 = 1.5*2^E + L1 and S2 = 1.5*2^(E-41) + L2, so adding a
// product |x| < 2^(E-12) is an error-free extraction of 3 + 3 operations with
// a one-add loop-carried dependency.  Out-of-range products (first product,
// growth, non-finite, extreme exponents) and the rare residual below the
// level-2 grid go to a TwoSum side expansion.
struct Bin {
    double s1, s2;
    uint32_t thi;   // high word of 2^(E-12); 0 = unanchored
    int e;
};
__device__ __forceinline__ double pow2hi(int e, uint32_t mant_hi) {   // (1 + mant) * 2^e, normal range
    return __hiloint2double(static_cast<int>((static_cast<uint32_t>(e + 1023) << 20) | mant_hi), 0);
}
// side expansion of one accumulator in shared memory: element i at side[i * BS]
__device__ __forceinline__ void side_grow(double* side, double x, int64_t* slot) {
    double e[KEXP];
#pragma unroll
    for (int i = 0; i < KEXP; ++i) e[i] = side[i * BS];
    grow(e, x, slot);
#pragma unroll
    for (int i = 0; i < KEXP; ++i) side[i * BS] = e[i];
}
__device__ unsigned long long g_slow[2];
__device__ __noinline__ Bin bin_slow(Bin b, double* side, double x, int64_t* slot) {
    atomicAdd(&g_slow[0], 1ull);
    const uint32_t hi = static_cast<uint32_t>(__double2hiint(x));
    const int ex = static_cast<int>((hi >> 20) & 0x7ff) - 1023;
    if (x == 0.0) return b;
    const int E = ex + 16;
    if (ex == 1024 || E > 1022 || E < -981) {   // non-finite or extreme: straight to the expansion
        side_grow(side, x, slot);
        return b;
    }
    if (b.thi) {   // re-anchor upwards: move the exact level sums into the expansion
        side_grow(side, __dsub_rn(b.s1, pow2hi(b.e, 0x80000u)), slot);
        side_grow(side, __dsub_rn(b.s2, pow2hi(b.e - 41, 0x80000u)), slot);
    }
    b.e = E;
    b.s1 = pow2hi(E, 0x80000u);
    b.s2 = pow2hi(E - 41, 0x80000u);
    b.thi = static_cast<uint32_t>(E - 12 + 1023) << 20;
    const double s1n = __dadd_rn(b.s1, x);
    const double r1 = __dsub_rn(x, __dsub_rn(s1n, b.s1));
    b.s1 = s1n;
    const double s2n = __dadd_rn(b.s2, r1);
    const double r2 = __dsub_rn(r1, __dsub_rn(s2n, b.s2));
    b.s2 = s2n;
    if (r2 != 0.0) side_grow(side, r2, slot);
    return b;
}
__device__ __noinline__ void side_grow_ni(double* side, double x, int64_t* slot) { atomicAdd(&g_slow[1], 1ull); side_grow(side, x, slot); }
__device__ __forceinline__ void bin_add(Bin& b, double* side, double x, int64_t* slot) {
    const uint32_t ah = static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu;
    if (ah < b.thi) {
        const double s1n = __dadd_rn(b.s1, x);
        const double r1 = __dsub_rn(x, __dsub_rn(s1n, b.s1));
        b.s1 = s1n;
        const double s2n = __dadd_rn(b.s2, r1);
        const double r2 = __dsub_rn(r1, __dsub_rn(s2n, b.s2));
        b.s2 = s2n;
        if (r2 != 0.0) side_grow_ni(side, r2, slot);
    } else {
        b = bin_slow(b, side, x, slot);
    }
}
__device__ __forceinline__ void bin_flush(Bin& b, double* side, int64_t* slot) {
    if (b.thi) {
        side_grow(side, __dsub_rn(b.s1, pow2hi(b.e, 0x80000u)), slot);
        side_grow(side, __dsub_rn(b.s2, pow2hi(b.e - 41, 0x80000u)), slot);
        b.s1 = pow2hi(b.e, 0x80000u);
        b.s2 = pow2hi(b.e - 41, 0x80000u);
    }
}

template <int ND, int BATCH = 0>
__device__ __forceinline__ void body(double (&acc)[2 * ND][KEXP], double2 t, double2 s, int64_t* const* sl0,
                                     int64_t* const* sl1) {
    if constexpr (BATCH) {
        double x[2 * ND];
        int64_t* sl[2 * ND];
        x[0] = __dmul_rn(t.x, s.x);
        x[1] = __dmul_rn(t.y, s.y);
        sl[0] = sl0[0];
        sl[1] = sl1[0];
        if constexpr (ND > 1) {
            x[2] = __dmul_rn(t.x, t.x);
            x[3] = __dmul_rn(t.y, t.y);
            sl[2] = sl0[ND - 1];
            sl[3] = sl1[ND - 1];
        }
        grow_batch<2 * ND>(acc, x, sl);
        return;
    }
    grow(acc[0], __dmul_rn(t.x, s.x), sl0[0]);
    grow(acc[1], __dmul_rn(t.y, s.y), sl1[0]);
    if (ND > 1) {
        grow(acc[2], __dmul_rn(t.x, t.x), sl0[ND - 1]);
        grow(acc[3], __dmul_rn(t.y, t.y), sl1[ND - 1]);
    }
}

// block combine as shipped: warp shuffles down to the 4 column classes, a
// shared-memory pass over the warps, one deposit per class and term
template <int ND>
__device__ __forceinline__ void flush(double (&acc)[2 * ND][KEXP], int64_t* const* sl0, int64_t* const* sl1) {
    __shared__ double sh[BS / 32][4][2 * ND][KEXP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int x = 0; x < 2 * ND; ++x) {
        int64_t* sl = (x & 1) ? sl1[x >> 1] : sl0[x >> 1];
        for (int off = 16; off >= 4; off >>= 1) {
            double t[KEXP];
            for (int i = 0; i < KEXP; ++i) t[i] = __shfl_down_sync(~0u, acc[x][i], off);
            if (lane < off)
                for (int i = 0; i < KEXP; ++i) grow(acc[x], t[i], sl);
        }
        if (lane < 4)
            for (int i = 0; i < KEXP; ++i) sh[warp][lane][x][i] = acc[x][i];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        for (int x = 0; x < 2 * ND; ++x) {
            int64_t* sl = (x & 1) ? sl1[x >> 1] : sl0[x >> 1];
            for (int w = 1; w < BS / 32; ++w)
                for (int i = 0; i < KEXP; ++i) grow(acc[x], sh[w][threadIdx.x][x][i], sl);
            for (int i = 0; i < KEXP; ++i)
                if (acc[x][i] != 0.0) digits_add_atomic(sl, acc[x][i]);
        }
    }
}

template <int ND, int DEPTH, int MINB, int BATCH = 0>
__global__ void __launch_bounds__(BS, MINB) k_reg(const double2* a, const double2* b, int64_t npk, int64_t* slots) {
    const int c0 = (threadIdx.x * 2) % M;
    int64_t* sl0[ND];
    int64_t* sl1[ND];
    for (int d = 0; d < ND; ++d) {
        sl0[d] = slots + (d * M + c0) * NSLOT;
        sl1[d] = slots + (d * M + c0 + 1) * NSLOT;
    }
    double acc[2 * ND][KEXP] = {};
    const int64_t stride = (int64_t)gridDim.x * BS;
    int64_t q = (int64_t)blockIdx.x * BS + threadIdx.x;
    double2 ta[DEPTH], sa[DEPTH];
#pragma unroll
    for (int k = 0; k < DEPTH; ++k)
        if (q + k * stride < npk) { ta[k] = a[q + k * stride]; sa[k] = b[q + k * stride]; }
    for (; q < npk; q += stride) {
        const double2 t = ta[0], s = sa[0];
#pragma unroll
        for (int k = 0; k + 1 < DEPTH; ++k) { ta[k] = ta[k + 1]; sa[k] = sa[k + 1]; }
        const int64_t qn = q + DEPTH * stride;
        if (qn < npk) { ta[DEPTH - 1] = a[qn]; sa[DEPTH - 1] = b[qn]; }
        body<ND, BATCH>(acc, t, s, sl0, sl1);
    }
    flush<ND>(acc, sl0, sl1);
}

template <int ND, int DEPTH, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_bin(const double2* a, const double2* b, int64_t npk, int64_t* slots) {
    const int c0 = (threadIdx.x * 2) % M;
    int64_t* sl0[ND];
    int64_t* sl1[ND];
    for (int d = 0; d < ND; ++d) {
        sl0[d] = slots + (d * M + c0) * NSLOT;
        sl1[d] = slots + (d * M + c0 + 1) * NSLOT;
    }
    __shared__ double side_sh[2 * ND][KEXP][BS];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) side_sh[x][i][threadIdx.x] = 0.0;
    Bin bin[2 * ND];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x) bin[x] = Bin{0.0, 0.0, 0u, 0};
    const int64_t stride = (int64_t)gridDim.x * BS;
    int64_t q = (int64_t)blockIdx.x * BS + threadIdx.x;
    double2 ta[DEPTH], sa[DEPTH];
#pragma unroll
    for (int k = 0; k < DEPTH; ++k)
        if (q + k * stride < npk) { ta[k] = a[q + k * stride]; sa[k] = b[q + k * stride]; }
    int trips = 0;
    for (; q < npk; q += stride) {
        const double2 t = ta[0], s = sa[0];
#pragma unroll
        for (int k = 0; k + 1 < DEPTH; ++k) { ta[k] = ta[k + 1]; sa[k] = sa[k + 1]; }
        const int64_t qn = q + DEPTH * stride;
        if (qn < npk) { ta[DEPTH - 1] = a[qn]; sa[DEPTH - 1] = b[qn]; }
        bin_add(bin[0], &side_sh[0][0][threadIdx.x], __dmul_rn(t.x, s.x), sl0[0]);
        bin_add(bin[1], &side_sh[1][0][threadIdx.x], __dmul_rn(t.y, s.y), sl1[0]);
        if (ND > 1) {
            bin_add(bin[2], &side_sh[2][0][threadIdx.x], __dmul_rn(t.x, t.x), sl0[ND - 1]);
            bin_add(bin[3], &side_sh[3][0][threadIdx.x], __dmul_rn(t.y, t.y), sl1[ND - 1]);
        }
        if (++trips == 1024) {
            trips = 0;
#pragma unroll
            for (int x = 0; x < 2 * ND; ++x) bin_flush(bin[x], &side_sh[x][0][threadIdx.x], (x & 1) ? sl1[x >> 1] : sl0[x >> 1]);
        }
    }
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x) bin_flush(bin[x], &side_sh[x][0][threadIdx.x], (x & 1) ? sl1[x >> 1] : sl0[x >> 1]);
    double acc[2 * ND][KEXP];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) acc[x][i] = side_sh[x][i][threadIdx.x];
    __syncthreads();
    flush<ND>(acc, sl0, sl1);
}

template <int ND, int S, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_bin_tma(const double2* a, const double2* b, int64_t npk, int64_t* slots) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double2* buf = reinterpret_cast<double2*>(smem + 128);
    const int c0 = (threadIdx.x * 2) % M;
    int64_t* sl0[ND];
    int64_t* sl1[ND];
    for (int d = 0; d < ND; ++d) {
        sl0[d] = slots + (d * M + c0) * NSLOT;
        sl1[d] = slots + (d * M + c0 + 1) * NSLOT;
    }
    __shared__ double side_sh[2 * ND][KEXP][BS];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) side_sh[x][i][threadIdx.x] = 0.0;
    Bin bin[2 * ND];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x) bin[x] = Bin{0.0, 0.0, 0u, 0};
    const int64_t nch = npk / BS, G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t k, int s) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[s], 2 * BS * 16);
            bulk_g2s(buf + (s * 2 + 0) * BS, a + ch * BS, BS * 16, &bar[s]);
            bulk_g2s(buf + (s * 2 + 1) * BS, b + ch * BS, BS * 16, &bar[s]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) issue(s, s);
    for (int64_t k = 0;; ++k) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch >= nch) break;
        const int s = static_cast<int>(k % S);
        while (!mbar_try_wait(&bar[s], static_cast<uint32_t>((k / S) & 1))) {
        }
        const double2 t = buf[(s * 2 + 0) * BS + threadIdx.x];
        const double2 u = buf[(s * 2 + 1) * BS + threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) issue(k + S, s);
        bin_add(bin[0], &side_sh[0][0][threadIdx.x], __dmul_rn(t.x, u.x), sl0[0]);
        bin_add(bin[1], &side_sh[1][0][threadIdx.x], __dmul_rn(t.y, u.y), sl1[0]);
        if (ND > 1) {
            bin_add(bin[2], &side_sh[2][0][threadIdx.x], __dmul_rn(t.x, t.x), sl0[ND - 1]);
            bin_add(bin[3], &side_sh[3][0][threadIdx.x], __dmul_rn(t.y, t.y), sl1[ND - 1]);
        }
        if ((k & 1023) == 1023) {
#pragma unroll
            for (int x = 0; x < 2 * ND; ++x) bin_flush(bin[x], &side_sh[x][0][threadIdx.x], (x & 1) ? sl1[x >> 1] : sl0[x >> 1]);
        }
    }
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x) bin_flush(bin[x], &side_sh[x][0][threadIdx.x], (x & 1) ? sl1[x >> 1] : sl0[x >> 1]);
    double acc[2 * ND][KEXP];
#pragma unroll
    for (int x = 0; x < 2 * ND; ++x)
#pragma unroll
        for (int i = 0; i < KEXP; ++i) acc[x][i] = side_sh[x][i][threadIdx.x];
    __syncthreads();
    flush<ND>(acc, sl0, sl1);
}

// TMA ring: chunk = BS packets (BS*16 bytes per input); S stages.
template <int ND, int S, int MINB, int BATCH = 0>
__global__ void __launch_bounds__(BS, MINB) k_tma(const double2* a, const double2* b, int64_t npk, int64_t* slots) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double2* buf = reinterpret_cast<double2*>(smem + 128);   // [S][2][BS]
    const int c0 = (threadIdx.x * 2) % M;
    int64_t* sl0[ND];
    int64_t* sl1[ND];
    for (int d = 0; d < ND; ++d) {
        sl0[d] = slots + (d * M + c0) * NSLOT;
        sl1[d] = slots + (d * M + c0 + 1) * NSLOT;
    }
    double acc[2 * ND][KEXP] = {};
    const int64_t nch = npk / BS;   // full chunks (the lab uses multiples)
    const int64_t G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t k, int s) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[s], 2 * BS * 16);
            bulk_g2s(buf + (s * 2 + 0) * BS, a + ch * BS, BS * 16, &bar[s]);
            bulk_g2s(buf + (s * 2 + 1) * BS, b + ch * BS, BS * 16, &bar[s]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) issue(s, s);
    for (int64_t k = 0;; ++k) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch >= nch) break;
        const int s = static_cast<int>(k % S);
        const uint32_t par = static_cast<uint32_t>((k / S) & 1);
        while (!mbar_try_wait(&bar[s], par)) {
        }
        const double2 t = buf[(s * 2 + 0) * BS + threadIdx.x];
        const double2 u = buf[(s * 2 + 1) * BS + threadIdx.x];
        __syncthreads();   // every thread has its packets: the stage may be refilled
        if (threadIdx.x == 0) issue(k + S, s);
        body<ND, BATCH>(acc, t, u, sl0, sl1);
    }
    flush<ND>(acc, sl0, sl1);
}

template <int S, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_tma_read(const double2* a, const double2* b, int64_t npk, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double2* buf = reinterpret_cast<double2*>(smem + 128);
    const int64_t nch = npk / BS, G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t k, int s) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[s], 2 * BS * 16);
            bulk_g2s(buf + (s * 2 + 0) * BS, a + ch * BS, BS * 16, &bar[s]);
            bulk_g2s(buf + (s * 2 + 1) * BS, b + ch * BS, BS * 16, &bar[s]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) issue(s, s);
    double acc = 0;
    for (int64_t k = 0;; ++k) {
        const int64_t ch = blockIdx.x + k * G;
        if (ch >= nch) break;
        const int s = static_cast<int>(k % S);
        while (!mbar_try_wait(&bar[s], static_cast<uint32_t>((k / S) & 1))) {
        }
        const double2 t = buf[(s * 2 + 0) * BS + threadIdx.x];
        const double2 u = buf[(s * 2 + 1) * BS + threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) issue(k + S, s);
        acc += t.x * u.x + t.y * u.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

template <int UNR>
__global__ void k_naive_u(const double2* a, const double2* b, int64_t npk, double* out) {
    double s0 = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < npk; q += UNR * stride) {
        double2 x[UNR], y[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < npk) { x[u] = a[q + u * stride]; y[u] = b[q + u * stride]; }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < npk) s0 += x[u].x * y[u].x + x[u].y * y[u].y;
    }
    if (s0 == 12345.678) out[0] = s0;
}

__global__ void k_naive(const double2* a, const double2* b, int64_t npk, double* out) {
    double s0 = 0, s1 = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < npk; q += stride) {
        const double2 x = a[q], y = b[q];
        s0 += x.x * y.x;
        s1 += x.y * y.y;
    }
    if (s0 + s1 == 12345.678) out[0] = s0;
}

int main() {
    const int64_t len = (int64_t)(1 << 21) * M;   // 16.8M doubles per vector (C2 shape)
    const int64_t npk = len / 2;
    double2 *a, *b;
    int64_t* slots;
    double* out;
    CK(cudaMalloc(&a, len * 8));
    CK(cudaMalloc(&b, len * 8));
    CK(cudaMalloc(&slots, 2 * M * NSLOT * 8));
    CK(cudaMalloc(&out, 8));
    {
        std::vector<double> h(len);
        uint64_t z = 88172645463325252ull;
        auto rnd = [&] {
            z ^= z << 13; z ^= z >> 7; z ^= z << 17;
            return (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2 - 1;
        };
        for (auto& v : h) v = rnd();
        CK(cudaMemcpy(a, h.data(), len * 8, cudaMemcpyHostToDevice));
        for (auto& v : h) v = rnd() * 1e-3;
        CK(cudaMemcpy(b, h.data(), len * 8, cudaMemcpyHostToDevice));
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* flush_buf;
    const size_t FL = 256ull << 20;
    CK(cudaMalloc(&flush_buf, FL));
    std::vector<double> ref;
    bool use_flush = true;
    auto check = [&](const char* name) {
        std::vector<int64_t> h(2 * M * NSLOT);
        CK(cudaMemcpy(h.data(), slots, h.size() * 8, cudaMemcpyDeviceToHost));
        std::vector<double> r;
        for (int d = 0; d < 2 * M; ++d) r.push_back(digits_round(h.data() + d * NSLOT));
        if (ref.empty()) ref = r;
        bool same = r == ref;
        if (!same) printf("  %s: MISMATCH\n", name);
    };
    const char* only = getenv("LAB_ONLY");
    const int lab_iters = getenv("LAB_ITERS") ? atoi(getenv("LAB_ITERS")) : 13;
    auto bench = [&](const char* name, auto f, bool exact, int nd) {
        if (only && !strstr(name, only)) return;
        float best = 1e9, tot = 0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int it = 0; it < lab_iters; ++it) {
            if (use_flush) CK(cudaMemsetAsync(flush_buf, it, FL));
            CK(cudaMemsetAsync(slots, 0, 2 * M * NSLOT * 8));
            cudaEventRecord(e0);
            f();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= (lab_iters > 3 ? 3 : 0)) { tot += ms; best = ms < best ? ms : best; }
        }
        CK(cudaGetLastError());
        const double avg = tot / (lab_iters > 3 ? lab_iters - 3 : lab_iters);
        printf("%-30s nd=%d avg %7.1f us  best %7.1f us  %6.0f GB/s\n", name, nd, avg * 1e3, best * 1e3,
               2.0 * len * 8 / (avg * 1e-3) / 1e9);
        if (exact) check(name);
        unsigned long long cnt[2];
        CK(cudaMemcpyFromSymbol(cnt, g_slow, 16));
        if (cnt[0] || cnt[1]) printf("    slow paths: anchor %llu  residual %llu (over 13 launches)\n", cnt[0], cnt[1]);
        unsigned long long z2[2] = {0, 0};
        CK(cudaMemcpyToSymbol(g_slow, z2, 16));
    };
    for (int nd : {1, 2, 3, 4}) {
        use_flush = nd <= 2;
        if (nd > 2) { nd -= 2; printf("-- no L2 flush between launches\n"); }
        ref.clear();
        char nm[64];
        bench("naive", [&] { k_naive<<<sms * 4, BS>>>(a, b, npk, out); }, false, nd);
        bench("naive u4 x4", [&] { k_naive_u<4><<<sms * 4, BS>>>(a, b, npk, out); }, false, nd);
        bench("naive u4 x8", [&] { k_naive_u<4><<<sms * 8, BS>>>(a, b, npk, out); }, false, nd);
        bench("cudaMemcpy a->flush (r+w)", [&] { cudaMemcpyAsync(flush_buf, a, len * 8, cudaMemcpyDeviceToDevice); }, false, nd);
        {
            const int sm = 128 + 4 * 2 * BS * 16;
            CK(cudaFuncSetAttribute(k_tma_read<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            bench("tma read s4 x4", [&] { k_tma_read<4, 4><<<sms * 4, BS, sm>>>(a, b, npk, out); }, false, nd);
            const int sm8 = 128 + 8 * 2 * BS * 16;
            CK(cudaFuncSetAttribute(k_tma_read<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8));
            bench("tma read s8 x2", [&] { k_tma_read<8, 2><<<sms * 2, BS, sm8>>>(a, b, npk, out); }, false, nd);
        }
#define REG(ND, DEP, MB)                                                                             \
    snprintf(nm, 64, "reg depth=%d minb=%d", DEP, MB);                                               \
    bench(nm, [&] { k_reg<ND, DEP, MB><<<sms * MB, BS>>>(a, b, npk, slots); }, true, ND);
#define TMA(ND, S, MB)                                                                                \
    {                                                                                                 \
        const int sm = 128 + S * 2 * BS * 16;                                                         \
        CK(cudaFuncSetAttribute(k_tma<ND, S, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));  \
        snprintf(nm, 64, "tma stages=%d minb=%d", S, MB);                                             \
        bench(nm, [&] { k_tma<ND, S, MB><<<sms * MB, BS, sm>>>(a, b, npk, slots); }, true, ND);       \
    }
#define REGB(ND, DEP, MB)                                                                            \
    snprintf(nm, 64, "reg batched depth=%d minb=%d", DEP, MB);                                       \
    bench(nm, [&] { k_reg<ND, DEP, MB, 1><<<sms * MB, BS>>>(a, b, npk, slots); }, true, ND);
#define TMAB(ND, S, MB)                                                                               \
    {                                                                                                 \
        const int sm = 128 + S * 2 * BS * 16;                                                         \
        CK(cudaFuncSetAttribute(k_tma<ND, S, MB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
        snprintf(nm, 64, "tma batched stages=%d minb=%d", S, MB);                                     \
        bench(nm, [&] { k_tma<ND, S, MB, 1><<<sms * MB, BS, sm>>>(a, b, npk, slots); }, true, ND);    \
    }
#define BIN(ND, DEP, MB)                                                                            \
    snprintf(nm, 64, "bin depth=%d minb=%d", DEP, MB);                                               \
    bench(nm, [&] { k_bin<ND, DEP, MB><<<sms * MB, BS>>>(a, b, npk, slots); }, true, ND);
#define BINT(ND, S, MB)                                                                               \
    {                                                                                                 \
        const int sm = 128 + S * 2 * BS * 16;                                                         \
        CK(cudaFuncSetAttribute(k_bin_tma<ND, S, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
        snprintf(nm, 64, "bin tma stages=%d minb=%d", S, MB);                                         \
        bench(nm, [&] { k_bin_tma<ND, S, MB><<<sms * MB, BS, sm>>>(a, b, npk, slots); }, true, ND);   \
    }
        if (nd == 1) {
            BIN(1, 1, 4) BIN(1, 2, 4) BINT(1, 2, 4) BINT(1, 4, 4) BINT(1, 4, 3) BINT(1, 4, 2)
        } else {
            BIN(2, 1, 4) BIN(2, 2, 4) BINT(2, 2, 4) BINT(2, 4, 4) BINT(2, 4, 3) BINT(2, 4, 2)
        }
        if (nd == 1) {
            REG(1, 1, 4) REG(1, 2, 4) TMA(1, 2, 4) TMA(1, 4, 3)
            REGB(1, 1, 4) REGB(1, 2, 4) REGB(1, 1, 3) REGB(1, 2, 3) TMAB(1, 2, 4) TMAB(1, 3, 4) TMAB(1, 4, 3) TMAB(1, 4, 2)
        } else {
            REG(2, 1, 4) REG(2, 2, 4) TMA(2, 2, 4) TMA(2, 4, 3)
            REGB(2, 1, 4) REGB(2, 2, 4) REGB(2, 1, 3) REGB(2, 2, 3) TMAB(2, 2, 4) TMAB(2, 3, 4) TMAB(2, 4, 3) TMAB(2, 4, 2)
        }
    }
    return 0;
}
