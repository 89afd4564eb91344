// exact.cuh -- exact (correctly rounded, order-independent) dot products.
//
// Replaces the reference's thread-blocked naive dot (execute.cpp:112-117,
// 141-157), whose result depends on the thread count (execute.hpp:23-24).
// An exact dot gives the same bits on 1 GPU, N GPUs and the CPU oracle
// (DESIGN.md "Parity").
//
// Representation
//   * per thread: a K-term floating-point expansion grown with TwoSum
//     (error-free); a residual that does not fit after K levels is deposited
//     exactly into the slot's long accumulator with integer atomics.
//   * long accumulator ("digits"): NDIG int64 words, word j counts units of
//     2^(32 j - 1074); three trailing counters record +inf / -inf / NaN
//     products.  Integer addition is associative, so digits from any number of
//     blocks or ranks (ncclInt64 sum) combine exactly.
//   * rounding: carry-normalise, take the top 64 bits plus a sticky bit and
//     round to nearest even, building the IEEE bits directly.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace mbg {

#ifdef __CUDACC__
// Programmatic dependent launch (sm_90+): a kernel launched with
// programmaticStreamSerialization may start while its predecessor drains;
// pdl_wait() blocks until the predecessor has completed and its writes are
// visible, pdl_trigger() lets the successor launch early.  Every solver kernel
// calls pdl_wait() before touching global state (including the stop word).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

constexpr int NDIG = 68;          // 68*32 bits >= 2098-bit double range + carry room
constexpr int NSLOT = 72;         // digits + 3 non-finite counters + pad (int64 words)
constexpr int IDX_PINF = NDIG, IDX_NINF = NDIG + 1, IDX_NAN = NDIG + 2;
constexpr int KEXP = 3;           // expansion length per thread accumulator

__host__ __device__ __forceinline__ uint64_t dbits(double x) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t b;
    __builtin_memcpy(&b, &x, 8);
    return b;
#endif
}

__host__ __device__ __forceinline__ double bitsd(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double x;
    __builtin_memcpy(&x, &b, 8);
    return x;
#endif
}

// Decompose a finite nonzero double into (word index j, three 32-bit chunks).
struct Chunks {
    int j;
    int64_t c0, c1, c2;
    bool neg;
};

__host__ __device__ __forceinline__ bool decompose(double x, Chunks& out, int& nonfinite_idx) {
    const uint64_t b = dbits(x);
    const int ex = static_cast<int>((b >> 52) & 0x7ff);
    uint64_t mant = b & ((1ull << 52) - 1);
    out.neg = (b >> 63) != 0;
    nonfinite_idx = -1;
    if (ex == 0x7ff) {
        nonfinite_idx = mant ? IDX_NAN : (out.neg ? IDX_NINF : IDX_PINF);
        return false;
    }
    int pos;
    if (ex == 0) {
        pos = 0;
    } else {
        mant |= 1ull << 52;
        pos = ex - 1;
    }
    if (!mant) return false;
    out.j = pos >> 5;
    const int sh = pos & 31;
    // mant << sh spans at most 85 bits: split into three 32-bit chunks
    const uint64_t lo = mant << sh;                         // low 64 bits
    const uint64_t hi = sh ? (mant >> (64 - sh)) : 0ull;    // bits 64..84
    out.c0 = static_cast<int64_t>(lo & 0xffffffffull);
    out.c1 = static_cast<int64_t>(lo >> 32);
    out.c2 = static_cast<int64_t>(hi);
    return true;
}

// Non-atomic deposit (fold kernels, host).
__host__ __device__ __forceinline__ void digits_add(int64_t* d, double x) {
    Chunks c;
    int nf;
    if (!decompose(x, c, nf)) {
        if (nf >= 0) d[nf] += 1;
        return;
    }
    if (c.neg) {
        d[c.j] -= c.c0; d[c.j + 1] -= c.c1; d[c.j + 2] -= c.c2;
    } else {
        d[c.j] += c.c0; d[c.j + 1] += c.c1; d[c.j + 2] += c.c2;
    }
}

#ifdef __CUDACC__
// Atomic deposit into a global slot (rare overflow path of the expansions).
__device__ __forceinline__ void digits_add_atomic(int64_t* d, double x) {
    Chunks c;
    int nf;
    auto* u = reinterpret_cast<unsigned long long*>(d);
    if (!decompose(x, c, nf)) {
        if (nf >= 0) atomicAdd(u + nf, 1ull);
        return;
    }
    const unsigned long long s0 = static_cast<unsigned long long>(c.neg ? -c.c0 : c.c0);
    const unsigned long long s1 = static_cast<unsigned long long>(c.neg ? -c.c1 : c.c1);
    const unsigned long long s2 = static_cast<unsigned long long>(c.neg ? -c.c2 : c.c2);
    if (s0) atomicAdd(u + c.j, s0);
    if (s1) atomicAdd(u + c.j + 1, s1);
    if (s2) atomicAdd(u + c.j + 2, s2);
}

// Lazy optimistic grow: not even a per-element finiteness test.  A non-finite
// running sum is sticky in a[0] (inf and NaN survive every later addition), so
// the caller tests a[0] once after its loop and re-walks the thread; the one
// side effect before that test -- the rare level-3 deposit -- is taken only
// while s0 is finite.  NEG = true deposits -e2 instead: the re-walk first
// replays the fast pass with NEG to cancel what it deposited (exactly: the
// replay repeats the same operations), then walks with the careful grow().
// Error-free addition s + e == a + b.  FAST: Dekker's FastTwoSum on the
// operands ordered by magnitude (one compare and two selects plus 3 fp64
// operations); else Knuth's 6-operation TwoSum.  The exact sum, hence every
// result bit, is the same either way.  Measured at ncu's locked base clock
// (tools/ncu_ab.sh): FastTwoSum makes the classical phi/psi pass 6 % faster and
// the Reordered four-dot pass 3 % slower (the selects lengthen its chains), so
// programs opt in (FAST_SUM).
template <bool FAST = false>
__device__ __forceinline__ void two_sum_lazy(double a, double b, double& s, double& e) {
    if constexpr (FAST) {
        const bool sw = fabs(b) > fabs(a);
        const double big = sw ? b : a, sml = sw ? a : b;
        s = __dadd_rn(big, sml);
        e = __dsub_rn(sml, __dsub_rn(s, big));
    } else {
        s = __dadd_rn(a, b);
        const double bb = __dsub_rn(s, a);
        e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    }
}

template <bool NEG = false, bool FAST = false>
__device__ __forceinline__ void grow_lazy(double (&a)[KEXP], double x, int64_t* slot) {
    double s0, e0, s1, e1;
    two_sum_lazy<FAST>(a[0], x, s0, e0);
    two_sum_lazy<FAST>(a[1], e0, s1, e1);
    a[0] = s0;
    a[1] = s1;
    if (e1 != 0.0 && isfinite(s0)) {
        double s2, e2;
        two_sum_lazy<FAST>(a[2], e1, s2, e2);
        a[2] = s2;
        if (e2 != 0.0) digits_add_atomic(slot, NEG ? -e2 : e2);
    }
}

// grow_lazy over N independent expansions as one basic block: levels 1-2 of
// all N run first (branch-free, so the N dependent chains interleave), then a
// single test for any level-2 error takes the rare level-3 path.  Exactly the
// per-expansion operations of grow_lazy, so the same values and deposits
// (integer deposits commute).  ncu on the Reordered 4-dot pass: 42 % of the
// stall samples were dependent-issue waits with a branch after every grow.
template <int N, bool NEG = false, bool FAST = false>
__device__ __forceinline__ void grow_lazy_batch(double (&acc)[N][KEXP], const double (&x)[N],
                                                int64_t* const (&slot)[N]) {
    double e1[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double s0, e0, s1;
        two_sum_lazy<FAST>(acc[k][0], x[k], s0, e0);
        two_sum_lazy<FAST>(acc[k][1], e0, s1, e1[k]);
        acc[k][0] = s0;
        acc[k][1] = s1;
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < N; ++k) any |= e1[k] != 0.0;
    if (any) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (e1[k] != 0.0 && isfinite(acc[k][0])) {
                double s2, e2;
                two_sum_lazy<FAST>(acc[k][2], e1[k], s2, e2);
                acc[k][2] = s2;
                if (e2 != 0.0) digits_add_atomic(slot[k], NEG ? -e2 : e2);
            }
        }
    }
}

// TwoSum-grow x into the expansion a[0..2]; the residual (if any) and any
// non-finite value go to the slot's long accumulator.
//
// Levels 1 and 2 always run (adding 0 is exact, so warps never diverge on
// data).  Level 3 runs only when level 2 leaves an error: for products of a
// normal dynamic range the bits of a thread's partial sum fit in 106 bits, so
// the second-level error is almost always exactly zero and the third TwoSum
// (and the atomic deposit after it) is a rarely taken branch.
__device__ __forceinline__ void grow(double (&a)[KEXP], double x, int64_t* slot) {
    static_assert(KEXP == 3, "grow is written for a 3-term expansion");
    double s0, e0;
    two_sum_lazy(a[0], x, s0, e0);
    if (!isfinite(s0)) {  // x non-finite, or the running sum would overflow
        digits_add_atomic(slot, x);
        return;
    }
    double s1, e1;
    two_sum_lazy(a[1], e0, s1, e1);
    a[0] = s0;
    a[1] = s1;
    if (e1 != 0.0) {
        double s2, e2;
        two_sum_lazy(a[2], e1, s2, e2);
        a[2] = s2;
        if (e2 != 0.0) digits_add_atomic(slot, e2);
    }
}
#endif

#ifdef __CUDACC__
// grow over N independent expansions as one basic block (see grow_lazy_batch):
// levels 1-2 of all N into temporaries and one test; if any expansion met a
// non-finite sum or a level-2 error, all N take grow()'s careful path from
// their untouched state -- the same result as N sequential grow() calls.
template <int N>
__device__ __forceinline__ void grow_batch(double (&acc)[N][KEXP], const double (&x)[N], int64_t* const (&slot)[N]) {
    double s0[N], s1[N];
    bool rare = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double e0, e1;
        two_sum_lazy(acc[k][0], x[k], s0[k], e0);
        two_sum_lazy(acc[k][1], e0, s1[k], e1);
        rare |= !isfinite(s0[k]) || e1 != 0.0;
    }
    if (!rare) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            acc[k][0] = s0[k];
            acc[k][1] = s1[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < N; ++k) grow(acc[k], x[k], slot[k]);
    }
}
#endif

// Carry-normalise in place: words 0..NDIG-2 in [0, 2^32), top word signed.
__host__ __device__ __forceinline__ void digits_normalize(int64_t* d) {
    int64_t carry = 0;
    for (int j = 0; j < NDIG - 1; ++j) {
        const int64_t v = d[j] + carry;
        carry = v >> 32;  // arithmetic shift = floor division
        d[j] = v & 0xffffffffll;
    }
    d[NDIG - 1] += carry;
}

__host__ __device__ __forceinline__ int bitlen32(uint64_t v) {
#ifdef __CUDA_ARCH__
    return 64 - __clzll(static_cast<long long>(v));
#else
    return v ? 64 - __builtin_clzll(v) : 0;
#endif
}

// Correctly rounded value of a slot (round to nearest, ties to even).
__host__ __device__ inline double digits_round(const int64_t* src) {
    const int64_t pinf = src[IDX_PINF], ninf = src[IDX_NINF], nan = src[IDX_NAN];
    if (nan || (pinf && ninf)) return bitsd(0x7ff8000000000000ull);
    if (pinf) return bitsd(0x7ff0000000000000ull);
    if (ninf) return bitsd(0xfff0000000000000ull);
    int64_t d[NDIG];
    for (int j = 0; j < NDIG; ++j) d[j] = src[j];
    digits_normalize(d);
    const bool neg = d[NDIG - 1] < 0;
    if (neg) {
        for (int j = 0; j < NDIG; ++j) d[j] = -d[j];
        digits_normalize(d);
    }
    int h = NDIG - 1;
    while (h >= 0 && d[h] == 0) --h;
    if (h < 0) return 0.0;
    const int L = bitlen32(static_cast<uint64_t>(d[h]));  // 1..32
    const int bitlen = 32 * h + L;
    uint64_t out;
    if (bitlen <= 53) {
        // exact: the bit pattern of mag * 2^-1074 is mag itself
        const uint64_t mag = (h >= 1 ? (static_cast<uint64_t>(d[1]) << 32) : 0ull) | static_cast<uint64_t>(d[0]);
        out = mag;
    } else {
        uint64_t top;      // top 64 bits of the magnitude, MSB set
        bool sticky;
        if (bitlen <= 64) {
            const uint64_t mag = (static_cast<uint64_t>(d[1]) << 32) | static_cast<uint64_t>(d[0]);
            top = mag << (64 - bitlen);
            sticky = false;
        } else {
            const uint64_t whi = (static_cast<uint64_t>(d[h]) << 32) | static_cast<uint64_t>(d[h - 1]);
            const uint64_t wlo = static_cast<uint64_t>(d[h - 2]);
            top = (whi << (32 - L)) | (wlo >> L);
            sticky = (wlo & ((1ull << L) - 1)) != 0;
            for (int j = 0; j < h - 2 && !sticky; ++j) sticky = d[j] != 0;
        }
        uint64_t keep = top >> 11;
        const bool rbit = (top >> 10) & 1;
        sticky = sticky || (top & 0x3ff) != 0;
        int shift = bitlen - 53;
        if (rbit && (sticky || (keep & 1))) ++keep;
        if (keep == (1ull << 53)) { keep >>= 1; ++shift; }
        const int biased = shift + 1;
        if (biased >= 2047)
            out = 0x7ff0000000000000ull;
        else
            out = (static_cast<uint64_t>(biased) << 52) | (keep & ((1ull << 52) - 1));
    }
    return bitsd(out | (neg ? 0x8000000000000000ull : 0ull));
}

#ifdef __CUDACC__
// Device rounding with every word in registers (fully unrolled; no local
// memory).  Same result as digits_round.
__device__ __forceinline__ double digits_round_regs(const int64_t* __restrict__ src) {
    const int64_t pinf = src[IDX_PINF], ninf = src[IDX_NINF], nan = src[IDX_NAN];
    int64_t d[NDIG];
#pragma unroll
    for (int j = 0; j < NDIG; ++j) d[j] = src[j];
    if (nan || (pinf && ninf)) return bitsd(0x7ff8000000000000ull);
    if (pinf) return bitsd(0x7ff0000000000000ull);
    if (ninf) return bitsd(0xfff0000000000000ull);
    int64_t carry = 0;
#pragma unroll
    for (int j = 0; j < NDIG - 1; ++j) {
        const int64_t v = d[j] + carry;
        carry = v >> 32;
        d[j] = v & 0xffffffffll;
    }
    d[NDIG - 1] += carry;
    const bool neg = d[NDIG - 1] < 0;
    if (neg) {
        carry = 0;
#pragma unroll
        for (int j = 0; j < NDIG - 1; ++j) {
            const int64_t v = -d[j] + carry;
            carry = v >> 32;
            d[j] = v & 0xffffffffll;
        }
        d[NDIG - 1] = -d[NDIG - 1] + carry;
    }
    // top nonzero word h and the two below it, plus a sticky flag for the rest
    int h = -1;
    uint64_t t0 = 0, t1 = 0, t2 = 0;
    bool below = false;   // any nonzero word strictly below h-2
    bool acc2 = false;    // OR of words 0..j-3 while scanning
#pragma unroll
    for (int j = 0; j < NDIG; ++j) {
        if (j >= 3) acc2 = acc2 || (d[j - 3] != 0);
        if (d[j] != 0) {
            h = j;
            t0 = static_cast<uint64_t>(d[j]);
            t1 = j >= 1 ? static_cast<uint64_t>(d[j - 1]) : 0ull;
            t2 = j >= 2 ? static_cast<uint64_t>(d[j - 2]) : 0ull;
            below = acc2;
        }
    }
    if (h < 0) return 0.0;
    const int L = bitlen32(t0);
    const int bitlen = 32 * h + L;
    uint64_t out;
    if (bitlen <= 64) {
        const uint64_t mag = h >= 1 ? ((t0 << 32) | t1) : t0;
        if (bitlen <= 53) {
            out = mag;
        } else {
            const int shift = bitlen - 53;
            uint64_t keep = mag >> shift;
            const bool rbit = (mag >> (shift - 1)) & 1;
            const bool sticky = (mag & ((1ull << (shift - 1)) - 1)) != 0;
            if (rbit && (sticky || (keep & 1))) ++keep;
            int sh = shift;
            if (keep == (1ull << 53)) { keep >>= 1; ++sh; }
            out = (static_cast<uint64_t>(sh + 1) << 52) | (keep & ((1ull << 52) - 1));
        }
    } else {
        const uint64_t whi = (t0 << 32) | t1;
        const uint64_t top = (whi << (32 - L)) | (t2 >> L);
        bool sticky = below || (t2 & ((1ull << L) - 1)) != 0;
        uint64_t keep = top >> 11;
        const bool rbit = (top >> 10) & 1;
        sticky = sticky || (top & 0x3ff) != 0;
        int shift = bitlen - 53;
        if (rbit && (sticky || (keep & 1))) ++keep;
        if (keep == (1ull << 53)) { keep >>= 1; ++shift; }
        const int biased = shift + 1;
        out = biased >= 2047 ? 0x7ff0000000000000ull
                             : (static_cast<uint64_t>(biased) << 52) | (keep & ((1ull << 52) - 1));
    }
    return bitsd(out | (neg ? 0x8000000000000000ull : 0ull));
}

// Warp-cooperative rounding of one slot (all 32 lanes call it; all return the
// same value).  Only the window of nonzero words is walked: lanes hold the
// words, a ballot finds the window [lo, hi], and the carry pass runs
// sequentially over it (typically < 12 words) with the words delivered by
// shuffles.  A negative sum is detected by the signed top word of the first
// pass and the pass repeats on the negated words.  Same result as digits_round.
__device__ __forceinline__ double warp_round_slot(const int64_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    // L2 loads: the slot was filled by other blocks' atomics
    const int64_t w0 = __ldcg(src + lane);
    const int64_t w1 = __ldcg(src + lane + 32);
    const int64_t w2 = lane + 64 < NDIG ? __ldcg(src + lane + 64) : 0;
    const int64_t pinf = __ldcg(src + IDX_PINF), ninf = __ldcg(src + IDX_NINF), nan = __ldcg(src + IDX_NAN);
    if (nan || (pinf && ninf)) return bitsd(0x7ff8000000000000ull);
    if (pinf) return bitsd(0x7ff0000000000000ull);
    if (ninf) return bitsd(0xfff0000000000000ull);
    const unsigned m0 = __ballot_sync(0xffffffffu, w0 != 0);
    const unsigned m1 = __ballot_sync(0xffffffffu, w1 != 0);
    const unsigned m2 = __ballot_sync(0xffffffffu, w2 != 0);
    if (!(m0 | m1 | m2)) return 0.0;
    const int lo = m0 ? __ffs(m0) - 1 : (m1 ? 32 + __ffs(m1) - 1 : 64 + __ffs(m2) - 1);
    const int hi = m2 ? 64 + 31 - __clz(m2) : (m1 ? 32 + 31 - __clz(m1) : 31 - __clz(m0));
    const int top = hi + 2 < NDIG - 1 ? hi + 2 : NDIG - 1;  // |word| < 2^44: carries reach <= 2 words up

    int h = -1;
    uint64_t t0 = 0, t1 = 0, t2 = 0;
    bool below = false;
    int64_t wtop = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int64_t sgn = pass ? -1 : 1;
        int64_t carry = 0;
        uint64_t p1 = 0, p2 = 0;   // the two previous normalised words
        bool acc = false;          // OR of words at least three below the current one
        h = -1;
        for (int j = lo; j <= top; ++j) {
            const int g = j >> 5;
            const int64_t mine = g == 0 ? w0 : (g == 1 ? w1 : w2);
            const int64_t dj = __shfl_sync(0xffffffffu, mine, j & 31) * sgn;
            const int64_t v = dj + carry;
            uint64_t word;
            if (j < top) {
                carry = v >> 32;
                word = static_cast<uint64_t>(v & 0xffffffffll);
            } else {
                wtop = v;
                word = static_cast<uint64_t>(v);
            }
            if (word != 0) {
                h = j;
                t0 = word;
                t1 = p1;
                t2 = p2;
                below = acc;
            }
            acc = acc || (p2 != 0);
            p2 = p1;
            p1 = word;
        }
        if (wtop >= 0) {
            const bool neg = pass == 1;
            if (h < 0) return 0.0;
            const int L = bitlen32(t0);
            const int bitlen = 32 * h + L;
            uint64_t out;
            if (bitlen <= 64) {
                // h <= 1: the window started at word 0 or 1 and t1 is word h-1
                const uint64_t mag = h >= 1 ? ((t0 << 32) | t1) : t0;
                if (bitlen <= 53) {
                    out = mag;
                } else {
                    const int shift = bitlen - 53;
                    uint64_t keep = mag >> shift;
                    const bool rbit = (mag >> (shift - 1)) & 1;
                    const bool sticky = (mag & ((1ull << (shift - 1)) - 1)) != 0;
                    if (rbit && (sticky || (keep & 1))) ++keep;
                    int sh = shift;
                    if (keep == (1ull << 53)) { keep >>= 1; ++sh; }
                    out = (static_cast<uint64_t>(sh + 1) << 52) | (keep & ((1ull << 52) - 1));
                }
            } else {
                const uint64_t whi = (t0 << 32) | t1;
                const uint64_t topbits = (whi << (32 - L)) | (t2 >> L);
                bool sticky = below || (t2 & ((1ull << L) - 1)) != 0;
                uint64_t keep = topbits >> 11;
                const bool rbit = (topbits >> 10) & 1;
                sticky = sticky || (topbits & 0x3ff) != 0;
                int shift = bitlen - 53;
                if (rbit && (sticky || (keep & 1))) ++keep;
                if (keep == (1ull << 53)) { keep >>= 1; ++shift; }
                const int biased = shift + 1;
                out = biased >= 2047 ? 0x7ff0000000000000ull
                                     : (static_cast<uint64_t>(biased) << 52) | (keep & ((1ull << 52) - 1));
            }
            return bitsd(out | (neg ? 0x8000000000000000ull : 0ull));
        }
    }
    return bitsd(0x7ff8000000000000ull);  // unreachable: the negated pass has a non-negative top
}
#endif

}  // namespace mbg
