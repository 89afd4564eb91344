/*
 * oracle.c -- CPU restatement of the multi-RHS BiCGStab hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked by the product.
 *
 * Compile with -ffp-contract=off: every multiply and add below must round
 * separately, exactly like the reference built with its CMake defaults
 * (proj/CMakeLists.txt:8-10, no -march => no FMA).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <time.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================================================================
 * RNG: SplitMix64 finaliser over a packed (seed, stream, a, b) key.
 * The reference has no RNG; this is the pin shared
 * with the product generator (paper_1907_12874_b200/csrc/generators.cpp).
 * ==================================================================== */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

uint64_t orc_hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
    h = mix64(h + a * 0xD1B54A32D192ED03ULL + 0x9E3779B97F4A7C15ULL);
    h = mix64(h + b * 0x8CB92BA72F3D8DD7ULL + 0x9E3779B97F4A7C15ULL);
    return h;
}

double orc_u01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return (double)(orc_hash4(seed, stream, a, b) >> 11) * 0x1.0p-53;
}

double orc_u11(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return 2.0 * orc_u01(seed, stream, a, b) - 1.0;
}

enum { ST_RHS = 1, ST_MAT = 2, ST_CNT = 3, ST_COL = 4, ST_VAL = 5 };

/* Host STREAM-style triad a = b + s*c over n doubles, all OpenMP threads, best of
 * reps: the host bandwidth recorded beside the CPU baseline. */
double orc_triad_gbs(long n, int reps) {
    double* a = (double*)malloc(sizeof(double) * (size_t)n);
    double* b = (double*)malloc(sizeof(double) * (size_t)n);
    double* c = (double*)malloc(sizeof(double) * (size_t)n);
    if (!a || !b || !c) { free(a); free(b); free(c); return 0.0; }
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) { a[i] = 0.0; b[i] = 1.0; c[i] = 2.0; }
    double best = 0.0;
    for (int r = 0; r < reps; ++r) {
        struct timespec t0, t1;
        clock_gettime(CLOCK_MONOTONIC, &t0);
#pragma omp parallel for schedule(static)
        for (long i = 0; i < n; ++i) a[i] = b[i] + 3.0 * c[i];
        clock_gettime(CLOCK_MONOTONIC, &t1);
        const double sec = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
        const double gbs = 24.0 * (double)n / sec / 1e9;
        if (gbs > best) best = gbs;
    }
    free(a); free(b); free(c);
    return best;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ======================================================================
 * Generators.  The 7-point layout follows gen_poisson_7pt
 * (generators.cpp:37-67): lexicographic rows, x fastest, neighbours in
 * ascending column order, constant diagonal regardless of boundary.
 * ==================================================================== */
static int stencil_row_count(int kind, int nx, int ny, int nz, int64_t row) {
    const int x = (int)(row % nx);
    const int y = (int)((row / nx) % ny);
    const int z = (int)(row / ((int64_t)nx * ny));
    if (kind == 2) {
        int cx = 1 + (x > 0) + (x < nx - 1);
        int cy = 1 + (y > 0) + (y < ny - 1);
        int cz = 1 + (z > 0) + (z < nz - 1);
        return cx * cy * cz;
    }
    return 1 + (x > 0) + (x < nx - 1) + (y > 0) + (y < ny - 1) + (z > 0) + (z < nz - 1);
}

int orc_gen_stencil(int kind, int nx, int ny, int nz, uint64_t seed, orc_csr* out) {
    if (nx < 1 || ny < 1 || nz < 1 || kind < 0 || kind > 3 || (kind == 3 && nz != 1)) return -1;
    const int64_t n = (int64_t)nx * ny * nz;
    const int64_t plane = (int64_t)nx * ny;
    out->n = n;
    out->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!out->off) return -2;
    out->off[0] = 0;
    for (int64_t i = 0; i < n; ++i) out->off[i + 1] = out->off[i] + stencil_row_count(kind, nx, ny, nz, i);
    out->nnz = out->off[n];
    out->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)out->nnz);
    out->val = (double*)malloc(sizeof(double) * (size_t)out->nnz);
    if (!out->col || !out->val) return -2;

#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < n; ++row) {
        const int x = (int)(row % nx);
        const int y = (int)((row / nx) % ny);
        const int z = (int)(row / plane);
        int64_t k = out->off[row];
        if (kind == 2) {
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (z + dz < 0 || z + dz >= nz || y + dy < 0 || y + dy >= ny ||
                            x + dx < 0 || x + dx >= nx)
                            continue;
                        const int64_t c = row + dz * plane + (int64_t)dy * nx + dx;
                        out->col[k] = (int32_t)c;
                        if (c == row)
                            out->val[k] = 26.0;
                        else
                            out->val[k] = -1.0 + 0.1 * orc_u11(seed, ST_MAT, (uint64_t)row, (uint64_t)c);
                        ++k;
                    }
        } else {
            const double west = kind == 1 ? -1.3 : -1.0;
            const double east = kind == 1 ? -0.7 : -1.0;
            if (z > 0)      { out->col[k] = (int32_t)(row - plane); out->val[k++] = -1.0; }
            if (y > 0)      { out->col[k] = (int32_t)(row - nx);    out->val[k++] = -1.0; }
            if (x > 0)      { out->col[k] = (int32_t)(row - 1);     out->val[k++] = west; }
            out->col[k] = (int32_t)row; out->val[k++] = kind == 3 ? 4.0 : 6.0;   /* 3: gen_poisson_5pt */
            if (x < nx - 1) { out->col[k] = (int32_t)(row + 1);     out->val[k++] = east; }
            if (y < ny - 1) { out->col[k] = (int32_t)(row + nx);    out->val[k++] = -1.0; }
            if (z < nz - 1) { out->col[k] = (int32_t)(row + plane); out->val[k++] = -1.0; }
        }
    }
    return 0;
}

static int banded_count(int64_t n, int64_t band, int kmin, int kmax, uint64_t seed, int64_t i) {
    int k = kmin + (int)(orc_hash4(seed, ST_CNT, (uint64_t)i, 0) % (uint64_t)(kmax - kmin + 1));
    const int64_t lo = i - band < 0 ? 0 : i - band;
    const int64_t hi = i + band > n - 1 ? n - 1 : i + band;
    const int64_t avail = hi - lo; /* candidates excluding the diagonal */
    if (k - 1 > avail) k = (int)avail + 1;
    return k;
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int orc_gen_banded(int64_t n, int64_t band, int kmin, int kmax, uint64_t seed, orc_csr* out) {
    if (n < 1 || kmin < 1 || kmax < kmin || band < 0) return -1;
    out->n = n;
    out->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!out->off) return -2;
    out->off[0] = 0;
    for (int64_t i = 0; i < n; ++i) out->off[i + 1] = out->off[i] + banded_count(n, band, kmin, kmax, seed, i);
    out->nnz = out->off[n];
    out->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)out->nnz);
    out->val = (double*)malloc(sizeof(double) * (size_t)out->nnz);
    if (!out->col || !out->val) return -2;

#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t lo = i - band < 0 ? 0 : i - band;
        const int64_t hi = i + band > n - 1 ? n - 1 : i + band;
        const uint64_t width = (uint64_t)(hi - lo + 1);
        const int k = (int)(out->off[i + 1] - out->off[i]);
        int32_t* cols = out->col + out->off[i];
        double* vals = out->val + out->off[i];
        int have = 0;
        cols[have++] = (int32_t)i;
        for (uint64_t j = 0; have < k; ++j) {
            const int64_t c = lo + (int64_t)(orc_hash4(seed, ST_COL, (uint64_t)i, j) % width);
            int dup = 0;
            for (int t = 0; t < have; ++t)
                if (cols[t] == (int32_t)c) { dup = 1; break; }
            if (!dup) cols[have++] = (int32_t)c;
        }
        qsort(cols, (size_t)k, sizeof(int32_t), cmp_i32);
        double s = 0.0;
        int diag = -1;
        for (int t = 0; t < k; ++t) {
            if (cols[t] == (int32_t)i) { diag = t; continue; }
            vals[t] = -orc_u01(seed, ST_VAL, (uint64_t)i, (uint64_t)cols[t]);
            s = s + fabs(vals[t]);
        }
        vals[diag] = 1.1 * s;
    }
    return 0;
}

void orc_csr_free(orc_csr* a) {
    free(a->off); free(a->col); free(a->val);
    a->off = NULL; a->col = NULL; a->val = NULL;
}

void orc_rhs(int64_t n, int m, uint64_t seed, double* b) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < m; ++c) b[i * m + c] = orc_u11(seed, ST_RHS, (uint64_t)i, (uint64_t)c);
}

/* ======================================================================
 * SpMV over the interleaved block: restates spmv_rows (spmv.cpp:27-50).
 * acc starts at 0.0, nonzeros in CSR order, separate multiply and add.
 * ==================================================================== */
void orc_spmv(const orc_csr* a, int m, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < a->n; ++i) {
        double acc[64];
        double* accp = m <= 64 ? acc : (double*)malloc(sizeof(double) * (size_t)m);
        for (int c = 0; c < m; ++c) accp[c] = 0.0;
        for (int64_t k = a->off[i]; k < a->off[i + 1]; ++k) {
            const double v = a->val[k];
            const double* xr = x + (int64_t)a->col[k] * m;
            for (int c = 0; c < m; ++c) accp[c] += v * xr[c];
        }
        for (int c = 0; c < m; ++c) y[i * m + c] = accp[c];
        if (accp != acc) free(accp);
    }
}

/* Restates run_rows' update branch (execute.cpp:104-111). */
void orc_spmv_transpose(const orc_csr* a, int m, const double* x, double* y) {
    memset(y, 0, sizeof(double) * (size_t)(a->n * m));
    for (int64_t i = 0; i < a->n; ++i) {
        const double* xr = x + i * m;
        for (int64_t k = a->off[i]; k < a->off[i + 1]; ++k) {
            const double v = a->val[k];
            double* yr = y + (int64_t)a->col[k] * m;
            for (int c = 0; c < m; ++c) yr[c] = yr[c] + v * xr[c];
        }
    }
}

void orc_update(int64_t n, int m, int nterms, const double* const* coeff,
                const double* const* src, double* out) {
    const int64_t len = n * m;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < len; ++e) {
        const int c = (int)(e % m);
        double acc = 0.0;
        for (int t = 0; t < nterms; ++t) acc += coeff[t][c] * src[t][e];
        out[e] = acc;
    }
}

/* ======================================================================
 * Exact dot product.
 *
 * Kulisch long accumulator: digit j holds a signed count of 2^(32j-1074).
 * Fast path: a 4-term floating-point expansion per accumulator (TwoSum
 * chain); any residual that does not fit, and the expansion itself at the
 * end, is deposited into the long accumulator exactly.  The result is the
 * correctly rounded exact sum, independent of order and thread count.
 * ==================================================================== */
#define NDIG 68
#define KEXP 4

typedef struct {
    int64_t d[NDIG];
    int64_t pinf, ninf, nan;
} kacc;

static void kacc_clear(kacc* k) { memset(k, 0, sizeof(*k)); }

static void kacc_add(kacc* k, double x) {
    uint64_t bits;
    memcpy(&bits, &x, sizeof bits);
    const int neg = (int)(bits >> 63);
    const int ex = (int)((bits >> 52) & 0x7ff);
    uint64_t mant = bits & ((1ULL << 52) - 1);
    if (ex == 0x7ff) {
        if (mant) k->nan++;
        else if (neg) k->ninf++;
        else k->pinf++;
        return;
    }
    int pos;
    if (ex == 0) pos = 0;
    else { mant |= 1ULL << 52; pos = ex - 1; }
    if (!mant) return;
    const int j = pos >> 5, sh = pos & 31;
    const unsigned __int128 v = (unsigned __int128)mant << sh;
    const int64_t c0 = (int64_t)(uint64_t)(v & 0xffffffffu);
    const int64_t c1 = (int64_t)(uint64_t)((v >> 32) & 0xffffffffu);
    const int64_t c2 = (int64_t)(uint64_t)(v >> 64);
    if (neg) { k->d[j] -= c0; k->d[j + 1] -= c1; k->d[j + 2] -= c2; }
    else     { k->d[j] += c0; k->d[j + 1] += c1; k->d[j + 2] += c2; }
}

static void kacc_merge(kacc* dst, const kacc* src) {
    for (int j = 0; j < NDIG; ++j) dst->d[j] += src->d[j];
    dst->pinf += src->pinf; dst->ninf += src->ninf; dst->nan += src->nan;
}

static void normalize(int64_t* d) {
    for (int j = 0; j < NDIG - 1; ++j) {
        const int64_t carry = d[j] >> 32; /* floor division */
        d[j] -= carry * 4294967296LL;
        d[j + 1] += carry;
    }
}

static int get_bit(const int64_t* d, int i) { return (int)((d[i >> 5] >> (i & 31)) & 1); }

/* Round the exact value held by k to the nearest double (ties to even). */
static double kacc_round(const kacc* k) {
    if (k->nan || (k->pinf && k->ninf)) return NAN;
    if (k->pinf) return INFINITY;
    if (k->ninf) return -INFINITY;
    int64_t d[NDIG];
    memcpy(d, k->d, sizeof d);
    normalize(d);
    int neg = d[NDIG - 1] < 0;
    if (neg) {
        for (int j = 0; j < NDIG; ++j) d[j] = -d[j];
        normalize(d);
    }
    int top = -1;
    for (int i = NDIG * 32 - 1; i >= 0; --i)
        if (get_bit(d, i)) { top = i; break; }
    if (top < 0) return 0.0;
    const int len = top + 1;
    double r;
    if (len <= 53) {
        uint64_t mag = 0;
        for (int i = 0; i < len; ++i) mag |= (uint64_t)get_bit(d, i) << i;
        r = ldexp((double)mag, -1074);
    } else {
        int shift = len - 53;
        uint64_t keep = 0;
        for (int i = 0; i < 53; ++i) keep |= (uint64_t)get_bit(d, shift + i) << i;
        const int half = get_bit(d, shift - 1);
        int sticky = 0;
        for (int i = 0; i < shift - 1 && !sticky; ++i) sticky = get_bit(d, i);
        if (half && (sticky || (keep & 1))) ++keep;
        if (keep == (1ULL << 53)) { keep >>= 1; ++shift; }
        r = ldexp((double)keep, shift - 1074);
    }
    return neg ? -r : r;
}

typedef struct {
    double a[KEXP];
} expansion;

static void exp_add(expansion* e, kacc* k, double x) {
    if (!isfinite(x)) { kacc_add(k, x); return; }
    for (int i = 0; i < KEXP; ++i) {
        const double s = e->a[i] + x;
        if (!isfinite(s)) { kacc_add(k, x); return; }
        const double bv = s - e->a[i];
        const double av = s - bv;
        const double err = (e->a[i] - av) + (x - bv);
        e->a[i] = s;
        x = err;
        if (x == 0.0) return;
    }
    kacc_add(k, x);
}

static void exp_flush(expansion* e, kacc* k) {
    for (int i = 0; i < KEXP; ++i) { kacc_add(k, e->a[i]); e->a[i] = 0.0; }
}

double orc_sum_exact(int64_t n, const double* v) {
    kacc k; kacc_clear(&k);
    expansion e; memset(&e, 0, sizeof e);
    for (int64_t i = 0; i < n; ++i) exp_add(&e, &k, v[i]);
    exp_flush(&e, &k);
    return kacc_round(&k);
}

void orc_dot_exact(int64_t n, int m, const double* a, const double* b, double* out) {
    kacc* total = (kacc*)calloc((size_t)m, sizeof(kacc));
#pragma omp parallel
    {
        kacc* loc = (kacc*)calloc((size_t)m, sizeof(kacc));
        expansion* ex = (expansion*)calloc((size_t)m, sizeof(expansion));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) {
                const double p = a[i * m + c] * b[i * m + c];
                exp_add(&ex[c], &loc[c], p);
            }
        for (int c = 0; c < m; ++c) exp_flush(&ex[c], &loc[c]);
#pragma omp critical
        for (int c = 0; c < m; ++c) kacc_merge(&total[c], &loc[c]);
        free(loc); free(ex);
    }
    for (int c = 0; c < m; ++c) out[c] = kacc_round(&total[c]);
    free(total);
}

/* ======================================================================
 * Solvers.  Schedules and term expansions: SURVEY.md Appendix C.
 * ==================================================================== */
typedef struct {
    int64_t n; int m; int64_t len;
} shape;

static double* vnew(const shape* s) { return (double*)calloc((size_t)s->len, sizeof(double)); }

#define UPD(S, OUT, NT, ...)                                                       \
    do {                                                                           \
        const double* _pairs[] = {__VA_ARGS__};                                    \
        const double* _c[4]; const double* _v[4];                                  \
        for (int _t = 0; _t < (NT); ++_t) { _c[_t] = _pairs[2 * _t]; _v[_t] = _pairs[2 * _t + 1]; } \
        orc_update((S)->n, (S)->m, (NT), _c, _v, (OUT));                           \
    } while (0)

static double hist_entry(double res2, double bb) {
    const double r = res2 > 0.0 ? res2 : 0.0;
    return sqrt(r / bb);
}

static int all_below(const double* v, const double* eps2, int m) {
    for (int c = 0; c < m; ++c)
        if (!(v[c] < eps2[c])) return 0;
    return 1;
}

/* first column whose denominator is zero or whose quotient is not finite */
static int bad_col(const double* den, const double* q, int m) {
    for (int c = 0; c < m; ++c)
        if ((den && den[c] == 0.0) || !isfinite(q[c])) return c;
    return -1;
}

/* "Lucky" exact convergence: the omega denominator vanishes because the
 * intermediate residual is exactly zero (e.g. A diagonal).
 * omega := 0 then, and the column has res2 = 0; otherwise a zero
 * denominator is a breakdown. */
static int lucky(double den, double sq) { return den == 0.0 && sq == 0.0; }

static int bad_omega(const double* den, const double* sq, const double* om, int m) {
    for (int c = 0; c < m; ++c)
        if ((den[c] == 0.0 && !lucky(den[c], sq[c])) || !isfinite(om[c])) return c;
    return -1;
}

int orc_method_preconditioned(int method) {
    return method == ORC_RBICGSTAB || method == ORC_PBICGSTAB || method == ORC_PPIPEBICGSTAB;
}

/* M^-1: identity = copy; synthetic(alpha) = alpha/2 passes
 * out = c*in, c = 2.0, 0.5, 2.0, ... and a last factor making the product 1. */
static void minv(const shape* S, int alpha, const double* c2, const double* ch, const double* c1,
                 const double* in, double* out) {
    if (alpha <= 2) {
        memcpy(out, in, sizeof(double) * (size_t)S->len);
        return;
    }
    const int k = alpha / 2;
    for (int i = 0; i < k; ++i) {
        const double* c = i < k - 1 ? ((i & 1) ? ch : c2) : (((k - 1) & 1) ? ch : c1);
        const double* src = i == 0 ? in : out;
        orc_update(S->n, S->m, 1, &c, &src, out);
    }
}

int orc_solve(const orc_csr* A, int m, const double* b, double* x, int method,
              int formulation, double tol, int fixed, int maxit, double* hist,
              orc_report* rep) {
    return orc_solve_pc(A, m, b, x, method, formulation, orc_method_preconditioned(method) ? 2 : 0,
                        tol, fixed, maxit, hist, rep);
}

int orc_solve_pc(const orc_csr* A, int m, const double* b, double* x, int method,
                 int formulation, int pa, double tol, int fixed, int maxit, double* hist,
                 orc_report* rep) {
    shape S = {A->n, m, A->n * m};
    if (method < 0 || method > 5) return -1;
    if (orc_method_preconditioned(method) ? (pa < 2 || (pa & 1)) : pa != 0) return -2;
    memset(rep, 0, sizeof *rep);
    double* one = (double*)malloc(sizeof(double) * m);
    double* mone = (double*)malloc(sizeof(double) * m);
    for (int c = 0; c < m; ++c) { one[c] = 1.0; mone[c] = -1.0; }
    double *bb = calloc(m, 8), *eps2 = calloc(m, 8), *rho = calloc(m, 8), *rhon = calloc(m, 8);
    double *alpha = calloc(m, 8), *nalpha = calloc(m, 8), *omega = calloc(m, 8), *nomega = calloc(m, 8);
    double *beta = calloc(m, 8), *nbo = calloc(m, 8), *oa = calloc(m, 8), *delta = calloc(m, 8);
    double *phi = calloc(m, 8), *psi = calloc(m, 8), *theta = calloc(m, 8), *eta = calloc(m, 8);
    double *pi = calloc(m, 8), *sigma = calloc(m, 8), *res2 = calloc(m, 8), *den = calloc(m, 8);
    double *two = calloc(m, 8), *half = calloc(m, 8), *sigmap = calloc(m, 8), *tau = calloc(m, 8);
    double *gam = calloc(m, 8), *kap = calloc(m, 8), *nu = calloc(m, 8), *cz2 = calloc(m, 8);
    double *cz3 = calloc(m, 8), *ndelta = calloc(m, 8);
    for (int c = 0; c < m; ++c) { two[c] = 2.0; half[c] = 0.5; }

    double* r = vnew(&S); double* r0 = vnew(&S); double* tmp = vnew(&S);
    double *p = NULL, *v = NULL, *s = NULL, *t = NULL, *z = NULL, *vh = NULL, *th = NULL;
    double *rt = NULL, *q = NULL, *w = NULL, *y = NULL, *tmp2 = NULL;
    double *u = NULL, *f0 = NULL, *ph = NULL, *sh = NULL, *qh = NULL, *rh = NULL, *wh = NULL, *zh = NULL;
#define MINV(IN, OUT) minv(&S, pa, two, half, one, (IN), (OUT))

    /* r0 = b - A x0 (Alg. 2 line 1-2) */
    orc_spmv(A, m, x, tmp);
    UPD(&S, r, 2, one, b, mone, tmp);
    UPD(&S, r0, 1, one, r);
    orc_dot_exact(S.n, m, b, b, bb);
    orc_dot_exact(S.n, m, r0, r0, rho);
    for (int c = 0; c < m; ++c) {
        eps2[c] = (tol * tol) * bb[c];
        hist[c] = hist_entry(rho[c], bb[c]);
    }
    int it = 0;
    if (!fixed && all_below(rho, eps2, m)) { rep->converged = 1; goto done; }

    if (method == ORC_BICGSTAB) {
        /* Alg. 2; schedule SURVEY.md Appendix C */
        p = vnew(&S); v = vnew(&S); s = vnew(&S); t = vnew(&S);
        UPD(&S, p, 1, one, r);
        for (it = 0; it < maxit; ++it) {
            orc_spmv(A, m, p, v);
            orc_dot_exact(S.n, m, v, r0, delta);
            for (int c = 0; c < m; ++c) { alpha[c] = rho[c] / delta[c]; nalpha[c] = -alpha[c]; }
            int bc = bad_col(delta, alpha, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; break; }
            UPD(&S, s, 2, one, r, nalpha, v);
            orc_spmv(A, m, s, t);
            orc_dot_exact(S.n, m, t, s, phi);
            orc_dot_exact(S.n, m, t, t, psi);
            orc_dot_exact(S.n, m, s, s, theta);
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(psi[c], theta[c]) ? 0.0 : phi[c] / psi[c];
                nomega[c] = -omega[c];
                res2[c] = theta[c] - omega[c] * phi[c];
            }
            bc = bad_omega(psi, theta, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, x, 3, one, x, alpha, p, omega, s);
            UPD(&S, r, 2, one, s, nomega, t);
            if (conv) { rep->converged = 1; ++it; break; }
            orc_dot_exact(S.n, m, r, r0, rhon);
            for (int c = 0; c < m; ++c) {
                beta[c] = (rhon[c] / rho[c]) * (alpha[c] / omega[c]);
                nbo[c] = -(beta[c] * omega[c]);
                rho[c] = rhon[c];
            }
            bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            UPD(&S, p, 3, one, r, beta, p, nbo, v);
        }
    } else if (method == ORC_RBICGSTAB) {
        /* Alg. 6 (identity M^-1), PAPER.md:1562-1598 with the footnote-5 fix */
        z = vnew(&S); vh = vnew(&S); v = vnew(&S); s = vnew(&S); th = vnew(&S);
        t = vnew(&S); rt = vnew(&S); q = vnew(&S);
        MINV(r0, z);                              /* z0 = M^-1 r0 */
        memcpy(vh, z, sizeof(double) * S.len);   /* v^0 = z0 */
        for (it = 0; it < maxit; ++it) {
            orc_spmv(A, m, vh, v);
            orc_dot_exact(S.n, m, v, r0, delta);
            MINV(v, s);                           /* s = M^-1 v */
            for (int c = 0; c < m; ++c) { alpha[c] = rho[c] / delta[c]; nalpha[c] = -alpha[c]; }
            int bc = bad_col(delta, alpha, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; break; }
            UPD(&S, th, 2, one, z, nalpha, s);
            orc_spmv(A, m, th, t);
            UPD(&S, rt, 2, one, r, nalpha, v);
            orc_dot_exact(S.n, m, t, rt, theta);
            orc_dot_exact(S.n, m, t, t, phi);
            orc_dot_exact(S.n, m, t, r0, psi);
            orc_dot_exact(S.n, m, rt, rt, eta);
            MINV(t, q);                           /* q = M^-1 t */
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(phi[c], eta[c]) ? 0.0 : theta[c] / phi[c];
                nomega[c] = -omega[c];
                res2[c] = eta[c] - omega[c] * theta[c];
            }
            bc = bad_omega(phi, eta, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, r, 2, one, rt, nomega, t);
            if (conv) {
                UPD(&S, x, 3, one, x, alpha, vh, omega, th);
                rep->converged = 1; ++it; break;
            }
            for (int c = 0; c < m; ++c) {
                rhon[c] = -(omega[c] * psi[c]);
                beta[c] = (rhon[c] / rho[c]) * (alpha[c] / omega[c]);
                nbo[c] = -(beta[c] * omega[c]);
                rho[c] = rhon[c];
            }
            bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            UPD(&S, x, 3, one, x, alpha, vh, omega, th);
            UPD(&S, z, 2, one, th, nomega, q);
            UPD(&S, vh, 3, one, z, beta, vh, nbo, s);
        }
    } else if (method == ORC_PIPEBICGSTAB) {
        /* Alg. 4 */
        w = vnew(&S); t = vnew(&S); p = vnew(&S); s = vnew(&S); z = vnew(&S);
        v = vnew(&S); q = vnew(&S); y = vnew(&S); tmp2 = vnew(&S);
        orc_spmv(A, m, r, w);
        orc_spmv(A, m, w, t);
        orc_dot_exact(S.n, m, r0, w, den);
        for (int c = 0; c < m; ++c) { alpha[c] = rho[c] / den[c]; beta[c] = 0.0; omega[c] = 0.0; }
        int bc = bad_col(den, alpha, m);
        if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; goto done; }
        for (it = 0; it < maxit; ++it) {
            for (int c = 0; c < m; ++c) { nbo[c] = -(beta[c] * omega[c]); nalpha[c] = -alpha[c]; }
            UPD(&S, p, 3, one, r, beta, p, nbo, s);
            UPD(&S, s, 3, one, w, beta, s, nbo, z);
            UPD(&S, z, 3, one, t, beta, z, nbo, v);
            UPD(&S, q, 2, one, r, nalpha, s);
            UPD(&S, y, 2, one, w, nalpha, z);
            orc_dot_exact(S.n, m, q, y, theta);
            orc_dot_exact(S.n, m, y, y, phi);
            orc_dot_exact(S.n, m, q, q, pi);
            orc_spmv(A, m, z, v);
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(phi[c], pi[c]) ? 0.0 : theta[c] / phi[c];
                nomega[c] = -omega[c];
                oa[c] = omega[c] * alpha[c];
                res2[c] = pi[c] - omega[c] * theta[c];
            }
            bc = bad_omega(phi, pi, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, x, 3, one, x, alpha, p, omega, q);
            UPD(&S, r, 2, one, q, nomega, y);
            if (conv) { rep->converged = 1; ++it; break; }
            if (formulation == ORC_BASIC) {
                /* split_basic peels the trailing pair (statement.cpp:58-85) */
                UPD(&S, tmp2, 2, nomega, t, oa, v);
                UPD(&S, w, 2, one, y, one, tmp2);
            } else {
                UPD(&S, w, 3, one, y, nomega, t, oa, v);
            }
            orc_dot_exact(S.n, m, r0, r, rhon);
            orc_dot_exact(S.n, m, r0, z, psi);
            orc_dot_exact(S.n, m, r0, w, sigma);
            orc_dot_exact(S.n, m, r0, s, delta);
            orc_spmv(A, m, w, t);
            for (int c = 0; c < m; ++c) {
                beta[c] = (alpha[c] / omega[c]) * (rhon[c] / rho[c]);
                den[c] = (sigma[c] + beta[c] * delta[c]) - (beta[c] * omega[c]) * psi[c];
                alpha[c] = rhon[c] / den[c];
                rho[c] = rhon[c];
            }
            bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            bc = bad_col(den, alpha, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; ++it; break; }
        }
    } else if (method == ORC_IBICGSTAB) {
        /* Alg. 3 (merged Improved BiCGStab).  Scalar
         * expression trees (pinned here, mirrored in scalar.cuh):
         *   rho' = (phi - omega*sigma_{j-1}) + (omega*alpha)*pi
         *   delta' = (rho'/rho)*alpha ; beta' = delta'/omega
         *   tau' = (sigma + beta'*tau) - delta'*pi ; alpha' = rho'/tau'
         *   z: coefficients alpha', beta'*(alpha'/alpha), -(alpha'*delta') */
        u = vnew(&S); f0 = vnew(&S); q = vnew(&S); v = vnew(&S); z = vnew(&S); s = vnew(&S); t = vnew(&S);
        orc_spmv(A, m, r, u);                  /* u0 = A r0 */
        orc_spmv_transpose(A, m, r0, f0);      /* f0 = A^T r0 */
        orc_dot_exact(S.n, m, r0, u, sigma);   /* sigma_0 = (r0, u0) */
        for (int c = 0; c < m; ++c) {
            phi[c] = rho[c];                   /* phi_0 = (r0, r0) */
            sigmap[c] = 0.0; pi[c] = 0.0; tau[c] = 0.0;
            rho[c] = 1.0; alpha[c] = 1.0; omega[c] = 1.0;
        }
        for (it = 0; it < maxit; ++it) {
            double* an = den;                  /* alpha_{j+1} */
            for (int c = 0; c < m; ++c) {
                rhon[c] = (phi[c] - omega[c] * sigmap[c]) + (omega[c] * alpha[c]) * pi[c];
                delta[c] = (rhon[c] / rho[c]) * alpha[c];
                beta[c] = delta[c] / omega[c];
                tau[c] = (sigma[c] + beta[c] * tau[c]) - delta[c] * pi[c];
                an[c] = rhon[c] / tau[c];
            }
            int bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            bc = bad_col(tau, an, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) {
                cz2[c] = beta[c] * (an[c] / alpha[c]);
                cz3[c] = -(an[c] * delta[c]);
                ndelta[c] = -delta[c];
                alpha[c] = an[c];
                nalpha[c] = -an[c];
                rho[c] = rhon[c];
            }
            UPD(&S, z, 3, alpha, r, cz2, z, cz3, v);
            UPD(&S, v, 3, one, u, beta, v, ndelta, q);
            UPD(&S, s, 2, one, r, nalpha, v);
            orc_spmv(A, m, v, q);
            UPD(&S, t, 2, one, u, nalpha, q);
            orc_dot_exact(S.n, m, r0, s, phi);
            orc_dot_exact(S.n, m, r0, q, pi);
            orc_dot_exact(S.n, m, f0, s, gam);
            orc_dot_exact(S.n, m, f0, t, eta);
            orc_dot_exact(S.n, m, s, t, theta);
            orc_dot_exact(S.n, m, t, t, kap);
            orc_dot_exact(S.n, m, s, s, nu);
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(kap[c], nu[c]) ? 0.0 : theta[c] / kap[c];
                nomega[c] = -omega[c];
                res2[c] = nu[c] - omega[c] * theta[c];
            }
            bc = bad_omega(kap, nu, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) {
                sigmap[c] = sigma[c];
                sigma[c] = gam[c] - omega[c] * eta[c];
                hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            }
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, r, 2, one, s, nomega, t);
            UPD(&S, x, 3, one, x, one, z, omega, s);
            if (conv) { rep->converged = 1; ++it; break; }
            orc_spmv(A, m, r, u);
        }
    } else if (method == ORC_PBICGSTAB) {
        /* Alg. 5 (merged preconditioned BiCGStab).  The x
         * update (independent of beta) runs before beta is formed. */
        p = vnew(&S); v = vnew(&S); s = vnew(&S); t = vnew(&S); ph = vnew(&S); sh = vnew(&S);
        UPD(&S, p, 1, one, r);
        for (it = 0; it < maxit; ++it) {
            MINV(p, ph);
            orc_spmv(A, m, ph, v);
            orc_dot_exact(S.n, m, v, r0, delta);
            for (int c = 0; c < m; ++c) { alpha[c] = rho[c] / delta[c]; nalpha[c] = -alpha[c]; }
            int bc = bad_col(delta, alpha, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; break; }
            UPD(&S, s, 2, one, r, nalpha, v);
            MINV(s, sh);
            orc_spmv(A, m, sh, t);
            orc_dot_exact(S.n, m, t, s, phi);
            orc_dot_exact(S.n, m, t, t, psi);
            orc_dot_exact(S.n, m, s, s, theta);
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(psi[c], theta[c]) ? 0.0 : phi[c] / psi[c];
                nomega[c] = -omega[c];
                res2[c] = theta[c] - omega[c] * phi[c];
            }
            bc = bad_omega(psi, theta, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, r, 2, one, s, nomega, t);
            UPD(&S, x, 3, one, x, alpha, ph, omega, sh);
            if (conv) { rep->converged = 1; ++it; break; }
            orc_dot_exact(S.n, m, r, r0, rhon);
            for (int c = 0; c < m; ++c) {
                beta[c] = (rhon[c] / rho[c]) * (alpha[c] / omega[c]);
                nbo[c] = -(beta[c] * omega[c]);
                rho[c] = rhon[c];
            }
            bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            UPD(&S, p, 3, one, r, beta, p, nbo, v);
        }
    } else if (method == ORC_PPIPEBICGSTAB) {
        /* Alg. 7 (merged preconditioned Pipelined BiCGStab)
         * (line 1: w^_0 = M^-1 w_0).  Expansions as Alg. 4. */
        rh = vnew(&S); w = vnew(&S); wh = vnew(&S); t = vnew(&S); ph = vnew(&S); sh = vnew(&S);
        qh = vnew(&S); s = vnew(&S); z = vnew(&S); q = vnew(&S); y = vnew(&S); zh = vnew(&S);
        v = vnew(&S); tmp2 = vnew(&S);
        MINV(r, rh);
        orc_spmv(A, m, rh, w);
        MINV(w, wh);
        orc_spmv(A, m, wh, t);
        orc_dot_exact(S.n, m, r0, w, den);
        for (int c = 0; c < m; ++c) { alpha[c] = rho[c] / den[c]; beta[c] = 0.0; omega[c] = 0.0; }
        int bc = bad_col(den, alpha, m);
        if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; goto done; }
        for (it = 0; it < maxit; ++it) {
            for (int c = 0; c < m; ++c) { nbo[c] = -(beta[c] * omega[c]); nalpha[c] = -alpha[c]; }
            UPD(&S, ph, 3, one, rh, beta, ph, nbo, sh);
            UPD(&S, sh, 3, one, wh, beta, sh, nbo, zh);
            UPD(&S, qh, 2, one, rh, nalpha, sh);
            UPD(&S, s, 3, one, w, beta, s, nbo, z);
            UPD(&S, z, 3, one, t, beta, z, nbo, v);
            UPD(&S, q, 2, one, r, nalpha, s);
            UPD(&S, y, 2, one, w, nalpha, z);
            orc_dot_exact(S.n, m, q, y, theta);
            orc_dot_exact(S.n, m, y, y, phi);
            orc_dot_exact(S.n, m, q, q, pi);
            MINV(z, zh);
            orc_spmv(A, m, zh, v);
            for (int c = 0; c < m; ++c) {
                omega[c] = lucky(phi[c], pi[c]) ? 0.0 : theta[c] / phi[c];
                nomega[c] = -omega[c];
                oa[c] = omega[c] * alpha[c];
                res2[c] = pi[c] - omega[c] * theta[c];
            }
            bc = bad_omega(phi, pi, omega, m);
            if (bc >= 0) { rep->breakdown = 2; rep->breakdown_col = bc; break; }
            for (int c = 0; c < m; ++c) hist[(int64_t)(it + 1) * m + c] = hist_entry(res2[c], bb[c]);
            const int conv = !fixed && all_below(res2, eps2, m);
            UPD(&S, x, 3, one, x, alpha, ph, omega, qh);
            if (conv) {
                UPD(&S, r, 2, one, q, nomega, y);
                rep->converged = 1; ++it; break;
            }
            if (formulation == ORC_BASIC) {
                UPD(&S, tmp2, 2, nomega, wh, oa, zh);
                UPD(&S, rh, 2, one, qh, one, tmp2);
            } else {
                UPD(&S, rh, 3, one, qh, nomega, wh, oa, zh);
            }
            UPD(&S, r, 2, one, q, nomega, y);
            if (formulation == ORC_BASIC) {
                UPD(&S, tmp2, 2, nomega, t, oa, v);
                UPD(&S, w, 2, one, y, one, tmp2);
            } else {
                UPD(&S, w, 3, one, y, nomega, t, oa, v);
            }
            orc_dot_exact(S.n, m, r0, r, rhon);
            orc_dot_exact(S.n, m, r0, z, psi);
            orc_dot_exact(S.n, m, r0, w, sigma);
            orc_dot_exact(S.n, m, r0, s, delta);
            MINV(w, wh);
            orc_spmv(A, m, wh, t);
            for (int c = 0; c < m; ++c) {
                beta[c] = (alpha[c] / omega[c]) * (rhon[c] / rho[c]);
                den[c] = (sigma[c] + beta[c] * delta[c]) - (beta[c] * omega[c]) * psi[c];
                alpha[c] = rhon[c] / den[c];
                rho[c] = rhon[c];
            }
            bc = bad_col(NULL, beta, m);
            if (bc >= 0) { rep->breakdown = 3; rep->breakdown_col = bc; break; }
            bc = bad_col(den, alpha, m);
            if (bc >= 0) { rep->breakdown = 1; rep->breakdown_col = bc; ++it; break; }
        }
    } else {
        it = -1;
    }
done:
    if (rep->breakdown) rep->breakdown_iter = it;
    rep->iterations = it < 0 ? 0 : it;
    free(one); free(mone); free(bb); free(eps2); free(rho); free(rhon); free(alpha); free(nalpha);
    free(omega); free(nomega); free(beta); free(nbo); free(oa); free(delta); free(phi); free(psi);
    free(theta); free(eta); free(pi); free(sigma); free(res2); free(den);
    free(r); free(r0); free(tmp); free(p); free(v); free(s); free(t); free(z); free(vh); free(th);
    free(rt); free(q); free(w); free(y); free(tmp2);
    free(two); free(half); free(sigmap); free(tau); free(gam); free(kap); free(nu); free(cz2); free(cz3);
    free(ndelta); free(u); free(f0); free(ph); free(sh); free(qh); free(rh); free(wh); free(zh);
#undef MINV
    return 0;
}
