// generators.cpp -- the BASELINE.json config matrices and right-hand sides.
//
// gen_poisson_7pt restates generators.cpp:37-67 of the reference (lexicographic
// rows, x fastest, ascending columns, constant diagonal 6, off-diagonals -1).
// The convection-diffusion, 27-point and random banded matrices and the RHS
// are the BASELINE.json configs with the pins of SURVEY.md Appendix A and
// DESIGN.md "Inputs" (counter-based RNG keyed by (seed, stream, row, col), so
// any partition or column subset regenerates identical values).  The CPU
// oracle (oracle/oracle.c) implements the same pins independently; tests
// compare the two bit for bit.
#include <algorithm>
#include <climits>
#include <cmath>
#include <thread>
#include <vector>

#include "common.hpp"

namespace mbg {
namespace {

uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27; z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ull));
    h = mix64(h + a * 0xD1B54A32D192ED03ull + 0x9E3779B97F4A7C15ull);
    h = mix64(h + b * 0x8CB92BA72F3D8DD7ull + 0x9E3779B97F4A7C15ull);
    return h;
}

double u01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return static_cast<double>(hash4(seed, stream, a, b) >> 11) * 0x1.0p-53;
}
double u11(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return 2.0 * u01(seed, stream, a, b) - 1.0;
}

enum : uint64_t { ST_RHS = 1, ST_MAT = 2, ST_CNT = 3, ST_COL = 4, ST_VAL = 5 };

template <class F>
void parallel_rows(int64_t n, F&& f) {
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    if (n < 65536) nt = 1;
    std::vector<std::thread> pool;
    const int64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const int64_t b = std::min<int64_t>(n, t * chunk), e = std::min<int64_t>(n, b + chunk);
        if (b >= e) continue;
        pool.emplace_back([&f, b, e] { for (int64_t i = b; i < e; ++i) f(i); });
    }
    for (auto& th : pool) th.join();
}

int stencil_count(int kind, int nx, int ny, int nz, int64_t row) {
    const int x = static_cast<int>(row % nx);
    const int y = static_cast<int>((row / nx) % ny);
    const int z = static_cast<int>(row / (static_cast<int64_t>(nx) * ny));
    if (kind == 2)
        return (1 + (x > 0) + (x < nx - 1)) * (1 + (y > 0) + (y < ny - 1)) * (1 + (z > 0) + (z < nz - 1));
    return 1 + (x > 0) + (x < nx - 1) + (y > 0) + (y < ny - 1) + (z > 0) + (z < nz - 1);
}

}  // namespace
}  // namespace mbg

extern "C" int mbg_gen_stencil(int kind, int nx, int ny, int nz, uint64_t seed, int64_t* nnz,
                               int64_t* off, int32_t* col, double* val) {
    using namespace mbg;
    try {
        if (kind < 0 || kind > 3) throw Invalid("gen_stencil: unknown kind");
        if (kind == 3 && nz != 1) throw Invalid("gen_stencil: the 5-point Poisson operator is 2-D (nz = 1)");
        if (nx < 1 || ny < 1 || nz < 1) throw Invalid("grid dimensions must be >= 1");
        const int64_t n = static_cast<int64_t>(nx) * ny * nz;
        if (n > INT32_MAX) throw Invalid("grid dimension overflow");
        const int64_t plane = static_cast<int64_t>(nx) * ny;
        std::vector<int64_t> own;
        int64_t* o = off;
        if (!o) { own.resize(n + 1); o = own.data(); }
        o[0] = 0;
        for (int64_t i = 0; i < n; ++i) o[i + 1] = o[i] + stencil_count(kind, nx, ny, nz, i);
        *nnz = o[n];
        if (!col || !val) return MBG_OK;
        parallel_rows(n, [&](int64_t row) {
            const int x = static_cast<int>(row % nx);
            const int y = static_cast<int>((row / nx) % ny);
            const int z = static_cast<int>(row / plane);
            int64_t k = o[row];
            if (kind == 2) {
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (z + dz < 0 || z + dz >= nz || y + dy < 0 || y + dy >= ny || x + dx < 0 ||
                                x + dx >= nx)
                                continue;
                            const int64_t c = row + dz * plane + static_cast<int64_t>(dy) * nx + dx;
                            col[k] = static_cast<int32_t>(c);
                            val[k] = c == row ? 26.0 : -1.0 + 0.1 * u11(seed, ST_MAT, row, c);
                            ++k;
                        }
            } else {
                const double west = kind == 1 ? -1.3 : -1.0, east = kind == 1 ? -0.7 : -1.0;
                auto put = [&](int64_t c, double v) { col[k] = static_cast<int32_t>(c); val[k] = v; ++k; };
                if (z > 0) put(row - plane, -1.0);
                if (y > 0) put(row - nx, -1.0);
                if (x > 0) put(row - 1, west);
                put(row, kind == 3 ? 4.0 : 6.0);   // kind 3: gen_poisson_5pt (generators.cpp:69-91)
                if (x < nx - 1) put(row + 1, east);
                if (y < ny - 1) put(row + nx, -1.0);
                if (z < nz - 1) put(row + plane, -1.0);
            }
        });
        return MBG_OK;
    } catch (const Invalid& e) {
        set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

extern "C" int mbg_gen_banded(int64_t n, int64_t band, int kmin, int kmax, uint64_t seed, int64_t* nnz,
                              int64_t* off, int32_t* col, double* val) {
    using namespace mbg;
    try {
        if (n < 1 || n > INT32_MAX || kmin < 1 || kmax < kmin || band < 0) throw Invalid("gen_banded: bad arguments");
        auto count = [&](int64_t i) {
            int k = kmin + static_cast<int>(hash4(seed, ST_CNT, i, 0) % static_cast<uint64_t>(kmax - kmin + 1));
            const int64_t lo = std::max<int64_t>(0, i - band), hi = std::min<int64_t>(n - 1, i + band);
            if (k - 1 > hi - lo) k = static_cast<int>(hi - lo) + 1;
            return k;
        };
        std::vector<int64_t> own;
        int64_t* o = off;
        if (!o) { own.resize(n + 1); o = own.data(); }
        o[0] = 0;
        for (int64_t i = 0; i < n; ++i) o[i + 1] = o[i] + count(i);
        *nnz = o[n];
        if (!col || !val) return MBG_OK;
        parallel_rows(n, [&](int64_t i) {
            const int64_t lo = std::max<int64_t>(0, i - band), hi = std::min<int64_t>(n - 1, i + band);
            const uint64_t width = static_cast<uint64_t>(hi - lo + 1);
            const int k = static_cast<int>(o[i + 1] - o[i]);
            int32_t* cs = col + o[i];
            double* vs = val + o[i];
            int have = 0;
            cs[have++] = static_cast<int32_t>(i);
            for (uint64_t j = 0; have < k; ++j) {
                const int32_t c = static_cast<int32_t>(lo + static_cast<int64_t>(hash4(seed, ST_COL, i, j) % width));
                if (std::find(cs, cs + have, c) == cs + have) cs[have++] = c;
            }
            std::sort(cs, cs + k);
            double s = 0.0;
            int diag = 0;
            for (int t = 0; t < k; ++t) {
                if (cs[t] == static_cast<int32_t>(i)) { diag = t; continue; }
                vs[t] = -u01(seed, ST_VAL, i, static_cast<uint64_t>(cs[t]));
                s = s + std::fabs(vs[t]);
            }
            vs[diag] = 1.1 * s;
        });
        return MBG_OK;
    } catch (const Invalid& e) {
        set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

extern "C" int mbg_gen_rhs(int64_t n, int m, uint64_t seed, double* b) {
    using namespace mbg;
    if (n < 0 || m < 1 || !b) { set_error("gen_rhs: bad arguments"); return MBG_ERR_INVALID; }
    parallel_rows(n, [&](int64_t i) {
        for (int c = 0; c < m; ++c) b[i * m + c] = u11(seed, ST_RHS, i, c);
    });
    return MBG_OK;
}
