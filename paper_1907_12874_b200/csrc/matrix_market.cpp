// matrix_market.cpp -- MatrixMarket ingest:
// coordinate real/integer, general/symmetric files -> host CSR that the
// device upload (and, for several GPUs, the general halo plan of plan.cpp)
// takes as is.
//
// Contract of core::read_matrix_market (proj/src/core/matrix_market.cpp:38-113,
// SPEC.md:83-91): banner / object / format / field / symmetry checks with the
// reference's "<name>:<line>: message" errors, square matrices only,
// symmetric files expanded to full storage, duplicate entries summed, rows
// sorted by column.  Duplicates are summed from 0.0 in FILE order (the
// reference sorts with the unstable std::sort, so its order for duplicates is
// unspecified; for distinct (row, col) pairs the two readers agree bit for bit).
//
// Built for large inputs: the file is read in one go and the entry lines are
// parsed by all host threads (std::from_chars), then bucketed by row with a
// stable counting sort -- no per-entry iostream and no global comparison sort.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"

namespace mbg {
namespace {

struct ParseError {
    int64_t line;
    std::string msg;
};

struct Triplet {
    int64_t row, col;
    double val;
};

std::string lower(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

const char* skip_ws(const char* p, const char* e) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    return p;
}

template <class T>
bool num(const char*& p, const char* e, T& out) {
    p = skip_ws(p, e);
    if (p < e && *p == '+') ++p;   // from_chars rejects a leading '+', istream accepts it
    auto r = std::from_chars(p, e, out);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
}

}  // namespace

struct MMatrix {
    int64_t n = 0;
    std::vector<int64_t> off;
    std::vector<int32_t> col;
    std::vector<double> val;
};

MMatrix read_matrix_market_text(const char* data, size_t size, const std::string& name) {
    const char* const end = data + size;
    auto fail = [&](int64_t line, const std::string& msg) -> void {
        throw std::runtime_error(name + ":" + std::to_string(line) + ": " + msg);
    };
    auto next_line = [&](const char*& p, const char*& le) -> bool {
        if (p >= end) return false;
        le = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        if (!le) le = end;
        return true;
    };
    const char* p = data;
    const char* le = nullptr;
    int64_t line_no = 1;
    if (!next_line(p, le)) fail(line_no, "empty file");
    bool symmetric = false;
    {
        std::string header(p, le);
        char b[64] = {0}, o[64] = {0}, f[64] = {0}, fl[64] = {0}, sy[64] = {0};
        std::sscanf(header.c_str(), "%63s %63s %63s %63s %63s", b, o, f, fl, sy);
        if (std::string(b) != "%%MatrixMarket") fail(line_no, "missing %%MatrixMarket banner");
        if (lower(o) != "matrix") fail(line_no, "object must be 'matrix'");
        if (lower(f) != "coordinate") fail(line_no, "only coordinate format supported");
        const std::string field = lower(fl);
        if (field != "real" && field != "integer") fail(line_no, "field must be 'real' or 'integer'");
        const std::string sym = lower(sy);
        symmetric = sym == "symmetric";
        if (!symmetric && sym != "general") fail(line_no, "symmetry must be 'general' or 'symmetric'");
        p = le + 1;
    }
    int64_t nr = 0, nc = 0, ne = 0;
    for (;;) {  // comments and empty lines up to the size line
        if (!next_line(p, le)) fail(line_no, "missing size line");
        ++line_no;
        if (p == le || *p == '%') {
            p = le + 1;
            continue;
        }
        const char* q = p;
        if (!num(q, le, nr) || !num(q, le, nc) || !num(q, le, ne)) fail(line_no, "malformed size line");
        p = le + 1;
        break;
    }
    if (nr != nc) fail(line_no, "matrix must be square");
    if (nr < 1) fail(line_no, "matrix must have at least one row");
    if (nr > INT32_MAX) fail(line_no, "matrix too large for 32-bit column indices");

    // split the remaining text into per-thread chunks at line boundaries
    const char* body = p < end ? p : end;
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<const char*> cut(nt + 1, end);
    cut[0] = body;
    for (unsigned t = 1; t < nt; ++t) {
        const char* c = body + (end - body) * static_cast<int64_t>(t) / nt;
        if (c < cut[t - 1]) c = cut[t - 1];
        const char* nl = c < end ? static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(end - c))) : nullptr;
        cut[t] = nl ? nl + 1 : end;
    }
    struct Chunk {
        std::vector<Triplet> ent;
        int64_t lines = 0;            // lines scanned
        int64_t entries = 0;          // entry lines seen (including a malformed one)
        int64_t bad_line = -1;        // local line index of the first error
        int64_t bad_entry = -1;       // its entry index within the chunk
        std::string bad_msg;
    };
    std::vector<Chunk> ch(nt);
    auto work = [&](unsigned t) {
        Chunk& c = ch[t];
        const char* q = cut[t];
        const char* e = cut[t + 1];
        while (q < e) {
            const char* l = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(e - q)));
            if (!l) l = e;
            if (q < l && *q != '%') {   // the reference skips empty and comment lines only
                int64_t i = 0, j = 0;
                double v = 0.0;
                const char* r = q;
                const char* msg = nullptr;
                if (!num(r, l, i) || !num(r, l, j) || !num(r, l, v)) msg = "malformed entry";
                else if (i < 1 || i > nr || j < 1 || j > nc) msg = "entry index out of range";
                if (msg) {
                    if (c.bad_line < 0) {
                        c.bad_line = c.lines;
                        c.bad_entry = c.entries;
                        c.bad_msg = msg;
                    }
                } else if (c.bad_line < 0) {
                    c.ent.push_back({i - 1, j - 1, v});
                }
                ++c.entries;
            }
            ++c.lines;
            q = l + 1;
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& x : th) x.join();
    }
    // first error among the first ne entry lines, in file order; else EOF check
    int64_t seen = 0, lines_before = line_no;
    bool enough = false;
    for (unsigned t = 0; t < nt && !enough; ++t) {
        if (ch[t].bad_line >= 0 && seen + ch[t].bad_entry < ne)
            fail(lines_before + ch[t].bad_line + 1, ch[t].bad_msg);
        if (seen + ch[t].entries >= ne) {
            enough = true;
        } else {
            seen += ch[t].entries;
            lines_before += ch[t].lines;
        }
    }
    if (!enough) fail(lines_before, "unexpected end of file");

    // keep the first ne entries (file order), expand symmetric ones
    std::vector<int64_t> cnt(static_cast<size_t>(nr) + 1, 0);
    int64_t left = ne;
    for (auto& c : ch) {
        const int64_t take = std::min<int64_t>(left, static_cast<int64_t>(c.ent.size()));
        c.ent.resize(static_cast<size_t>(take));
        left -= take;
        for (const auto& e : c.ent) {
            ++cnt[e.row + 1];
            if (symmetric && e.row != e.col) ++cnt[e.col + 1];
        }
    }
    for (int64_t i = 0; i < nr; ++i) cnt[i + 1] += cnt[i];
    std::vector<int32_t> tcol(static_cast<size_t>(cnt[nr]));
    std::vector<double> tval(static_cast<size_t>(cnt[nr]));
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (const auto& c : ch)
        for (const auto& e : c.ent) {
            int64_t k = pos[e.row]++;
            tcol[k] = static_cast<int32_t>(e.col);
            tval[k] = e.val;
            if (symmetric && e.row != e.col) {
                k = pos[e.col]++;
                tcol[k] = static_cast<int32_t>(e.row);
                tval[k] = e.val;
            }
        }
    // per row: stable sort by column, sum duplicates (file order) from 0.0
    MMatrix out;
    out.n = nr;
    out.off.assign(static_cast<size_t>(nr) + 1, 0);
    std::vector<int64_t> rowlen(static_cast<size_t>(nr), 0);
    auto rows = [&](int64_t r0, int64_t r1) {
        std::vector<int64_t> idx;
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t b = cnt[r], e = cnt[r + 1];
            idx.resize(static_cast<size_t>(e - b));
            for (int64_t k = b; k < e; ++k) idx[k - b] = k;
            std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return tcol[x] < tcol[y]; });
            // write compacted (col, sum) back in place over [b, ...)
            std::vector<std::pair<int32_t, double>> tmp;
            tmp.reserve(idx.size());
            for (size_t a = 0; a < idx.size();) {
                const int32_t c = tcol[idx[a]];
                double s = 0.0;
                while (a < idx.size() && tcol[idx[a]] == c) s = s + tval[idx[a++]];
                tmp.emplace_back(c, s);
            }
            for (size_t a = 0; a < tmp.size(); ++a) {
                tcol[b + static_cast<int64_t>(a)] = tmp[a].first;
                tval[b + static_cast<int64_t>(a)] = tmp[a].second;
            }
            rowlen[r] = static_cast<int64_t>(tmp.size());
        }
    };
    {
        std::vector<std::thread> th;
        const int64_t per = (nr + nt - 1) / nt;
        for (unsigned t = 1; t < nt; ++t)
            if (static_cast<int64_t>(t) * per < nr)
                th.emplace_back(rows, static_cast<int64_t>(t) * per, std::min<int64_t>(nr, (t + 1) * per));
        rows(0, std::min<int64_t>(nr, per));
        for (auto& x : th) x.join();
    }
    for (int64_t r = 0; r < nr; ++r) out.off[r + 1] = out.off[r] + rowlen[r];
    out.col.resize(static_cast<size_t>(out.off[nr]));
    out.val.resize(static_cast<size_t>(out.off[nr]));
    for (int64_t r = 0; r < nr; ++r) {
        std::memcpy(out.col.data() + out.off[r], tcol.data() + cnt[r], static_cast<size_t>(rowlen[r]) * 4);
        std::memcpy(out.val.data() + out.off[r], tval.data() + cnt[r], static_cast<size_t>(rowlen[r]) * 8);
    }
    if (out.off[nr] > INT32_MAX - 64) fail(line_no, "nnz >= 2^31 is not supported");
    return out;
}

MMatrix read_matrix_market_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw std::runtime_error(path + ": cannot open file");
    const std::streamsize sz = in.tellg();
    in.seekg(0);
    std::string buf(static_cast<size_t>(sz > 0 ? sz : 0), '\0');
    if (sz > 0 && !in.read(buf.data(), sz)) throw std::runtime_error(path + ": read error");
    return read_matrix_market_text(buf.data(), buf.size(), path);
}

}  // namespace mbg

// ---- C ABI ---------------------------------------------------------------------
extern "C" int mbg_mm_read(const char* path, void** handle, int64_t* n, int64_t* nnz) {
    try {
        if (!path || !handle) throw mbg::Invalid("mm_read: null argument");
        auto m = std::make_unique<mbg::MMatrix>(mbg::read_matrix_market_file(path));
        if (n) *n = m->n;
        if (nnz) *nnz = m->off.back();
        *handle = m.release();
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}

extern "C" int mbg_mm_copy(const void* handle, int64_t* offsets, int32_t* cols, double* vals) {
    if (!handle) {
        mbg::set_error("mm_copy: null handle");
        return MBG_ERR_INVALID;
    }
    const auto* m = static_cast<const mbg::MMatrix*>(handle);
    if (offsets) std::memcpy(offsets, m->off.data(), m->off.size() * sizeof(int64_t));
    if (cols) std::memcpy(cols, m->col.data(), m->col.size() * sizeof(int32_t));
    if (vals) std::memcpy(vals, m->val.data(), m->val.size() * sizeof(double));
    return MBG_OK;
}

extern "C" void mbg_mm_free(void* handle) { delete static_cast<mbg::MMatrix*>(handle); }

extern "C" int mbg_mm_write(const char* path, int64_t n, const int64_t* off, const int32_t* col,
                            const double* val) {
    try {
        if (!path || !off) throw mbg::Invalid("mm_write: null argument");
        FILE* f = std::fopen(path, "w");
        if (!f) throw std::runtime_error(std::string(path) + ": cannot open file for writing");
        std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
        std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(n), static_cast<long long>(n),
                     static_cast<long long>(off[n]));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = off[i]; k < off[i + 1]; ++k)
                std::fprintf(f, "%lld %d %.17g\n", static_cast<long long>(i + 1), col[k] + 1, val[k]);
        if (std::fclose(f) != 0) throw std::runtime_error(std::string(path) + ": write error");
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        mbg::set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}
