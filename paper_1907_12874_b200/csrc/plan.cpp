// plan.cpp -- row partition and halo plan for the distributed SpMM.
//
// The paper distributes contiguous row blocks across processes (Fig. 1,
// PAPER.md:60-78) and exchanges the boundary rows of the vector before each
// SpMV; the reference only models this analytically
// (SPEC.md:112).  This is the executable plan: local CSR renumbered to
// [owned rows | halo rows], per-peer send lists and receive windows, and the
// interior / boundary row split used to overlap the exchange.
#include <algorithm>
#include <limits>

#include "comm.hpp"

namespace mbg {

HaloPlan build_halo_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val,
                         int nparts, const int64_t* begin, int my) {
    if (nparts < 1 || my < 0 || my >= nparts) throw Invalid("partition: bad part index");
    if (begin[0] != 0 || begin[nparts] != n) throw Invalid("partition: bounds must cover [0, n)");
    for (int p = 0; p < nparts; ++p)
        if (begin[p] > begin[p + 1]) throw Invalid("partition: bounds must be non-decreasing");
    const int64_t rb = begin[my], re = begin[my + 1];
    HaloPlan pl;
    pl.n_own = re - rb;
    const int64_t nnz = off[re] - off[rb];
    if (nnz > std::numeric_limits<int32_t>::max()) throw Invalid("partition: local nnz exceeds int32");

    std::vector<int64_t> halo;
    for (int64_t i = rb; i < re; ++i)
        for (int64_t k = off[i]; k < off[i + 1]; ++k) {
            const int64_t g = col[k];
            if (g < rb || g >= re) halo.push_back(g);
        }
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
    pl.n_halo = static_cast<int64_t>(halo.size());
    pl.halo_global = halo;
    if (pl.n_own + pl.n_halo > std::numeric_limits<int32_t>::max())
        throw Invalid("partition: local rows exceed int32");

    pl.nnz = nnz;
    pl.off.resize(pl.n_own + 1);
    pl.col.resize(nnz);
    pl.val.assign(val + off[rb], val + off[re]);
    pl.off[0] = 0;
    for (int64_t i = rb; i < re; ++i) {
        bool bnd = false;
        for (int64_t k = off[i]; k < off[i + 1]; ++k) {
            const int64_t g = col[k];
            int64_t l;
            if (g >= rb && g < re) {
                l = g - rb;
            } else {
                l = pl.n_own + (std::lower_bound(halo.begin(), halo.end(), g) - halo.begin());
                bnd = true;
            }
            pl.col[k - off[rb]] = static_cast<int32_t>(l);
        }
        pl.off[i - rb + 1] = static_cast<int32_t>(off[i + 1] - off[rb]);
        (bnd ? pl.boundary : pl.interior).push_back(static_cast<int32_t>(i - rb));
    }

    // Local numbering note: owned columns keep their relative order and halo
    // columns are appended, so a row's column list may no longer be sorted in
    // local numbering -- the nonzeros keep their global CSR order, which is
    // what fixes the summation order (spmv.cpp:40-46).
    for (int q = 0; q < nparts; ++q) {
        if (q == my) continue;
        HaloPlan::Peer peer;
        peer.part = q;
        const int64_t qb = begin[q], qe = begin[q + 1];
        auto lo = std::lower_bound(halo.begin(), halo.end(), qb);
        auto hi = std::lower_bound(halo.begin(), halo.end(), qe);
        peer.recv_offset = lo - halo.begin();
        peer.recv_count = hi - lo;
        std::vector<int64_t> need;
        for (int64_t i = qb; i < qe; ++i)
            for (int64_t k = off[i]; k < off[i + 1]; ++k) {
                const int64_t g = col[k];
                if (g >= rb && g < re) need.push_back(g);
            }
        std::sort(need.begin(), need.end());
        need.erase(std::unique(need.begin(), need.end()), need.end());
        for (int64_t g : need) peer.send_rows.push_back(static_cast<int32_t>(g - rb));
        if (peer.recv_count || !peer.send_rows.empty()) pl.peers.push_back(std::move(peer));
    }
    return pl;
}

// Halo plan of A^T for the same row partition (IBiCGStab's f0 = A^T r0,
// PAPER.md:1441-1447, across ranks).  Row j of A^T lists the nonzeros A(i, j)
// in ascending source row i -- the summation order of spmv_transpose
// (spmv.cpp:76-90) -- so the ordinary distributed SpMM on this operator
// reproduces the reference bit for bit.  Its halo is the rows i of other
// ranks that couple to an owned column j; built from the full host CSR in
// one O(nnz) pass, without forming the global transpose.
HaloPlan build_transpose_plan(int64_t n, const int64_t* off, const int32_t* col, const double* val, int nparts,
                              const int64_t* begin, int my) {
    if (nparts < 1 || my < 0 || my >= nparts) throw Invalid("partition: bad part index");
    const int64_t rb = begin[my], re = begin[my + 1];
    HaloPlan pl;
    pl.n_own = re - rb;
    // pass 1: row lengths of the local A^T and the halo source rows
    std::vector<int64_t> len(static_cast<size_t>(pl.n_own), 0);
    std::vector<int64_t> halo;
    for (int64_t i = 0; i < n; ++i) {
        bool touches = false;
        for (int64_t k = off[i]; k < off[i + 1]; ++k) {
            const int64_t j = col[k];
            if (j >= rb && j < re) {
                ++len[j - rb];
                touches = true;
            }
        }
        if (touches && (i < rb || i >= re)) halo.push_back(i);   // ascending already
    }
    pl.n_halo = static_cast<int64_t>(halo.size());
    pl.halo_global = halo;
    int64_t nnz = 0;
    for (int64_t v : len) nnz += v;
    if (nnz > std::numeric_limits<int32_t>::max() || pl.n_own + pl.n_halo > std::numeric_limits<int32_t>::max())
        throw Invalid("partition: local transpose exceeds int32");
    pl.nnz = nnz;
    pl.off.assign(static_cast<size_t>(pl.n_own) + 1, 0);
    for (int64_t j = 0; j < pl.n_own; ++j) pl.off[j + 1] = pl.off[j] + static_cast<int32_t>(len[j]);
    pl.col.resize(static_cast<size_t>(nnz));
    pl.val.resize(static_cast<size_t>(nnz));
    // pass 2: fill in ascending source row order
    std::vector<int32_t> pos(pl.off.begin(), pl.off.end() - 1);
    std::vector<char> bnd(static_cast<size_t>(pl.n_own), 0);
    size_t hcur = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t li;
        const bool own = i >= rb && i < re;
        if (own) {
            li = static_cast<int32_t>(i - rb);
        } else {
            while (hcur < halo.size() && halo[hcur] < i) ++hcur;
            li = (hcur < halo.size() && halo[hcur] == i) ? static_cast<int32_t>(pl.n_own + hcur) : -1;
        }
        for (int64_t k = off[i]; k < off[i + 1]; ++k) {
            const int64_t j = col[k];
            if (j < rb || j >= re) continue;
            const int32_t q = pos[j - rb]++;
            pl.col[q] = li;
            pl.val[q] = val[k];
            if (!own) bnd[j - rb] = 1;
        }
    }
    for (int64_t j = 0; j < pl.n_own; ++j) (bnd[j] ? pl.boundary : pl.interior).push_back(static_cast<int32_t>(j));
    // peers: receive the halo rows owned by q; send my rows i with a nonzero in q's columns
    for (int q = 0; q < nparts; ++q) {
        if (q == my) continue;
        HaloPlan::Peer peer;
        peer.part = q;
        const int64_t qb = begin[q], qe = begin[q + 1];
        auto lo = std::lower_bound(halo.begin(), halo.end(), qb);
        auto hi = std::lower_bound(halo.begin(), halo.end(), qe);
        peer.recv_offset = lo - halo.begin();
        peer.recv_count = hi - lo;
        for (int64_t i = rb; i < re; ++i)
            for (int64_t k = off[i]; k < off[i + 1]; ++k)
                if (col[k] >= qb && col[k] < qe) {
                    peer.send_rows.push_back(static_cast<int32_t>(i - rb));
                    break;
                }
        if (peer.recv_count || !peer.send_rows.empty()) pl.peers.push_back(std::move(peer));
    }
    return pl;
}

}  // namespace mbg
