// traffic.cpp -- vector-transfer analyzer, basic splitter, per-method
// schedules and the HBM byte model.
//
// analyze_traffic restates statement.cpp:25-56 (reads = ids consumed before
// being produced in the group, writes = distinct outputs); split_basic
// restates statement.cpp:58-85 (singleton groups; updates touching >= 4
// distinct vectors peel their trailing operand pair into a temporary).  The
// schedules are the merged listings of SURVEY.md Appendix C; summing them
// reproduces Table 2.
#include <set>
#include <vector>

#include "common.hpp"
#include "solver.hpp"

namespace mbg {

namespace {

void check_group(const mbg_statement* st, int ns) {
    if (ns < 0 || (ns > 0 && !st)) throw Invalid("statement group: bad statement array");
    for (int i = 0; i < ns; ++i) {
        if (st[i].kind == MBG_STMT_UPDATE) {
            if (st[i].out < 0) throw Invalid("statement group: dangling operand id");
            if (st[i].nterms < 0 || st[i].nterms > MBG_MAX_TERMS)
                throw Invalid("statement group: too many terms");
            for (int t = 0; t < st[i].nterms; ++t)
                if (st[i].term_vec[t] < 0) throw Invalid("statement group: dangling operand id");
        } else if (st[i].kind == MBG_STMT_DOT) {
            if (st[i].left < 0 || st[i].right < 0) throw Invalid("statement group: dangling operand id");
            if (st[i].slot < 0) throw Invalid("statement group: negative dot slot");
        } else {
            throw Invalid("statement group: unknown statement kind");
        }
    }
}

void analyze(const mbg_statement* st, int ns, int* reads, int* writes) {
    std::set<int> produced, rd, wr;
    auto consume = [&](int id) {
        if (!produced.count(id)) rd.insert(id);
    };
    for (int i = 0; i < ns; ++i) {
        if (st[i].kind == MBG_STMT_UPDATE) {
            for (int t = 0; t < st[i].nterms; ++t) consume(st[i].term_vec[t]);
            produced.insert(st[i].out);
            wr.insert(st[i].out);
        } else {
            consume(st[i].left);
            consume(st[i].right);
        }
    }
    *reads = static_cast<int>(rd.size());
    *writes = static_cast<int>(wr.size());
}

// split_basic: returns the list of singleton groups (each one statement)
std::vector<mbg_statement> split(const mbg_statement* st, int ns, int first_temp) {
    std::vector<mbg_statement> out;
    for (int i = 0; i < ns; ++i) {
        if (st[i].kind != MBG_STMT_UPDATE) {
            out.push_back(st[i]);
            continue;
        }
        mbg_statement cur = st[i];
        int next_temp = first_temp;
        for (;;) {
            std::set<int> inv{cur.out};
            for (int t = 0; t < cur.nterms; ++t) inv.insert(cur.term_vec[t]);
            if (inv.size() < 4 || cur.nterms < 2) break;
            mbg_statement peeled{};
            peeled.kind = MBG_STMT_UPDATE;
            peeled.out = next_temp++;
            peeled.nterms = 2;
            for (int t = 0; t < 2; ++t) {
                peeled.term_vec[t] = cur.term_vec[cur.nterms - 2 + t];
                peeled.term_coeff[t] = cur.term_coeff[cur.nterms - 2 + t];
            }
            out.push_back(peeled);
            cur.nterms -= 2;
            cur.term_vec[cur.nterms] = peeled.out;
            cur.term_coeff[cur.nterms] = nullptr;  // constant 1
            cur.nterms += 1;
        }
        out.push_back(cur);
    }
    return out;
}

mbg_statement U(int out, std::initializer_list<int> terms) {
    mbg_statement s{};
    s.kind = MBG_STMT_UPDATE;
    s.out = out;
    for (int v : terms) s.term_vec[s.nterms++] = v;
    return s;
}
mbg_statement Dt(int l, int r, int slot) {
    mbg_statement s{};
    s.kind = MBG_STMT_DOT;
    s.left = l;
    s.right = r;
    s.slot = slot;
    return s;
}

// vector ids for the schedule tables
enum { X, P, R, R0, V, S, T, Z, VH, TH, RT, Q, W, Y, U_, F0, PH, SH, QH, RH, WH, ZH, TEMP = 100 };

using Group = std::vector<mbg_statement>;

// SURVEY.md Appendix C (merged listings); identity M^-1 copies are separate.
std::vector<Group> schedule(int method) {
    switch (method) {
        case MBG_BICGSTAB:  // Alg. 2
            return {{Dt(V, R0, 0)},
                    {U(S, {R, V})},
                    {Dt(T, S, 0), Dt(T, T, 1), Dt(S, S, 2)},
                    {U(X, {X, P, S}), U(R, {S, T}), Dt(R, R0, 0)},
                    {U(P, {R, P, V})}};
        case MBG_RBICGSTAB:  // Alg. 6
            return {{Dt(V, R0, 0)},
                    {U(TH, {Z, S})},
                    {U(RT, {R, V}), Dt(T, RT, 0), Dt(T, T, 1), Dt(T, R0, 2), Dt(RT, RT, 3)},
                    {U(R, {RT, T})},
                    {U(X, {X, VH, TH}), U(Z, {TH, Q}), U(VH, {Z, VH, S})}};
        case MBG_PIPEBICGSTAB:  // Alg. 4
            return {{U(P, {R, P, S}), U(S, {W, S, Z}), U(Z, {T, Z, V}), U(Q, {R, S}), U(Y, {W, Z}),
                     Dt(Q, Y, 0), Dt(Y, Y, 1), Dt(Q, Q, 2)},
                    {U(X, {X, P, Q}), U(R, {Q, Y})},
                    {U(W, {Y, T, V}), Dt(R0, R, 0), Dt(R0, Z, 1), Dt(R0, W, 2), Dt(R0, S, 3)}};
        case MBG_IBICGSTAB:  // Alg. 3, PAPER.md:1455-1471 (Eq. (15): 20 transfers, one 7-dot reduction)
            return {{U(Z, {R, Z, V}), U(V, {U_, V, Q}), U(S, {R, V})},
                    {U(T, {U_, Q}), Dt(R0, S, 0), Dt(R0, Q, 1), Dt(F0, S, 2), Dt(F0, T, 3), Dt(S, T, 4),
                     Dt(T, T, 5), Dt(S, S, 6)},
                    {U(R, {S, T}), U(X, {X, Z, S})}};
        case MBG_PBICGSTAB:  // Alg. 5, PAPER.md:1536-1556 (Eq. (17): 19 transfers + 2 M^-1)
            return {{Dt(V, R0, 0)},
                    {U(S, {R, V})},
                    {Dt(T, S, 0), Dt(T, T, 1), Dt(S, S, 2)},
                    {U(R, {S, T}), Dt(R, R0, 0)},
                    {U(X, {X, PH, SH})},
                    {U(P, {R, P, V})}};
        case MBG_PPIPEBICGSTAB:  // Alg. 7, PAPER.md:1611-1631 (Eq. (19): 34 transfers + 2 M^-1)
            return {{U(PH, {RH, PH, SH}), U(SH, {WH, SH, ZH}), U(QH, {RH, SH})},
                    {U(S, {W, S, Z}), U(Z, {T, Z, V}), U(Q, {R, S}), U(Y, {W, Z}), Dt(Q, Y, 0), Dt(Y, Y, 1),
                     Dt(Q, Q, 2)},
                    {U(X, {X, PH, QH}), U(RH, {QH, WH, ZH})},
                    {U(R, {Q, Y}), U(W, {Y, T, V}), Dt(R0, R, 0), Dt(R0, Z, 1), Dt(R0, W, 2), Dt(R0, S, 3)}};
    }
    throw Invalid("unknown method");
}


// Fused formulation: dots fused into SpMM epilogues read one aux
// vector there (aux_reads); identity M^-1 copies are elided (s = v, q = t);
// Alg. 4 lines 7 + 12 run as one pass.
std::vector<Group> schedule_fused(int method, int* aux_reads, int* spmm_dots) {
    switch (method) {
        case MBG_BICGSTAB:
            // theta = (s,s) computed where s is produced; same transfers as merged
            *aux_reads = 0;
            spmm_dots[0] = spmm_dots[1] = 0;
            return {{Dt(V, R0, 0)},
                    {U(S, {R, V}), Dt(S, S, 2)},
                    {Dt(T, S, 0), Dt(T, T, 1)},
                    {U(X, {X, P, S}), U(R, {S, T}), Dt(R, R0, 0)},
                    {U(P, {R, P, V})}};
        case MBG_RBICGSTAB:
            *aux_reads = 1;                 // r0 in v = A vh
            spmm_dots[0] = 1;
            spmm_dots[1] = 0;
            // rt = r - alpha v lives in registers only: the 4-dot pass reads r, v,
            // t, r0 and stores nothing (modelled by dots over the same vectors);
            // r = rt - omega t is formed in the x / z / vh pass from r, v, t
            return {{U(TH, {Z, V})},
                    {Dt(T, R, 0), Dt(T, T, 1), Dt(T, R0, 2), Dt(V, V, 3)},
                    {U(X, {X, VH, TH}), U(Z, {TH, T}), U(VH, {Z, VH, V}), U(R, {R, V, T})}};
        case MBG_PIPEBICGSTAB:
            *aux_reads = 0;
            spmm_dots[0] = spmm_dots[1] = 0;
            // q = r - alpha s, y = w - alpha z in registers only: the line-4 pass
            // dots them where they are formed (modelled by dots over the vectors
            // they come from) and the line-7/12 pass recomputes them from r, w,
            // s, z -- Alg. 4 lines 7 + 12 in one pass, 22 transfers
            return {{U(P, {R, P, S}), U(S, {W, S, Z}), U(Z, {T, Z, V}), Dt(R, S, 0), Dt(W, Z, 1), Dt(R, W, 2)},
                    {U(X, {X, P, R, S}), U(R, {R, S, W, Z}), U(W, {W, Z, T, V}), Dt(R0, R, 0), Dt(R0, Z, 1),
                     Dt(R0, W, 2), Dt(R0, S, 3)}};
    }
    throw Invalid("unknown method");
}

}  // namespace

bool preconditioned(int method) {
    return method == MBG_RBICGSTAB || method == MBG_PBICGSTAB || method == MBG_PPIPEBICGSTAB;
}

double spmv_traffic_bytes(int64_t n, int64_t nnz, int m) {
    const double dn = static_cast<double>(n), dz = static_cast<double>(nnz);
    return 8.0 * m * (dn + dz) + 4.0 * (dn + 3.0 * dz);
}

double spmv_compulsory_bytes(int64_t n, int64_t nnz, int m) {
    const double dn = static_cast<double>(n), dz = static_cast<double>(nnz);
    return 16.0 * m * dn + 12.0 * dz + 4.0 * (dn + 1.0);
}

// Per-iteration totals, SPEC.md:236-244 form: reads/writes exclude the
// preconditioner, whose applications are returned separately (each costs
// precond_alpha transfers; identity copies elided by the fused formulation).
void method_schedule_pc(int method, int formulation, int precond_alpha, int* reads, int* writes, int* spmvs,
                        int* precond_apps, int* nred, int* dots) {
    if (method < 0 || method > 5) throw Invalid("unknown method");
    int r = 0, w = 0, k = 0;
    const int apps = preconditioned(method) ? 2 : 0;
    *precond_apps = (formulation == MBG_FUSED && precond_alpha == 2) ? 0 : apps;
    *spmvs = 2;
    if (formulation == MBG_FUSED && method <= MBG_PIPEBICGSTAB) {
        int aux = 0, sd[2] = {0, 0};
        for (const auto& g : schedule_fused(method, &aux, sd)) {
            int gr, gw;
            analyze(g.data(), static_cast<int>(g.size()), &gr, &gw);
            r += gr;
            w += gw;
        }
        r += aux;
        // reductions in iteration order
        std::vector<int> red;
        if (method == MBG_BICGSTAB) red = {1, 3, 1};
        else if (method == MBG_RBICGSTAB) red = {1, 4};
        else red = {3, 4};
        for (size_t i = 0; i < red.size(); ++i)
            if (dots && i < 8) dots[i] = red[i];
        *reads = r;
        *writes = w;
        *nred = static_cast<int>(red.size());
        return;
    }
    // the fused formulation of Alg. 3 / 5 / 7 is the merged schedule (with
    // identity M^-1 applications elided)
    for (const auto& g : schedule(method)) {
        if (formulation == MBG_BASIC) {
            for (const auto& st : split(g.data(), static_cast<int>(g.size()), TEMP)) {
                int gr, gw;
                analyze(&st, 1, &gr, &gw);
                r += gr;
                w += gw;
                if (st.kind == MBG_STMT_DOT) {
                    if (dots && k < 8) dots[k] = 1;
                    ++k;
                }
            }
        } else {
            int gr, gw;
            analyze(g.data(), static_cast<int>(g.size()), &gr, &gw);
            r += gr;
            w += gw;
            int nd = 0;
            for (const auto& st : g) nd += st.kind == MBG_STMT_DOT;
            if (nd) {
                if (dots && k < 8) dots[k] = nd;
                ++k;
            }
        }
    }
    *reads = r;
    *writes = w;
    *nred = k;
}

// Legacy totals: the preconditioner's transfers folded into reads/writes
// (alpha/2 read + alpha/2 write per application; 1 + 1 for an identity copy).
void method_schedule(int method, int formulation, int* reads, int* writes, int* spmvs, int* nred, int* dots) {
    const int pa = preconditioned(method) ? 2 : 0;
    int apps = 0;
    method_schedule_pc(method, formulation, pa, reads, writes, spmvs, &apps, nred, dots);
    *reads += apps * pa / 2;
    *writes += apps * pa / 2;
}

double iteration_bytes(int method, int formulation, int precond_alpha, int64_t n, int64_t nnz, int m) {
    int r, w, s, apps, k, d[8];
    method_schedule_pc(method, formulation, precond_alpha, &r, &w, &s, &apps, &k, d);
    return static_cast<double>(r + w + apps * precond_alpha) * 8.0 * static_cast<double>(n) * m +
           s * spmv_compulsory_bytes(n, nnz, m);
}

}  // namespace mbg

extern "C" int mbg_analyze_traffic(const mbg_statement* st, int ns, int* reads, int* writes) {
    try {
        mbg::check_group(st, ns);
        mbg::analyze(st, ns, reads, writes);
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    }
}

extern "C" int mbg_split_basic_traffic(const mbg_statement* st, int ns, int first_temp, int* reads,
                                       int* writes, int* ngroups) {
    try {
        mbg::check_group(st, ns);
        auto parts = mbg::split(st, ns, first_temp);
        int r = 0, w = 0;
        for (const auto& s : parts) {
            int gr, gw;
            mbg::analyze(&s, 1, &gr, &gw);
            r += gr;
            w += gw;
        }
        *reads = r;
        *writes = w;
        *ngroups = static_cast<int>(parts.size());
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    }
}

extern "C" int mbg_method_schedule(int method, int formulation, int* reads, int* writes, int* spmvs,
                                   int* nreductions, int* dots_per_reduction) {
    try {
        if (formulation != MBG_MERGED && formulation != MBG_BASIC && formulation != MBG_FUSED)
            throw mbg::Invalid("unknown formulation");
        mbg::method_schedule(method, formulation, reads, writes, spmvs, nreductions, dots_per_reduction);
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    }
}

extern "C" int mbg_method_schedule_pc(int method, int formulation, int precond_alpha, int* reads, int* writes,
                                      int* spmvs, int* precond_applications, int* nreductions,
                                      int* dots_per_reduction) {
    try {
        if (formulation != MBG_MERGED && formulation != MBG_BASIC && formulation != MBG_FUSED)
            throw mbg::Invalid("unknown formulation");
        if (mbg::preconditioned(method) ? (precond_alpha < 2 || precond_alpha % 2) : precond_alpha != 0)
            throw mbg::Invalid("method_schedule: preconditioner presence mismatch");
        mbg::method_schedule_pc(method, formulation, precond_alpha, reads, writes, spmvs, precond_applications,
                                nreductions, dots_per_reduction);
        return MBG_OK;
    } catch (const mbg::Invalid& e) {
        mbg::set_error(e.what());
        return MBG_ERR_INVALID;
    }
}

extern "C" double mbg_spmv_traffic_bytes(int64_t n, int64_t nnz, int m) {
    return mbg::spmv_traffic_bytes(n, nnz, m);
}

extern "C" double mbg_spmv_compulsory_bytes(int64_t n, int64_t nnz, int m) {
    return mbg::spmv_compulsory_bytes(n, nnz, m);
}
