// host_code.cpp -- host side of libmetldpc: validation of the edge-indexed H,
// the device layout build (degree-1 split of P:34 / P:64-68), the alist reader
// (S:55-63), the fp32 phi tables of DESIGN.md N2 and error reporting.
// Compiled with -ffp-contract=off: the phi tables are fp64 closed forms rounded
// to fp32 in the exact expression order DESIGN.md N2 states.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"

namespace metldpc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

metldpc_status fail(metldpc_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

metldpc_status build_layout(int32_t n, int32_t m, int64_t E, const int64_t* cn_ptr,
                            const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                            HostLayout* out, uint32_t flags) {
    if (n <= 0 || m < 0) return fail(METLDPC_EINVAL, "n must be > 0 and m >= 0");
    if (E < 0 || E >= (int64_t(1) << 31)) return fail(METLDPC_EUNSUPPORTED, "num_edges must be in [0, 2^31)");
    if (!cn_ptr || !vn_ptr || (E > 0 && (!edge_vn || !vn_edge)))
        return fail(METLDPC_EINVAL, "NULL array");
    if (cn_ptr[0] != 0 || cn_ptr[m] != E) return fail(METLDPC_EFORMAT, "cn_ptr must start at 0 and end at num_edges");
    if (vn_ptr[0] != 0 || vn_ptr[n] != E) return fail(METLDPC_EFORMAT, "vn_ptr must start at 0 and end at num_edges");
    for (int32_t j = 0; j < m; ++j)
        if (cn_ptr[j + 1] < cn_ptr[j]) return fail(METLDPC_EFORMAT, "cn_ptr not non-decreasing at CN " + std::to_string(j));
    for (int32_t v = 0; v < n; ++v)
        if (vn_ptr[v + 1] < vn_ptr[v]) return fail(METLDPC_EFORMAT, "vn_ptr not non-decreasing at VN " + std::to_string(v));
    std::vector<int32_t> deg(n, 0);
    for (int64_t e = 0; e < E; ++e) {
        int32_t v = edge_vn[e];
        if (v < 0 || v >= n)
            return fail(METLDPC_EFORMAT, "edge " + std::to_string(e) + ": VN index " + std::to_string(v) +
                                             " out of range n=" + std::to_string(n));
        deg[v]++;
    }
    // duplicate (VN, CN) pairs within a row
    {
        std::vector<int32_t> seen(n, -1);
        for (int32_t j = 0; j < m; ++j)
            for (int64_t e = cn_ptr[j]; e < cn_ptr[j + 1]; ++e) {
                if (seen[edge_vn[e]] == j)
                    return fail(METLDPC_EFORMAT, "duplicate edge (CN " + std::to_string(j) + ", VN " +
                                                     std::to_string(edge_vn[e]) + ")");
                seen[edge_vn[e]] = j;
            }
    }
    for (int32_t v = 0; v < n; ++v) {
        if (deg[v] == 0) return fail(METLDPC_EFORMAT, "VN " + std::to_string(v) + " has degree 0");
        if (vn_ptr[v + 1] - vn_ptr[v] != deg[v])
            return fail(METLDPC_EFORMAT, "CSR/CSC mismatch: VN " + std::to_string(v) + " degree");
    }
    // CSC: permutation of edge ids, each slot of column v pointing at an edge of v
    {
        std::vector<uint8_t> hit(E, 0);
        for (int32_t v = 0; v < n; ++v)
            for (int64_t k = vn_ptr[v]; k < vn_ptr[v + 1]; ++k) {
                int64_t e = vn_edge[k];
                if (e < 0 || e >= E) return fail(METLDPC_EFORMAT, "vn_edge[" + std::to_string(k) + "] out of range");
                if (hit[e]) return fail(METLDPC_EFORMAT, "vn_edge is not a permutation (edge " + std::to_string(e) + ")");
                hit[e] = 1;
                if (edge_vn[e] != v)
                    return fail(METLDPC_EFORMAT, "CSR/CSC mismatch: CSC slot " + std::to_string(k) + " of VN " +
                                                     std::to_string(v) + " points at an edge of VN " +
                                                     std::to_string(edge_vn[e]));
            }
    }
    // Degree-1 VNs are skipped during iterations unless METLDPC_CODE_NO_SKIP asks for
    // the paper's "without skipping" variant (Table 1 left columns): then every VN is iterated.
    const int32_t min_act = (flags & METLDPC_CODE_NO_SKIP) ? 1 : 2;
    HostLayout& L = *out;
    L = HostLayout();
    L.n = n; L.m = m; L.E = E;
    L.vmap.assign(n, 0);
    int32_t n_a = 0;
    for (int32_t v = 0; v < n; ++v) {
        if (deg[v] >= min_act) { L.vmap[v] = n_a++; L.act_vn.push_back(v); }
        L.max_vn_deg = std::max(L.max_vn_deg, deg[v]);
    }
    L.n_a = n_a;
    // N3: the fixed-point VN sum of an active VN is exact only while deg * 30 * 2^17 stays
    // inside the 32-bit accumulator (deg <= kMaxVnDeg)
    if (L.max_vn_deg > kMaxVnDeg)
        return fail(METLDPC_EUNSUPPORTED, "VN degree " + std::to_string(L.max_vn_deg) + " > " +
                                              std::to_string(kMaxVnDeg) + " (fixed-point VN sum, DESIGN.md N3)");
    // canonical active-edge id: rank among active edges in the caller's CSR order
    std::vector<int32_t> canon(E, -1);
    int64_t tc = 0;
    for (int64_t e = 0; e < E; ++e)
        if (deg[edge_vn[e]] >= min_act) canon[e] = int32_t(tc++);
    // CN relabelling by degree class (stable): key 2D + nd for D <= 16, nd <= 1; else generic
    std::vector<int32_t> cnd(m, 0);
    for (int32_t j = 0; j < m; ++j) {
        int32_t d = int32_t(cn_ptr[j + 1] - cn_ptr[j]);
        if (d > kMaxCnDeg)
            return fail(METLDPC_EUNSUPPORTED, "CN " + std::to_string(j) + " has degree " + std::to_string(d) +
                                                  " > " + std::to_string(kMaxCnDeg));
        for (int64_t e = cn_ptr[j]; e < cn_ptr[j + 1]; ++e) cnd[j] += (deg[edge_vn[e]] < min_act);
    }
    const int generic_key = 2 * (kMaxUnrolledCnDeg + 1);
    auto cls_key = [&](int32_t j) {
        const int d = int(cn_ptr[j + 1] - cn_ptr[j]);
        return (d <= kMaxUnrolledCnDeg && cnd[j] <= 1) ? 2 * d + cnd[j] : generic_key;
    };
    std::vector<std::vector<int32_t>> buckets(generic_key + 1);
    for (int32_t j = 0; j < m; ++j) buckets[cls_key(j)].push_back(j);
    // An exact class with one degree-1 slot lists its CNs by the original index of that degree-1
    // VN, so consecutive degree-1 slots q hold VNs in ascending original order: a frame's priors
    // then land in whole 32-byte sectors of the blocked lam1 layout.
    for (int key = 1; key < generic_key; key += 2) {
        auto& bk = buckets[key];
        if (bk.size() < 2) continue;
        std::vector<std::pair<int32_t, int32_t>> kv;
        kv.reserve(bk.size());
        for (int32_t j : bk) {
            int32_t v1 = -1;
            for (int64_t e = cn_ptr[j]; e < cn_ptr[j + 1]; ++e)
                if (deg[edge_vn[e]] < min_act) v1 = edge_vn[e];
            kv.emplace_back(v1, j);
        }
        std::stable_sort(kv.begin(), kv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t i = 0; i < bk.size(); ++i) bk[i] = kv[i].second;
    }
    std::vector<int32_t> order;
    order.reserve(m);
    for (int key = 0; key <= generic_key; ++key) {
        if (buckets[key].empty()) continue;
        HostLayout::CnClass c{key < generic_key ? key / 2 : -1, key < generic_key ? key % 2 : -1,
                              int32_t(order.size()), int32_t(buckets[key].size())};
        order.insert(order.end(), buckets[key].begin(), buckets[key].end());
        L.classes.push_back(c);
    }
    L.cn_new.assign(m, 0);
    for (int32_t jn = 0; jn < m; ++jn) L.cn_new[order[jn]] = jn;
    std::vector<int32_t> act_id(E, -1);
    L.cn_aptr.assign(m + 1, 0);
    L.cn_dptr.assign(m + 1, 0);
    L.perm_r.reserve(size_t(tc));
    int32_t t = 0, n_1 = 0;
    for (int32_t jn = 0; jn < m; ++jn) {
        const int32_t j = order[jn];

        L.cn_aptr[jn] = t;
        L.cn_dptr[jn] = n_1;
        L.max_cn_deg = std::max(L.max_cn_deg, int32_t(cn_ptr[j + 1] - cn_ptr[j]));
        for (int64_t e = cn_ptr[j]; e < cn_ptr[j + 1]; ++e) {
            int32_t v = edge_vn[e];
            if (deg[v] >= min_act) {
                act_id[e] = t++;
                L.a_vn.push_back(L.vmap[v]);
                L.perm_r.push_back(canon[e]);
            } else {
                L.vmap[v] = ~n_1;
                n_1++;
            }
        }
    }
    L.cn_aptr[m] = t;
    L.cn_dptr[m] = n_1;
    L.E_it = t;
    L.n_1 = n_1;
    L.vn_aptr.assign(n_a + 1, 0);
    L.vn_aedge.reserve(size_t(t));
    for (int32_t a = 0; a < n_a; ++a) {
        int32_t v = L.act_vn[a];
        L.vn_aptr[a] = int32_t(L.vn_aedge.size());
        for (int64_t k = vn_ptr[v]; k < vn_ptr[v + 1]; ++k) L.vn_aedge.push_back(act_id[vn_edge[k]]);
    }
    L.vn_aptr[n_a] = int32_t(L.vn_aedge.size());
    L.csr_ptr.assign(cn_ptr, cn_ptr + m + 1);
    L.csr_vn.assign(edge_vn, edge_vn + E);
    return METLDPC_OK;
}

void fill_info(const HostLayout& L, metldpc_code_info_t* info) {
    info->n = L.n;
    info->m = L.m;
    info->edges = L.E;
    info->iter_edges = L.E_it;
    info->n_active = L.n_a;
    info->n_deg1 = L.n_1;
    info->max_cn_deg = L.max_cn_deg;
    info->max_vn_deg = L.max_vn_deg;
}

// ------------------------------------------------------------------ phi tables (N2)

static double phi_d(double y) { return std::log1p(2.0 / std::expm1(y)); }     // -ln tanh(y/2)
static double dphi_d(double y) { return -1.0 / std::sinh(y); }

static void knot(int J, int b, double* y0, double* h) {
    int e = kPhiELo + (b >> J);
    int j = b & ((1 << J) - 1);
    *y0 = std::ldexp(1.0 + double(j) / double(1 << J), e);
    *h = std::ldexp(1.0, e - J);
}

void phi_table_exact(float* out) {
    for (int b = 0; b < kPhiBinsExact; ++b) {
        double y0, h;
        knot(kPhiJExact, b, &y0, &h);
        double y1 = y0 + h;
        double f0 = phi_d(y0), f1 = phi_d(y1);
        double m0 = h * dphi_d(y0), m1 = h * dphi_d(y1);
        double c2 = 3.0 * (f1 - f0) - 2.0 * m0 - m1;
        double c3 = 2.0 * (f0 - f1) + m0 + m1;
        out[4 * b + 0] = float(f0);
        out[4 * b + 1] = float(m0);
        out[4 * b + 2] = float(c2);
        out[4 * b + 3] = float(c3);
    }
}

void phi_table_lut(float* out) {
    for (int b = 0; b < kPhiBinsLut; ++b) {
        double y0, h;
        knot(kPhiJLut, b, &y0, &h);
        double f0 = phi_d(y0), f1 = phi_d(y0 + h);
        out[2 * b + 0] = float(f0);
        out[2 * b + 1] = float(f1 - f0);
    }
}

float phi_top() { return float(phi_d(std::ldexp(1.0, kPhiELo))); }

std::vector<float> phi_device_table(int rule) {
    const bool ex = (rule == METLDPC_RULE_EXACT);
    const int nb = ex ? kPhiBinsExact : kPhiBinsLut, per = ex ? 4 : 2;
    std::vector<float> base(size_t(nb) * per);
    if (ex) phi_table_exact(base.data());
    else phi_table_lut(base.data());
    // coefficients pre-scaled by 2^(J q) (exact: power-of-two scaling of an fp32 value), so the
    // kernel evaluates the polynomial in t / 2^J -- bit-identical results (kernels.cu phi_dev)
    const int J = ex ? kPhiJExact : kPhiJLut;
    const int zb = ex ? kPhiZeroBinsExact : kPhiZeroBinsLut;            // zero bins for [2^6, 2^7)
    std::vector<float> dev(size_t(nb + zb) * kPhiCopies * per, 0.0f);
    for (int b = 0; b < nb; ++b)
        for (int k = 0; k < kPhiCopies; ++k)
            for (int q = 0; q < per; ++q)
                dev[(size_t(b) * kPhiCopies + k) * per + q] = std::ldexp(base[size_t(b) * per + q], J * q);
    return dev;
}

// ------------------------------------------------------------------ MD product table (N6)

// Cayley-Dickson product of two d-vectors, (a1, a2)(b1, b2) = (a1 b1 - conj(b2) a2,
// b2 a1 + a2 conj(b1)), on doubles; basis products are read off e_p * e_q.
static void cd_conj(const double* a, int d, double* out) {
    out[0] = a[0];
    for (int i = 1; i < d; ++i) out[i] = -a[i];
}
static void cd_mul_vec(const double* a, const double* b, int d, double* out) {
    if (d == 1) { out[0] = a[0] * b[0]; return; }
    const int h = d / 2;
    double t1[8], t2[8], cb2[8], cb1[8];
    cd_conj(b + h, h, cb2);
    cd_conj(b, h, cb1);
    cd_mul_vec(a, b, h, t1);
    cd_mul_vec(cb2, a + h, h, t2);
    for (int i = 0; i < h; ++i) out[i] = t1[i] - t2[i];
    cd_mul_vec(b + h, a, h, t1);
    cd_mul_vec(a + h, cb1, h, t2);
    for (int i = 0; i < h; ++i) out[h + i] = t1[i] + t2[i];
}

void md_product_table(int d, int8_t* kp, int8_t* ks) {
    for (int p = 0; p < d; ++p)
        for (int q = 0; q < d; ++q) {
            double ep[8] = {0}, eq[8] = {0}, r[8];
            ep[p] = 1.0;
            eq[q] = 1.0;
            cd_mul_vec(ep, eq, d, r);
            for (int i = 0; i < d; ++i)
                if (r[i] != 0.0) {           // e_p e_q = sgn e_i
                    kp[i * d + q] = int8_t(p);
                    ks[i * d + q] = int8_t(r[i] > 0 ? 1 : -1);
                }
        }
}

// ------------------------------------------------------------------ alist

struct LineReader {
    std::istream& in;
    int line = 0;
    std::string cur;
    explicit LineReader(std::istream& s) : in(s) {}
    bool next(std::vector<long long>& vals) {
        while (std::getline(in, cur)) {
            ++line;
            std::istringstream ss(cur);
            vals.clear();
            std::string tok;
            bool any = false;
            while (ss >> tok) {
                char* end = nullptr;
                long long v = std::strtoll(tok.c_str(), &end, 10);
                if (!end || *end != '\0') { vals.assign(1, LLONG_MIN); return true; }
                vals.push_back(v);
                any = true;
            }
            if (any) return true;
        }
        return false;
    }
};

metldpc_status parse_alist(const char* path, int32_t* n_out, int32_t* m_out, std::vector<int64_t>* cn_ptr,
                           std::vector<int32_t>* edge_vn, std::vector<int64_t>* vn_ptr,
                           std::vector<int64_t>* vn_edge) {
    std::ifstream f(path);
    if (!f) return fail(METLDPC_EINVAL, std::string("cannot open alist file ") + path);
    LineReader R(f);
    std::vector<long long> v;
    auto bad = [&](const std::string& what) {
        return fail(METLDPC_EFORMAT, "alist line " + std::to_string(R.line) + ": " + what);
    };
    auto is_bad_tok = [&]() { return !v.empty() && v[0] == LLONG_MIN; };
    if (!R.next(v) || is_bad_tok() || v.size() != 2) return bad("expected 'n m'");
    long long n = v[0], m = v[1];
    if (n <= 0 || m < 0 || n > (1LL << 30) || m > (1LL << 30)) return bad("n, m out of range");
    if (!R.next(v) || is_bad_tok() || v.size() != 2) return bad("expected 'max_vn_deg max_cn_deg'");
    std::vector<long long> vdeg, cdeg;
    if (!R.next(vdeg) || (long long)vdeg.size() != n) return bad("expected n VN degrees");
    if (!R.next(cdeg) || (long long)cdeg.size() != m) return bad("expected m CN degrees");
    std::vector<std::vector<int32_t>> vn_lists(n), cn_lists(m);
    for (long long i = 0; i < n; ++i) {
        if (!R.next(v) || is_bad_tok()) return bad("expected CN list of VN " + std::to_string(i + 1));
        std::vector<int32_t> lst;
        for (long long x : v) {
            if (x == 0) continue;  // zero padding allowed by the format
            if (x < 1 || x > m) return bad("CN index " + std::to_string(x) + " out of range m=" + std::to_string(m));
            lst.push_back(int32_t(x - 1));
        }
        if ((long long)lst.size() != vdeg[i]) return bad("VN " + std::to_string(i + 1) + " degree mismatch");
        vn_lists[i] = std::move(lst);
    }
    for (long long j = 0; j < m; ++j) {
        if (!R.next(v) || is_bad_tok()) return bad("expected VN list of CN " + std::to_string(j + 1));
        std::vector<int32_t> lst;
        for (long long x : v) {
            if (x == 0) continue;
            if (x < 1 || x > n) return bad("VN index " + std::to_string(x) + " >= n=" + std::to_string(n));
            lst.push_back(int32_t(x - 1));
        }
        if ((long long)lst.size() != cdeg[j]) return bad("CN " + std::to_string(j + 1) + " degree mismatch");
        cn_lists[j] = std::move(lst);
    }
    *n_out = int32_t(n);
    *m_out = int32_t(m);
    cn_ptr->assign(m + 1, 0);
    edge_vn->clear();
    for (long long j = 0; j < m; ++j) {
        (*cn_ptr)[j] = int64_t(edge_vn->size());
        for (int32_t x : cn_lists[j]) edge_vn->push_back(x);
    }
    (*cn_ptr)[m] = int64_t(edge_vn->size());
    // CSC: for each VN, its CN list order; find the CSR edge id of (cn, vn)
    int64_t E = int64_t(edge_vn->size());
    vn_ptr->assign(n + 1, 0);
    vn_edge->assign(E, -1);
    int64_t k = 0;
    for (long long i = 0; i < n; ++i) {
        (*vn_ptr)[i] = k;
        for (int32_t j : vn_lists[i]) {
            int64_t found = -1;
            for (int64_t e = (*cn_ptr)[j]; e < (*cn_ptr)[j + 1]; ++e)
                if ((*edge_vn)[e] == int32_t(i)) { found = e; break; }
            if (found < 0)
                return fail(METLDPC_EFORMAT, "alist: VN " + std::to_string(i + 1) + " lists CN " + std::to_string(j + 1) +
                                                 " but that CN does not list it");
            if (k >= E) return fail(METLDPC_EFORMAT, "alist: VN lists have more entries than CN lists");
            (*vn_edge)[k++] = found;
        }
    }
    (*vn_ptr)[n] = k;
    if (k != E) return fail(METLDPC_EFORMAT, "alist: VN and CN lists disagree on the edge count");
    return METLDPC_OK;
}

}  // namespace metldpc

using namespace metldpc;

extern "C" {

const char* metldpc_last_error(void) { return g_last_error.c_str(); }

const char* metldpc_status_string(metldpc_status s) {
    switch (s) {
        case METLDPC_OK: return "ok";
        case METLDPC_EINVAL: return "invalid argument";
        case METLDPC_EFORMAT: return "malformed parity-check matrix";
        case METLDPC_ENOMEM: return "out of memory";
        case METLDPC_ECUDA: return "CUDA error";
        case METLDPC_EUNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

metldpc_status metldpc_code_check(int32_t n, int32_t m, int64_t num_edges, const int64_t* cn_ptr,
                                  const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                                  metldpc_code_info_t* info_out) {
    HostLayout L;
    metldpc_status s = build_layout(n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge, &L, 0);
    if (s == METLDPC_OK && info_out) fill_info(L, info_out);
    return s;
}

int32_t metldpc_phi_table(int32_t rule, float* out, int32_t cap) {
    int32_t need = (rule == METLDPC_RULE_EXACT) ? kPhiBinsExact * 4 + 1 : kPhiBinsLut * 2 + 1;
    if (!out || cap < need) return need;
    if (rule == METLDPC_RULE_EXACT) phi_table_exact(out);
    else phi_table_lut(out);
    out[need - 1] = phi_top();
    return need;
}

}  // extern "C"
