/*
 * bp_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, CPU reference of the
 * syndrome belief-propagation decoder of arXiv 1711.01783 (PAPER.md "Methods",
 * Steps 1-5, Eqs. (1)-(5), lines 115-146).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path in
 * paper_1711_01783_b200/csrc; both follow DESIGN.md ("Numerics contract").
 *
 * Two precisions of the same algorithm:
 *   M2 (fp64)  the plain definition: phi(y) = log1p(2/expm1(y)) from libm.
 *   M3 (fp32)  replay of the kernel precision: phi from the fp32 table of
 *              DESIGN.md section N2, evaluated exactly as written there.
 * Hard decisions are taken in the precision of the run (N0).
 *
 * Algorithm per iteration l = 1..N (flooding; every CN reads only l-1 state):
 *   CN phase (Eqs. 2-3 in the LLR sign/phi form, with the syndrome sign
 *     sigma_j = 1 - 2 S_B[j]; reading R1):
 *       inputs in slot order k = 0..d-1 -- the active edges of row j in CSR
 *       order, then its degree-1 edges in CSR order (reading R9);
 *       x_k = L_v - r_e (posterior form of Eq. 4, reading R10) for an active
 *       edge, x_k = lambda_v for a degree-1 VN (Eq. 4 with an empty product:
 *       degree-1 VNs are skipped during iterations);
 *       p_k = phi(|x_k|); n_k = [x_k < 0];
 *       forward sums P_0 = 0, P_{k+1} = P_k + p_k; backward sums Q_{d-1} = 0,
 *       Q_k = Q_{k+1} + p_{k+1}; S_k = P_k + Q_k;
 *       o_k = (-1)^(XOR_{k'!=k} n_k' XOR s_j) * min(phi(S_k), R_MAX).
 *   VN phase (Eq. 4/5): L_i = lambda_i + sum of r over C_i -- in fp64 (M2) a left
 *       fold in the caller's CSC slot order; in fp32 (M3) an exact fixed-point sum
 *       with 2^-17 resolution (N3, see vn_phase32).
 *   Decisions (Step 5, Eq. 5): c_i = [L_i < 0] for active VNs,
 *       c_v = [lambda_v + rho_v < 0] for degree-1 VNs (rho = their CN output; in
 *       fp32 (M3) the unclamped rho, compared in the phi domain: DESIGN.md N1);
 *       a tie (exact zero) gives 0 -- "if q_i^l > 1, c_i = 1".
 *   Syndrome test (Step 5): stop at the first l with H c^T = S_B when early
 *       termination is on; otherwise run N iterations and test once.
 *   Variant ORC_NO_SKIP (Table 1 "without skipping"): degree-1 VNs are iterated
 *       like the others, so "active" means degree >= 1 in everything above.
 * LLR convention lambda = ln P(0)/P(1) = -ln q^0 (Eq. 1 ratio q = q(1)/q(0)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define R_MAX 30.0
#define PHI_E_LO (-44)
#define PHI_E_HI 6
/* bins per binade 2^J: EXACT J = 4 (cubic), PHI_LUT J = 5 (linear) -- DESIGN.md N2 */
#define PHI_J_EXACT 4
#define PHI_J_LUT 5
#define PHI_NBIN_MAX (((PHI_E_HI) - (PHI_E_LO)) << PHI_J_LUT)
static int phi_j(int rule) { return rule == 0 ? PHI_J_EXACT : PHI_J_LUT; }
static int phi_nbin(int rule) { return ((PHI_E_HI) - (PHI_E_LO)) << phi_j(rule); }

enum { RULE_EXACT = 0, RULE_PHI_LUT = 1 };

/* Variant bit or-ed into the `rule` argument of the decoders (and the `variant`
 * argument of orc_graph_sizes): iterate degree-1 VNs like every other VN -- the
 * paper's "without skipping" column of Table 1.  A degree-1 VN then
 * keeps a message r and a posterior L = lambda + r like any VN (Eq. 4/5), and
 * its CN input is the extrinsic L - r (R26). */
#define ORC_NO_SKIP 0x100

/* Variant bit of the fp32 decoder (M3) only: 16-bit message storage (R28 / N7).
 * The paper fixes no precision for the stored messages and names global-memory access as
 * the cost that dominates.  The CN output o of iteration l is kept for the next
 * iteration as the integer rint(2^10 o) (round half to even; |o| <= R_MAX = 30 gives
 * |rint(2^10 o)| <= 30720 < 2^15), i.e. the stored message is rint(2^10 o) * 2^-10, within
 * 2^-11 of o.  The VN sum of Eq. (4)/(5) of iteration l is taken over the unrounded outputs
 * o (N3); the extrinsic of iteration l + 1, x = L - r (R10), reads the stored message. */
#define ORC_MSG16 0x200

/* ------------------------------------------------------------------ phi */

/* phi(y) = ln((e^y + 1)/(e^y - 1)) = -ln tanh(y/2); phi(0) = +inf, phi(inf) = 0. */
double orc_phi_def(double y) {
    if (y <= 0.0) return INFINITY;
    return log1p(2.0 / expm1(y));
}

/* phi'(y) = -1/sinh(y) */
static double dphi_def(double y) { return -1.0 / sinh(y); }

/* Bin b covers [y0, y0 + h): y0 = 2^e (1 + j/2^J), h = 2^(e-J), e = -44 + (b >> J), j = b mod 2^J. */
static void bin_knots(int J, int b, double* y0, double* h) {
    int e = PHI_E_LO + (b >> J);
    int j = b & ((1 << J) - 1);
    *y0 = ldexp(1.0 + (double)j / (double)(1 << J), e);
    *h = ldexp(1.0, e - J);
}

/* DESIGN.md N2: the fp32 phi table of each rule (EXACT 800 bins, PHI_LUT 1600 bins).
 *   EXACT  : 4 floats per bin, cubic Hermite on t in [0,1):
 *            c0 = f0, c1 = m0, c2 = 3(f1-f0) - 2 m0 - m1, c3 = 2(f0-f1) + m0 + m1,
 *            f = phi(knot), m = h * phi'(knot), evaluated in double, rounded.
 *   PHI_LUT: 2 floats per bin, linear: c0 = f0, c1 = f1 - f0.
 * Returns the number of floats written (cap permitting). */
int orc_phi_table(int rule, float* out, int cap) {
    int per = (rule == RULE_EXACT) ? 4 : 2;
    int need = phi_nbin(rule) * per;
    if (!out || cap < need) return need;
    for (int b = 0; b < phi_nbin(rule); ++b) {
        double y0, h;
        bin_knots(phi_j(rule), b, &y0, &h);
        double y1 = y0 + h;
        double f0 = orc_phi_def(y0), f1 = orc_phi_def(y1);
        if (rule == RULE_EXACT) {
            double m0 = h * dphi_def(y0), m1 = h * dphi_def(y1);
            double c2 = 3.0 * (f1 - f0) - 2.0 * m0 - m1;
            double c3 = 2.0 * (f0 - f1) + m0 + m1;
            out[4 * b + 0] = (float)f0;
            out[4 * b + 1] = (float)m0;
            out[4 * b + 2] = (float)c2;
            out[4 * b + 3] = (float)c3;
        } else {
            out[2 * b + 0] = (float)f0;
            out[2 * b + 1] = (float)(f1 - f0);
        }
    }
    return need;
}

static float g_tab[2][PHI_NBIN_MAX * 4];
static int g_tab_ready[2];
static float g_phi_top;  /* phi(2^-44) rounded to fp32 */

/* Builds both fp32 tables; the Python loader calls it once before any
 * (possibly multi-threaded) decode, so the lazy path below never races. */
void orc_init(void) {
    orc_phi_table(RULE_EXACT, g_tab[0], PHI_NBIN_MAX * 4);
    orc_phi_table(RULE_PHI_LUT, g_tab[1], PHI_NBIN_MAX * 4);
    g_phi_top = (float)orc_phi_def(ldexp(1.0, PHI_E_LO));
    g_tab_ready[0] = g_tab_ready[1] = 1;
}

static void ensure_tables(void) {
    if (!g_tab_ready[0] || !g_tab_ready[1]) orc_init();
}

/* M3: fp32 phi of DESIGN.md N2 (y >= 0). */
float orc_phi32(int rule, float y) {
    ensure_tables();
    uint32_t bits;
    memcpy(&bits, &y, 4);
    const uint32_t lo = (uint32_t)(127 + PHI_E_LO) << 23;
    const uint32_t hi = (uint32_t)(127 + PHI_E_HI) << 23;
    if (bits < lo) return g_phi_top;
    if (bits >= hi) return 0.0f;
    int J = phi_j(rule);
    uint32_t idx = (bits - lo) >> (23 - J);
    float t = (float)(bits & ((1u << (23 - J)) - 1u)) * (1.0f / (float)(1u << (23 - J)));
    if (rule == RULE_EXACT) {
        const float* c = &g_tab[0][4 * idx];
        return fmaf(fmaf(fmaf(c[3], t, c[2]), t, c[1]), t, c[0]);
    }
    const float* c = &g_tab[1][2 * idx];
    return fmaf(c[1], t, c[0]);
}

/* M2: fp64 phi.  EXACT is the definition; PHI_LUT is the same piecewise-linear
 * semi-log table rule with its knots kept in double (reading R4/R5). */
double orc_phi64(int rule, double y) {
    if (rule == RULE_EXACT) return orc_phi_def(y);
    if (y < ldexp(1.0, PHI_E_LO)) return orc_phi_def(ldexp(1.0, PHI_E_LO));
    if (y >= ldexp(1.0, PHI_E_HI)) return 0.0;
    int e;
    double mant = frexp(y, &e);          /* y = mant * 2^e, mant in [0.5, 1) */
    e -= 1;                               /* y = (2 mant) 2^e, 2 mant in [1, 2) */
    double pos = (2.0 * mant - 1.0) * (double)(1 << PHI_J_LUT);
    int j = (int)floor(pos);
    double t = pos - (double)j;
    int b = ((e - PHI_E_LO) << PHI_J_LUT) + j;
    double y0, h;
    bin_knots(PHI_J_LUT, b, &y0, &h);
    double f0 = orc_phi_def(y0), f1 = orc_phi_def(y0 + h);
    return f0 + t * (f1 - f0);
}

/* ------------------------------------------------------------------ graph */

typedef struct {
    int n, m;
    const int64_t* cn_ptr; const int32_t* edge_vn;
    const int64_t* vn_ptr; const int64_t* vn_edge;
    int64_t E;
    int32_t* vdeg;        /* [n] */
    int64_t* act_id;      /* [E] active-edge id of CSR edge e, or -1 for a degree-1 edge */
    int32_t* vn_act;      /* [n] active index of VN or -1 */
    int64_t E_it;
    int32_t n_a;
    int32_t* act_vn;      /* [n_a] VN of active index */
    int max_cdeg;         /* largest CN degree */
} graph_t;

static int graph_build(graph_t* g, int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                       const int64_t* vn_ptr, const int64_t* vn_edge, int variant) {
    /* a VN is iterated ("active") if its degree is >= 2, or >= 1 without skipping */
    const int min_act = (variant & ORC_NO_SKIP) ? 1 : 2;
    memset(g, 0, sizeof(*g));
    g->n = n; g->m = m; g->cn_ptr = cn_ptr; g->edge_vn = edge_vn; g->vn_ptr = vn_ptr; g->vn_edge = vn_edge;
    g->E = cn_ptr[m];
    g->vdeg = calloc((size_t)n, sizeof(int32_t));
    g->act_id = malloc((size_t)(g->E > 0 ? g->E : 1) * sizeof(int64_t));
    g->vn_act = malloc((size_t)n * sizeof(int32_t));
    for (int64_t e = 0; e < g->E; ++e) {
        if (edge_vn[e] < 0 || edge_vn[e] >= n) return -1;
        g->vdeg[edge_vn[e]]++;
    }
    g->n_a = 0;
    for (int v = 0; v < n; ++v) {
        if (g->vdeg[v] == 0) return -2;                      /* degree-0 VN: rejected */
        if (vn_ptr[v + 1] - vn_ptr[v] != g->vdeg[v]) return -3; /* CSR/CSC mismatch */
        g->vn_act[v] = (g->vdeg[v] >= min_act) ? g->n_a++ : -1;
    }
    g->act_vn = malloc((size_t)(g->n_a > 0 ? g->n_a : 1) * sizeof(int32_t));
    for (int v = 0; v < n; ++v) if (g->vn_act[v] >= 0) g->act_vn[g->vn_act[v]] = v;
    g->max_cdeg = 1;
    for (int j = 0; j < m; ++j)
        if (cn_ptr[j + 1] - cn_ptr[j] > g->max_cdeg) g->max_cdeg = (int)(cn_ptr[j + 1] - cn_ptr[j]);
    g->E_it = 0;
    for (int64_t e = 0; e < g->E; ++e)
        g->act_id[e] = (g->vdeg[edge_vn[e]] >= min_act) ? g->E_it++ : -1;
    return 0;
}

static void graph_free(graph_t* g) {
    free(g->vdeg); free(g->act_id); free(g->vn_act); free(g->act_vn);
}

int orc_graph_sizes(int variant, int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                    const int64_t* vn_ptr, const int64_t* vn_edge, int64_t* E_it, int32_t* n_a) {
    graph_t g;
    int rc = graph_build(&g, n, m, cn_ptr, edge_vn, vn_ptr, vn_edge, variant);
    if (rc == 0) { *E_it = g.E_it; *n_a = g.n_a; }
    graph_free(&g);
    return rc;
}

static int synd_bit(const uint32_t* s, int j) { return (int)((s[j >> 5] >> (j & 31)) & 1u); }

/* Step 5: S_A = H c^T compared with S_B. Returns 1 if equal. */
static int syndrome_matches(const graph_t* g, const uint8_t* c, const uint32_t* synd) {
    for (int j = 0; j < g->m; ++j) {
        int par = 0;
        for (int64_t e = g->cn_ptr[j]; e < g->cn_ptr[j + 1]; ++e) par ^= c[g->edge_vn[e]];
        if (par != synd_bit(synd, j)) return 0;
    }
    return 1;
}

void orc_syndrome(int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                  const uint8_t* c, uint8_t* s_out) {
    (void)n;
    for (int j = 0; j < m; ++j) {
        int par = 0;
        for (int64_t e = cn_ptr[j]; e < cn_ptr[j + 1]; ++e) par ^= c[edge_vn[e]];
        s_out[j] = (uint8_t)par;
    }
}

/* ------------------------------------------------------------------ decoders */

/* The decoder is written once per precision as a macro-free pair of functions
 * so each reads as the plain algorithm in its own type. */

/* ---- fp32 (M3) ---- */
static void cn_phase32(const graph_t* g, int rule, const float* lam, const uint32_t* synd,
                       const float* r_old, const float* L_old, float* r_new, uint8_t* dec1 /*[n]*/) {
    int D = g->max_cdeg;
    float* x = malloc(sizeof(float) * (size_t)D);
    float* p = malloc(sizeof(float) * (size_t)D);
    float* P = malloc(sizeof(float) * (size_t)(D + 1));
    float* Q = malloc(sizeof(float) * (size_t)D);
    int64_t* slot_e = malloc(sizeof(int64_t) * (size_t)D);
    for (int j = 0; j < g->m; ++j) {
        int d = 0;
        /* slot order: active edges (CSR order), then degree-1 edges (CSR order) */
        for (int64_t e = g->cn_ptr[j]; e < g->cn_ptr[j + 1]; ++e)
            if (g->act_id[e] >= 0) slot_e[d++] = e;
        for (int64_t e = g->cn_ptr[j]; e < g->cn_ptr[j + 1]; ++e)
            if (g->act_id[e] < 0) slot_e[d++] = e;
        if (d == 0) continue;
        int par = synd_bit(synd, j);
        for (int k = 0; k < d; ++k) {
            int64_t e = slot_e[k];
            int v = g->edge_vn[e];
            if (g->act_id[e] >= 0) x[k] = L_old[g->vn_act[v]] - r_old[g->act_id[e]];
            else x[k] = lam[v];
            p[k] = orc_phi32(rule, fabsf(x[k]));
            par ^= (x[k] < 0.0f);
        }
        P[0] = 0.0f;
        for (int k = 0; k < d; ++k) P[k + 1] = P[k] + p[k];
        Q[d - 1] = 0.0f;
        for (int k = d - 2; k >= 0; --k) Q[k] = Q[k + 1] + p[k + 1];
        for (int k = 0; k < d; ++k) {
            float S = P[k] + Q[k];
            int neg = par ^ (x[k] < 0.0f);
            int64_t e = slot_e[k];
            if (g->act_id[e] >= 0) {
                float mag = fminf(orc_phi32(rule, S), (float)R_MAX);
                r_new[g->act_id[e]] = neg ? -mag : mag;
            } else {
                /* Step 5 for the degree-1 VN v (N1): c_v = [lambda_v + rho_v < 0]
                 * for the unclamped CN output rho_v = (-1)^neg phi(S_k).  Since
                 * |rho_v| = phi(S_k), |lambda_v| = phi(p_k) and phi is decreasing,
                 * |rho_v| > |lambda_v| <=> S_k < p_k: equal signs decide by that sign,
                 * opposite signs by the larger magnitude, an exact tie gives 0. */
                int nl = x[k] < 0.0f;
                dec1[g->edge_vn[e]] = nl ? (uint8_t)(neg || p[k] < S) : (uint8_t)(neg && S < p[k]);
            }
        }
    }
    free(x); free(p); free(P); free(Q); free(slot_e);
}

/* DESIGN.md N3 (fp32 replay): the sum of Eq. (4)/(5) over C_i is taken exactly in
 * fixed point -- each message rounded to the nearest multiple of 2^-17 (ties to even),
 * the integers added exactly, the total converted to fp32 (round to nearest) and scaled:
 * L_i = lambda_i + (float)(sum_k rint(2^17 r_k)) * 2^-17.  An exact integer sum has no
 * order, so the result is independent of the order the messages arrive in. */
#define VN_FIX_BITS 17
static void vn_phase32(const graph_t* g, const float* lam, const float* r_new, float* L_new) {
    for (int a = 0; a < g->n_a; ++a) {
        int v = g->act_vn[a];
        int64_t acc = 0;
        for (int64_t k = g->vn_ptr[v]; k < g->vn_ptr[v + 1]; ++k) {
            float scaled = r_new[g->act_id[g->vn_edge[k]]] * (float)(1 << VN_FIX_BITS);   /* exact */
            acc += (int64_t)rintf(scaled);
        }
        float sum = (float)acc * (1.0f / (float)(1 << VN_FIX_BITS));
        L_new[a] = lam[v] + sum;
    }
}

static void decide32(const graph_t* g, const float* L, const uint8_t* dec1, uint8_t* c) {
    for (int v = 0; v < g->n; ++v)
        c[v] = (g->vn_act[v] >= 0) ? (L[g->vn_act[v]] < 0.0f) : dec1[v];
}

/* DESIGN.md N7: the stored copy of the messages under ORC_MSG16 (see above). */
static void store_msg16(float* r, int64_t E_it) {
    /* the integer q = rint(2^10 r) is what is stored (q = 0 reads back as +0); both products exact */
    for (int64_t e = 0; e < E_it; ++e) r[e] = (float)(int32_t)rintf(r[e] * 1024.0f) * (1.0f / 1024.0f);
}

static int all_finite32(const float* a, int n) {
    for (int i = 0; i < n; ++i) if (!isfinite(a[i])) return 0;
    return 1;
}

/* M3 decode of one frame.  r_trace/L_trace (optional) receive r^l [E_it] and
 * L^l [n_a] after every iteration l = 1..iters (active-edge CSR order /
 * active-VN ascending order).  Returns 0, or <0 on a malformed graph. */
int orc_decode_f32(int rule, int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                   const int64_t* vn_ptr, const int64_t* vn_edge,
                   const float* lam, const uint32_t* synd, int max_iter, int early_term,
                   uint8_t* bits_out, int32_t* iters_out, uint8_t* conv_out,
                   float* r_trace, float* L_trace) {
    graph_t g;
    int rc = graph_build(&g, n, m, cn_ptr, edge_vn, vn_ptr, vn_edge, rule);
    const int msg16 = (rule & ORC_MSG16) != 0;
    rule &= 0xff;
    if (rc) { graph_free(&g); return rc; }
    memset(bits_out, 0, (size_t)n);
    if (!all_finite32(lam, n)) { *iters_out = -1; *conv_out = 0; graph_free(&g); return 0; }
    size_t Ea = (size_t)(g.E_it > 0 ? g.E_it : 1), Na = (size_t)(g.n_a > 0 ? g.n_a : 1);
    float* r_old = calloc(Ea, 4); float* r_new = calloc(Ea, 4);
    float* L_old = malloc(Na * 4); float* L_new = malloc(Na * 4);
    uint8_t* dec1 = calloc((size_t)n, 1);
    for (int a = 0; a < g.n_a; ++a) L_old[a] = lam[g.act_vn[a]];   /* Step 2: L^0 = lambda, r^0 = 0 */
    int it = 0, conv = 0;
    for (int l = 1; l <= max_iter; ++l) {
        cn_phase32(&g, rule, lam, synd, r_old, L_old, r_new, dec1);
        vn_phase32(&g, lam, r_new, L_new);
        if (msg16) store_msg16(r_new, g.E_it);   /* what iteration l + 1 reads (N7) */
        decide32(&g, L_new, dec1, bits_out);
        if (r_trace) memcpy(r_trace + (size_t)(l - 1) * g.E_it, r_new, (size_t)g.E_it * 4);
        if (L_trace) memcpy(L_trace + (size_t)(l - 1) * g.n_a, L_new, (size_t)g.n_a * 4);
        float* t;
        t = r_old; r_old = r_new; r_new = t;
        t = L_old; L_old = L_new; L_new = t;
        it = l;
        if (early_term && syndrome_matches(&g, bits_out, synd)) { conv = 1; break; }
    }
    if (!early_term || !conv) conv = syndrome_matches(&g, bits_out, synd);
    *iters_out = it;
    *conv_out = (uint8_t)conv;
    free(r_old); free(r_new); free(L_old); free(L_new); free(dec1);
    graph_free(&g);
    return 0;
}

/* ---- fp64 (M2) ---- */
static void cn_phase64(const graph_t* g, int rule, const double* lam, const uint32_t* synd,
                       const double* r_old, const double* L_old, double* r_new, double* rho) {
    int D = g->max_cdeg;
    double* x = malloc(sizeof(double) * (size_t)D);
    double* p = malloc(sizeof(double) * (size_t)D);
    double* P = malloc(sizeof(double) * (size_t)(D + 1));
    double* Q = malloc(sizeof(double) * (size_t)D);
    int64_t* slot_e = malloc(sizeof(int64_t) * (size_t)D);
    for (int j = 0; j < g->m; ++j) {
        int d = 0;
        for (int64_t e = g->cn_ptr[j]; e < g->cn_ptr[j + 1]; ++e)
            if (g->act_id[e] >= 0) slot_e[d++] = e;
        for (int64_t e = g->cn_ptr[j]; e < g->cn_ptr[j + 1]; ++e)
            if (g->act_id[e] < 0) slot_e[d++] = e;
        if (d == 0) continue;
        int par = synd_bit(synd, j);
        for (int k = 0; k < d; ++k) {
            int64_t e = slot_e[k];
            int v = g->edge_vn[e];
            x[k] = (g->act_id[e] >= 0) ? L_old[g->vn_act[v]] - r_old[g->act_id[e]] : lam[v];
            p[k] = orc_phi64(rule, fabs(x[k]));
            par ^= (x[k] < 0.0);
        }
        P[0] = 0.0;
        for (int k = 0; k < d; ++k) P[k + 1] = P[k] + p[k];
        Q[d - 1] = 0.0;
        for (int k = d - 2; k >= 0; --k) Q[k] = Q[k + 1] + p[k + 1];
        for (int k = 0; k < d; ++k) {
            int64_t e = slot_e[k];
            /* R_MAX clamps the stored messages only (R6); a degree-1 VN's CN output is not
             * stored, its decision takes the unclamped posterior lambda + rho (N1) */
            double mag = orc_phi64(rule, P[k] + Q[k]);
            if (g->act_id[e] >= 0) mag = fmin(mag, R_MAX);
            double o = (par ^ (x[k] < 0.0)) ? -mag : mag;
            if (g->act_id[e] >= 0) r_new[g->act_id[e]] = o;
            else rho[g->edge_vn[e]] = o;
        }
    }
    free(x); free(p); free(P); free(Q); free(slot_e);
}

static void vn_phase64(const graph_t* g, const double* lam, const double* r_new, double* L_new) {
    for (int a = 0; a < g->n_a; ++a) {
        int v = g->act_vn[a];
        double acc = lam[v];
        for (int64_t k = g->vn_ptr[v]; k < g->vn_ptr[v + 1]; ++k) acc += r_new[g->act_id[g->vn_edge[k]]];
        L_new[a] = acc;
    }
}

static void decide64(const graph_t* g, const double* lam, const double* L, const double* rho, uint8_t* c) {
    for (int v = 0; v < g->n; ++v)
        c[v] = (g->vn_act[v] >= 0) ? (L[g->vn_act[v]] < 0.0) : ((lam[v] + rho[v]) < 0.0);
}

int orc_decode_f64(int rule, int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                   const int64_t* vn_ptr, const int64_t* vn_edge,
                   const double* lam, const uint32_t* synd, int max_iter, int early_term,
                   uint8_t* bits_out, int32_t* iters_out, uint8_t* conv_out,
                   double* r_trace, double* L_trace, double* post_out /*[n] or NULL*/) {
    graph_t g;
    int rc = graph_build(&g, n, m, cn_ptr, edge_vn, vn_ptr, vn_edge, rule);
    rule &= 0xff;
    if (rc) { graph_free(&g); return rc; }
    memset(bits_out, 0, (size_t)n);
    for (int i = 0; i < n; ++i)
        if (!isfinite(lam[i])) { *iters_out = -1; *conv_out = 0; graph_free(&g); return 0; }
    size_t Ea = (size_t)(g.E_it > 0 ? g.E_it : 1), Na = (size_t)(g.n_a > 0 ? g.n_a : 1);
    double* r_old = calloc(Ea, 8); double* r_new = calloc(Ea, 8);
    double* L_old = malloc(Na * 8); double* L_new = malloc(Na * 8);
    double* rho = calloc((size_t)n, 8);
    for (int a = 0; a < g.n_a; ++a) L_old[a] = lam[g.act_vn[a]];
    int it = 0, conv = 0;
    for (int l = 1; l <= max_iter; ++l) {
        cn_phase64(&g, rule, lam, synd, r_old, L_old, r_new, rho);
        vn_phase64(&g, lam, r_new, L_new);
        decide64(&g, lam, L_new, rho, bits_out);
        if (r_trace) memcpy(r_trace + (size_t)(l - 1) * g.E_it, r_new, (size_t)g.E_it * 8);
        if (L_trace) memcpy(L_trace + (size_t)(l - 1) * g.n_a, L_new, (size_t)g.n_a * 8);
        double* t;
        t = r_old; r_old = r_new; r_new = t;
        t = L_old; L_old = L_new; L_new = t;
        it = l;
        if (early_term && syndrome_matches(&g, bits_out, synd)) { conv = 1; break; }
    }
    if (!early_term || !conv) conv = syndrome_matches(&g, bits_out, synd);
    if (post_out)   /* Eq. (5) posterior LLR of every VN at the last iteration */
        for (int v = 0; v < n; ++v)
            post_out[v] = (g.vn_act[v] >= 0) ? L_old[g.vn_act[v]] : lam[v] + rho[v];
    *iters_out = it;
    *conv_out = (uint8_t)conv;
    free(r_old); free(r_new); free(L_old); free(L_new); free(rho);
    graph_free(&g);
    return 0;
}

/* One fp64 iteration from a given state (r^{l-1}, L^{l-1}) -> (r^l, L^l):
 * the teacher-forced step used to bound the fp32 replay against the fp64
 * definition one iteration at a time (parity). */
int orc_step_f64(int rule, int n, int m, const int64_t* cn_ptr, const int32_t* edge_vn,
                 const int64_t* vn_ptr, const int64_t* vn_edge,
                 const double* lam, const uint32_t* synd, const double* r_in, const double* L_in,
                 double* r_out, double* L_out) {
    graph_t g;
    int rc = graph_build(&g, n, m, cn_ptr, edge_vn, vn_ptr, vn_edge, rule);
    rule &= 0xff;
    if (rc) { graph_free(&g); return rc; }
    double* rho = calloc((size_t)n, 8);
    cn_phase64(&g, rule, lam, synd, r_in, L_in, r_out, rho);
    vn_phase64(&g, lam, r_out, L_out);
    free(rho);
    graph_free(&g);
    return 0;
}

/* ------------------------------------------------------------------ LLR from MD output */

/* DESIGN.md reading R13: lambda_i = 2 sqrt(snr (1 + snr)) * |x|_blk * v_i
 * (sigma_X^2 = 1, bit 0 <-> +).  fp32 replay: c = (float)(2 sqrt(snr(1+snr)))
 * computed in double from the float snr; xb = xnorm[i/d] or (float)sqrt(d);
 * lambda = (c * xb) * v in fp32, in that order. */
void orc_llr_from_md_f32(int n, int d, float snr, const float* v, const float* xnorm, float* out) {
    double s = (double)snr;
    float c = (float)(2.0 * sqrt(s * (1.0 + s)));
    float xd = (float)sqrt((double)d);
    for (int i = 0; i < n; ++i) {
        float xb = xnorm ? xnorm[i / d] : xd;
        float cx = c * xb;
        out[i] = cx * v[i];
    }
}

void orc_llr_from_md_f64(int n, int d, double snr, const double* v, const double* xnorm, double* out) {
    double c = 2.0 * sqrt(snr * (1.0 + snr));
    for (int i = 0; i < n; ++i) out[i] = c * (xnorm ? xnorm[i / d] : sqrt((double)d)) * v[i];
}

/* ------------------------------------------------------------------ MD on the raw block (NEXT #1) */

/* Basis products of the d-dimensional Cayley-Dickson algebra (d = 1, 2, 4, 8) with
 * (a1, a2)(b1, b2) = (a1 b1 - conj(b2) a2, b2 a1 + a2 conj(b1)): e_p e_q = sgn * e_r.
 * Built recursively on basis indices (oracle's own implementation). */
static void cd_basis(int d, int p, int q, int* r, int* sgn) {
    if (d == 1) { *r = 0; *sgn = 1; return; }
    int h = d / 2;
    int pa = p >= h, qa = q >= h, pl = p % h, ql = q % h;
    int rr, ss;
    if (!pa && !qa) {            /* (a1,0)(b1,0) = (a1 b1, 0) */
        cd_basis(h, pl, ql, &rr, &ss); *r = rr; *sgn = ss;
    } else if (!pa && qa) {      /* (a1,0)(0,b2) = (0, b2 a1) */
        cd_basis(h, ql, pl, &rr, &ss); *r = h + rr; *sgn = ss;
    } else if (pa && !qa) {      /* (0,a2)(b1,0) = (0, a2 conj(b1)) */
        cd_basis(h, pl, ql, &rr, &ss); *r = h + rr; *sgn = ss * ((ql == 0) ? 1 : -1);
    } else {                     /* (0,a2)(0,b2) = (-conj(b2) a2, 0) */
        cd_basis(h, ql, pl, &rr, &ss); *r = rr; *sgn = -ss * ((ql == 0) ? 1 : -1);
    }
}

/* DESIGN.md N6: (a b)_i = sum over q of sgn * a_p * b_q with e_p e_q = sgn e_i, evaluated
 * as acc = fmaf(sgn * a_p, b_q, acc) for q = 0..d-1 from acc = 0; lambda_i = c * (alpha x)_i
 * with c = (float)(2 sqrt(snr (1 + snr))) -- since M(alpha) is linear, c |x| (alpha x^)_i =
 * c (alpha x)_i (R13 without the normalisation). */
void orc_md_alice_f32(int n, int d, float snr, const float* x, const float* alpha, float* out) {
    int kp[8][8], ks[8][8];
    for (int i = 0; i < d; ++i)
        for (int q = 0; q < d; ++q)
            for (int p = 0; p < d; ++p) {
                int r, sg;
                cd_basis(d, p, q, &r, &sg);
                if (r == i) { kp[i][q] = p; ks[i][q] = sg; }
            }
    double s = (double)snr;
    float c = (float)(2.0 * sqrt(s * (1.0 + s)));
    for (int b = 0; b < n / d; ++b) {
        const float* a = alpha + (size_t)b * d;
        const float* xb = x + (size_t)b * d;
        for (int i = 0; i < d; ++i) {
            float acc = 0.0f;
            for (int q = 0; q < d; ++q) {
                float ap = ks[i][q] > 0 ? a[kp[i][q]] : -a[kp[i][q]];
                acc = fmaf(ap, xb[q], acc);
            }
            out[(size_t)b * d + i] = c * acc;
        }
    }
}

/* Basis table for tests: k[i*d + q] = p, s[i*d + q] = sgn. */
void orc_md_table(int d, int* k, int* sg) {
    for (int i = 0; i < d; ++i)
        for (int q = 0; q < d; ++q)
            for (int p = 0; p < d; ++p) {
                int r, s2;
                cd_basis(d, p, q, &r, &s2);
                if (r == i) { k[i * d + q] = p; sg[i * d + q] = s2; }
            }
}
