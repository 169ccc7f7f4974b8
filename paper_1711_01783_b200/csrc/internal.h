// internal.h -- private structures of libmetldpc (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/metldpc.h"

namespace metldpc {

constexpr int kMaxCnDeg = 32;          // templated CN kernel bound (metldpc.h: EUNSUPPORTED above)
// DESIGN.md N3: deg * (2^22 + 30 * 2^17) < 2^32, so the biased fixed-point VN sum never wraps
constexpr int kMaxVnDeg = 512;
constexpr float kRMax = 30.0f;         // DESIGN.md R6
// phi tables (N2): 2^J bins per binade on [2^-44, 2^6); EXACT J = 4 (cubic,
// 4 floats/bin), PHI_LUT J = 5 (linear, 2 floats/bin).
constexpr int kPhiELo = -44, kPhiEHi = 6;
constexpr int kPhiJExact = 4, kPhiJLut = 5;
constexpr int kPhiBinsExact = (kPhiEHi - kPhiELo) << kPhiJExact;   // 800
constexpr int kPhiBinsLut = (kPhiEHi - kPhiELo) << kPhiJLut;       // 1600
constexpr uint32_t kPhiLoBits = uint32_t(127 + kPhiELo) << 23;     // 2^-44
constexpr uint32_t kPhiHiBits = uint32_t(127 + kPhiEHi) << 23;     // 2^6
// The device copy appends one binade of all-zero bins, [2^6, 2^7): phi = 0 there as above, so
// a sum S < 2^7 (every S of a check of total degree <= 5: S <= 4 phi(2^-44) = 124.8) needs no
// upper clamp (kernels.cu phi_pair<RULE, false>).
constexpr int kPhiZeroBinsExact = 1 << kPhiJExact, kPhiZeroBinsLut = 1 << kPhiJLut;
// Device copy: each bin (plus one all-zero sentinel bin) replicated kPhiCopies times,
// interleaved, so the 8 threads of a quarter-warp LDS phase read 8 distinct bank groups.
#ifndef METLDPC_PHI_COPIES
#define METLDPC_PHI_COPIES 8
#endif
constexpr int kPhiCopies = METLDPC_PHI_COPIES;

void set_error(const std::string& msg);
metldpc_status fail(metldpc_status s, const std::string& msg);

// Host layout of H (DESIGN.md section 6 "Data layout").
//   CN label        j' in [0, m): CNs relabelled so every degree class is one contiguous
//                   range (classes by total degree D = 0..16, then one class for 17..32),
//                   ascending original index within a class (classes with one degree-1
//                   slot: ascending original index of the degree-1 VN)
//   active VN index a in [0, n_a): VNs of degree >= 2, ascending original index
//   active edge id  t in [0, E_it): edges of active VNs, CN-major in j' order, CSR order
//                   within a row (perm_r maps t to the canonical active-edge CSR order)
//   degree-1 slot   q in [0, n_1): edges of degree-1 VNs, same order (so a class with one
//                   degree-1 slot has them in ascending original VN order)
struct HostLayout {
    int32_t n = 0, m = 0;
    int64_t E = 0, E_it = 0;
    int32_t n_a = 0, n_1 = 0, max_cn_deg = 0, max_vn_deg = 0;
    std::vector<int32_t> cn_aptr;   // [m+1] active-edge offsets per CN
    std::vector<int32_t> cn_dptr;   // [m+1] degree-1 slot offsets per CN
    std::vector<int32_t> a_vn;      // [E_it] active VN index of active edge t
    std::vector<int32_t> vn_aptr;   // [n_a+1] offsets into vn_aedge
    std::vector<int32_t> vn_aedge;  // [E_it] active edge ids of active VN a, caller's CSC order
    std::vector<int32_t> vmap;      // [n] a (>= 0) for active VNs, ~q (< 0) for degree-1
    std::vector<int32_t> act_vn;    // [n_a] original VN id of active index
    std::vector<int32_t> cn_new;    // [m] original CN id -> j'
    std::vector<int32_t> perm_r;    // [E_it] t -> canonical active-edge id
    std::vector<int32_t> csr_ptr;   // [m+1] caller's CSR row offsets (int32)
    std::vector<int32_t> csr_vn;    // [E]   caller's CSR edge VNs
    // CN degree classes: contiguous j' ranges with one total degree D <= 16 and nd <= 1
    // degree-1 slots (a kernel instantiation per (D, nd), registers sized for it), or the
    // generic class (D = -1: nd >= 2 or degree 17..32).
    struct CnClass { int D, nd; int32_t begin, count; };
    std::vector<CnClass> classes;
};

constexpr int kMaxUnrolledCnDeg = 16;

// Validates the edge-indexed CSR/CSC and builds the layout.  Returns OK/EFORMAT/EUNSUPPORTED.
metldpc_status build_layout(int32_t n, int32_t m, int64_t E, const int64_t* cn_ptr,
                            const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                            HostLayout* out, uint32_t flags);

void fill_info(const HostLayout& L, metldpc_code_info_t* info);

// fp32 phi tables (N2), generated here independently of the oracle.
void phi_table_exact(float* out /*kPhiBinsExact*4*/);
void phi_table_lut(float* out /*kPhiBinsLut*2*/);
// replicated device layout [bin 0..nbins (sentinel)][copy][coefficients]
std::vector<float> phi_device_table(int rule);
float phi_top();
// Cayley-Dickson basis table for d in {1,2,4,8}: (a b)_i = sum_q ks[i d + q] a_{kp[i d + q]} b_q.
void md_product_table(int d, int8_t* kp, int8_t* ks);

}  // namespace metldpc

struct metldpc_code_s {
    int device = 0;
    metldpc::HostLayout host;
    // device copies (int32)
    int32_t* d_cn_aptr = nullptr;
    int32_t* d_cn_dptr = nullptr;
    int32_t* d_a_vn = nullptr;
    int32_t* d_vn_aptr = nullptr;
    int32_t* d_vn_aedge = nullptr;
    int32_t* d_vmap = nullptr;
    int32_t* d_cn_new = nullptr;
    int32_t* d_csr_ptr = nullptr;   // original CSR (int32) for the syndrome kernel (Step 1)
    int32_t* d_csr_vn = nullptr;
    float* d_phi_exact = nullptr;   // (kPhiBinsExact + kPhiZeroBinsExact) * 8 copies * 4
    float* d_phi_lut = nullptr;     // (kPhiBinsLut + kPhiZeroBinsLut) * 8 copies * 2
    int num_sms = 148;
};
