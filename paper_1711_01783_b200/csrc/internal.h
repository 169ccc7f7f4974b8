// internal.h -- private structures of libmetldpc (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/metldpc.h"

namespace metldpc {

constexpr int kMaxCnDeg = 32;          // templated CN kernel bound (metldpc.h: EUNSUPPORTED above)
constexpr float kRMax = 30.0f;         // DESIGN.md R6
constexpr int kPhiELo = -44, kPhiEHi = 6, kPhiJ = 5;
constexpr int kPhiBins = (kPhiEHi - kPhiELo) << kPhiJ;      // 1600
constexpr uint32_t kPhiLoBits = uint32_t(127 + kPhiELo) << 23;  // 2^-44
constexpr uint32_t kPhiHiBits = uint32_t(127 + kPhiEHi) << 23;  // 2^6

void set_error(const std::string& msg);
metldpc_status fail(metldpc_status s, const std::string& msg);

// Host layout of H (DESIGN.md section 6 "Data layout").
//   active VN index a in [0, n_a): VNs of degree >= 2, ascending original index
//   active edge id  t in [0, E_it): CSR edges of active VNs, CSR order
//   degree-1 slot   q in [0, n_1): CSR edges of degree-1 VNs, CSR order
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
    // CN degree classes: CNs grouped by total-degree window so each class kernel
    // gets a register budget sized for its own degree (kernels.cu k_cn_update).
    struct CnClass { int dlo, dhi; int32_t begin, count; };
    std::vector<CnClass> classes;
    std::vector<int32_t> cls_cn;    // [m] CN ids, grouped by class, ascending within a class
};

// Degree windows of the CN classes: [0,4] [5,8] [9,12] [13,16] unrolled; [17,32] generic.
constexpr int kNumCnWindows = 5;
constexpr int kCnWinLo[kNumCnWindows] = {0, 5, 9, 13, 17};
constexpr int kCnWinHi[kNumCnWindows] = {4, 8, 12, 16, 32};

// Validates the edge-indexed CSR/CSC and builds the layout.  Returns OK/EFORMAT/EUNSUPPORTED.
metldpc_status build_layout(int32_t n, int32_t m, int64_t E, const int64_t* cn_ptr,
                            const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                            HostLayout* out);

void fill_info(const HostLayout& L, metldpc_code_info_t* info);

// fp32 phi tables (N2), generated here independently of the oracle.
void phi_table_exact(float* out /*kPhiBins*4*/);
void phi_table_lut(float* out /*kPhiBins*2*/);
float phi_top();

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
    int32_t* d_cls_cn = nullptr;
    float* d_phi_exact = nullptr;   // kPhiBins * 4
    float* d_phi_lut = nullptr;     // kPhiBins * 2
    int num_sms = 148;
};
