// kernels.cu -- sm_100a kernels of the batched syndrome BP decoder (arXiv 1711.01783).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false: every fp32
// operation below is the one DESIGN.md N1-N5 writes, no FMA contraction; the
// only fused multiply-adds are the explicit __fmaf_rn of the phi table (N2).
//
// Mapping: one warp = one node (CN or VN) x 32 codeword lanes.
// All 32 threads of a warp therefore run the same degree -> no divergence, and
// every per-lane access is one full 128-byte line of a codeword-interleaved
// array.  CN and VN kernels are persistent (grid = SMs x resident CTAs) so each
// CTA loads the phi table into shared memory once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "internal.h"
#include "kernels.cuh"

namespace metldpc {

#define FULL 0xffffffffu

// ------------------------------------------------------------------ phi (N2)

// Device table layout: [bin 0..NB-1, NB..NB+ZB-1 zero bins][copy 0..7][coefficients]; a thread
// reads copy (lane & 7), so the 8 threads of an LDS phase hit 8 distinct bank groups
// whatever their bins (no shared-memory bank conflicts, 1 wavefront per phase).
template <int RULE>
struct PhiT;
template <>
struct PhiT<METLDPC_RULE_EXACT> {      // cubic Hermite, 16 bins per binade
    static constexpr int J = kPhiJExact, ENTRY = 16, NB = kPhiBinsExact, ZB = kPhiZeroBinsExact;
    static constexpr int STRIDE = kPhiCopies * ENTRY;                        // bytes per bin
    static constexpr int BIAS = int(kPhiLoBits >> (23 - J)) * STRIDE;       // bin(2^-44) * STRIDE
    static constexpr int TAB_BYTES = (NB + ZB) * STRIDE;
};
template <>
struct PhiT<METLDPC_RULE_PHI_LUT> {    // linear, 32 bins per binade
    static constexpr int J = kPhiJLut, ENTRY = 8, NB = kPhiBinsLut, ZB = kPhiZeroBinsLut;
    static constexpr int STRIDE = kPhiCopies * ENTRY;
    static constexpr int BIAS = int(kPhiLoBits >> (23 - J)) * STRIDE;
    static constexpr int TAB_BYTES = (NB + ZB) * STRIDE;
};

// phi(y), y >= 0, exactly as DESIGN.md N2: clamping the bit pattern to [2^-44, 2^6]
// reproduces both out-of-range rules with no selects (u = 2^-44: bin 0, t = 0, c0 =
// (float)phi(2^-44) = PHI_TOP; u = 2^6: the first zero bin, +0).  The bin's byte
// offset is (u >> (23 - J)) * STRIDE = (u with the low 23-J bits cleared) >> 12.
// The device table stores the coefficients pre-scaled by powers of two, c_k * 2^(J k),
// and the polynomial runs in ts = t / 2^J = bits(1.0 | low mantissa bits) - 1 (exact):
// scaling by a power of two commutes with rounding, so every Horner intermediate is the
// oracle's times 2^(J k) and the result is bit-identical to N2 as written.
// (a & m) | c in one LOP3: c is kept in a register (an immediate would split the op in two).
template <uint32_t M>
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(M), "r"(c));
    return d;
}

// 1.0f as an opaque register value (see and_or).
__device__ __forceinline__ uint32_t one_bits() {
    uint32_t c;
    asm("mov.b32 %0, 0x3F800000;" : "=r"(c));
    return c;
}

// Bit pattern of y clamped to [2^-44, 2^6].  For y >= +0 (or y = |x|) the float order is the
// order of the bit patterns, so this equals the integer clamp of N2; as FMNMX it folds the
// |x| of the callers into an operand modifier.  (A NaN, only possible in an invalid frame
// whose lane is discarded, clamps to 2^-44.)
__device__ __forceinline__ uint32_t phi_clamp_bits(float y) {
    return __float_as_uint(fminf(fmaxf(y, __uint_as_float(kPhiLoBits)), __uint_as_float(kPhiHiBits)));
}

// tabk: 32-bit shared-window address of this lane's table copy minus BIAS (phi_tab_lane).
template <int RULE>
__device__ __forceinline__ float phi_dev(uint32_t tabk, float y, uint32_t one) {
    using P = PhiT<RULE>;
    constexpr uint32_t LOW = (1u << (23 - P::J)) - 1u;
    const uint32_t u = phi_clamp_bits(y);
    uint32_t e;   // tabk + bin * STRIDE as one IMAD (FMA pipe) after the shift
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e) : "r"(u >> (23 - P::J)), "n"(P::STRIDE), "r"(tabk));
    const float ts = __fsub_rn(__uint_as_float(and_or<LOW>(u, one)), 1.0f);
    if constexpr (RULE == METLDPC_RULE_EXACT) {
        float4 c;
        asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w) : "r"(e));
        return __fmaf_rn(__fmaf_rn(__fmaf_rn(c.w, ts, c.z), ts, c.y), ts, c.x);
    } else {
        float2 c;
        asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(c.x), "=f"(c.y) : "r"(e));
        return __fmaf_rn(c.y, ts, c.x);
    }
}

// The table copy of this lane as a 32-bit shared-window address with the bin bias folded
// in, held opaquely in one register (the bin offset then costs SHF + LEA).
template <int RULE>
__device__ __forceinline__ uint32_t phi_tab_lane(const char* smem, int lane) {
    const uint32_t a = uint32_t(__cvta_generic_to_shared(smem)) + uint32_t((lane & (kPhiCopies - 1)) * PhiT<RULE>::ENTRY) -
                       uint32_t(PhiT<RULE>::BIAS);
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(a));
    return r;
}

// phi(y) of the selected rule read from copy 0 of the device table in global memory -- the
// same N2 formula as phi_dev, for the once-per-frame users (the degree-1 priors of k_scatter).
template <int RULE>
__device__ __forceinline__ float phi_gmem_rule(const float* tab, float y) {
    using P = PhiT<RULE>;
    constexpr uint32_t LOW = (1u << (23 - P::J)) - 1u;
    const uint32_t u = phi_clamp_bits(y);
    const char* e = reinterpret_cast<const char*>(tab) + size_t((u >> (23 - P::J)) - (kPhiLoBits >> (23 - P::J))) * P::STRIDE;
    const float ts = __fsub_rn(__uint_as_float((u & LOW) | 0x3F800000u), 1.0f);
    if constexpr (RULE == METLDPC_RULE_EXACT) {
        const float4 c = __ldg(reinterpret_cast<const float4*>(e));
        return __fmaf_rn(__fmaf_rn(__fmaf_rn(c.w, ts, c.z), ts, c.y), ts, c.x);
    } else {
        const float2 c = __ldg(reinterpret_cast<const float2*>(e));
        return __fmaf_rn(c.y, ts, c.x);
    }
}

// lam1 layout: [n_1 / 8][B lanes][8].  Lane b's priors of 8 consecutive
// degree-1 slots fill one 32-byte sector, so a frame's priors are written in whole sectors (the
// refill wave writes one lane at a time); a ring stage of 24 consecutive checks is 3 contiguous
// blocks (one bulk copy).  The slot inside the sector is XOR-swizzled by lane, so the 32 lanes
// of a warp reading one slot hit 32 distinct shared-memory banks.
__host__ __device__ __forceinline__ size_t lam1_idx(int q, int b, int B) {
    return size_t(q >> 3) * size_t(8 * B) + size_t(b) * 8 + size_t((q & 7) ^ ((b >> 2) & 7));
}

// Degree-1 prior as the CN kernels read it (N1): phi(|lambda|) with the sign bit
// [lambda < 0] (an input of -0 carries no sign, R2).
__device__ __forceinline__ float lam1_phi_form(const CodeDev& cd, float lam) {
    const float ph = (cd.rule == METLDPC_RULE_EXACT) ? phi_gmem_rule<METLDPC_RULE_EXACT>(cd.phi, fabsf(lam))
                                                     : phi_gmem_rule<METLDPC_RULE_PHI_LUT>(cd.phi, fabsf(lam));
    return __uint_as_float(__float_as_uint(ph) | (lam < 0.0f ? 0x80000000u : 0u));
}

template <int RULE>
__device__ __forceinline__ void load_phi_table(char* smem, const float* phi) {
    using P = PhiT<RULE>;
    for (int i = threadIdx.x; i < P::TAB_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = __ldg(reinterpret_cast<const uint4*>(phi) + i);
}

// ------------------------------------------------------------------ check-node update (a2 + a4)

// The CN classes of one iteration are independent (disjoint CNs and r rows; the VN sums are
// order-free integer atomics), so each class launch lets the next one start on SMs it has
// released (programmatic dependent launch).  Every class kernel waits for its predecessor at
// its very end, so the finish kernel, a normal launch after the last class, still sees all
// of them complete.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_previous() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Whether the group has finished (every lane latched), read once per block so that every
// thread of the block takes the same early exit (one barrier).
__device__ __forceinline__ bool block_done(const Group& g) {
    __shared__ int s_done;
    if (threadIdx.x == 0) s_done = *reinterpret_cast<volatile int*>(g.done);
    __syncthreads();
    return s_done != 0;
}

struct CnCtl {
    int check;   // test the syndrome of iteration l-1 (reads L^{l-1}, degree-1 bits[rpar])
    int rpar, wpar;
    int dev;     // 1: take l from Group::iter (CUDA-graph loop); check = et && l >= 2
    int et;
};

// Resolves the iteration controls of a CN launch (host-given or device-driven).
__device__ __forceinline__ CnCtl cn_ctl(CnCtl k, const Group& g) {
    if (k.dev) {
        const int l = *reinterpret_cast<volatile int*>(g.iter);
        k.check = k.et && l >= 2;
        k.rpar = (l - 1) & 1;
        k.wpar = l & 1;
    }
    return k;
}

constexpr int kCnThreads = 512;   // 2 CTAs x 16 warps per SM (the replicated table is 100 KB)

// DESIGN.md N1 for one CN and one lane (fp32, slot order: actives, then the degree-1
// slot): Eqs. (2)-(3) in sign/phi form with the syndrome sign (R1).
// Returns the syndrome-test bit (N4) of iteration l-1; writes r for active slots and
// the degree-1 decision bit.
// Fixed-point VN-sum term of a message (N3): bits(fmaf(o, 2^17, 1.5 * 2^23)) =
// 0x4B400000 + rint(2^17 o) exactly for |2^17 o| < 2^22 (|o| <= 30); the finish kernel
// removes the 0x4B400000 bias (degree times, modulo 2^32).
__device__ __forceinline__ uint32_t vn_fix(float o) {
    return __float_as_uint(__fmaf_rn(o, 131072.0f, 12582912.0f));
}

// Degree-1 decision (Step 5; N1): bit = [lambda + rho < 0] for the
// unclamped posterior, with |rho| = phi(S) and |lambda| = phi(p), p = phi(|lambda|) the
// stored prior.  phi is a decreasing involution, so |rho| > |lambda| <=> S < p and the
// decision needs no phi(S): equal signs give that sign, opposite signs the sign of the
// larger magnitude, an exact tie 0.  nl / nr: sign bits (bit 31) of lambda and rho.
__device__ __forceinline__ uint32_t d1_decision(uint32_t nl, uint32_t nr, float p, float S) {
    nl >>= 31;
    nr >>= 31;
    return nl ? (nr | uint32_t(p < S)) : (nr & uint32_t(S < p));
}

// ------------------------------------------------------------------ two-lane (fp32x2) helpers

// sm_100a packed fp32 pairs: FADD2 / FFMA2 round each element to nearest like FADD / FFMA,
// so a pair op is bit-identical to two scalar ops; it halves the instruction count of the
// two codeword lanes a thread carries.
__device__ __forceinline__ unsigned long long f2pack(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pack(a)), "l"(f2pack(b)));
    return f2unpack(r);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pack(a)), "l"(f2pack(b)));
    return f2unpack(r);
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pack(a)), "l"(f2pack(b)), "l"(f2pack(c)));
    return f2unpack(r);
}

// phi of two lanes: integer bin/mantissa work per lane, ts - 1 as one FADD2.  UPPER = false:
// the caller guarantees y < 2^7 (the zero bins above 2^6 then give phi = 0 with no clamp).
template <int RULE, bool UPPER = true>
__device__ __forceinline__ float2 phi_pair(uint32_t tabk, float y0, float y1, uint32_t one) {
    using P = PhiT<RULE>;
    constexpr uint32_t LOW = (1u << (23 - P::J)) - 1u;
    const uint32_t u0 = UPPER ? phi_clamp_bits(y0) : __float_as_uint(fmaxf(y0, __uint_as_float(kPhiLoBits)));
    const uint32_t u1 = UPPER ? phi_clamp_bits(y1) : __float_as_uint(fmaxf(y1, __uint_as_float(kPhiLoBits)));
    uint32_t e0, e1;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e0) : "r"(u0 >> (23 - P::J)), "n"(P::STRIDE), "r"(tabk));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(e1) : "r"(u1 >> (23 - P::J)), "n"(P::STRIDE), "r"(tabk));
    const float2 ts = f2add(make_float2(__uint_as_float(and_or<LOW>(u0, one)), __uint_as_float(and_or<LOW>(u1, one))),
                            make_float2(-1.0f, -1.0f));
    float2 r;
    if constexpr (RULE == METLDPC_RULE_EXACT) {
        float4 c0, c1;
        asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(c0.x), "=f"(c0.y), "=f"(c0.z), "=f"(c0.w) : "r"(e0));
        asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(c1.x), "=f"(c1.y), "=f"(c1.z), "=f"(c1.w) : "r"(e1));
        r.x = __fmaf_rn(__fmaf_rn(__fmaf_rn(c0.w, ts.x, c0.z), ts.x, c0.y), ts.x, c0.x);
        r.y = __fmaf_rn(__fmaf_rn(__fmaf_rn(c1.w, ts.y, c1.z), ts.y, c1.y), ts.y, c1.x);
    } else {
        float2 c0, c1;
        asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(c0.x), "=f"(c0.y) : "r"(e0));
        asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(c1.x), "=f"(c1.y) : "r"(e1));
        r.x = __fmaf_rn(c0.y, ts.x, c0.x);
        r.y = __fmaf_rn(c1.y, ts.y, c1.x);
    }
    return r;
}

// DESIGN.md N1 for one CN and the two lanes (l, l + 32) of a thread (slot order: actives, then the
// degree-1 slot; Eqs. (2)-(3), in sign/phi form with the syndrome sign, R1), the two
// lanes' identical fp32 operations as packed pairs.  Returns the syndrome-test bits (N4) of
// iteration l - 1; stores r for the active slots and returns the degree-1 decision bits.
// Fixed-point VN-sum term of a message (N3): bits(fmaf(o, 2^17, 1.5 * 2^23)) = 0x4B400000 +
// rint(2^17 o) exactly for |2^17 o| < 2^22 (|o| <= 30); the finish kernel removes the bias.
// 16-bit message storage (R28 / N7), the two lanes of a thread in one 32-bit word
// (lane l in the low half, lane l + 32 in the high half).  A stored half-word is w = q + 0x8080
// for the message q * 2^-10, q = rint(2^10 o): fmaf(o, 2^10, 2^23 + 0x8080) = 2^23 + w exactly
// (|q| <= 30720), so w is the low half of its bit pattern, and byte-filling a row with 0x80
// stores q = 0 (r^0 = 0, Step 2).  Read back: PRMT puts w under the exponent of 2^23, one
// exact FADD2 removes 2^23 + 0x8080.
constexpr float kMsg16Magic = 8421504.0f;   // 2^23 + 0x8080
__device__ __forceinline__ float2 msg16_q(uint32_t w) {
    uint32_t a, b;
    const uint32_t e = 0x4B000000u;   // bits of 2^23
    asm("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(a) : "r"(w), "r"(e));
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(b) : "r"(w), "r"(e));
    return f2sub(make_float2(__uint_as_float(a), __uint_as_float(b)), make_float2(kMsg16Magic, kMsg16Magic));
}
__device__ __forceinline__ uint32_t msg16_pack(float2 o) {
    const float2 f = f2fma(o, make_float2(1024.0f, 1024.0f), make_float2(kMsg16Magic, kMsg16Magic));
    uint32_t w;
    asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(w) : "r"(__float_as_uint(f.x)), "r"(__float_as_uint(f.y)));
    return w;
}

// MSG = 0: r rows of fp32 (pr: float row pointer, ro: the messages).  MSG = 1: 16-bit rows
// (pr: the thread's word of the row as uint32_t*, ro: the integers q of the stored messages,
// x = fmaf(q, -2^-10, L) = the single rounding of L - q 2^-10, N7).
template <int RULE, int NA, int ND, int MSG = 0>
__device__ __forceinline__ uint2 cn_pair(uint32_t tabk, const float2 (&Lv)[NA > 0 ? NA : 1],
                                         const float2 (&ro)[NA > 0 ? NA : 1], float2 lam, uint2 sbit, uint2 d1prev,
                                         void* prv, float* pla, const uint32_t (&offs)[NA > 0 ? NA : 1],
                                         uint2& d1bit) {
    float* pr = static_cast<float*>(prv);
    constexpr int D = NA + ND;
    const uint32_t one = one_bits();
    const float2 zero2 = make_float2(0.0f, 0.0f);
    float2 p[D], P[D];
    uint32_t xb0[D], xb1[D];
    uint32_t par0 = sbit.x << 31, par1 = sbit.y << 31;
    uint32_t lw0 = 0, lw1 = 0;   // XOR of the L words: bit 31 = parity of the active decisions
#pragma unroll
    for (int s = 0; s < NA; ++s) {
        const float2 x = MSG ? f2fma(ro[s], make_float2(-0.0009765625f, -0.0009765625f), Lv[s])
                             : f2sub(Lv[s], ro[s]);                       // extrinsic q = L - r (R10)
        // [L < 0] and [x < 0] are the sign bits: L and x are never -0 (see k_scatter)
        lw0 ^= __float_as_uint(Lv[s].x);
        lw1 ^= __float_as_uint(Lv[s].y);
        xb0[s] = __float_as_uint(x.x);
        xb1[s] = __float_as_uint(x.y);
        par0 ^= xb0[s];
        par1 ^= xb1[s];
        p[s] = phi_pair<RULE>(tabk, fabsf(x.x), fabsf(x.y), one);
    }
    if constexpr (ND > 0) {          // degree-1 prior in phi form (N1): sign = [lambda < 0], |.| = phi(|lambda|)
        xb0[NA] = __float_as_uint(lam.x);
        xb1[NA] = __float_as_uint(lam.y);
        par0 ^= xb0[NA];
        par1 ^= xb1[NA];
        p[NA] = make_float2(fabsf(lam.x), fabsf(lam.y));
    }
    P[0] = zero2;
    if constexpr (D > 1) P[1] = p[0];
#pragma unroll
    for (int s = 2; s < D; ++s) P[s] = f2add(P[s - 1], p[s - 1]);
    float2 Q = zero2;
#pragma unroll
    for (int s = D - 1; s >= 0; --s) {
        const float2 S = (s == D - 1) ? P[s] : (s == 0 ? Q : f2add(P[s], Q));
        if (s >= NA) {   // Step 5 for the degree-1 VN (N1): no phi(S) needed
            d1bit = make_uint2(d1_decision(xb0[s], par0 ^ xb0[s], p[s].x, S.x),
                               d1_decision(xb1[s], par1 ^ xb1[s], p[s].y, S.y));
            if (s > 0) Q = f2add(Q, p[s]);
            continue;
        }
        // S <= (D - 1) phi(2^-44) = 31.2 (D - 1) < 2^7 for D <= 5: no upper clamp needed
        const float2 ph = phi_pair<RULE, (D > 5)>(tabk, S.x, S.y, one);
        const float2 o = make_float2(
            __uint_as_float(__float_as_uint(fminf(ph.x, kRMax)) | ((par0 ^ xb0[s]) & 0x80000000u)),
            __uint_as_float(__float_as_uint(fminf(ph.y, kRMax)) | ((par1 ^ xb1[s]) & 0x80000000u)));
        if (s < NA) {
            // Unpredicated: a latched or padding lane's r and accumulator columns are never
            // read for that lane again (k_finish keeps its L and clears the accumulator), and
            // full 256-byte rows avoid partial-sector writes.
            const float2 fx = f2fma(o, make_float2(131072.0f, 131072.0f), make_float2(12582912.0f, 12582912.0f));
            // VN sums of both lanes (Eq. 4, N3; of the unrounded o with 16-bit storage) in one
            // 64-bit RED on the thread's pair word of the accumulator row (offs = pair position)
            atomicAdd(reinterpret_cast<unsigned long long*>(pla + offs[s] + 64),
                      (static_cast<unsigned long long>(__float_as_uint(fx.y)) << 32) | __float_as_uint(fx.x));
            if constexpr (MSG) __stcs(reinterpret_cast<unsigned int*>(prv) + s * 32, msg16_pack(o));   // stored message (N7)
            else __stcs(reinterpret_cast<float2*>(pr) + s * 32, o);                            // pair row: lanes l, l + 32
        }
        if (s > 0) Q = f2add(Q, p[s]);
    }
    return make_uint2((lw0 >> 31) ^ sbit.x ^ d1prev.x, (lw1 >> 31) ^ sbit.y ^ d1prev.y);
}

// One degree class (CN labels [begin, begin + count), NA active + ND <= 1 degree-1 slots)
// for 64-lane groups.  Work unit = a tile of ts consecutive CNs owned by one warp that
// covers both 32-lane chunks (each thread: lanes `lane` and `lane + 32`, two independent
// dependency chains; NA > 4 runs 1 CTA per SM with up to 128 registers).
// The tile's metadata is one coalesced load per array and its active-edge VN indices
// (pre-scaled to row offsets) are staged in shared memory.
template <int NA>
__host__ __device__ constexpr int cn_tile_min_blocks() { return NA <= 4 ? 2 : 1; }   // NA > 4: 128 registers

template <int RULE, int NA, int ND, int MSG = 0>
__global__ void __launch_bounds__(kCnThreads, cn_tile_min_blocks<NA>()) k_cn_tile(CodeDev cd, Group g, CnCtl karg,
                                                                                  int begin, int count, int ts) {
    using PT = PhiT<RULE>;
    constexpr int LPT = 2;                     // lanes l and l + 32 per thread (pair rows)
    constexpr int UPT = 2 / LPT;               // units per tile
    constexpr int NAS = NA > 0 ? NA : 1;
    constexpr int STAGE = (NA <= 4 ? 32 : 8) * NAS;
    extern __shared__ __align__(16) char smem[];
    __shared__ uint32_t s_unsat[2], s_act[2], s_fresh[2];
    pdl_launch_dependents();
    if (block_done(g)) {
        pdl_wait_previous();
        return;
    }
    const CnCtl k = cn_ctl(karg, g);
    load_phi_table<RULE>(smem, cd.phi);
    if (threadIdx.x < 2) {
        s_unsat[threadIdx.x] = 0u;
        s_act[threadIdx.x] = g.act[threadIdx.x];
        s_fresh[threadIdx.x] = g.fresh[threadIdx.x];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tabk = phi_tab_lane<RULE>(smem, lane);
    int* s_idx = reinterpret_cast<int*>(smem + PT::TAB_BYTES) + warp * STAGE;
    const uint32_t am0 = s_act[0], am1 = s_act[1];
    const int wpb = blockDim.x >> 5;
    const int ntiles = (count + ts - 1) / ts;
    uint32_t un0 = 0, un1 = 0;
    for (int u = blockIdx.x * wpb + warp; u < ntiles * UPT; u += gridDim.x * wpb) {
        const int tile = u / UPT;
        const int c0 = (UPT == 2) ? (u & 1) : 0;            // first chunk of this unit
        const uint32_t amA = c0 ? am1 : am0;                  // mask of chunk c0
        if ((LPT == 2 ? (am0 | am1) : amA) == 0u) continue;
        const int j0 = begin + tile * ts;
        const int nt = min(ts, begin + count - j0);
        const bool on = lane < nt;
        const int a_l = on ? __ldg(cd.cn_aptr + j0 + lane) : 0;
        const int d_l = on ? __ldg(cd.cn_dptr + j0 + lane) : 0;
        const uint2 sw_l = on ? __ldg(reinterpret_cast<const uint2*>(g.synd_t) + (j0 + lane)) : make_uint2(0, 0);
        if constexpr (NA + ND == 0) {          // empty rows: satisfied iff S_B[j] = 0
            for (int i = 0; i < nt; ++i) {
                un0 |= __shfl_sync(FULL, sw_l.x, i);
                un1 |= __shfl_sync(FULL, sw_l.y, i);
            }
            continue;
        } else {
            const int A0 = __shfl_sync(FULL, a_l, 0);
            if constexpr (NA > 0) {
                __syncwarp();
                for (int e = lane; e < nt * NA; e += 32) s_idx[e] = __ldg(cd.a_vn + A0 + e) * 128;
                __syncwarp();
            }
            for (int i = 0; i < nt; ++i) {
                const int ab = __shfl_sync(FULL, a_l, i);
                const int q0 = __shfl_sync(FULL, d_l, i);
                const uint32_t swx = __shfl_sync(FULL, sw_l.x, i), swy = __shfl_sync(FULL, sw_l.y, i);
                const int* idx = s_idx + (ab - A0);
                float* pr = g.r + (size_t(ab) * 64 + 2 * lane);   // pair rows: lanes lane, lane + 32 adjacent
                float Lv[LPT][NAS], ro[LPT][NAS], lam[LPT];
                uint32_t offs[NAS];   // pair position of the thread in the VN's row (one IMAD.WIDE.U32 per gather)
#pragma unroll
                for (int s = 0; s < NA; ++s) {
                    offs[s] = uint32_t(idx[s]) + 2u * uint32_t(lane);
                    const float2 lv = __ldg(reinterpret_cast<const float2*>(g.L + offs[s]));
                    Lv[0][s] = lv.x;
                    Lv[1][s] = lv.y;
                    if constexpr (MSG) {   // 16-bit row: the thread's word holds lanes lane, lane + 32 (N7)
                        const float2 q = msg16_q(__ldcs(reinterpret_cast<const unsigned int*>(g.r) + size_t(ab + s) * 32 + lane));
                        ro[0][s] = q.x;
                        ro[1][s] = q.y;
                    } else {
                        const float2 q = __ldcs(reinterpret_cast<const float2*>(pr) + s * 32);   // r^0 = 0: zeroed at group begin
                        ro[0][s] = q.x;
                        ro[1][s] = q.y;
                    }
                }
                if (s_fresh[0] | s_fresh[1]) {   // lane refill: r^0 = 0 for a frame starting in this pass
#pragma unroll
                    for (int h = 0; h < LPT; ++h)
                        if ((s_fresh[c0 + h] >> lane) & 1u)
#pragma unroll
                            for (int s = 0; s < NA; ++s) ro[h][s] = 0.0f;
                }
                uint2 wv = make_uint2(0, 0);
                if constexpr (ND > 0) {
#pragma unroll
                    for (int h = 0; h < LPT; ++h) lam[h] = __ldcs(g.lam1 + lam1_idx(q0, (c0 + h) * 32 + lane, 64));
                    if (k.check) wv = __ldg(reinterpret_cast<const uint2*>(g.d1bits) + (size_t(k.rpar) * cd.n_1 + q0));
                } else {
#pragma unroll
                    for (int h = 0; h < LPT; ++h) lam[h] = 0.0f;
                }
                uint32_t chk[LPT], b[LPT];
                {
                    float2 L2[NAS], r2[NAS];
#pragma unroll
                    for (int s = 0; s < NA; ++s) {
                        L2[s] = make_float2(Lv[0][s], Lv[1][s]);
                        r2[s] = make_float2(ro[0][s], ro[1][s]);
                    }
                    uint2 d1 = make_uint2(0, 0);
                    void* prv = MSG ? static_cast<void*>(reinterpret_cast<unsigned int*>(g.r) + size_t(ab) * 32 + lane)
                                    : static_cast<void*>(pr);
                    const uint2 c2 = cn_pair<RULE, NA, ND, MSG>(
                        tabk, L2, r2, make_float2(lam[0], lam[1]), make_uint2((swx >> lane) & 1u, (swy >> lane) & 1u),
                        make_uint2((wv.x >> lane) & 1u, (wv.y >> lane) & 1u), prv, g.L, offs, d1);
                    chk[0] = c2.x;
                    chk[1] = c2.y;
                    b[0] = d1.x;
                    b[1] = d1.y;
                }
#pragma unroll
                for (int h = 0; h < LPT; ++h) {
                    const uint32_t bal = __ballot_sync(FULL, chk[h]);
                    if (c0 + h) un1 |= bal;
                    else un0 |= bal;
                }
                if constexpr (ND > 0) {
                    uint32_t bal[LPT];
#pragma unroll
                    for (int h = 0; h < LPT; ++h) bal[h] = __ballot_sync(FULL, b[h]);
                    if (lane == 0) {
                        uint32_t* wp = g.d1bits + (size_t(k.wpar) * cd.n_1 + q0) * 2 + c0;
#pragma unroll
                        for (int h = 0; h < LPT; ++h) {
                            const uint32_t amh = (c0 + h) ? am1 : am0;
                            wp[h] = (amh == FULL) ? bal[h] : ((bal[h] & amh) | (wp[h] & ~amh));
                        }
                    }
                }
            }
        }
    }
    if (k.check && lane == 0) {
        if (un0 & am0) atomicOr(&s_unsat[0], un0 & am0);
        if (un1 & am1) atomicOr(&s_unsat[1], un1 & am1);
    }
    __syncthreads();
    if (k.check && threadIdx.x < 2 && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
    pdl_wait_previous();
}

// ------------------------------------------------------------------ TMA-pipelined CN tiles

// Exact-degree classes with 1..4 active slots and <= 1 degree-1 slot (at C3: 97 % of the
// CNs, all of the inner checks) for 64-lane groups.  Same arithmetic as k_cn_tile (cn_pair),
// different data movement.  In an exact-degree class CN j owns r rows abase + (j - begin) NA
// .. + NA and lambda row dbase + (j - begin), so a warp's DRAM stream is known in advance:
// one lane per warp issues 1D bulk copies (cp.async.bulk on the TMA unit, no registers held,
// evict-first L2 policy) of the next CN's NA + ND rows into a 2-stage shared-memory ring that
// completes on an mbarrier, while the warp computes the current CN from the previous stage.
// The L gathers stay direct loads (L2 hits; staging them by TMA as well, prefetching them
// into registers or L1 all measured slower -- DESIGN.md section 7).  The tile's VN row offsets
// are staged one tile ahead (double buffer).  One CTA per SM shares a single phi table; its
// warp count is what the rings leave room for.
#ifndef METLDPC_PIPE_STAGES
#define METLDPC_PIPE_STAGES 2   // shared-memory ring depth (3 stages measured no better)
#endif
#ifndef METLDPC_PIPE_WARPS
#define METLDPC_PIPE_WARPS 32   // warps per CTA cap (at most what the rings leave room for)
#endif
#ifndef METLDPC_RING_CW
#define METLDPC_RING_CW 24      // compute warps of the CN ring kernel (+ 1 producer warp; a multiple of 8)
#endif
#ifndef METLDPC_RING_CW_CORE
#define METLDPC_RING_CW_CORE 15 // compute warps of the ring kernel for classes with 5..16 active slots
#endif
#ifndef METLDPC_RING_STAGES
#define METLDPC_RING_STAGES 6   // CTA ring depth cap (k_cn_ring)
#endif
constexpr int kPipeStages = METLDPC_PIPE_STAGES;
constexpr int kSmemPerSm = 232448;     // opt-in dynamic shared memory per block (227 KB)

template <int NA, int ND, int MSG = 0>
struct PipeCfg {
    static constexpr int RB = MSG ? 128 : 256;                        // bytes per r row (64 lanes)
    static constexpr int STG = NA * RB;                               // bytes per stage: r rows
    static constexpr int IDX = 32 * NA;                               // ints per staged tile
    static constexpr int WARP_BYTES = (2 * IDX * 4 + kPipeStages * STG + kPipeStages * 8 + 127) / 128 * 128;
    static constexpr int TAB = (PhiT<METLDPC_RULE_EXACT>::TAB_BYTES > PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES)
                                   ? PhiT<METLDPC_RULE_EXACT>::TAB_BYTES
                                   : PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES;
    static constexpr int W0 = (kSmemPerSm - TAB - 64) / WARP_BYTES;
    // NA = 4 (the no-skip layouts' inner checks) spills at 64 registers (32 warps): 24 warps with
    // 80 registers measured 810 vs 715 Mb/s on no-skip C3
    static constexpr int WCAP = NA >= 4 ? 24 : METLDPC_PIPE_WARPS;
    static constexpr int WARPS = W0 > WCAP ? WCAP : W0;
    static constexpr int THREADS = WARPS * 32;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Streams read once per iteration (r, lambda): evict-first, so the L / accumulator rows stay in L2.
__device__ __forceinline__ void tma_load_1d_ef(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

template <int RULE, int NA, int ND, int MSG = 0>
__global__ void __launch_bounds__(PipeCfg<NA, ND, MSG>::THREADS, 1)
    k_cn_pipe(CodeDev cd, Group g, CnCtl karg, int begin, int count) {
    using PT = PhiT<RULE>;
    using PC = PipeCfg<NA, ND, MSG>;
    constexpr int TS = 32;                     // CNs per tile
    extern __shared__ __align__(16) char smem[];
    __shared__ uint32_t s_unsat[2], s_act[2], s_fresh[2];
    pdl_launch_dependents();
    if (block_done(g)) {
        pdl_wait_previous();
        return;
    }
    const CnCtl k = cn_ctl(karg, g);
    load_phi_table<RULE>(smem, cd.phi);
    if (threadIdx.x < 2) {
        s_unsat[threadIdx.x] = 0u;
        s_act[threadIdx.x] = g.act[threadIdx.x];
        s_fresh[threadIdx.x] = g.fresh[threadIdx.x];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* wb = smem + PT::TAB_BYTES + warp * PC::WARP_BYTES;
    int* s_idx = reinterpret_cast<int*>(wb);                         // [2][IDX]
    char* stage = wb + 2 * PC::IDX * 4;                              // [kPipeStages][STG]
    const uint32_t stage_a = smem_addr(stage);
    const uint32_t bar_a = smem_addr(stage + kPipeStages * PC::STG);
    if (lane == 0) {
        for (int st = 0; st < kPipeStages; ++st) mbar_init(bar_a + 8 * st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t tabk = phi_tab_lane<RULE>(smem, lane);
    const uint32_t am0 = s_act[0], am1 = s_act[1];
    const bool any_fresh = (s_fresh[0] | s_fresh[1]) != 0u;   // lane refill: frames starting now
    const int abase = __ldg(cd.cn_aptr + begin);
    const int dbase = ND ? __ldg(cd.cn_dptr + begin) : 0;
    const int ntiles = (count + TS - 1) / TS;
    const int GW = gridDim.x * PC::WARPS;
    const int gw = blockIdx.x * PC::WARPS + warp;
    const uint64_t pol = l2_evict_first_policy();
    auto stage_idx = [&](int tile, int b) {   // VN row offsets (a * 128 floats) of a tile
        const int jt = tile * TS, nt = min(TS, count - jt);
        for (int e = lane; e < nt * NA; e += 32) s_idx[b * PC::IDX + e] = __ldg(cd.a_vn + abase + jt * NA + e) * 128;
    };
    // producer cursor (tile, index) runs kPipeStages - 1 CNs ahead of the consumer
    int pt = gw, pi = 0;
    uint32_t np = 0, nc = 0;
    auto produce = [&]() {
        if (pt >= ntiles) return;
        const int jl = pt * TS + pi;
        if (lane == 0) {
            const uint32_t st = np % kPipeStages;
            const uint32_t bar = bar_a + 8 * st, dst = stage_a + st * PC::STG;
            mbar_expect_tx(bar, PC::STG);
            tma_load_1d_ef(dst, reinterpret_cast<const char*>(g.r) + size_t(abase + jl * NA) * PC::RB, NA * PC::RB, bar, pol);
        }
        ++np;
        if (++pi == min(TS, count - pt * TS)) { pi = 0; pt += GW; }
    };
    if (gw < ntiles) stage_idx(gw, 0);
    __syncwarp();
    for (int st = 0; st < kPipeStages - 1; ++st) produce();
    uint32_t un0 = 0, un1 = 0;
    int cb = 0;
    for (int tile = gw; tile < ntiles; tile += GW, cb ^= 1) {
        const int jt = tile * TS;                           // class-local index of the tile's first CN
        const int nt = min(TS, count - jt);
        const bool on = lane < nt;
        // the next tile's row offsets: its buffer last held the previous tile, finished
        if (tile + GW < ntiles) stage_idx(tile + GW, cb ^ 1);
        const uint2 sw_l = on ? __ldg(reinterpret_cast<const uint2*>(g.synd_t) + (begin + jt + lane)) : make_uint2(0, 0);
        uint2 wv_l = make_uint2(0, 0);
        if constexpr (ND > 0)
            if (k.check && on)
                wv_l = __ldg(reinterpret_cast<const uint2*>(g.d1bits) + (size_t(k.rpar) * cd.n_1 + dbase + jt + lane));
        __syncwarp();
        uint2 d1w = make_uint2(0u, 0u);   // degree-1 decision words of CN `lane` of the tile
        for (int i = 0; i < nt; ++i) {
            produce();
            const uint32_t st = nc % kPipeStages, ph = (nc / kPipeStages) & 1u;
            ++nc;
            const uint32_t swx = __shfl_sync(FULL, sw_l.x, i), swy = __shfl_sync(FULL, sw_l.y, i);
            uint2 wv = make_uint2(0, 0);
            if constexpr (ND > 0) {
                wv.x = __shfl_sync(FULL, wv_l.x, i);
                wv.y = __shfl_sync(FULL, wv_l.y, i);
            }
            const int jl = jt + i;
            const int* idx = s_idx + cb * PC::IDX + i * NA;
            uint32_t offs[NA];
            float2 L2[NA], r2[NA];
#pragma unroll
            for (int s = 0; s < NA; ++s) {
                offs[s] = uint32_t(idx[s]) + 2u * uint32_t(lane);
                L2[s] = __ldg(reinterpret_cast<const float2*>(g.L + offs[s]));   // L2-resident gathers, pair rows
            }
            mbar_wait(bar_a + 8 * st, ph);
            const float* sr = reinterpret_cast<const float*>(stage + st * PC::STG);
#pragma unroll
            for (int s = 0; s < NA; ++s) {
                if constexpr (MSG) r2[s] = msg16_q(reinterpret_cast<const uint32_t*>(sr)[s * 32 + lane]);   // q (N7)
                else r2[s] = reinterpret_cast<const float2*>(sr + s * 64)[lane];
            }
            // r^0 = 0 for a lane whose frame starts in this pass (Step 2), applied in registers:
            // the ring stages are written only by the TMA (async proxy), never by the threads
            if (any_fresh) {
                const bool f0 = (s_fresh[0] >> lane) & 1u, f1 = (s_fresh[1] >> lane) & 1u;
#pragma unroll
                for (int s = 0; s < NA; ++s) {
                    if (f0) r2[s].x = 0.0f;
                    if (f1) r2[s].y = 0.0f;
                }
            }
            float2 lam = make_float2(0.0f, 0.0f);
            if constexpr (ND > 0)   // blocked lam1 rows: two direct loads (this kernel is the METLDPC_RING=0 path)
                lam = make_float2(__ldcs(g.lam1 + lam1_idx(dbase + jl, lane, 64)), __ldcs(g.lam1 + lam1_idx(dbase + jl, lane + 32, 64)));
            void* pr = MSG ? static_cast<void*>(reinterpret_cast<unsigned int*>(g.r) + (size_t(abase + jl * NA) * 32 + lane))
                           : static_cast<void*>(g.r + (size_t(abase + jl * NA) * 64 + 2 * lane));
            uint2 d1 = make_uint2(0, 0);
            const uint2 c2 = cn_pair<RULE, NA, ND, MSG>(tabk, L2, r2, lam, make_uint2((swx >> lane) & 1u, (swy >> lane) & 1u),
                                                        make_uint2((wv.x >> lane) & 1u, (wv.y >> lane) & 1u), pr, g.L, offs, d1);
            un0 |= __ballot_sync(FULL, c2.x);
            un1 |= __ballot_sync(FULL, c2.y);
            if constexpr (ND > 0) {
                const uint32_t b0 = __ballot_sync(FULL, d1.x), b1 = __ballot_sync(FULL, d1.y);
                if (lane == i) { d1w.x = b0; d1w.y = b1; }   // lane i keeps CN i's words
            }
            __syncwarp();   // every lane has read stage st before it is refilled
        }
        if constexpr (ND > 0) {   // the tile's degree-1 decision words: one coalesced 8-byte store per lane
            if (on) {
                uint2* wp = reinterpret_cast<uint2*>(g.d1bits) + (size_t(k.wpar) * cd.n_1 + dbase + jt + lane);
                if ((am0 & am1) != FULL) {   // keep the words of lanes not iterating
                    const uint2 o = *wp;
                    d1w.x = (d1w.x & am0) | (o.x & ~am0);
                    d1w.y = (d1w.y & am1) | (o.y & ~am1);
                }
                *wp = d1w;
            }
        }
    }
    if (k.check && lane == 0) {
        if (un0 & am0) atomicOr(&s_unsat[0], un0 & am0);
        if (un1 & am1) atomicOr(&s_unsat[1], un1 & am1);
    }
    __syncthreads();
    if (k.check && threadIdx.x < 2 && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
    pdl_wait_previous();
}

// ------------------------------------------------------------------ CTA-ring CN kernel

// Same classes and arithmetic as k_cn_pipe (cn_pair), different data movement.  One CTA per SM
// of 31 compute warps and one producer warp.  A ring stage holds CW = 31 consecutive CNs of the
// class, compute warp w taking CN w of the stage.  In an exact-degree class everything those
// CNs read is contiguous in HBM -- their r rows, lambda rows, active-VN indices, S_B words and
// (from l = 2) the degree-1 decision words of iteration l - 1 -- so the producer moves a whole
// stage with five bulk copies (TMA, one mbarrier), instead of two copies per CN issued by every
// compute warp in between its own work, and a compute warp's per-CN overhead shrinks to one
// barrier wait, a few shared-memory reads and one release arrive.  The L gathers stay direct
// loads (L2-resident rows).
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int NA, int ND, int MSG>
struct RingCfg {

    // compute warps = CNs per stage: 64 registers for the inner classes (NA <= 4), up to 128 for
    // the core classes (NA > 4, 16 warps per SM)
    static constexpr int CW = NA <= 4 ? METLDPC_RING_CW : METLDPC_RING_CW_CORE;
    static constexpr int SC = CW;                                     // CNs per stage
    static_assert(ND == 0 || SC % 8 == 0, "a stage's lam1 rows must be whole blocks of 8 slots");
    static constexpr int RB = MSG ? 128 : 256;                        // r row bytes (64 lanes)
    // word arrays are copied from the 16-byte-aligned word at or below the first one needed
    // (lead 0..3 words) and rounded up to 16 bytes; the device arrays are padded for it
    static constexpr int IDX_BYTES = ((SC * NA + 8) * 4 + 15) / 16 * 16;
    static constexpr int W_BYTES = ((SC * 2 + 8) * 4 + 15) / 16 * 16;
    static constexpr int OFF_R = 0;
    static constexpr int OFF_L1 = OFF_R + SC * NA * RB;
    static constexpr int OFF_IDX = OFF_L1 + ND * SC * 256;
    static constexpr int OFF_SY = OFF_IDX + IDX_BYTES;
    static constexpr int OFF_D1 = OFF_SY + W_BYTES;
    static constexpr int STG = OFF_D1 + ND * W_BYTES;
    static constexpr int TAB = (PhiT<METLDPC_RULE_EXACT>::TAB_BYTES > PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES)
                                   ? PhiT<METLDPC_RULE_EXACT>::TAB_BYTES
                                   : PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES;
    static constexpr int S0 = (kSmemPerSm - TAB - 256) / STG;
    static constexpr int STAGES = S0 > METLDPC_RING_STAGES ? METLDPC_RING_STAGES : S0;
    static constexpr int SMEM = TAB + STAGES * STG + 256;             // + 2 x STAGES mbarriers
    static constexpr int THREADS = (CW + 1) * 32;
};

// 16-byte-aligned bulk copy of words [w0, w0 + n) of `base` (a padded device array): returns the
// bytes copied; the words land at dst + 4 * (w0 & 3).
__device__ __forceinline__ uint32_t ring_copy_words(uint32_t dst, const uint32_t* base, long w0, int n, uint32_t bar,
                                                    uint64_t pol) {
    const long a = w0 & ~3L;
    const uint32_t bytes = uint32_t(((w0 - a) + n + 3) & ~3L) * 4u;
    tma_load_1d_ef(dst, base + a, bytes, bar, pol);
    return bytes;
}
__device__ __forceinline__ uint32_t ring_words_bytes(long w0, int n) { return uint32_t(((w0 & 3) + n + 3) & ~3L) * 4u; }

template <int RULE, int NA, int ND, int MSG = 0>
__global__ void __launch_bounds__(RingCfg<NA, ND, MSG>::THREADS, 1)
    k_cn_ring(CodeDev cd, Group g, CnCtl karg, int begin, int count) {
    using PT = PhiT<RULE>;
    using RC = RingCfg<NA, ND, MSG>;
    constexpr int CW = RC::CW, S = RC::STAGES, SC = RC::SC;
    extern __shared__ __align__(16) char smem[];
    __shared__ uint32_t s_unsat[2], s_act[2], s_fresh[2];
    pdl_launch_dependents();
    if (block_done(g)) {
        pdl_wait_previous();
        return;
    }
    const CnCtl k = cn_ctl(karg, g);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* ring = smem + PT::TAB_BYTES;
    const uint32_t ring_a = smem_addr(ring);
    const uint32_t full_a = smem_addr(ring + S * RC::STG), empty_a = full_a + 8 * S;
    if (threadIdx.x < 2) {
        s_unsat[threadIdx.x] = 0u;
        s_act[threadIdx.x] = g.act[threadIdx.x];
        s_fresh[threadIdx.x] = g.fresh[threadIdx.x];
    }
    if (threadIdx.x == 32 * CW) {
        for (int st = 0; st < S; ++st) {
            mbar_init(full_a + 8 * st, 1);
            mbar_init(empty_a + 8 * st, CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int abase = __ldg(cd.cn_aptr + begin);
    const int dbase = ND ? __ldg(cd.cn_dptr + begin) : 0;
    // Stages are aligned to the lam1 blocks: stage gs covers class positions [gs SC - lo, (gs + 1) SC - lo),
    // lo = dbase mod 8, so every stage's degree-1 slots are whole 8-slot blocks (the first stage is
    // lo checks short).  Without degree-1 slots lo = 0.
    const int lo = ND ? (dbase & 7) : 0;
    const int nst = (count + lo + SC - 1) / SC;
    const bool d1in = ND > 0 && k.check;           // degree-1 decisions of l - 1 for the syndrome test
    load_phi_table<RULE>(smem, cd.phi);
    __syncthreads();
    if (warp == CW) {                              // ---- producer warp
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int slot = 0, use = 0;
            for (int gs = blockIdx.x; gs < nst; gs += gridDim.x) {
                if (use) mbar_wait(empty_a + 8 * slot, (use - 1) & 1);
                const int j0 = max(gs * SC - lo, 0), ncn = min((gs + 1) * SC - lo, count) - j0;
                const uint32_t dst = ring_a + slot * RC::STG, bar = full_a + 8 * slot;
                const long wi = long(abase) + long(j0) * NA, ws = (long(begin) + j0) * 2,
                           wd = (long(k.rpar) * cd.n_1 + dbase + j0) * 2;
                uint32_t bytes = uint32_t(ncn) * NA * RC::RB + ring_words_bytes(wi, ncn * NA) + ring_words_bytes(ws, ncn * 2);
                const int nblk = (j0 + ncn - (gs * SC - lo) + 7) >> 3;   // lam1 blocks of the stage
                if constexpr (ND > 0) bytes += uint32_t(nblk) * 2048u + (d1in ? ring_words_bytes(wd, ncn * 2) : 0u);
                mbar_expect_tx(bar, bytes);
                tma_load_1d_ef(dst + RC::OFF_R, reinterpret_cast<const char*>(g.r) + size_t(abase + j0 * NA) * RC::RB,
                               uint32_t(ncn) * NA * RC::RB, bar, pol);
                if constexpr (ND > 0)   // whole lam1 blocks from slot dbase + gs SC - lo (a multiple of 8)
                    tma_load_1d_ef(dst + RC::OFF_L1, g.lam1 + size_t((dbase - lo) / 8 + gs * (SC / 8)) * 512, uint32_t(nblk) * 2048u,
                                   bar, pol);
                ring_copy_words(dst + RC::OFF_IDX, reinterpret_cast<const uint32_t*>(cd.a_vn), wi, ncn * NA, bar, pol);
                ring_copy_words(dst + RC::OFF_SY, g.synd_t, ws, ncn * 2, bar, pol);
                if constexpr (ND > 0)
                    if (d1in) ring_copy_words(dst + RC::OFF_D1, g.d1bits, wd, ncn * 2, bar, pol);
                if (++slot == S) {
                    slot = 0;
                    ++use;
                }
            }
        }
    } else {                                       // ---- compute warps: CN `warp` of every stage
        const uint32_t tabk = phi_tab_lane<RULE>(smem, lane);
        const uint32_t am0 = s_act[0], am1 = s_act[1];
        const bool any_fresh = (s_fresh[0] | s_fresh[1]) != 0u;
        const bool f0 = (s_fresh[0] >> lane) & 1u, f1 = (s_fresh[1] >> lane) & 1u;
        uint32_t un0 = 0, un1 = 0;
        int slot = 0;
        uint32_t phase = 0;   // parity of the slot's current use
        for (int gs = blockIdx.x; gs < nst; gs += gridDim.x) {
            const int j0 = max(gs * SC - lo, 0);
            const int jl = gs * SC - lo + warp;          // class position of this warp's check
            const int wl = jl - j0;                      // its index among the stage's copied rows
            mbar_wait(full_a + 8 * slot, phase);
            if (jl >= 0 && jl < count) {
                const char* sp = ring + slot * RC::STG;
                const int* sidx = reinterpret_cast<const int*>(sp + RC::OFF_IDX) + ((abase + j0 * NA) & 3) + wl * NA;
                uint32_t offs[NA];
                float2 L2[NA], r2[NA];
#pragma unroll
                for (int s = 0; s < NA; ++s) {
                    offs[s] = uint32_t(sidx[s]) * 128u + 2u * uint32_t(lane);
                    L2[s] = __ldg(reinterpret_cast<const float2*>(g.L + offs[s]));   // L2-resident gathers, pair rows
                }
                const uint32_t* ssy = reinterpret_cast<const uint32_t*>(sp + RC::OFF_SY) + (((begin + j0) * 2) & 3) + wl * 2;
                const uint32_t swx = ssy[0], swy = ssy[1];
                uint2 wv = make_uint2(0, 0);
                if constexpr (ND > 0)
                    if (d1in) {
                        const uint32_t* sd =
                            reinterpret_cast<const uint32_t*>(sp + RC::OFF_D1) + ((long(k.rpar) * cd.n_1 + dbase + j0) * 2 & 3) + wl * 2;
                        wv = make_uint2(sd[0], sd[1]);
                    }
                const float* sr = reinterpret_cast<const float*>(sp + RC::OFF_R + wl * NA * RC::RB);
#pragma unroll
                for (int s = 0; s < NA; ++s) {
                    if constexpr (MSG) r2[s] = msg16_q(reinterpret_cast<const uint32_t*>(sr)[s * 32 + lane]);
                    else r2[s] = reinterpret_cast<const float2*>(sr + s * 64)[lane];
                }
                if (any_fresh) {   // r^0 = 0 for a frame starting in this pass (Step 2), in registers
#pragma unroll
                    for (int s = 0; s < NA; ++s) {
                        if (f0) r2[s].x = 0.0f;
                        if (f1) r2[s].y = 0.0f;
                    }
                }
                float2 lam = make_float2(0.0f, 0.0f);
                if constexpr (ND > 0) {
                    const float* sl = reinterpret_cast<const float*>(sp + RC::OFF_L1 + (warp >> 3) * 2048) + lane * 8 +
                                      ((warp & 7) ^ ((lane >> 2) & 7));
                    lam = make_float2(sl[0], sl[256]);
                }
                void* pr = MSG ? static_cast<void*>(reinterpret_cast<unsigned int*>(g.r) + (size_t(abase + jl * NA) * 32 + lane))
                               : static_cast<void*>(g.r + (size_t(abase + jl * NA) * 64 + 2 * lane));
                uint2 d1 = make_uint2(0, 0);
                const uint2 c2 = cn_pair<RULE, NA, ND, MSG>(tabk, L2, r2, lam,
                                                            make_uint2((swx >> lane) & 1u, (swy >> lane) & 1u),
                                                            make_uint2((wv.x >> lane) & 1u, (wv.y >> lane) & 1u), pr, g.L, offs, d1);
                un0 |= __ballot_sync(FULL, c2.x);
                un1 |= __ballot_sync(FULL, c2.y);
                if constexpr (ND > 0) {
                    const uint2 b = make_uint2(__ballot_sync(FULL, d1.x), __ballot_sync(FULL, d1.y));
                    if (lane == 0) {
                        uint2* wp = reinterpret_cast<uint2*>(g.d1bits) + (size_t(k.wpar) * cd.n_1 + dbase + jl);
                        if ((am0 & am1) != FULL) {
                            // keep the words of lanes not iterating, without a read on the warp's path:
                            // AND clears the iterating lanes' 0 bits, OR sets their 1 bits (two
                            // fire-and-forget reductions, applied in order; the words are read again
                            // only by the next pass)
                            unsigned int* w = reinterpret_cast<unsigned int*>(wp);
                            atomicAnd(w, b.x | ~am0);
                            atomicOr(w, b.x & am0);
                            atomicAnd(w + 1, b.y | ~am1);
                            atomicOr(w + 1, b.y & am1);
                        } else {
                            *wp = b;
                        }
                    }
                }
            }
            __syncwarp();                           // the warp has read the stage
            if (lane == 0) mbar_arrive(empty_a + 8 * slot);
            if (++slot == S) {
                slot = 0;
                phase ^= 1u;
            }
        }
        if (k.check && lane == 0) {
            if (un0 & am0) atomicOr(&s_unsat[0], un0 & am0);
            if (un1 & am1) atomicOr(&s_unsat[1], un1 & am1);
        }
    }
    __syncthreads();
    if (k.check && threadIdx.x < 2 && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
    pdl_wait_previous();
}

// Generic class: any lane count, CNs with more than one degree-1 slot or total degree
// 17..32 (rare in MET ensembles); one CN x one 32-lane chunk per warp item, run-time
// degree, arrays in local memory.  Same arithmetic (N1).
template <int RULE>
__global__ void __launch_bounds__(kCnThreads, 2) k_cn_generic(CodeDev cd, Group g, CnCtl karg, int begin, int count) {
    using PT = PhiT<RULE>;
    extern __shared__ __align__(16) char smem[];
    __shared__ uint32_t s_unsat[4], s_act[4];
    pdl_launch_dependents();
    if (block_done(g)) {
        pdl_wait_previous();
        return;
    }
    const CnCtl k = cn_ctl(karg, g);
    load_phi_table<RULE>(smem, cd.phi);
    if (threadIdx.x < g.C) { s_unsat[threadIdx.x] = 0u; s_act[threadIdx.x] = g.act[threadIdx.x]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t tabk = phi_tab_lane<RULE>(smem, lane);
    const int wpb = blockDim.x >> 5;
    const int lc = __ffs(g.C) - 1;
    const long total = long(count) << lc;
    for (long item = long(blockIdx.x) * wpb + (threadIdx.x >> 5); item < total; item += long(gridDim.x) * wpb) {
        const int c = int(item & (g.C - 1));
        const uint32_t amask = s_act[c];
        // a chunk is skipped only with its pair chunk: every lane of a pair word must receive its
        // VN's deg terms for the 64-bit accumulator to decode (k_finish)
        if (!(amask | (g.B == 32 ? 0u : s_act[c ^ 1]))) continue;
        const int j = begin + int(item >> lc);
        const size_t off = size_t(c) * 32 + lane;
        const size_t po = size_t(lpos(int(off), g.B));   // pair position of the lane (r, L, accumulator rows)
        const int ab = __ldg(cd.cn_aptr + j), na = __ldg(cd.cn_aptr + j + 1) - ab;
        const int db = __ldg(cd.cn_dptr + j), d = na + (__ldg(cd.cn_dptr + j + 1) - db);
        const uint32_t sbit = (__ldg(g.synd_t + size_t(j) * g.C + c) >> lane) & 1u;
        const int idx = (lane < na) ? __ldg(cd.a_vn + ab + lane) : 0;
        const uint32_t one = one_bits();
        float p[kMaxCnDeg], P[kMaxCnDeg];
        uint32_t negmask = 0, chk = sbit;
        for (int s = 0; s < d; ++s) {
            float x;
            if (s < na) {
                const int v = __shfl_sync(FULL, idx, s);
                const float Lv = __ldg(g.L + size_t(v) * 2 * g.B + po);
                if (g.msg16) {   // 16-bit row (N7): half-word c of word `lane`; x = L - q 2^-10 (one rounding)
                    const uint32_t w = ((g.fresh[c] >> lane) & 1u) ? 0x8080u
                        : uint32_t(__ldcs(reinterpret_cast<const unsigned short*>(g.r) + size_t(ab + s) * 64 + 2 * lane + c));
                    const float q = __fsub_rn(__uint_as_float(0x4B000000u | w), kMsg16Magic);
                    x = __fmaf_rn(q, -0.0009765625f, Lv);
                } else {
                    const float ro = ((g.fresh[c] >> lane) & 1u) ? 0.0f : __ldcs(g.r + size_t(ab + s) * g.B + po);
                    x = __fsub_rn(Lv, ro);
                }
                chk ^= uint32_t(Lv < 0.0f);
            } else {
                const int q = db + (s - na);
                x = __ldcs(g.lam1 + lam1_idx(q, int(off), g.B));
                if (k.check) chk ^= (__ldg(g.d1bits + (size_t(k.rpar) * cd.n_1 + q) * g.C + c) >> lane) & 1u;
            }
            if (s < na) {
                negmask |= (__float_as_uint(__fadd_rn(x, 0.0f)) >> 31) << s;   // = [x < 0]
                p[s] = phi_dev<RULE>(tabk, fabsf(x), one);
            } else {   // degree-1 prior in phi form (N1): sign bit = [lambda < 0], |x| = phi(|lambda|)
                negmask |= (__float_as_uint(x) >> 31) << s;
                p[s] = fabsf(x);
            }
        }
        if (k.check) {
            const uint32_t mm = __ballot_sync(FULL, chk) & amask;
            if (mm && lane == 0) atomicOr(&s_unsat[c], mm);
        }
        float acc = 0.0f;
        for (int s = 0; s < d; ++s) { P[s] = acc; acc = __fadd_rn(acc, p[s]); }
        const uint32_t par = sbit ^ (__popc(negmask) & 1u);
        const bool act = (amask >> lane) & 1u;
        float Q = 0.0f;
        for (int s = d - 1; s >= 0; --s) {
            const float S = __fadd_rn(P[s], Q);
            if (s >= na) {   // Step 5 for a degree-1 VN (N1): no phi(S) needed
                const uint32_t nl = (negmask >> s) & 1u, nr = par ^ nl;
                const uint32_t bal = __ballot_sync(FULL, d1_decision(nl << 31, nr << 31, p[s], S));
                if (lane == 0) {
                    uint32_t* w = g.d1bits + (size_t(k.wpar) * cd.n_1 + db + (s - na)) * g.C + c;
                    *w = (amask == FULL) ? bal : ((bal & amask) | (*w & ~amask));
                }
                if (s > 0) Q = __fadd_rn(Q, p[s]);
                continue;
            }
            const float mag = fminf(phi_dev<RULE>(tabk, S, one), kRMax);
            const float o = __uint_as_float(__float_as_uint(mag) | ((par ^ ((negmask >> s) & 1u)) << 31));
            {
                const int v = __shfl_sync(FULL, idx, s);      // whole warp: lane s may be an idle lane
                {   // unpredicated, as the pair kernels: each lane's accumulator gets exactly deg terms
                    (void)act;
                    if (g.msg16)
                        __stcs(reinterpret_cast<unsigned short*>(g.r) + size_t(ab + s) * 64 + 2 * lane + c,
                               (unsigned short)(__float_as_uint(__fmaf_rn(o, 1024.0f, kMsg16Magic)) & 0xFFFFu));
                    else
                        __stcs(g.r + size_t(ab + s) * g.B + po, o);
                    float* acc = g.L + size_t(v) * 2 * g.B + g.B;
                    if (g.B == 32)
                        atomicAdd(reinterpret_cast<unsigned int*>(acc + off), vn_fix(o));
                    else   // the lane's half of its pair word, as a 64-bit add (the same sum as the pair kernels' REDs)
                        atomicAdd(reinterpret_cast<unsigned long long*>(acc + (po & ~size_t(1))),
                                  static_cast<unsigned long long>(vn_fix(o)) << (32 * (po & 1)));
                }
            }
            if (s > 0) Q = __fadd_rn(Q, p[s]);
        }
    }
    __syncthreads();
    if (k.check && threadIdx.x < g.C && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
    pdl_wait_previous();
}

// ------------------------------------------------------------------ syndrome test only (a4 at l = N)

__global__ void __launch_bounds__(256) k_check(CodeDev cd, Group g, int par) {
    __shared__ uint32_t s_unsat[4], s_act[4];
    if (threadIdx.x < g.C) { s_unsat[threadIdx.x] = 0u; s_act[threadIdx.x] = g.act[threadIdx.x]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int lc = __ffs(g.C) - 1;
    const long total = long(cd.m) << lc;
    for (long item = long(blockIdx.x) * wpb + (threadIdx.x >> 5); item < total; item += long(gridDim.x) * wpb) {
        const int j = int(item >> lc), c = int(item & (g.C - 1));
        const uint32_t amask = s_act[c];
        if (!amask) continue;
        const size_t off = size_t(c) * 32 + lane;
        const int ab = __ldg(cd.cn_aptr + j), ae = __ldg(cd.cn_aptr + j + 1);
        const int db = __ldg(cd.cn_dptr + j), de = __ldg(cd.cn_dptr + j + 1);
        uint32_t chk = (__ldg(g.synd_t + size_t(j) * g.C + c) >> lane) & 1u;
        const int po = lpos(int(off), g.B);
        for (int t = ab; t < ae; ++t) chk ^= uint32_t(__ldg(g.L + size_t(__ldg(cd.a_vn + t)) * 2 * g.B + po) < 0.0f);
        for (int q = db; q < de; ++q) chk ^= (__ldg(g.d1bits + (size_t(par) * cd.n_1 + q) * g.C + c) >> lane) & 1u;
        const uint32_t mm = __ballot_sync(FULL, chk) & amask;
        if (mm && lane == 0) atomicOr(&s_unsat[c], mm);
    }
    __syncthreads();
    if (threadIdx.x < g.C && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
}

// ------------------------------------------------------------------ variable-node update (a3)

// Eq. (4)/(5), N3: the CN pass has accumulated, per active VN a and lane b, the
// exact fixed-point sum sum_k bits(fmaf(r_k, 2^17, 1.5 * 2^23)) (mod 2^32); remove the
// degree x 0x4B400000 bias, L = lambda + (float)sum * 2^-17 for lanes still iterating,
// and clear the accumulator for the next iteration.  Four lanes per thread (128-bit).
__global__ void __launch_bounds__(256) k_finish(CodeDev cd, Group g) {
    __shared__ uint32_t s_act[4];
    pdl_launch_dependents();
    pdl_wait_previous();   // may be launched ahead of the latch it follows
    if (block_done(g)) return;
    if (threadIdx.x < g.C) s_act[threadIdx.x] = g.act[threadIdx.x];
    __syncthreads();
    const int qpr = g.B >> 2;                           // float4 quads per row half
    const long total = long(cd.n_a) * qpr;
    for (long t = long(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += long(gridDim.x) * blockDim.x) {
        const int a = int(t / qpr), q = int(t - long(a) * qpr);
        const int deg = __ldg(cd.vn_aptr + a + 1) - __ldg(cd.vn_aptr + a);
        const uint32_t bias = uint32_t(deg) * 0x4B400000u;
        float4* Lrow = reinterpret_cast<float4*>(g.L + size_t(a) * 2 * g.B);
        uint4* Arow = reinterpret_cast<uint4*>(g.L + size_t(a) * 2 * g.B + g.B);
        const uint4 acc = Arow[q];
        const float4 lam = __ldg(reinterpret_cast<const float4*>(g.lam_a + size_t(a) * g.B) + q);
        // positions 4q .. 4q + 3 of the pair rows; their lanes and fixed-point sums
        int sx, sy, sz, sw;
        uint32_t m;
        if (g.B == 32) {
            m = (s_act[0] >> (q * 4)) & 0xFu;
            sx = int(acc.x - bias);
            sy = int(acc.y - bias);
            sz = int(acc.z - bias);
            sw = int(acc.w - bias);
        } else {
            // words (x, y) and (z, w): lanes t, t + 32 and t + 1, t + 33 of the 64-lane block
            const int blk = (q * 4) & ~63, t = ((q * 4) & 63) >> 1;
            const uint32_t lo = s_act[blk >> 5] >> t, hi = s_act[(blk >> 5) + 1] >> t;
            m = (lo & 1u) | ((hi & 1u) << 1) | ((lo & 2u) << 1) | ((hi & 2u) << 2);
            // 64-bit word = (deg bias + sum_hi) 2^32 + (deg bias + sum_lo) mod 2^64: the low sum
            // is exact mod 2^32 (|sum| < 2^31), and its carry into the high word follows from it
            const unsigned long long dB = static_cast<unsigned long long>(uint32_t(deg)) * 0x4B400000ull;
            sx = int(acc.x - bias);
            sy = int(acc.y - bias - uint32_t((dB + static_cast<unsigned long long>(static_cast<long long>(sx))) >> 32));
            sz = int(acc.z - bias);
            sw = int(acc.w - bias - uint32_t((dB + static_cast<unsigned long long>(static_cast<long long>(sz))) >> 32));
        }
        float4 L = (m == 0xFu) ? make_float4(0.f, 0.f, 0.f, 0.f) : Lrow[q];   // all 4 lanes rewritten: skip the read
        const float sc = 1.0f / 131072.0f;
        if (m & 1u) L.x = __fadd_rn(lam.x, __fmul_rn(__int2float_rn(sx), sc));
        if (m & 2u) L.y = __fadd_rn(lam.y, __fmul_rn(__int2float_rn(sy), sc));
        if (m & 4u) L.z = __fadd_rn(lam.z, __fmul_rn(__int2float_rn(sz), sc));
        if (m & 8u) L.w = __fadd_rn(lam.w, __fmul_rn(__int2float_rn(sw), sc));
        if (m) Lrow[q] = L;
        Arow[q] = make_uint4(0u, 0u, 0u, 0u);
    }
}

// ------------------------------------------------------------------ 64-lane tiled syndrome check

// Syndrome test of iteration l = N (N4) for 64-lane groups: warp per tile of 32 CNs.
__global__ void __launch_bounds__(256) k_check64(CodeDev cd, Group g, int par) {
    __shared__ uint32_t s_unsat[2], s_act[2];
    if (threadIdx.x < 2) { s_unsat[threadIdx.x] = 0u; s_act[threadIdx.x] = g.act[threadIdx.x]; }
    __syncthreads();
    const uint32_t am0 = s_act[0], am1 = s_act[1];
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int ntiles = (cd.m + 31) >> 5;
    const float* Ll = g.L + 2 * lane;   // pair rows: lanes lane, lane + 32 adjacent
    uint32_t un0 = 0, un1 = 0;
    if (am0 | am1) {
        for (int tile = blockIdx.x * wpb + (threadIdx.x >> 5); tile < ntiles; tile += gridDim.x * wpb) {
            const int j0 = tile * 32;
            const int nt = min(32, cd.m - j0);
            const bool on = lane < nt;
            const int a_l = on ? __ldg(cd.cn_aptr + j0 + lane) : 0, ae_l = on ? __ldg(cd.cn_aptr + j0 + lane + 1) : 0;
            const int d_l = on ? __ldg(cd.cn_dptr + j0 + lane) : 0, de_l = on ? __ldg(cd.cn_dptr + j0 + lane + 1) : 0;
            const uint2 sw_l = on ? __ldg(reinterpret_cast<const uint2*>(g.synd_t) + (j0 + lane)) : make_uint2(0, 0);
            for (int i = 0; i < nt; ++i) {
                const int ab = __shfl_sync(FULL, a_l, i), na = __shfl_sync(FULL, ae_l, i) - ab;
                const int db = __shfl_sync(FULL, d_l, i), nd = __shfl_sync(FULL, de_l, i) - db;
                uint32_t c0 = (__shfl_sync(FULL, sw_l.x, i) >> lane) & 1u;
                uint32_t c1 = (__shfl_sync(FULL, sw_l.y, i) >> lane) & 1u;
                const int idx = (lane < na) ? __ldg(cd.a_vn + ab + lane) * 128 : 0;
                for (int s = 0; s < na; ++s) {
                    const int o = __shfl_sync(FULL, idx, s);
                    const float2 lv = __ldg(reinterpret_cast<const float2*>(Ll + o));
                    c0 ^= uint32_t(lv.x < 0.0f);
                    c1 ^= uint32_t(lv.y < 0.0f);
                }
                for (int q = db; q < db + nd; ++q) {
                    const uint2 w = __ldg(reinterpret_cast<const uint2*>(g.d1bits) + (size_t(par) * cd.n_1 + q));
                    c0 ^= (w.x >> lane) & 1u;
                    c1 ^= (w.y >> lane) & 1u;
                }
                un0 |= __ballot_sync(FULL, c0);
                un1 |= __ballot_sync(FULL, c1);
            }
        }
    }
    if (lane == 0) {
        if (un0 & am0) atomicOr(&s_unsat[0], un0 & am0);
        if (un1 & am1) atomicOr(&s_unsat[1], un1 & am1);
    }
    __syncthreads();
    if (threadIdx.x < 2 && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
}

// ------------------------------------------------------------------ latch (a4 bookkeeping)

// Lanes still active whose tested iteration l had no unsatisfied check converged at l
// (R11, R12).  final_: iteration l = N, every remaining active lane ends here.
__global__ void k_latch(Group g, int l, int final_) {
    const int c = threadIdx.x;   // one thread per chunk
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    if (c < g.C) {
        const uint32_t a = g.act[c], u = g.unsat[c];
        const uint32_t ok = a & ~u;
        const uint32_t end = final_ ? a : ok;
        for (int b = 0; b < 32; ++b)
            if ((end >> b) & 1u) {
                g.iters[c * 32 + b] = l;
                g.conv[c * 32 + b] = uint8_t((ok >> b) & 1u);
            }
        const uint32_t na = final_ ? 0u : (a & u);
        g.act[c] = na;
        g.unsat[c] = 0u;
        if (na) atomicOr(&s_any, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *g.done = s_any ? 0 : 1;
}

// Graph-loop versions: latch the lanes converged at l - 1 after CN pass l (ET), and
// advance l, leaving the WHILE condition = (l <= N && some lane still iterating).
__global__ void k_latch_dev(Group g, int et) {
    pdl_launch_dependents();
    pdl_wait_previous();   // launched programmatically after the CN classes: their results first
    const int l = *reinterpret_cast<volatile int*>(g.iter);
    if (!et || l < 2) return;
    const int c = threadIdx.x;
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    if (c < g.C) {
        const uint32_t a = g.act[c], u = g.unsat[c];
        const uint32_t ok = a & ~u;
        for (int b = 0; b < 32; ++b)
            if ((ok >> b) & 1u) {
                g.iters[c * 32 + b] = l - 1;
                g.conv[c * 32 + b] = 1;
            }
        const uint32_t na = a & u;
        g.act[c] = na;
        g.unsat[c] = 0u;
        if (na) atomicOr(&s_any, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *g.done = s_any ? 0 : 1;
}

__global__ void k_loop_ctl(Group g, cudaGraphConditionalHandle h) {
    pdl_wait_previous();
    const int l = *g.iter + 1;
    *g.iter = l;
    cudaGraphSetConditional(h, (l <= *g.maxit && !*reinterpret_cast<volatile int*>(g.done)) ? 1u : 0u);
}

// ------------------------------------------------------------------ group init (a1)

// llr [nb][n] frame-major -> lam_a / L / lam1 [slot][B]: 32 VNs x 32 lanes tile transposed
// through shared memory so both the read and the write are 128-byte lines.
__global__ void __launch_bounds__(256) k_scatter(CodeDev cd, Group g, const float* __restrict__ llr, int nb) {
    __shared__ float tile[32][33];
    const int i0 = blockIdx.x * 32, c = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int rr = w; rr < 32; rr += 8) {
        const int fl = c * 32 + rr, i = i0 + lane;
        tile[rr][lane] = (fl < nb && i < cd.n) ? __ldcs(llr + size_t(fl) * cd.n + i) : 0.0f;
    }
    __syncthreads();
    const size_t off = size_t(c) * 32 + lane;
    const bool valid_lane = (c * 32 + lane) < nb;
    for (int ii = w; ii < 32; ii += 8) {
        const int i = i0 + ii;
        if (i >= cd.n) break;
        const float val = tile[lane][ii];
        const uint32_t bad = __ballot_sync(FULL, valid_lane && !isfinite(val));
        if (bad && lane == 0) atomicOr(g.invalid + c, bad);
        const int v = __ldg(cd.vmap + i);
        if (v >= 0) {
            // lambda + 0: an input -0 becomes +0 (same value; R2 gives it no sign).  Then no L^l
            // and no extrinsic L - r is ever -0 (L^l = lambda + sum, x = L - r with L != -0), so
            // the CN kernels read [L < 0] and [x < 0] straight from the sign bits.
            const float lz = __fadd_rn(val, 0.0f);
            const int po = lpos(int(off), g.B);
            g.lam_a[size_t(v) * g.B + po] = lz;
            g.L[size_t(v) * 2 * g.B + po] = lz;                      // L^0 = lambda (Step 2)
            g.L[size_t(v) * 2 * g.B + g.B + po] = 0.0f;              // empty VN-sum accumulator (its half)
        } else {
            g.lam1[lam1_idx(~v, int(off), g.B)] = lam1_phi_form(cd, val);
        }
    }
}

// S_B [nb][W] LSB-first -> synd_t[j][c]: 32 x 32 bit transpose by ballots.
__global__ void __launch_bounds__(256) k_pack_syndrome(CodeDev cd, Group g, const uint32_t* __restrict__ synd, int nb) {
    const int W = (cd.m + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const long item = long(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (item >= long(W) * g.C) return;
    const int wd = int(item / g.C), c = int(item % g.C);
    const int fl = c * 32 + lane;
    const uint32_t word = (fl < nb) ? __ldg(synd + size_t(fl) * W + wd) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const uint32_t bal = __ballot_sync(FULL, (word >> b) & 1u);
        if (lane == b) mine = bal;
    }
    const int j = wd * 32 + lane;
    if (j < cd.m) g.synd_t[size_t(__ldg(cd.cn_new + j)) * g.C + c] = mine;
}

__global__ void k_init_ctl(Group g, int nb, int N) {
    if (threadIdx.x == 0) {
        *g.iter = 1;
        *g.maxit = N;
    }
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < g.B; b += blockDim.x) {
        const bool valid = b < nb;
        const bool bad = (g.invalid[b >> 5] >> (b & 31)) & 1u;
        g.iters[b] = (valid && bad) ? -1 : 0;
        g.conv[b] = 0;
    }
    if (threadIdx.x < g.C) {
        const int c = threadIdx.x;
        const int lo = c * 32;
        uint32_t vm = (nb >= lo + 32) ? FULL : (nb > lo ? ((1u << (nb - lo)) - 1u) : 0u);
        const uint32_t a = vm & ~g.invalid[c];
        g.act[c] = a;
        g.unsat[c] = 0u;
        if (a) atomicOr(&s_any, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) *g.done = s_any ? 0 : 1;
}

// ------------------------------------------------------------------ finalize (a5)

// Hard bits in original VN order: active VNs from sign(L), degree-1 VNs from the bits of
// their final iteration's parity; packed LSB-first per frame ("de-permutate").
__global__ void __launch_bounds__(256) k_finalize(CodeDev cd, Group g, int nb, uint32_t* __restrict__ bits_out,
                                                  int32_t* __restrict__ iters_out, uint8_t* __restrict__ conv_out) {
    const int NW = (cd.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int wblk = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int c = blockIdx.y;
    const int fl = c * 32 + lane;
    const int it = g.iters[fl];
    if (blockIdx.x == 0 && threadIdx.x < 32 && fl < nb) {
        iters_out[fl] = it;
        conv_out[fl] = g.conv[fl];
    }
    if (wblk >= NW) return;
    const size_t off = size_t(c) * 32 + lane;
    const int par = it & 1;
    uint32_t word = 0;
    const int i0 = wblk * 32;
    for (int ii = 0; ii < 32; ++ii) {
        const int i = i0 + ii;
        if (i >= cd.n) break;
        const int v = __ldg(cd.vmap + i);
        uint32_t b;
        if (v >= 0) {
            b = g.L[size_t(v) * 2 * g.B + lpos(int(off), g.B)] < 0.0f;
        } else {
            const uint32_t w0 = g.d1bits[(size_t(0) * cd.n_1 + ~v) * g.C + c];
            const uint32_t w1 = g.d1bits[(size_t(1) * cd.n_1 + ~v) * g.C + c];
            b = ((par ? w1 : w0) >> lane) & 1u;
        }
        word |= b << ii;
    }
    if (it < 0) word = 0;
    if (fl < nb) bits_out[size_t(fl) * NW + wblk] = word;
}

// ------------------------------------------------------------------ lane refill (streaming decode, a6)

// A streaming decode keeps every lane of a 64-lane group busy: a lane whose frame has
// latched (converged, or N iterations and the final test done) is given the next frame of
// the queue in a refill wave, while the other lanes keep iterating.  Each lane counts its
// own iterations (lane_l); the CN kernels need no per-lane state beyond the `fresh` mask
// (r^0 = 0 for a frame's first pass): the degree-1 decision buffers stay indexed by the
// global pass parity, and the buffer that holds a lane's final decisions is recorded per
// lane (lane_fbuf) when it latches.  A frame's arithmetic never depends on its lane or on
// the other lanes, so every frame decodes bit-identically to group mode (tests).

__global__ void k_stream_init(Group g) {
    const int b = threadIdx.x;
    if (b < g.C) {
        g.act[b] = 0u;
        g.unsat[b] = 0u;
        g.invalid[b] = 0u;
        g.fresh[b] = 0u;
        g.newm[b] = 0u;
        g.fin[b] = (g.B - 32 * b >= 32) ? FULL : ((1u << (g.B - 32 * b)) - 1u);   // every lane is free
    }
    if (b < g.B) {
        g.lane_frame[b] = -1;
        g.lane_l[b] = 0;
        g.lane_fbuf[b] = 0;
    }
    if (b == 0) {
        *g.iter = 1;
        *g.done = 0;
    }
}

// After CN pass l: per lane, latch a frame whose decisions of its iteration l_b - 1 satisfy
// every check (ET), or whose final test (pass N + 1) is done; else count the iteration.
// Requests a refill wave (IF node) once wave_min lanes wait or no lane iterates.
// Also the end of the pass: advances the global pass counter and sets the WHILE condition (loop
// while any lane iterates or waits for its refill wave).  The condition is taken before the refill
// wave of this pass; a wave that retires the last lanes costs one empty pass at the end of a decode.
// (The pass cap only guards against a host-path queue that never fills: a correct run ends long
// before it, when every frame has been decoded.)
__global__ void k_latch_stream(Group g, StreamJob* job, cudaGraphConditionalHandle if_h,
                               cudaGraphConditionalHandle while_h) {
    __shared__ uint32_t s_act[4], s_fin[4];
    pdl_launch_dependents();
    pdl_wait_previous();
    const int b = threadIdx.x, c = b >> 5, bit = b & 31;
    const int l = *reinterpret_cast<volatile int*>(g.iter);
    const int N = job->N;
    bool act = false, finished = false;
    if (b < g.B) {
        act = (g.act[c] >> bit) & 1u;
        if (act) {
            const int lb = g.lane_l[b];
            const bool passed = !((g.unsat[c] >> bit) & 1u);
            if (lb >= 2 && passed) {
                g.iters[b] = lb - 1;
                g.conv[b] = 1;
                finished = true;
            } else if (lb > N) {
                g.iters[b] = N;
                g.conv[b] = 0;
                finished = true;
            } else {
                g.lane_l[b] = lb + 1;
            }
            if (finished) g.lane_fbuf[b] = (l - 1) & 1;   // decisions of global pass l - 1
        }
    }
    const uint32_t a_bal = __ballot_sync(FULL, act && !finished), f_bal = __ballot_sync(FULL, finished);
    if (bit == 0 && c < g.C) {
        s_act[c] = a_bal;
        s_fin[c] = g.fin[c] | f_bal;
    }
    __syncthreads();
    if (b == 0) {
        int nact = 0, nfin = 0;
        for (int q = 0; q < g.C; ++q) {
            g.act[q] = s_act[q];
            g.fin[q] = s_fin[q];
            g.unsat[q] = 0u;
            g.fresh[q] = 0u;
            nact += __popc(s_act[q]);
            nfin += __popc(s_fin[q]);
        }
        cudaGraphSetConditional(if_h, (nfin > 0 && (nfin >= job->wave_min || nact == 0)) ? 1u : 0u);
        *g.iter = l + 1;
        const uint32_t passes = g.stat[0] + 1u;
        g.stat[0] = passes;
        cudaGraphSetConditional(while_h, ((nact + nfin) > 0 && passes < uint32_t(job->max_passes)) ? 1u : 0u);
    }
}

// Refill wave 1/4: outputs of the finished lanes (as k_finalize, per lane: frame lane_frame,
// degree-1 decisions from buffer lane_fbuf).
// Lanes of a chunk set in `mask` (and, if need_frame, holding a frame), listed in shared memory
// in lane order by the first C warps of the block (lane index, frame); returns the count.
__device__ __forceinline__ int list_lanes(const Group& g, const uint32_t* mask, bool need_frame, int* s_b, int* s_f,
                                          int* s_cnt) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int f = -1;
    bool in = false;
    uint32_t bal = 0;
    if (w < g.C) {
        const int b = w * 32 + lane;
        in = (mask[w] >> lane) & 1u;
        if (in) f = g.lane_frame[b];
        if (need_frame) in = in && f >= 0;
        bal = __ballot_sync(FULL, in);
        if (lane == 0) s_cnt[w] = __popc(bal);
    }
    __syncthreads();
    if (w < g.C && in) {
        int pos = __popc(bal & ((1u << lane) - 1u));   // rank in the chunk
        for (int q = 0; q < w; ++q) pos += s_cnt[q];
        s_b[pos] = w * 32 + lane;
        s_f[pos] = f;
    }
    __syncthreads();
    int tot = 0;
    for (int q = 0; q < g.C; ++q) tot += s_cnt[q];
    return tot;
}

// Refill wave 1/4: hard bits (original VN order, packed) of the lanes whose frame finished.  A warp
// owns one word of 32 VNs (thread = VN, one coalesced index load) and serves every finished lane
// of the group from it: per lane one load per thread (the VN's L entry or degree-1 decision word,
// the lane's column) and one ballot -- four lanes' loads in flight at a time.
__global__ void __launch_bounds__(256) k_finalize_lanes(CodeDev cd, Group g, StreamJob* job) {
    __shared__ int s_b[128], s_f[128], s_cnt[4];
    const int NW = (cd.n + 31) >> 5;
    const int nfin = list_lanes(g, g.fin, true, s_b, s_f, s_cnt);
    if (nfin == 0) return;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0)
        for (int q = threadIdx.x; q < nfin; q += blockDim.x) {
            job->iters[s_f[q]] = g.iters[s_b[q]];
            job->conv[s_f[q]] = g.conv[s_b[q]];
        }
    const int wblk = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (wblk >= NW) return;
    const int i = wblk * 32 + lane;
    const int v = (i < cd.n) ? __ldg(cd.vmap + i) : 0;
    const bool act = v >= 0 && i < cd.n, d1 = v < 0 && i < cd.n;
    const float* Lv = g.L + size_t(act ? v : 0) * 2 * g.B;
    const size_t d1off = size_t(d1 ? ~v : 0) * g.C;
    for (int q0 = 0; q0 < nfin; q0 += 4) {
        uint32_t bits[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = min(q0 + u, nfin - 1);
            const int b = s_b[q], c = b >> 5;
            const int par = g.lane_fbuf[b];
            uint32_t bit = 0;
            if (act) bit = Lv[lpos(b, g.B)] < 0.0f;
            else if (d1) bit = (g.d1bits[size_t(par) * cd.n_1 * g.C + d1off + c] >> (b & 31)) & 1u;
            bits[u] = bit;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t word = __ballot_sync(FULL, bits[u]);
            const int q = q0 + u;
            if (q < nfin && lane == u) {
                const int b = s_b[q];
                job->bits[size_t(s_f[q]) * NW + wblk] = (g.iters[b] < 0) ? 0u : word;
            }
        }
    }
}

// Refill wave 2/4: the finished lanes take the next frames of the queue (in lane order),
// among those whose inputs are on the device (f < avail).  A freed lane that gets no frame
// stays free (in `fin`, lane_frame = -1) while the queue still has frames to come, so a
// later wave can fill it; once every frame is claimed it retires.
__global__ void k_refill_assign(Group g, StreamJob* job) {
    __shared__ int s_base, s_take, s_pending;
    __shared__ uint32_t s_new[4];
    const int b = threadIdx.x, c = b >> 5, bit = b & 31;
    const bool freed = b < g.B && ((g.fin[c] >> bit) & 1u);
    uint32_t rank = 0, cnt = 0;
    for (int q = 0; q < g.C; ++q) {
        const uint32_t m = g.fin[q];
        if (q < c) rank += __popc(m);
        cnt += __popc(m);
    }
    if (freed) rank += __popc(g.fin[c] & ((1u << bit) - 1u));
    if (b == 0) {
        // claim up to cnt frames from [next, min(avail, nframes)) (one CAS loop per wave; the
        // K workspaces of a decode share the queue)
        const int nf = job->nframes;
        const int avail = min(*reinterpret_cast<volatile int*>(&job->avail), nf);
        int cur = *reinterpret_cast<volatile int*>(&job->next), take = 0;
        while (cnt) {
            take = min(int(cnt), avail - cur);
            if (take <= 0) { take = 0; break; }
            const int prev = atomicCAS(&job->next, cur, cur + take);
            if (prev == cur) break;
            cur = prev;
        }
        s_base = cur;
        s_take = take;
        s_pending = (cur + take) < nf;
    }
    __syncthreads();
    const int f = s_base + int(rank);
    const bool got = freed && int(rank) < s_take;
    if (freed) {
        g.lane_frame[b] = got ? f : -1;
        g.lane_l[b] = got ? 1 : 0;
    }
    const uint32_t nb = __ballot_sync(FULL, got);
    const uint32_t wait = __ballot_sync(FULL, freed && !got);
    if (bit == 0 && c < g.C) s_new[c] = nb;
    __syncthreads();
    if (b < g.C) g.newm[b] = s_new[b];
    if (bit == 0 && c < g.C) {
        g.fin[c] = s_pending ? wait : 0u;   // free lanes waiting for frames still to come
        g.invalid[c] &= ~nb;
    }
}

// Refill wave 3/4: lambda of the new frames into their lanes' columns (lam_a, L = lambda,
// accumulator 0, lam1).  Work item = (new lane, 32 consecutive VNs): one coalesced load of the
// frame's LLRs and of the VN indices, then one store per thread into the VN's row; four items'
// loads in flight per warp.  (The S_B bits follow in k_refill_synd.)
__global__ void __launch_bounds__(256) k_refill_scatter(CodeDev cd, Group g, StreamJob* job) {
    __shared__ int s_b[128], s_f[128], s_cnt[4];
    const int nnew = list_lanes(g, g.newm, false, s_b, s_f, s_cnt);
    if (nnew == 0) return;
    const int lane = threadIdx.x & 31;
    const int ntiles = (cd.n + 31) / 32;
    const long total = long(nnew) * ntiles;
    const long GW = long(gridDim.x) * (blockDim.x >> 5);
    for (long t0 = long(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); t0 < total; t0 += 4 * GW) {
        float val[4];
        int vm[4], bb[4], ii[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long t = t0 + u * GW;
            const int q = t < total ? int(t / ntiles) : 0;
            const int i = t < total ? int(t - long(q) * ntiles) * 32 + lane : cd.n;
            bb[u] = s_b[q];
            ii[u] = i;
            val[u] = (i < cd.n) ? __ldcv(job->llr + size_t(s_f[q]) * cd.n + i) : 0.0f;
            vm[u] = (i < cd.n) ? __ldg(cd.vmap + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = bb[u];
            if (__ballot_sync(FULL, ii[u] < cd.n && !isfinite(val[u])) && lane == 0) atomicOr(g.invalid + (b >> 5), 1u << (b & 31));
            if (ii[u] >= cd.n) continue;
            const int v = vm[u];
            if (v >= 0) {
                const float lz = __fadd_rn(val[u], 0.0f);   // -0 -> +0, as k_scatter
                const int po = lpos(b, g.B);
                g.lam_a[size_t(v) * g.B + po] = lz;
                g.L[size_t(v) * 2 * g.B + po] = lz;
                g.L[size_t(v) * 2 * g.B + g.B + po] = 0.0f;
            } else {
                g.lam1[lam1_idx(~v, b, g.B)] = lam1_phi_form(cd, val[u]);
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_refill_synd(CodeDev cd, Group g, StreamJob* job) {
    const int W = (cd.m + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const long item = long(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (item >= long(W) * g.C) return;
    const int wd = int(item / g.C), c = int(item % g.C);
    const uint32_t nm = g.newm[c];
    if (!nm) return;
    const int f = ((nm >> lane) & 1u) ? g.lane_frame[c * 32 + lane] : -1;
    const uint32_t word = (f >= 0) ? __ldcv(job->synd + size_t(f) * W + wd) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int bb = 0; bb < 32; ++bb) {
        const uint32_t bal = __ballot_sync(FULL, (word >> bb) & 1u);
        if (lane == bb) mine = bal;
    }
    const int j = wd * 32 + lane;
    if (j < cd.m) {
        uint32_t* p = g.synd_t + size_t(__ldg(cd.cn_new + j)) * g.C + c;
        *p = (*p & ~nm) | (mine & nm);
    }
}

// Refill wave 4/4: start the new frames (fresh: r^0 = 0 in their first pass); a frame with a
// non-finite LLR is not decoded (iterations = -1, R24) and waits for the next wave's outputs.
__global__ void k_refill_activate(Group g) {
    const int b = threadIdx.x, c = b >> 5, bit = b & 31;
    if (b == 0) g.stat[1] += 1u;
    if (b >= g.B) return;
    const uint32_t nm = g.newm[c];
    if (!((nm >> bit) & 1u)) return;
    const bool bad = (g.invalid[c] >> bit) & 1u;
    if (bad) {
        g.iters[b] = -1;
        g.conv[b] = 0;
        g.lane_fbuf[b] = 0;
        atomicOr(g.fin + c, 1u << bit);
    } else {
        g.iters[b] = 0;
        g.conv[b] = 0;
        atomicOr(g.act + c, 1u << bit);
        atomicOr(g.fresh + c, 1u << bit);
    }
    atomicAnd(g.newm + c, ~(1u << bit));
}

// ------------------------------------------------------------------ LLR from MD output (a1, R13)

// v and out may alias (the host-buffer path converts the staged v in place), so neither is
// __restrict__ and v is read through the coherent path.
__global__ void __launch_bounds__(256) k_md_llr(int64_t total, int n, int d, float c, const float* v,
                                                const float* __restrict__ xnorm, float* out, float xd) {
    const int nb = n / d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = e / n;
        const int i = int(e - f * n);
        const float xb = xnorm ? __ldg(xnorm + f * nb + i / d) : xd;
        const float cx = __fmul_rn(c, xb);
        out[e] = __fmul_rn(cx, v[e]);
    }
}

// ------------------------------------------------------------------ MD front end

// Alice's LLRs from her raw block x and Bob's rotation alpha: M(alpha) is
// linear, so c |x| (alpha x^)_i = c (alpha x)_i -- DESIGN.md N6: (alpha x)_i evaluated as
// acc = fmaf(+-alpha_p, x_q, acc) for q = 0..D-1 from 0, lambda_i = c * acc.
template <int D>
__global__ void __launch_bounds__(256) k_md_alice(int64_t nblk, float c, const float* __restrict__ x,
                                                  const float* __restrict__ alpha, float* __restrict__ out,
                                                  MdTable t) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nblk; b += int64_t(gridDim.x) * blockDim.x) {
        float a[D], xv[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            a[i] = __ldg(alpha + b * D + i);
            xv[i] = __ldcs(x + b * D + i);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            float acc = 0.0f;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const float ap = (t.ks[i * D + q] > 0) ? a[t.kp[i * D + q]] : -a[t.kp[i * D + q]];
                acc = __fmaf_rn(ap, xv[q], acc);
            }
            out[b * D + i] = __fmul_rn(c, acc);
        }
    }
}

// S = H c^T for frame-major bit-packed words (Step 1: Bob's syndrome of U; also a
// checker of any decided word).  Warp = 32 consecutive CNs of one frame.
__global__ void __launch_bounds__(256) k_syndrome(const int32_t* __restrict__ csr_ptr, const int32_t* __restrict__ csr_vn,
                                                  int n, int m, int batch, const uint32_t* __restrict__ bits,
                                                  uint32_t* __restrict__ synd) {
    const int W = (m + 31) >> 5, NW = (n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const long items = long(W) * batch;
    for (long it = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items;
         it += (long(gridDim.x) * blockDim.x) >> 5) {
        const int f = int(it / W), w = int(it - long(f) * W);
        const int j = w * 32 + lane;
        uint32_t par = 0;
        if (j < m) {
            const uint32_t* bf = bits + size_t(f) * NW;
            for (int e = __ldg(csr_ptr + j); e < __ldg(csr_ptr + j + 1); ++e) {
                const int v = __ldg(csr_vn + e);
                par ^= (__ldg(bf + (v >> 5)) >> (v & 31)) & 1u;
            }
        }
        const uint32_t word = __ballot_sync(FULL, par);
        if (lane == 0) synd[size_t(f) * W + w] = word;
    }
}

void launch_md_alice(int64_t nblk, int d, float c, const float* x, const float* alpha, float* out, const MdTable& t,
                     cudaStream_t s) {
    const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((nblk + 255) / 256, 148 * 16)));
    switch (d) {
        case 1: k_md_alice<1><<<grid, 256, 0, s>>>(nblk, c, x, alpha, out, t); break;
        case 2: k_md_alice<2><<<grid, 256, 0, s>>>(nblk, c, x, alpha, out, t); break;
        case 4: k_md_alice<4><<<grid, 256, 0, s>>>(nblk, c, x, alpha, out, t); break;
        default: k_md_alice<8><<<grid, 256, 0, s>>>(nblk, c, x, alpha, out, t); break;
    }
}

void launch_syndrome(const int32_t* csr_ptr, const int32_t* csr_vn, int n, int m, int batch, const uint32_t* bits,
                     uint32_t* synd, cudaStream_t s) {
    const long warps = long((m + 31) / 32) * batch;
    const unsigned grid = unsigned(std::max<long>(1, std::min<long>((warps + 7) / 8, 148 * 16)));
    k_syndrome<<<grid, 256, 0, s>>>(csr_ptr, csr_vn, n, m, batch, bits, synd);
}

// ------------------------------------------------------------------ batch counters (a7)

__global__ void k_counters(int batch, const int32_t* __restrict__ iters, const uint8_t* __restrict__ conv,
                           unsigned long long* __restrict__ out) {
    unsigned long long f = 0, cv = 0, it = 0, bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < batch; i += gridDim.x * blockDim.x) {
        const int t = iters[i];
        f += 1;
        cv += conv[i] ? 1 : 0;
        if (t >= 0) it += unsigned(t);
        else bad += 1;
    }
    for (int o = 16; o > 0; o >>= 1) {
        f += __shfl_xor_sync(FULL, f, o);
        cv += __shfl_xor_sync(FULL, cv, o);
        it += __shfl_xor_sync(FULL, it, o);
        bad += __shfl_xor_sync(FULL, bad, o);
    }
    if ((threadIdx.x & 31) == 0 && f) {
        atomicAdd(out + 0, f);
        atomicAdd(out + 1, cv);
        atomicAdd(out + 2, it);
        atomicAdd(out + 3, bad);
    }
}

void launch_counters(int batch, const int32_t* iters, const uint8_t* conv, int64_t* out, cudaStream_t s) {
    const int blocks = std::min(64, (batch + 255) / 256);
    k_counters<<<blocks, 256, 0, s>>>(batch, iters, conv, reinterpret_cast<unsigned long long*>(out));
}

// ------------------------------------------------------------------ launchers

template <int RULE, int NA, int ND, int MSG>
static void* cn_tile_fn() { return reinterpret_cast<void*>(&k_cn_tile<RULE, NA, ND, MSG>); }

template <int RULE, int MSG, int D = 0>
static void* cn_tile_kernel(int d, int nd) {
    if constexpr (D <= kMaxUnrolledCnDeg) {
        if (d == D) {
            if constexpr (D == 0) return cn_tile_fn<RULE, 0, 0, MSG>();
            else return nd ? cn_tile_fn<RULE, D - 1, 1, MSG>() : cn_tile_fn<RULE, D, 0, MSG>();
        }
        return cn_tile_kernel<RULE, MSG, D + 1>(d, nd);
    } else {
        return nullptr;
    }
}

static void* cn_kernel(int rule, int D, int nd, int msg16) {
    if (D < 0)
        return rule == METLDPC_RULE_EXACT ? reinterpret_cast<void*>(&k_cn_generic<METLDPC_RULE_EXACT>)
                                          : reinterpret_cast<void*>(&k_cn_generic<METLDPC_RULE_PHI_LUT>);
    if (msg16)
        return rule == METLDPC_RULE_EXACT ? cn_tile_kernel<METLDPC_RULE_EXACT, 1>(D, nd)
                                          : cn_tile_kernel<METLDPC_RULE_PHI_LUT, 1>(D, nd);
    return rule == METLDPC_RULE_EXACT ? cn_tile_kernel<METLDPC_RULE_EXACT, 0>(D, nd)
                                      : cn_tile_kernel<METLDPC_RULE_PHI_LUT, 0>(D, nd);
}

template <int RULE, int MSG>
static void* cn_pipe_kernel_m(int na, int nd) {
    switch (na * 2 + nd) {
        case 2: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 1, 0, MSG>);
        case 3: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 1, 1, MSG>);
        case 4: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 2, 0, MSG>);
        case 5: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 2, 1, MSG>);
        case 6: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 3, 0, MSG>);
        case 7: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 3, 1, MSG>);
        case 8: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 4, 0, MSG>);
        case 9: return reinterpret_cast<void*>(&k_cn_pipe<RULE, 4, 1, MSG>);
    }
    return nullptr;
}

template <int RULE, int MSG, int NA = 5>
static void* cn_ring_core_kernel(int na) {   // core classes: 5..16 active slots, no degree-1 slot
    if constexpr (NA <= kMaxUnrolledCnDeg) {
        if (na == NA) return reinterpret_cast<void*>(&k_cn_ring<RULE, NA, 0, MSG>);
        return cn_ring_core_kernel<RULE, MSG, NA + 1>(na);
    } else {
        return nullptr;
    }
}

template <int RULE, int MSG>
static void* cn_ring_kernel_m(int na, int nd) {
    if (na > 4) return nd == 0 ? cn_ring_core_kernel<RULE, MSG>(na) : nullptr;
    switch (na * 2 + nd) {
        case 2: return reinterpret_cast<void*>(&k_cn_ring<RULE, 1, 0, MSG>);
        case 3: return reinterpret_cast<void*>(&k_cn_ring<RULE, 1, 1, MSG>);
        case 4: return reinterpret_cast<void*>(&k_cn_ring<RULE, 2, 0, MSG>);
        case 5: return reinterpret_cast<void*>(&k_cn_ring<RULE, 2, 1, MSG>);
        case 6: return reinterpret_cast<void*>(&k_cn_ring<RULE, 3, 0, MSG>);
        case 7: return reinterpret_cast<void*>(&k_cn_ring<RULE, 3, 1, MSG>);
        case 8: return reinterpret_cast<void*>(&k_cn_ring<RULE, 4, 0, MSG>);
        case 9: return reinterpret_cast<void*>(&k_cn_ring<RULE, 4, 1, MSG>);
    }
    return nullptr;
}

// CTA-ring kernel (k_cn_ring) for the pipelined classes (default; METLDPC_RING=0 selects the
// per-warp pipeline k_cn_pipe for A/B).  Measured (C3, CN phase per 64-lane group-iteration,
// same call): fp32 0.443 vs 0.450 ms, 16-bit messages 0.381 vs 0.406 ms.
static bool cn_use_ring() {
    static const bool on = [] {
        const char* e = std::getenv("METLDPC_RING");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int NA, int ND, int MSG>
static void ring_geom(int* threads, size_t* smem) {
    *threads = RingCfg<NA, ND, MSG>::THREADS;
    *smem = size_t(RingCfg<NA, ND, MSG>::SMEM);
}

template <int MSG, int NA = 5>
static void cn_ring_core_geom(int na, int* threads, size_t* smem) {
    if constexpr (NA <= kMaxUnrolledCnDeg) {
        if (na == NA) return ring_geom<NA, 0, MSG>(threads, smem);
        return cn_ring_core_geom<MSG, NA + 1>(na, threads, smem);
    } else {
        *threads = 0;
        *smem = 0;
    }
}

template <int MSG>
static void cn_ring_geom_m(int D, int nd, int* threads, size_t* smem) {
    if (D - nd > 4) return cn_ring_core_geom<MSG>(D - nd, threads, smem);
    switch ((D - nd) * 2 + nd) {
        case 2: ring_geom<1, 0, MSG>(threads, smem); return;
        case 3: ring_geom<1, 1, MSG>(threads, smem); return;
        case 4: ring_geom<2, 0, MSG>(threads, smem); return;
        case 5: ring_geom<2, 1, MSG>(threads, smem); return;
        case 6: ring_geom<3, 0, MSG>(threads, smem); return;
        case 7: ring_geom<3, 1, MSG>(threads, smem); return;
        case 8: ring_geom<4, 0, MSG>(threads, smem); return;
        case 9: ring_geom<4, 1, MSG>(threads, smem); return;
    }
    *threads = 0;
    *smem = 0;
}

static void* cn_pipe_kernel(int rule, int na, int nd, int msg16) {
    if (cn_use_ring()) {
        if (rule == METLDPC_RULE_EXACT)
            return msg16 ? cn_ring_kernel_m<METLDPC_RULE_EXACT, 1>(na, nd) : cn_ring_kernel_m<METLDPC_RULE_EXACT, 0>(na, nd);
        return msg16 ? cn_ring_kernel_m<METLDPC_RULE_PHI_LUT, 1>(na, nd) : cn_ring_kernel_m<METLDPC_RULE_PHI_LUT, 0>(na, nd);
    }
    if (rule == METLDPC_RULE_EXACT)
        return msg16 ? cn_pipe_kernel_m<METLDPC_RULE_EXACT, 1>(na, nd) : cn_pipe_kernel_m<METLDPC_RULE_EXACT, 0>(na, nd);
    return msg16 ? cn_pipe_kernel_m<METLDPC_RULE_PHI_LUT, 1>(na, nd) : cn_pipe_kernel_m<METLDPC_RULE_PHI_LUT, 0>(na, nd);
}

// Pipelined kernel for classes with 1..4 active slots and <= 1 degree-1 slot (64-lane
// groups); METLDPC_PIPE=0 selects the register-only k_cn_tile instead (A/B experiments).
bool cn_use_pipe(int D, int nd) {
    static const bool on = [] {
        const char* e = std::getenv("METLDPC_PIPE");
        return !(e && e[0] == '0');
    }();
    // core classes (5..16 active slots, no degree-1 slot) in the ring kernel too (default;
    // METLDPC_RING_CORE=0: the register-only tiled kernel).  Measured (r0.1de C3, fixed N, same
    // call): CN phase fp32 0.463 vs 0.473 ms, 16-bit 0.378 vs 0.393 ms.
    static const bool core = [] {
        const char* e = std::getenv("METLDPC_RING_CORE");
        return !(e && e[0] == '0');
    }();
    if (!on || D < 0 || nd > 1 || D - nd < 1) return false;
    if (D - nd <= 4) return true;
    return core && cn_use_ring() && nd == 0 && D <= kMaxUnrolledCnDeg;
}

template <int NA, int ND, int MSG>
static void pipe_geom(int rule, int* threads, size_t* smem) {
    using PC = PipeCfg<NA, ND, MSG>;
    *threads = PC::THREADS;
    *smem = size_t(rule == METLDPC_RULE_EXACT ? PhiT<METLDPC_RULE_EXACT>::TAB_BYTES : PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES) +
            size_t(PC::WARPS) * PC::WARP_BYTES;
}

template <int MSG>
static void cn_pipe_geom_m(int rule, int D, int nd, int* threads, size_t* smem) {
    switch ((D - nd) * 2 + nd) {
        case 2: pipe_geom<1, 0, MSG>(rule, threads, smem); return;
        case 3: pipe_geom<1, 1, MSG>(rule, threads, smem); return;
        case 4: pipe_geom<2, 0, MSG>(rule, threads, smem); return;
        case 5: pipe_geom<2, 1, MSG>(rule, threads, smem); return;
        case 6: pipe_geom<3, 0, MSG>(rule, threads, smem); return;
        case 7: pipe_geom<3, 1, MSG>(rule, threads, smem); return;
        case 8: pipe_geom<4, 0, MSG>(rule, threads, smem); return;
        case 9: pipe_geom<4, 1, MSG>(rule, threads, smem); return;
    }
    *threads = 0;
    *smem = 0;
}

static void cn_pipe_geom(int rule, int D, int nd, int msg16, int* threads, size_t* smem) {
    if (cn_use_ring()) {
        if (msg16) cn_ring_geom_m<1>(D, nd, threads, smem);
        else cn_ring_geom_m<0>(D, nd, threads, smem);
        return;
    }
    if (msg16) cn_pipe_geom_m<1>(rule, D, nd, threads, smem);
    else cn_pipe_geom_m<0>(rule, D, nd, threads, smem);
}

int cn_tile_max(int D, int nd) { return (D - nd) <= 4 ? 32 : 8; }
int cn_units_per_tile(int, int) { return 1; }

size_t cn_smem(int rule, int D, int nd) {
    const size_t tab = size_t(rule == METLDPC_RULE_EXACT ? PhiT<METLDPC_RULE_EXACT>::TAB_BYTES
                                                         : PhiT<METLDPC_RULE_PHI_LUT>::TAB_BYTES);
    if (D < 0) return tab;
    const int na = std::max(1, D - nd);
    return tab + size_t(kCnThreads / 32) * cn_tile_max(D, nd) * na * sizeof(int);
}

int cn_blocks_per_sm(int rule, int D, int nd, int msg16) {
    if (cn_use_pipe(D, nd)) {
        void* f = cn_pipe_kernel(rule, D - nd, nd, msg16);
        int th;
        size_t sm;
        cn_pipe_geom(rule, D, nd, msg16, &th, &sm);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        return 1;
    }
    int nb = 0;
    void* f = cn_kernel(rule, D, nd, msg16);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cn_smem(rule, D, nd)));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kCnThreads, cn_smem(rule, D, nd)) != cudaSuccess) nb = 1;
    return nb > 0 ? nb : 1;
}

int finish_blocks_per_sm() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_finish, 256, 0) != cudaSuccess) nb = 1;
    return nb > 0 ? nb : 1;
}

void launch_scatter(const CodeDev& cd, const Group& g, const float* llr, int nb, cudaStream_t s) {
    dim3 grid((cd.n + 31) / 32, g.C);
    k_scatter<<<grid, 256, 0, s>>>(cd, g, llr, nb);
}

void launch_pack_syndrome(const CodeDev& cd, const Group& g, const uint32_t* synd, int nb, cudaStream_t s) {
    const long items = long((cd.m + 31) / 32) * g.C;
    k_pack_syndrome<<<unsigned((items + 7) / 8), 256, 0, s>>>(cd, g, synd, nb);
}

void launch_init_ctl(const Group& g, int nb, int N, cudaStream_t s) { k_init_ctl<<<1, 128, 0, s>>>(g, nb, N); }

static void launch_small(void* f, dim3 grid, dim3 block, void** args, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (pdl) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    cudaLaunchKernelExC(&cfg, f, args);
}

void launch_latch_dev(const Group& g, bool et, cudaStream_t s, bool pdl) {
    int e = et ? 1 : 0;
    void* args[] = {const_cast<Group*>(&g), &e};
    launch_small(reinterpret_cast<void*>(&k_latch_dev), dim3(1), dim3(32), args, s, pdl);
}

void launch_stream_init(const Group& g, cudaStream_t s) { k_stream_init<<<1, 128, 0, s>>>(g); }

void launch_latch_stream(const Group& g, StreamJob* job, unsigned long long if_handle, unsigned long long while_handle,
                         cudaStream_t s, bool pdl) {
    cudaGraphConditionalHandle h = cudaGraphConditionalHandle(if_handle);
    cudaGraphConditionalHandle hw = cudaGraphConditionalHandle(while_handle);
    void* args[] = {const_cast<Group*>(&g), &job, &h, &hw};
    launch_small(reinterpret_cast<void*>(&k_latch_stream), dim3(1), dim3(128), args, s, pdl);
}


// Host path: frames [0, avail) of the queue are on the device (launched on the copy stream
// after their H2D copies and LLR conversion, so stream order makes the data visible first).
__global__ void k_publish(StreamJob* job, int avail) {
    __threadfence();
    atomicMax(&job->avail, avail);
}

void launch_publish(StreamJob* job, int avail, cudaStream_t s) { k_publish<<<1, 1, 0, s>>>(job, avail); }

void launch_refill_wave(const CodeDev& cd, const Group& g, StreamJob* job, cudaStream_t s) {
    const int NW = (cd.n + 31) / 32, W = (cd.m + 31) / 32;
    k_finalize_lanes<<<unsigned((NW + 7) / 8), 256, 0, s>>>(cd, g, job);
    k_refill_assign<<<1, 128, 0, s>>>(g, job);
    k_refill_scatter<<<148 * 8, 256, 0, s>>>(cd, g, job);
    k_refill_synd<<<unsigned((long(W) * g.C + 7) / 8), 256, 0, s>>>(cd, g, job);
    k_refill_activate<<<1, 128, 0, s>>>(g);
}

void launch_loop_ctl(const Group& g, unsigned long long cond_handle, cudaStream_t s, bool pdl) {
    cudaGraphConditionalHandle h = cudaGraphConditionalHandle(cond_handle);
    void* args[] = {const_cast<Group*>(&g), &h};
    launch_small(reinterpret_cast<void*>(&k_loop_ctl), dim3(1), dim3(1), args, s, pdl);
}

// Optional persisting-L2 window over the group's L / accumulator rows (set by the decoder
// when the device supports it).
static cudaError_t launch_with_window(void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s,
                                      const L2Window& w, bool pdl = false) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (w.bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = w.base;
        attr[na].val.accessPolicyWindow.num_bytes = w.bytes;
        attr[na].val.accessPolicyWindow.hitRatio = w.hit_ratio;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    if (pdl) {   // programmatic dependent launch: may start while the previous CN class drains
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, f, args);
}

void launch_cn(const CodeDev& cd, const Group& g, int rule, int D, int nd, int begin, int count, int ts, int grid,
               int l, bool check, cudaStream_t s, const L2Window& w, bool pdl) {
    CnCtl k{check ? 1 : 0, (l - 1) & 1, l & 1, l == 0 ? 1 : 0, check ? 1 : 0};
    if (cn_use_pipe(D, nd)) {
        void* f = cn_pipe_kernel(rule, D - nd, nd, g.msg16);
        int th;
        size_t sm;   // the smem attribute was set by cn_blocks_per_sm
        cn_pipe_geom(rule, D, nd, g.msg16, &th, &sm);
        void* args[] = {const_cast<CodeDev*>(&cd), const_cast<Group*>(&g), &k, &begin, &count};
        launch_with_window(f, dim3(grid), dim3(th), args, sm, s, w, pdl);
        return;
    }
    void* f = cn_kernel(rule, D, nd, g.msg16);
    if (D < 0) {
        void* args[] = {const_cast<CodeDev*>(&cd), const_cast<Group*>(&g), &k, &begin, &count};
        launch_with_window(f, dim3(grid), dim3(kCnThreads), args, cn_smem(rule, D, nd), s, w, pdl);
    } else {
        void* args[] = {const_cast<CodeDev*>(&cd), const_cast<Group*>(&g), &k, &begin, &count, &ts};
        launch_with_window(f, dim3(grid), dim3(kCnThreads), args, cn_smem(rule, D, nd), s, w, pdl);
    }
}

void launch_finish(const CodeDev& cd, const Group& g, int grid, cudaStream_t s, const L2Window& w, bool pdl) {
    void* args[] = {const_cast<CodeDev*>(&cd), const_cast<Group*>(&g)};
    launch_with_window(reinterpret_cast<void*>(&k_finish), dim3(grid), dim3(256), args, 0, s, w, pdl);
}

void launch_check(const CodeDev& cd, const Group& g, int grid, int l, cudaStream_t s) {
    if (g.B == 64) k_check64<<<grid, 256, 0, s>>>(cd, g, l & 1);
    else k_check<<<grid, 256, 0, s>>>(cd, g, l & 1);
}

void launch_latch(const Group& g, int l, bool final_, cudaStream_t s) { k_latch<<<1, 32, 0, s>>>(g, l, final_ ? 1 : 0); }

void launch_finalize(const CodeDev& cd, const Group& g, int nb, uint32_t* bits_out, int32_t* iters_out,
                     uint8_t* conv_out, cudaStream_t s) {
    const int NW = (cd.n + 31) / 32;
    dim3 grid((NW + 7) / 8, g.C);
    k_finalize<<<grid, 256, 0, s>>>(cd, g, nb, bits_out, iters_out, conv_out);
}

void launch_md_llr(int64_t total, int n, int d, float c, const float* v, const float* xnorm, float* out,
                   cudaStream_t s) {
    const float xd = float(std::sqrt(double(d)));
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    k_md_llr<<<unsigned(blocks), 256, 0, s>>>(total, n, d, c, v, xnorm, out, xd);
}

}  // namespace metldpc

namespace metldpc {
const int kCnThreadsHost = kCnThreads;
}
