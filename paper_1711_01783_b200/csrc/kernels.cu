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
#include <cmath>

#include "internal.h"
#include "kernels.cuh"

namespace metldpc {

#define FULL 0xffffffffu

// ------------------------------------------------------------------ phi (N2)

template <int RULE>
__device__ __forceinline__ float phi_dev(const float* __restrict__ tab, float y, float top) {
    const uint32_t u = __float_as_uint(y);
    const uint32_t uc = min(max(u, kPhiLoBits), kPhiHiBits - 1u);
    const uint32_t idx = (uc - kPhiLoBits) >> (23 - kPhiJ);
    const float t = __fmul_rn(__uint2float_rn(uc & ((1u << (23 - kPhiJ)) - 1u)), 1.0f / float(1u << (23 - kPhiJ)));
    float v;
    if constexpr (RULE == METLDPC_RULE_EXACT) {
        const float4 c = reinterpret_cast<const float4*>(tab)[idx];
        v = __fmaf_rn(__fmaf_rn(__fmaf_rn(c.w, t, c.z), t, c.y), t, c.x);
    } else {
        const float2 c = reinterpret_cast<const float2*>(tab)[idx];
        v = __fmaf_rn(c.y, t, c.x);
    }
    v = (u < kPhiLoBits) ? top : v;
    v = (u >= kPhiHiBits) ? 0.0f : v;
    return v;
}

// ------------------------------------------------------------------ check-node update (a2 + a4)

struct CnCtl {
    int check;   // test the syndrome of iteration l-1 (reads L^{l-1}, degree-1 bits[rpar])
    int first;   // l == 1: r^0 = 0 (not read)
    int rpar, wpar;
};

// One CN j, one 32-lane chunk c, total degree d (active edges first, then degree-1):
// DESIGN.md N1 in registers.  Eqs. (2)-(3), with the syndrome sign (R1).
// FIXED: d == D known at compile time (fully unrolled, arrays in registers);
// otherwise d <= D at run time (generic path for rare high-degree CNs).
template <int RULE, int D, bool FIXED>
__device__ __forceinline__ void cn_item(const CodeDev& cd, const Group& g, const float* tab, const CnCtl& k,
                                        int j, int c, int lane, uint32_t amask, int ab, int na, int db, int d_rt,
                                        uint32_t* s_unsat) {
    const int d = FIXED ? D : d_rt;
    const int B = g.B, C = g.C;
    const size_t off = size_t(c) * 32 + lane;
    const int sbit = (__ldg(g.synd_t + size_t(j) * C + c) >> lane) & 1;
    if constexpr (FIXED && D == 0) {   // empty row: satisfied iff S_B[j] = 0
        if (k.check) {
            const uint32_t mm = __ballot_sync(FULL, sbit) & amask;
            if (mm && lane == 0) atomicOr(&s_unsat[c], mm);
        }
        return;
    } else {
        const int idx = (lane < na) ? __ldg(cd.a_vn + ab + lane) : 0;
        float p[D], P[D], lam1[D];
        uint32_t negmask = 0;
        int chk = sbit;
#pragma unroll
        for (int s = 0; s < d; ++s) {
            float x;
            if (s < na) {
                const int v = __shfl_sync(FULL, idx, s);
                const float Lv = __ldg(g.L + size_t(v) * B + off);
                const float ro = k.first ? 0.0f : __ldcs(g.r + size_t(ab + s) * B + off);
                x = __fsub_rn(Lv, ro);                                  // extrinsic, R10
                chk ^= int(Lv < 0.0f);                                  // c_v^{l-1}, N4
            } else {
                const int q = db + (s - na);
                x = __ldcs(g.lam1 + size_t(q) * B + off);               // degree-1 VN sends its prior
                lam1[s] = x;
                if (k.check) chk ^= int((__ldg(g.d1bits + (size_t(k.rpar) * cd.n_1 + q) * C + c) >> lane) & 1u);
            }
            negmask |= uint32_t(x < 0.0f) << s;
            p[s] = phi_dev<RULE>(tab, fabsf(x), cd.phi_top);
        }
        if (k.check) {
            const uint32_t mm = __ballot_sync(FULL, chk) & amask;
            if (mm && lane == 0) atomicOr(&s_unsat[c], mm);
        }
        float acc = 0.0f;
#pragma unroll
        for (int s = 0; s < d; ++s) { P[s] = acc; acc = __fadd_rn(acc, p[s]); }
        const uint32_t par = uint32_t(sbit) ^ (__popc(negmask) & 1u);
        const bool act = (amask >> lane) & 1u;
        float Q = 0.0f;
#pragma unroll
        for (int s = d - 1; s >= 0; --s) {
            const float S = __fadd_rn(P[s], Q);
            const float mag = fminf(phi_dev<RULE>(tab, S, cd.phi_top), kRMax);
            const float o = (par ^ ((negmask >> s) & 1u)) ? -mag : mag;
            if (s < na) {
                if (act) __stcs(g.r + size_t(ab + s) * B + off, o);
            } else {
                const int q = db + (s - na);
                const uint32_t bal = __ballot_sync(FULL, __fadd_rn(lam1[s], o) < 0.0f);   // Step 5 for VN_b
                if (lane == 0) {
                    uint32_t* w = g.d1bits + (size_t(k.wpar) * cd.n_1 + q) * C + c;
                    *w = (amask == FULL) ? bal : ((bal & amask) | (*w & ~amask));
                }
            }
            Q = __fadd_rn(Q, p[s]);
        }
    }
}

template <int RULE, int D, int DHI>
__device__ __forceinline__ void cn_dispatch(int d, const CodeDev& cd, const Group& g, const float* tab,
                                            const CnCtl& k, int j, int c, int lane, uint32_t amask, int ab,
                                            int na, int db, uint32_t* s_unsat) {
    if constexpr (D <= DHI) {
        if (d == D) {
            cn_item<RULE, D, true>(cd, g, tab, k, j, c, lane, amask, ab, na, db, d, s_unsat);
            return;
        }
        cn_dispatch<RULE, D + 1, DHI>(d, cd, g, tab, k, j, c, lane, amask, ab, na, db, s_unsat);
    }
}

// One CN degree class (CNs with total degree in [DLO, DHI], listed in cls_cn).
// DHI <= 16: unrolled per degree; DHI == 32: generic run-time-degree path.
template <int RULE, int DLO, int DHI>
__global__ void __launch_bounds__(256) k_cn_update(CodeDev cd, Group g, CnCtl k, const int32_t* __restrict__ cls_cn,
                                                   int count) {
    extern __shared__ __align__(16) float s_tab[];
    __shared__ uint32_t s_unsat[4], s_act[4];
    if (*reinterpret_cast<volatile int*>(g.done)) return;
    constexpr int tabn4 = (RULE == METLDPC_RULE_EXACT) ? kPhiBins : kPhiBins / 2;   // float4 units
    for (int i = threadIdx.x; i < tabn4; i += blockDim.x)
        reinterpret_cast<float4*>(s_tab)[i] = __ldg(reinterpret_cast<const float4*>(cd.phi) + i);
    if (threadIdx.x < g.C) { s_unsat[threadIdx.x] = 0u; s_act[threadIdx.x] = g.act[threadIdx.x]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int lc = __ffs(g.C) - 1;  // C is a power of two
    const long total = long(count) << lc;
    for (long item = long(blockIdx.x) * wpb + (threadIdx.x >> 5); item < total; item += long(gridDim.x) * wpb) {
        const int c = int(item & (g.C - 1));
        const uint32_t amask = s_act[c];
        if (!amask) continue;
        const int j = __ldg(cls_cn + (item >> lc));
        const int ab = __ldg(cd.cn_aptr + j), na = __ldg(cd.cn_aptr + j + 1) - ab;
        const int db = __ldg(cd.cn_dptr + j), d = na + (__ldg(cd.cn_dptr + j + 1) - db);
        if constexpr (DHI <= 16) {
            cn_dispatch<RULE, DLO, DHI>(d, cd, g, s_tab, k, j, c, lane, amask, ab, na, db, s_unsat);
        } else {
            cn_item<RULE, DHI, false>(cd, g, s_tab, k, j, c, lane, amask, ab, na, db, d, s_unsat);
        }
    }
    __syncthreads();
    if (k.check && threadIdx.x < g.C && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
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
        for (int t = ab; t < ae; ++t) chk ^= uint32_t(__ldg(g.L + size_t(__ldg(cd.a_vn + t)) * g.B + off) < 0.0f);
        for (int q = db; q < de; ++q) chk ^= (__ldg(g.d1bits + (size_t(par) * cd.n_1 + q) * g.C + c) >> lane) & 1u;
        const uint32_t mm = __ballot_sync(FULL, chk) & amask;
        if (mm && lane == 0) atomicOr(&s_unsat[c], mm);
    }
    __syncthreads();
    if (threadIdx.x < g.C && s_unsat[threadIdx.x]) atomicOr(g.unsat + threadIdx.x, s_unsat[threadIdx.x]);
}

// ------------------------------------------------------------------ variable-node update (a3)

// L_a = lambda_a + sum of r over C_a, left fold in the caller's CSC slot order (Eq. 4/5, N3).
__global__ void __launch_bounds__(256) k_vn_update(CodeDev cd, Group g) {
    __shared__ uint32_t s_act[4];
    if (*reinterpret_cast<volatile int*>(g.done)) return;
    if (threadIdx.x < g.C) s_act[threadIdx.x] = g.act[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int lc = __ffs(g.C) - 1;
    const int B = g.B;
    const long total = long(cd.n_a) << lc;
    for (long item = long(blockIdx.x) * wpb + (threadIdx.x >> 5); item < total; item += long(gridDim.x) * wpb) {
        const int a = int(item >> lc), c = int(item & (g.C - 1));
        const uint32_t amask = s_act[c];
        if (!amask) continue;
        const size_t off = size_t(c) * 32 + lane;
        const int vb = __ldg(cd.vn_aptr + a), ve = __ldg(cd.vn_aptr + a + 1);
        float acc = __ldg(g.lam_a + size_t(a) * B + off);
        for (int base = vb; base < ve; base += 32) {
            const int cnt = min(32, ve - base);
            const int eid = (lane < cnt) ? __ldg(cd.vn_aedge + base + lane) : 0;
            int s = 0;
            for (; s + 8 <= cnt; s += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcs(g.r + size_t(__shfl_sync(FULL, eid, s + u)) * B + off);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
            }
            for (; s < cnt; ++s) acc = __fadd_rn(acc, __ldcs(g.r + size_t(__shfl_sync(FULL, eid, s)) * B + off));
        }
        if ((amask >> lane) & 1u) g.L[size_t(a) * B + off] = acc;
    }
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
            g.lam_a[size_t(v) * g.B + off] = val;
            g.L[size_t(v) * g.B + off] = val;                       // L^0 = lambda (Step 2)
        } else {
            g.lam1[size_t(~v) * g.B + off] = val;
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
    if (j < cd.m) g.synd_t[size_t(j) * g.C + c] = mine;
}

__global__ void k_init_ctl(Group g, int nb) {
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
            b = g.L[size_t(v) * g.B + off] < 0.0f;
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

// ------------------------------------------------------------------ LLR from MD output (a1, R13)

__global__ void __launch_bounds__(256) k_md_llr(int64_t total, int n, int d, float c, const float* __restrict__ v,
                                                const float* __restrict__ xnorm, float* __restrict__ out,
                                                float xd) {
    const int nb = n / d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = e / n;
        const int i = int(e - f * n);
        const float xb = xnorm ? __ldg(xnorm + f * nb + i / d) : xd;
        const float cx = __fmul_rn(c, xb);
        out[e] = __fmul_rn(cx, __ldg(v + e));
    }
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

template <int RULE, int W>
static void* cn_fn() { return reinterpret_cast<void*>(&k_cn_update<RULE, kCnWinLo[W], kCnWinHi[W]>); }

template <int RULE>
static void* cn_kernel_rule(int win) {
    switch (win) {
        case 0: return cn_fn<RULE, 0>();
        case 1: return cn_fn<RULE, 1>();
        case 2: return cn_fn<RULE, 2>();
        case 3: return cn_fn<RULE, 3>();
        default: return cn_fn<RULE, 4>();
    }
}

static void* cn_kernel(int rule, int win) {
    return rule == METLDPC_RULE_EXACT ? cn_kernel_rule<METLDPC_RULE_EXACT>(win)
                                      : cn_kernel_rule<METLDPC_RULE_PHI_LUT>(win);
}

static size_t cn_smem(int rule) {
    return size_t(kPhiBins) * (rule == METLDPC_RULE_EXACT ? 4 : 2) * sizeof(float);
}

int cn_window(int dlo) {
    for (int w = 0; w < kNumCnWindows; ++w)
        if (kCnWinLo[w] == dlo) return w;
    return kNumCnWindows - 1;
}

int cn_blocks_per_sm(int rule, int win) {
    int nb = 0;
    void* f = cn_kernel(rule, win);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cn_smem(rule)));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 256, cn_smem(rule)) != cudaSuccess) nb = 1;
    return nb > 0 ? nb : 1;
}

int vn_blocks_per_sm() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_vn_update, 256, 0) != cudaSuccess) nb = 1;
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

void launch_init_ctl(const Group& g, int nb, cudaStream_t s) { k_init_ctl<<<1, 128, 0, s>>>(g, nb); }

void launch_cn(const CodeDev& cd, const Group& g, int rule, int win, const int32_t* cls_cn, int count, int grid,
               int l, bool check, cudaStream_t s) {
    CnCtl k{check ? 1 : 0, l == 1 ? 1 : 0, (l - 1) & 1, l & 1};
    void* f = cn_kernel(rule, win);
    void* args[] = {const_cast<CodeDev*>(&cd), const_cast<Group*>(&g), &k, const_cast<int32_t**>(&cls_cn), &count};
    cudaLaunchKernel(f, dim3(grid), dim3(256), args, cn_smem(rule), s);
}

void launch_vn(const CodeDev& cd, const Group& g, int grid, cudaStream_t s) {
    k_vn_update<<<grid, 256, 0, s>>>(cd, g);
}

void launch_check(const CodeDev& cd, const Group& g, int grid, int l, cudaStream_t s) {
    k_check<<<grid, 256, 0, s>>>(cd, g, l & 1);
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
