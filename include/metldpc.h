/*
 * metldpc.h -- C ABI of the B200-native batched syndrome belief-propagation
 * decoder for long, low-rate multi-edge-type LDPC codes (arXiv 1711.01783).
 *
 * Citations: P:L = PAPER.md line L; S:L = SPEC.md line L; DESIGN.md Rn =
 * reading n, Nn = numerics-contract clause n.
 *
 * Conventions for every call
 *  - Every call returns metldpc_status (METLDPC_OK = 0) unless stated; no C++
 *    exception crosses the ABI.  On error, metldpc_last_error() returns a
 *    thread-local one-line detail (e.g. "alist line 17: VN index 4 >= n=3").
 *  - Argument and shape errors are returned before any work is enqueued
 *    (S:200).  Nothing is written to outputs on error.
 *  - Ownership: the library owns handles; the caller owns every buffer it
 *    passes.  Host arrays passed to *_create are copied.  "dev" pointers are
 *    CUDA device pointers on the handle's device (e.g. torch data_ptr()).
 *  - Streams: cuda_stream is a cudaStream_t cast to uintptr_t (0 = legacy
 *    default stream).  Stream-ordered calls return once the work is enqueued;
 *    outputs are valid after the stream synchronises.
 *  - Thread safety: a code is immutable and may be shared by any number of
 *    decoders and threads.  A decoder is used by one host thread at a time.
 *  - Bit vectors are packed LSB-first into uint32 words: bit i of a vector is
 *    (w[i >> 5] >> (i & 31)) & 1.
 *  - LLR convention (R2): lambda = ln P(c=0)/P(c=1) = -ln q^0 with
 *    q^0 the ratio of Eq. (1); decided bit is 1 iff the posterior
 *    LLR is < 0 (Step 5: "If q_i^l > 1, c_i = 1, otherwise 0").
 */
#ifndef METLDPC_H
#define METLDPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    METLDPC_OK = 0,
    METLDPC_EINVAL = 1,        /* bad argument (NULL, size, range, batch > max_batch, ...) */
    METLDPC_EFORMAT = 2,       /* malformed H: index out of range, duplicate edge, degree-0 VN,
                                  CSR/CSC mismatch, alist syntax            */
    METLDPC_ENOMEM = 3,        /* host or device allocation failed                            */
    METLDPC_ECUDA = 4,         /* CUDA runtime error (detail in metldpc_last_error)          */
    METLDPC_EUNSUPPORTED = 5   /* valid but outside this build (CN degree > 32, no sm_100 GPU) */
} metldpc_status;

typedef struct metldpc_code_s* metldpc_code;        /* immutable H + device layout          */
typedef struct metldpc_decoder_s* metldpc_decoder;  /* per-device workspace                  */

/* Check-node rule (R4, R5, N1, N2). */
typedef enum {
    METLDPC_RULE_EXACT = 0,    /* Eqs. (2)-(3) exactly, sign/phi form, fp32 cubic phi table   */
    METLDPC_RULE_PHI_LUT = 1   /* the P:146 lookup-table LLR update (linear phi table)        */
} metldpc_cn_rule;

typedef struct {
    int32_t rule;              /* metldpc_cn_rule; default METLDPC_RULE_EXACT                 */
    int32_t max_iter;          /* N >= 1 (100/150/200); default 100                    */
    int32_t early_term;        /* 1 = per-frame syndrome early termination (default, R12);
                                  0 = fixed N, the paper's Figure-1 flow               */
    int32_t lanes_per_group;   /* codewords interleaved per group: 32, 64 or 128; default 64
                                  (coalesced when a multiple of 32)               */
    int32_t groups_in_flight;  /* lane groups decoded concurrently on their own streams, 1..8;
                                  default 1 (each has its own ~1 GB workspace at C3).  With 1
                                  the decoder keeps its posterior / VN-sum rows in a persisting
                                  L2 window (it sets the context's
                                  cudaLimitPersistingL2CacheSize; METLDPC_L2PERSIST=0
                                  disables)                                                   */
    int32_t lane_refill;       /* 1 = streaming decode (needs early_term, 64-lane groups): a lane
                                  whose frame has latched takes the next frame of the batch in
                                  a refill wave while the other lanes keep iterating, so a
                                  group no longer waits for its slowest frame; per-frame
                                  results are identical to group mode.  Default 1 (used by
                                  metldpc_decode when early_term and lanes_per_group = 64;
                                  the host-buffer calls and profiling use group mode).     */
    int32_t msg_bits;          /* storage width of the edge messages r between iterations:
                                  32 (fp32, default) or 16 (R28 / N7: rint(2^10 r)
                                  in 16 bits, within 2^-11 of the CN output, which the VN sum
                                  of the same iteration uses unrounded; halves the dominant
                                  HBM stream).  16 needs lanes_per_group = 64.         */
} metldpc_config_t;

typedef struct {
    int32_t n, m;              /* VNs, CNs (H is m x n, R = (n - m)/n)                */
    int64_t edges;             /* Table 1 "Total Number of Edges"                            */
    int64_t iter_edges;        /* Table 1 "Number of Edges to pass messages": edges of VNs of
                                  degree > 1                                        */
    int32_t n_active;          /* VNs of degree > 1 (Table 1 "Updated VNs")                  */
    int32_t n_deg1;            /* degree-1 VNs (Table 1 "Ignored VNs")           */
    int32_t max_cn_deg, max_vn_deg;
} metldpc_code_info_t;

/* Kernel-level accounting of one decoder (bench / tests). */
typedef struct {
    int64_t launches;          /* this library's kernel launches since the last reset        */
    int64_t cn_launches;       /* k_cn_update launches                                        */
    int64_t vn_launches;       /* k_vn_update launches                                        */
    double  cn_ms;             /* summed CUDA-event time of k_cn_update launches (profiling on) */
    double  vn_ms;             /* same for k_vn_update                                        */
    int64_t cn_lane_iters;     /* sum over CN launches of lanes in the launched group         */
} metldpc_profile_t;

/* ---------------------------------------------------------------- 1. code (H) */

/* Load H stored edge-indexed (BASELINE north_star; "store H in two files"):
 * edges numbered 0..E-1 in CSR (check-major) order; cn_ptr[m+1] (int64, cn_ptr[0] = 0,
 * cn_ptr[m] = E) row offsets; edge_vn[E] the VN (0..n-1) of CSR edge e; vn_ptr[n+1]
 * column offsets; vn_edge[E] the CSR edge id of CSC slot k.  The CSC slot order of a
 * column is the order in which its messages are summed (R9/N3).
 * Host arrays, copied.  Validates (EFORMAT): indices in range, no duplicate (VN, CN)
 * pair, no degree-0 VN (R23), vn_edge a permutation consistent with edge_vn and
 * vn_ptr.  EUNSUPPORTED if a CN has degree > 32 or no sm_100 device is present.
 * The layout build (active/degree-1 split) runs on the host; arrays are
 * uploaded to `device`. */
metldpc_status metldpc_code_create(int32_t device, int32_t n, int32_t m, int64_t num_edges,
                                   const int64_t* cn_ptr, const int32_t* edge_vn,
                                   const int64_t* vn_ptr, const int64_t* vn_edge,
                                   metldpc_code* out);

/* Code-layout flags of metldpc_code_create_ex. */
#define METLDPC_CODE_NO_SKIP 1u  /* iterate degree-1 VNs like every other VN: the paper's "without
                                    skipping" variant (Table 1 left columns).  Their
                                    messages are then stored and summed (posterior form, R10), so
                                    n_active = n, iter_edges = edges and n_deg1 = 0; the decoded
                                    word may differ from the skipping decoder's by the rounding of
                                    L - r vs lambda (R26). */

/* metldpc_code_create with layout flags (0 = metldpc_code_create; EINVAL on unknown bits). */
metldpc_status metldpc_code_create_ex(int32_t device, int32_t n, int32_t m, int64_t num_edges,
                                      const int64_t* cn_ptr, const int32_t* edge_vn,
                                      const int64_t* vn_ptr, const int64_t* vn_edge,
                                      uint32_t flags, metldpc_code* out);

/* Same from a MacKay alist text file: "n m", "max_vn max_cn", VN degrees,
 * CN degrees, then n lines of 1-based CN lists and m lines of 1-based VN lists.
 * Edges are numbered in CSR order of the CN lists; the CSC order of a column is the
 * order of its VN line.  EFORMAT with the offending line number on any error. */
metldpc_status metldpc_code_load_alist(int32_t device, const char* path, metldpc_code* out);

/* Host-only validation + layout statistics, no GPU touched (used by CPU tests). */
metldpc_status metldpc_code_check(int32_t n, int32_t m, int64_t num_edges,
                                  const int64_t* cn_ptr, const int32_t* edge_vn,
                                  const int64_t* vn_ptr, const int64_t* vn_edge,
                                  metldpc_code_info_t* info_out);

metldpc_status metldpc_code_info(metldpc_code code, metldpc_code_info_t* out);

/* (EUNSUPPORTED also if a VN has degree > 512: the exact fixed-point VN sum of DESIGN.md N3
 * would overflow its 32-bit accumulator.) */

/* Destroy after every decoder using it. NULL is a no-op. */
void metldpc_code_destroy(metldpc_code code);

/* ---------------------------------------------------------------- decoder */

void metldpc_config_default(metldpc_config_t* cfg);

/* Workspace for batches of up to max_batch frames.  Frames are decoded in lane groups
 * (lanes_per_group frames), groups_in_flight groups at a time, each through its own group
 * workspace (~ E_it x lanes x 4 B of edge messages plus node arrays: ~1.05 GB for the
 * rate-0.1 n = 10^6 code at 64 lanes), so device memory does not grow with max_batch; the
 * host-buffer paths add 2 x groups_in_flight staging slots on first use.  cfg may be NULL
 * (defaults). */
metldpc_status metldpc_decoder_create(metldpc_code code, int32_t max_batch,
                                      const metldpc_config_t* cfg, metldpc_decoder* out);
void metldpc_decoder_destroy(metldpc_decoder dec);

/* ---------------------------------------------------------------- 2. LLRs from MD output */

/* Per-bit LLRs from d-dimensional multidimensional-reconciliation output (
 * DESIGN.md R13, N5):  lambda_i = 2 sqrt(snr (1 + snr)) * xnorm[i/d] * v_i  in fp32 as
 * c = (float)(2 sqrt(snr(1+snr))) (double), lambda = (c * xnorm) * v.
 *   v       dev fp32 [batch][n]   Alice's rotated, normalised blocks V (frame-major)
 *   xnorm   dev fp32 [batch][n/d] |x| of each block, or NULL => sqrt(d)
 *   llr_out dev fp32 [batch][n]   may alias v
 * d in {1,2,4,8} and n % d == 0; snr > 0 and finite; 0 <= batch <= max_batch. */
metldpc_status metldpc_llr_from_md(metldpc_decoder dec, int32_t batch, int32_t d, float snr,
                                   const float* v, const float* xnorm, float* llr_out,
                                   uintptr_t cuda_stream);

/* Alice's LLRs straight from her raw Gaussian block and Bob's rotation (the
 * GPU MD front end): with M(alpha) w = alpha * w the d-dimensional
 * division-algebra product (Cayley-Dickson: (a1,a2)(b1,b2) = (a1 b1 - conj(b2) a2,
 * b2 a1 + a2 conj(b1))), lambda = c |x| M(alpha) x/|x| = c M(alpha) x, c = 2 sqrt(snr(1+snr))
 * (R13).  fp32 per DESIGN.md N6: (alpha x)_i = fmaf left fold over the d terms, then * c.
 *   x       dev fp32 [batch][n]  Alice's raw block values X
 *   alpha   dev fp32 [batch][n]  Bob's rotation coefficients, d per block (as sent)
 *   llr_out dev fp32 [batch][n]  may alias x. */
metldpc_status metldpc_md_alice_llr(metldpc_decoder dec, int32_t batch, int32_t d, float snr,
                                    const float* x, const float* alpha, float* llr_out,
                                    uintptr_t cuda_stream);

/* S = H c^T (Step 1: Bob's syndrome S_B of his string U; equally the S_A test of a
 * decided word).  bits dev u32 [batch][ceil(n/32)], synd_out dev u32 [batch][ceil(m/32)],
 * both LSB-first in the caller's VN / CN order. */
metldpc_status metldpc_syndrome(metldpc_decoder dec, int32_t batch, const uint32_t* bits,
                                uint32_t* synd_out, uintptr_t cuda_stream);

/* ---------------------------------------------------------------- 3. decode */

/* Syndrome BP decoding of a batch (P:117-146 Steps 2-5, flooding schedule, degree-1
 * VNs skipped during iterations):
 *   llr        dev fp32 [batch][n]         lambda per frame, original VN order
 *   syndrome   dev u32  [batch][ceil(m/32)] Bob's S_B per frame (Step 1)
 *   max_iter   1..cfg.max_iter, or 0 => cfg.max_iter
 *   bits_out   dev u32  [batch][ceil(n/32)] hard decisions c, original VN order (Step 5,
 *                                c = [posterior LLR < 0]; a degree-1 VN's posterior
 *                                is lambda + its unclamped CN output, N1 / R27)
 *   iters_out  dev i32  [batch]  first l in 1..max_iter with H c^l = S_B (early_term),
 *                                else max_iter; -1 if the frame's lambda has a non-finite
 *                                value (R24; bits are then 0)
 *   converged_out dev u8 [batch] 1 iff H c = S_B for the returned c
 * Results are latched per frame at the first syndrome match (R12), so they do not
 * depend on batch composition, lane, group size, device or lane refill (cfg.lane_refill:
 * frames stream through the lanes, each freed lane taking the next frame of the batch).
 * 0 <= batch <= max_batch. */
metldpc_status metldpc_decode(metldpc_decoder dec, int32_t batch,
                              const float* llr, const uint32_t* syndrome, int32_t max_iter,
                              uint32_t* bits_out, int32_t* iters_out, uint8_t* converged_out,
                              uintptr_t cuda_stream);

/* The same from HOST buffers (the end-to-end path, Figure 1 incl. H2D/D2H):
 * the library stages each lane group through device buffers on its own streams,
 * overlapping the copies of group g+1 / g-1 with the decoding of group g.  Host
 * buffers should be pinned (cudaHostRegister / torch pin_memory) for full speed.
 * Synchronous: returns when the outputs are in host memory. */
metldpc_status metldpc_decode_host(metldpc_decoder dec, int32_t batch,
                                   const float* llr_host, const uint32_t* syndrome_host,
                                   int32_t max_iter, uint32_t* bits_host, int32_t* iters_host,
                                   uint8_t* converged_host);

/* Alice's whole hot path from HOST MD output (V -> LLR -> decode -> U): per lane
 * group, H2D of v / xnorm / S_B, metldpc_llr_from_md, decode, D2H of the results, with
 * the copies of neighbouring groups overlapping the decode (as metldpc_decode_host).
 *   v_host [batch][n], xnorm_host [batch][n/d] or NULL, syndrome_host [batch][ceil(m/32)];
 *   outputs as metldpc_decode_host.  Synchronous. */
metldpc_status metldpc_decode_md_host(metldpc_decoder dec, int32_t batch, int32_t d, float snr,
                                      const float* v_host, const float* xnorm_host,
                                      const uint32_t* syndrome_host, int32_t max_iter,
                                      uint32_t* bits_host, int32_t* iters_host, uint8_t* converged_host);

/* Frame counters of a decoded batch (FER accounting; R17):
 * counters_out dev i64 [4] += { frames, converged frames, sum of iterations over valid
 * frames, invalid frames } computed from iters/converged (dev, [batch]) by a kernel.
 * Multi-GPU runs all-reduce this buffer (NCCL) -- the only cross-GPU exchange. */
metldpc_status metldpc_batch_counters(metldpc_decoder dec, int32_t batch, const int32_t* iters,
                                      const uint8_t* converged, int64_t* counters_out,
                                      uintptr_t cuda_stream);

/* ---------------------------------------------------------------- debug / accounting */

/* Copy the message state of `lane` (0 <= lane < lanes_per_group) of the LAST lane group
 * decoded by this decoder to host memory: r_out [iter_edges] in active-edge CSR order
 * (CSR order with degree-1 edges removed), L_out [n_active] in ascending VN index order.
 * With early_term = 0 and max_iter = l this is (r^l, L^l).  Synchronises the device. */
metldpc_status metldpc_debug_dump(metldpc_decoder dec, int32_t lane, float* r_out, float* L_out);

/* Run k (>= 1) further iterations on the state left by the last decode (P:117-146 Steps 3-4;
 * SURVEY 8(b) debug hook): the valid lanes of the last lane group are re-activated and k plain
 * iterations (CN update, VN update; no syndrome test, no latch) are enqueued on cuda_stream.
 * With early_term = 0 and max_iter = l - 1, metldpc_debug_dump before and after one step
 * gives (r^{l-1}, L^{l-1}) and (r^l, L^l) -- the teacher-forced comparison with the fp64
 * definition.  EINVAL before any decode or after a streaming (lane-refill) decode. */
metldpc_status metldpc_debug_step(metldpc_decoder dec, int32_t k, uintptr_t cuda_stream);

/* The fp32 phi table of a rule (N2), host computed, no GPU touched:
 * EXACT 800 x 4 floats (c0..c3 per bin, 16 bins per binade), PHI_LUT 1600 x 2 floats
 * (c0, c1, 32 bins per binade), then one trailing float PHI_TOP.  Returns the number of
 * floats needed; writes if cap allows. */
int32_t metldpc_phi_table(int32_t rule, float* out, int32_t cap);

/* Profiling: when enabled, CN/VN launches are bracketed by CUDA events on the
 * decode stream and their durations summed (adds a host sync per decode call). */
metldpc_status metldpc_set_profiling(metldpc_decoder dec, int32_t enable);
metldpc_status metldpc_get_profile(metldpc_decoder dec, metldpc_profile_t* out);
metldpc_status metldpc_reset_profile(metldpc_decoder dec);

const char* metldpc_status_string(metldpc_status s);
const char* metldpc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* METLDPC_H */
