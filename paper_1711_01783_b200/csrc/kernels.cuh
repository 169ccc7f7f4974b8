// kernels.cuh -- launch interface of the sm_100a kernels (private).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace metldpc {

// Position of lane b in a "pair" row (r rows and the VN-sum accumulator rows): inside each block
// of 64 lanes, lanes t and t + 32 are adjacent (word t of the thread that carries both lanes), so
// a thread moves its two lanes with one 8-byte access and adds both fixed-point terms with one
// 64-bit RED (N3, section 6).  32-lane groups keep lane order.
__host__ __device__ __forceinline__ int lpos(int b, int B) {
    return B == 32 ? b : (b & ~63) | ((b & 31) << 1) | ((b >> 5) & 1);
}

// Device state of the lane group being decoded.  Arrays are codeword-interleaved:
// element (slot s, lane b) lives at s * B + b, B = lanes per group (32/64/128), so
// a warp (32 consecutive lanes) touches one full 128-byte line per slot
// ("when the number of simultaneously decoded codewords is an integer
// multiple of 32, both of the variable nodes and check nodes memory access are
// consecutive").  C = B / 32 lane chunks; bit vectors over lanes are uint32 per chunk.
struct Group {
    int B, C;
    int msg16;         // 1: r rows hold 16-bit messages (N7; 64-lane groups only)
    float* r;          // [E_it][B]   CN->VN messages r_ji of active edges (Eqs. 2-3), lane b at
                       //             lpos(b); with msg16 [E_it][32] uint32 words, word t = lanes t
                       //             (low), t + 32 (high) -- the same pair order
    float* L;          // [n_a][2][B] row of VN a: posterior LLR L (Eq. 5) at +0 (lane order), the
                       //             fixed-point accumulator of the next L at +B: B = 32 uint32 per
                       //             lane; B = 64 / 128 one uint64 per lane pair (t, t + 32) of each
                       //             64-lane block, low word lane t (N3)
    float* lam_a;      // [n_a][B]    channel LLR of active VNs (Eq. 1)
    float* lam1;       // [n_1][B]    degree-1 priors in phi form: phi(|lambda|), sign bit [lambda < 0]
                       //             (N1), CSR slot order
    uint32_t* d1bits;  // [2][n_1][C] hard bits of degree-1 VNs, by iteration parity
    uint32_t* synd_t;  // [m][C]      S_B bits, lane-transposed
    uint32_t* act;     // [C]  lanes still iterating
    uint32_t* unsat;   // [C]  lanes with an unsatisfied check in the tested iteration
    uint32_t* invalid; // [C]  lanes with a non-finite LLR
    int32_t* iters;    // [B]
    uint8_t* conv;     // [B]
    int32_t* done;     // [1]  all lanes latched
    int32_t* iter;     // [1]  current iteration l (graph-driven loop; 1-based)
    int32_t* maxit;    // [1]  N of the running decode
    // lane refill (streaming decode; all zero / unused in group mode)
    uint32_t* fresh;   // [C]  lanes whose frame starts in this pass: r^0 = 0 (Step 2)
    uint32_t* fin;     // [C]  lanes whose frame finished and awaits the refill wave
    uint32_t* newm;    // [C]  lanes given a new frame by the running refill wave
    int32_t* lane_l;   // [B]  pass number of the lane's current frame (its iteration l)
    int32_t* lane_frame;  // [B] frame index of the lane in the batch (-1: none)
    int32_t* lane_fbuf;   // [B] d1bits buffer holding the lane's final degree-1 decisions
    uint32_t* stat;    // [2]  streaming passes and refill waves run (kernel-launch accounting)
};

// Frame queue of a streaming decode (device memory, shared by the K workspaces): the
// batch's buffers, the next unassigned frame and the refill threshold.
struct StreamJob {
    const float* llr;      // [nframes][n]
    const uint32_t* synd;  // [nframes][W]
    uint32_t* bits;        // [nframes][NW]
    int32_t* iters;        // [nframes]
    uint8_t* conv;         // [nframes]
    int32_t nframes;
    int32_t next;          // atomically advanced by the refill waves (frames claimed)
    int32_t N;             // max_iter
    int32_t wave_min;      // refill once this many lanes have finished (or none iterates)
    int32_t avail;         // frames [0, avail) have their inputs on the device (host path:
                           // raised chunk by chunk by k_publish on the copy stream)
    int32_t max_passes;    // hang guard: a workspace's loop stops after this many passes
};

struct CodeDev {
    int32_t n, m, n_a, n_1;
    int64_t E_it;
    const int32_t* cn_aptr;
    const int32_t* cn_dptr;
    const int32_t* a_vn;
    const int32_t* vn_aptr;
    const int32_t* vn_aedge;
    const int32_t* vmap;
    const int32_t* cn_new;  // original CN id -> relabelled id
    const float* phi;      // table of the selected rule
    float phi_top;
    int rule;              // METLDPC_RULE_EXACT / METLDPC_RULE_PHI_LUT
};

// returns the number of CTAs per SM the CN kernel reaches (for persistent grids)
struct L2Window {          // persisting-L2 access window (bytes == 0: none)
    void* base = nullptr;
    size_t bytes = 0;
    float hit_ratio = 1.0f;
};

// CN class kernels: total degree D in 0..16 with nd <= 1 degree-1 slots (tiled, unrolled)
// or D = -1 (generic: more degree-1 slots or degree 17..32)
int cn_blocks_per_sm(int rule, int D, int nd, int msg16);
int cn_tile_max(int D, int nd);          // CNs per warp tile the kernel stages
int cn_units_per_tile(int D, int nd);    // warp units per tile (1: both chunks, 2: one each)
extern const int kCnThreadsHost;
size_t cn_smem(int rule, int D, int nd);
int finish_blocks_per_sm();

void launch_scatter(const CodeDev& cd, const Group& g, const float* llr, int nb, cudaStream_t s);
void launch_pack_syndrome(const CodeDev& cd, const Group& g, const uint32_t* synd, int nb, cudaStream_t s);
void launch_init_ctl(const Group& g, int nb, int N, cudaStream_t s);
// Device-driven iteration control for the CUDA-graph loop (l read from Group::iter).
void launch_latch_dev(const Group& g, bool et, cudaStream_t s, bool pdl = false);
void launch_loop_ctl(const Group& g, unsigned long long cond_handle, cudaStream_t s, bool pdl = false);
// lane refill (streaming decode)
void launch_stream_init(const Group& g, cudaStream_t s);
// per-lane latch + end of a streaming pass (pass counter, WHILE condition), IF condition of the wave
void launch_latch_stream(const Group& g, StreamJob* job, unsigned long long if_handle, unsigned long long while_handle,
                         cudaStream_t s, bool pdl = false);
void launch_refill_wave(const CodeDev& cd, const Group& g, StreamJob* job, cudaStream_t s);
void launch_publish(StreamJob* job, int avail, cudaStream_t s);
// l >= 1: iteration given by the host; l == 0: read from Group::iter (graph body), with
// et telling whether iterations >= 2 test the syndrome.
void launch_cn(const CodeDev& cd, const Group& g, int rule, int D, int nd, int begin, int count, int ts, int grid,
               int l, bool check, cudaStream_t s, const L2Window& w, bool pdl = false);
bool cn_use_pipe(int D, int nd);   // class runs the TMA-pipelined kernel
void launch_finish(const CodeDev& cd, const Group& g, int grid, cudaStream_t s, const L2Window& w, bool pdl = false);
void launch_check(const CodeDev& cd, const Group& g, int grid, int l, cudaStream_t s);
void launch_latch(const Group& g, int l, bool final_, cudaStream_t s);
void launch_finalize(const CodeDev& cd, const Group& g, int nb, uint32_t* bits_out, int32_t* iters_out,
                     uint8_t* conv_out, cudaStream_t s);
struct MdTable {
    int8_t kp[64], ks[64];
};
void launch_md_alice(int64_t blocks_total, int d, float c, const float* x, const float* alpha, float* out,
                     const MdTable& t, cudaStream_t s);
void launch_syndrome(const int32_t* csr_ptr, const int32_t* csr_vn, int n, int m, int batch, const uint32_t* bits,
                     uint32_t* synd, cudaStream_t s);
void launch_counters(int batch, const int32_t* iters, const uint8_t* conv, int64_t* out, cudaStream_t s);
void launch_md_llr(int64_t total, int n, int d, float c, const float* v, const float* xnorm, float* out,
                   cudaStream_t s);

}  // namespace metldpc
