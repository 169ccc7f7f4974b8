// decoder.cu -- C ABI of libmetldpc: code upload, decoder workspace, the batch
// scheduler and the host-buffer end-to-end path.
//
// Schedule of one lane group (Figure 1 with per-frame early termination):
//   scatter LLRs / syndromes -> init
//   for l = 1..N:  CN update (tests iteration l-1 if ET) -> latch (ET) -> VN update
//   syndrome test of iteration N -> final latch -> finalize (bits, iterations, flags)
// Kernels early-exit once every lane of the group is latched.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.cuh"

namespace metldpc {
metldpc_status parse_alist(const char* path, int32_t* n_out, int32_t* m_out, std::vector<int64_t>* cn_ptr,
                           std::vector<int32_t>* edge_vn, std::vector<int64_t>* vn_ptr,
                           std::vector<int64_t>* vn_edge);
}

using namespace metldpc;

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(METLDPC_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
    } while (0)

struct metldpc_decoder_s {
    metldpc_code code = nullptr;
    metldpc_config_t cfg{};
    int32_t max_batch = 0;
    int B = 64, C = 2;
    struct ClassLaunch { int D, nd; int32_t begin, count; int ts, grid; };
    std::vector<ClassLaunch> cn_classes;
    int vn_grid = 0, chk_grid = 0;
    // K lane-group workspaces decoded concurrently on K streams (their CN and VN kernels
    // interleave on the GPU: the issue-bound CN pass of one group overlaps the HBM-bound VN
    // pass of another).
    struct Workspace {
        float *r = nullptr, *L = nullptr, *lam_a = nullptr, *lam1 = nullptr;
        uint32_t *d1bits = nullptr, *synd_t = nullptr, *ctl = nullptr;  // ctl: act[4] unsat[4] invalid[4]
                                                                          // iter maxit . . fresh[4] fin[4] newm[4]
        int32_t *lane_l = nullptr, *lane_frame = nullptr, *lane_fbuf = nullptr;   // lane refill
        int32_t* iters = nullptr;
        uint8_t* conv = nullptr;
        int32_t* done = nullptr;
    };
    int K = 1;
    std::vector<Workspace> ws;
    std::vector<L2Window> l2w;                      // per workspace: persisting window over L rows
    // CUDA-graph iteration loop per workspace: a conditional WHILE node whose
    // body is CN classes -> latch -> finish -> loop control; built on first use.
    std::vector<cudaGraphExec_t> loop_exec;
    std::vector<cudaGraphExec_t> stream_exec;       // lane-refill graph per workspace
    StreamJob* job = nullptr;                       // frame queue of a streaming decode (device)
    bool stream_used = false;                       // a streaming decode ran (device-side counters)
    int use_graph = 1;
    std::vector<cudaStream_t> gs;                   // one stream per workspace (K > 1)
    std::vector<cudaEvent_t> fork_ev, join_ev;
    int last_ws = 0;                                // workspace of the last group decoded
    int last_nb = 0;                                // its frames (group mode)
    bool last_streaming = false;                    // the last decode was a streaming decode
    // host-path staging: 2 rounds x K groups
    struct Staging {
        float* llr = nullptr;
        uint32_t* synd = nullptr;
        uint32_t* bits = nullptr;
        int32_t* iters = nullptr;
        uint8_t* conv = nullptr;
        float* xnorm = nullptr;
    };
    std::vector<Staging> st;
    size_t st_xnorm_cap = 0;                        // floats per group-mode slot's xnorm buffer
    struct HostStream {                             // streaming host path: up to kHostStreamCap frames
        float* llr = nullptr;
        uint32_t* synd = nullptr;
        uint32_t* bits = nullptr;
        int32_t* iters = nullptr;
        uint8_t* conv = nullptr;
        float* xnorm = nullptr;
        size_t xnorm_cap = 0;
    } hs;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    // accounting
    int profiling = 0;
    metldpc_profile_t prof{};
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, size_t>> ev_pending;  // (0 = cn, 1 = vn), start index; stop = start + 1
    size_t ev_used = 0;
};

namespace {

template <class T>
metldpc_status dalloc(T** p, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? METLDPC_ENOMEM : METLDPC_ECUDA,
                    std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    return METLDPC_OK;
}

template <class T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

CodeDev code_dev(const metldpc_code c, int rule) {
    CodeDev cd;
    cd.n = c->host.n;
    cd.m = c->host.m;
    cd.n_a = c->host.n_a;
    cd.n_1 = c->host.n_1;
    cd.E_it = c->host.E_it;
    cd.cn_aptr = c->d_cn_aptr;
    cd.cn_dptr = c->d_cn_dptr;
    cd.a_vn = c->d_a_vn;
    cd.vn_aptr = c->d_vn_aptr;
    cd.vn_aedge = c->d_vn_aedge;
    cd.vmap = c->d_vmap;
    cd.cn_new = c->d_cn_new;
    cd.phi = (rule == METLDPC_RULE_EXACT) ? c->d_phi_exact : c->d_phi_lut;
    cd.phi_top = phi_top();
    cd.rule = rule;
    return cd;
}

Group group_of(metldpc_decoder d, int k) {
    const auto& w = d->ws[size_t(k)];
    Group g;
    g.B = d->B;
    g.C = d->C;
    g.msg16 = d->cfg.msg_bits == 16 ? 1 : 0;
    g.r = w.r;
    g.L = w.L;
    g.lam_a = w.lam_a;
    g.lam1 = w.lam1;
    g.d1bits = w.d1bits;
    g.synd_t = w.synd_t;
    g.act = w.ctl;
    g.unsat = w.ctl + 4;
    g.invalid = w.ctl + 8;
    g.iters = w.iters;
    g.conv = w.conv;
    g.done = w.done;
    g.iter = reinterpret_cast<int32_t*>(w.ctl + 12);
    g.maxit = reinterpret_cast<int32_t*>(w.ctl + 13);
    g.fresh = w.ctl + 16;
    g.fin = w.ctl + 20;
    g.newm = w.ctl + 24;
    g.lane_l = w.lane_l;
    g.lane_frame = w.lane_frame;
    g.lane_fbuf = w.lane_fbuf;
    g.stat = w.ctl + 14;
    return g;
}

template <class T>
metldpc_status upload(T** dst, const std::vector<T>& src) {
    metldpc_status s = dalloc(dst, src.size());
    if (s) return s;
    if (!src.empty()) CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return METLDPC_OK;
}

// 16 bytes of zero padding after an index array: the CN ring kernel copies word ranges rounded
// up to 16 bytes (kernels.cu ring_copy_words)
std::vector<int32_t> padded(const std::vector<int32_t>& v) {
    std::vector<int32_t> p(v);
    p.resize(v.size() + 8, 0);
    return p;
}

metldpc_status check_device(int32_t device, int* num_sms) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(METLDPC_EUNSUPPORTED, "no CUDA device available");
    }
    if (device < 0 || device >= count) return fail(METLDPC_EINVAL, "device index out of range");
    cudaDeviceProp p;
    CUDA_TRY(cudaGetDeviceProperties(&p, device));
    if (p.major != 10) return fail(METLDPC_EUNSUPPORTED, std::string("built for sm_100a; device is ") + p.name);
    *num_sms = p.multiProcessorCount;
    return METLDPC_OK;
}

// Resident-CTA share of each persistent kernel when K groups are in flight.  Measured
// (round 1, C3): sizing every kernel for the whole GPU (split 1) beats splitting the SMs
// between the groups -- the gain of K > 1 is filling each kernel's ramp/tail and the
// launch gaps with another group's work.  METLDPC_GRID_SPLIT overrides (experiments).
int grid_split(int /*K*/) {
    const char* e = std::getenv("METLDPC_GRID_SPLIT");
    if (e && *e) return std::max(1, std::atoi(e));
    return 1;
}

// Records a kernel-timing event pair when profiling (CUDA events on the launch stream).
size_t ev_begin(metldpc_decoder d, int kind, cudaStream_t s) {
    if (!d->profiling) return size_t(-1);
    while (d->ev_used + 2 > d->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        d->ev_pool.push_back(e);
    }
    size_t i = d->ev_used;
    d->ev_used += 2;
    cudaEventRecord(d->ev_pool[i], s);
    d->ev_pending.push_back({kind, i});
    return i;
}

void ev_end(metldpc_decoder d, size_t i, cudaStream_t s) {
    if (i == size_t(-1)) return;
    cudaEventRecord(d->ev_pool[i + 1], s);
}

void ev_collect(metldpc_decoder d) {
    if (d->ev_pending.empty()) return;
    cudaEventSynchronize(d->ev_pool[d->ev_pending.back().second + 1]);
    for (auto& pr : d->ev_pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, d->ev_pool[pr.second], d->ev_pool[pr.second + 1]);
        (pr.first == 0 ? d->prof.cn_ms : d->prof.vn_ms) += ms;
    }
    d->ev_pending.clear();
    d->ev_used = 0;
}

// A lane group in three phases so K groups can be interleaved on K streams.
struct GroupJob {
    int k;                       // workspace
    const float* llr;            // frame-major inputs, offset to the group's first frame
    const uint32_t* synd;
    int nb;                      // frames in the group (<= B)
    uint32_t* bits_out;
    int32_t* iters_out;
    uint8_t* conv_out;
    cudaStream_t s;
    cudaEvent_t ready = nullptr;   // optional: inputs staged (host path); waited on by the group's stream
    cudaEvent_t done = nullptr;    // optional: recorded on the group's stream after finalize
};

// The CN classes of one pass: the small register-only classes first and the pipelined ones
// last, each launch after the first programmatically dependent on its predecessor, so a
// class's tail overlaps the next class's start (METLDPC_PDL=0: plain stream order).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("METLDPC_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void launch_cn_classes(metldpc_decoder d, const CodeDev& cd, const Group& g, int l, bool check, cudaStream_t s,
                       const L2Window& w) {
    const bool pdl_on = pdl_enabled();
    int n = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (const auto& c : d->cn_classes) {
            if (cn_use_pipe(c.D, c.nd) != (pass == 1)) continue;
            launch_cn(cd, g, d->cfg.rule, c.D, c.nd, c.begin, c.count, c.ts, c.grid, l, check, s, w, pdl_on && n > 0);
            ++n;
        }
}

metldpc_status group_begin(metldpc_decoder d, const GroupJob& j, int N) {
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, j.k);
    CUDA_TRY(cudaMemsetAsync(d->ws[size_t(j.k)].ctl + 8, 0, 4 * sizeof(uint32_t), j.s));
    // r^0 = 0 (Step 2): the CN kernels read r unconditionally (~0.2 % of a decode's traffic);
    // a 16-bit row stores the message 0 as the half-word 0x8080 (N7, kernels.cu msg16_q)
    if (g.msg16) CUDA_TRY(cudaMemsetAsync(g.r, 0x80, size_t(cd.E_it) * size_t(g.B) * 2, j.s));
    else CUDA_TRY(cudaMemsetAsync(g.r, 0, size_t(cd.E_it) * size_t(g.B) * sizeof(float), j.s));
    launch_scatter(cd, g, j.llr, j.nb, j.s);
    launch_pack_syndrome(cd, g, j.synd, j.nb, j.s);
    launch_init_ctl(g, j.nb, N, j.s);
    d->prof.launches += 3;
    return METLDPC_OK;
}

// Iteration l: CN update (all degree classes; tests iteration l-1 when ET is on), latch,
// VN update.
void group_iter(metldpc_decoder d, const GroupJob& j, int l) {
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, j.k);
    const bool et = d->cfg.early_term != 0;
    size_t e = ev_begin(d, 0, j.s);
    launch_cn_classes(d, cd, g, l, et && l >= 2, j.s, d->l2w[size_t(j.k)]);
    d->prof.launches += int64_t(d->cn_classes.size());
    ev_end(d, e, j.s);
    d->prof.cn_launches++;
    d->prof.cn_lane_iters += j.nb;
    if (et && l >= 2) {
        launch_latch(g, l - 1, false, j.s);
        d->prof.launches++;
    }
    e = ev_begin(d, 1, j.s);
    launch_finish(cd, g, d->vn_grid, j.s, d->l2w[size_t(j.k)]);
    ev_end(d, e, j.s);
    d->prof.vn_launches++;
    d->prof.launches++;
}

metldpc_status group_end(metldpc_decoder d, const GroupJob& j, int N) {
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, j.k);
    launch_check(cd, g, d->chk_grid, N, j.s);
    launch_latch(g, N, true, j.s);
    launch_finalize(cd, g, j.nb, j.bits_out, j.iters_out, j.conv_out, j.s);
    d->prof.launches += 3;
    d->last_ws = j.k;
    d->last_nb = j.nb;
    d->last_streaming = false;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

// Builds (once per workspace) the graph  while (l <= N && lanes left) { CN classes; latch;
// finish; l++ }  with the iteration number and N in device memory (Group::iter / maxit).
metldpc_status loop_graph(metldpc_decoder d, int k, cudaGraphExec_t* out) {
    if (d->loop_exec[size_t(k)]) {
        *out = d->loop_exec[size_t(k)];
        return METLDPC_OK;
    }
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, k);
    const bool et = d->cfg.early_term != 0;
    cudaGraph_t graph;
    CUDA_TRY(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    CUDA_TRY(cudaGraphConditionalHandleCreate(&h, graph, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CUDA_TRY(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t cs;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    launch_cn_classes(d, cd, g, 0, et, cs, d->l2w[size_t(k)]);
    const bool pdl = pdl_enabled();
    launch_latch_dev(g, et, cs, pdl);
    launch_finish(cd, g, d->vn_grid, cs, d->l2w[size_t(k)], pdl);
    launch_loop_ctl(g, (unsigned long long)h, cs, pdl);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return fail(METLDPC_ECUDA, std::string("loop graph capture: ") + cudaGetErrorString(e));
    }
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(METLDPC_ECUDA, std::string("loop graph instantiate: ") + cudaGetErrorString(e));
    d->loop_exec[size_t(k)] = exec;
    *out = exec;
    return METLDPC_OK;
}

// The iteration loop of one group: the CUDA graph (one launch, device-side trip count and
// early exit) unless profiling needs per-iteration events (host-enqueued loop).
metldpc_status group_loop(metldpc_decoder d, const GroupJob& j, int N) {
    if (d->use_graph && !d->profiling) {
        cudaGraphExec_t exec;
        metldpc_status st = loop_graph(d, j.k, &exec);
        if (st) return st;
        CUDA_TRY(cudaGraphLaunch(exec, j.s));
        const size_t per_iter = d->cn_classes.size() + 3;
        d->prof.launches += int64_t(per_iter) * N;      // upper bound (the loop may stop early)
        d->prof.cn_launches += N;
        d->prof.vn_launches += N;
        d->prof.cn_lane_iters += int64_t(j.nb) * N;
        return METLDPC_OK;
    }
    for (int l = 1; l <= N; ++l) group_iter(d, j, l);
    return METLDPC_OK;
}

// Lane-refill graph of workspace k ("refill ... from a frame queue", per lane):
//   while (some lane iterates or waits) {
//       CN classes; latch (per lane, pass counter++, loop condition); finish;
//       if (wave) { finalize finished lanes; assign next frames; scatter; syndrome; activate } }
// The refill wave is an IF node, so passes without a wave cost nothing extra.
metldpc_status stream_graph(metldpc_decoder d, int k, cudaGraphExec_t* out) {
    if (d->stream_exec[size_t(k)]) {
        *out = d->stream_exec[size_t(k)];
        return METLDPC_OK;
    }
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, k);
    cudaGraph_t graph;
    CUDA_TRY(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle hw;
    CUDA_TRY(cudaGraphConditionalHandleCreate(&hw, graph, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp{};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CUDA_TRY(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    cudaGraphConditionalHandle hi;
    CUDA_TRY(cudaGraphConditionalHandleCreate(&hi, body, 0u, cudaGraphCondAssignDefault));
    cudaStream_t cs;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    auto fail_capture = [&](cudaError_t e, const char* what) {
        cudaStreamDestroy(cs);
        cudaGraphDestroy(graph);
        return fail(METLDPC_ECUDA, std::string(what) + cudaGetErrorString(e));
    };
    // part A: one pass (CN classes, per-lane latch, finish)
    cudaError_t e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) return fail_capture(e, "stream graph capture: ");
    launch_cn_classes(d, cd, g, 0, true, cs, d->l2w[size_t(k)]);
    launch_latch_stream(g, d->job, (unsigned long long)hi, (unsigned long long)hw, cs, pdl_enabled());
    launch_finish(cd, g, d->vn_grid, cs, d->l2w[size_t(k)], pdl_enabled());
    cudaGraph_t cap;
    if ((e = cudaStreamEndCapture(cs, &cap)) != cudaSuccess) return fail_capture(e, "stream graph capture: ");
    // the last node of part A (a single-stream capture is a chain: the node without successors)
    size_t nn = 0;
    cudaGraphGetNodes(body, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(body, nodes.data(), &nn);
    cudaGraphNode_t last = nullptr;
    for (auto nd : nodes) {
        size_t nout = 0;
        cudaGraphNodeGetDependentNodes(nd, nullptr, &nout);
        if (nout == 0) last = nd;
    }
    // IF node: the refill wave
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    if ((e = cudaGraphAddNode(&inode, body, &last, 1, &ip)) != cudaSuccess) return fail_capture(e, "stream graph IF: ");
    cudaGraph_t wave = ip.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(cs, wave, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
        return fail_capture(e, "stream graph capture: ");
    launch_refill_wave(cd, g, d->job, cs);
    if ((e = cudaStreamEndCapture(cs, &cap)) != cudaSuccess) return fail_capture(e, "stream graph capture: ");
    cudaStreamDestroy(cs);
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(METLDPC_ECUDA, std::string("stream graph instantiate: ") + cudaGetErrorString(e));
    d->stream_exec[size_t(k)] = exec;
    *out = exec;
    return METLDPC_OK;
}

bool stream_mode(metldpc_decoder d) {
    return d->cfg.lane_refill && d->job && d->cfg.early_term && d->use_graph && !d->profiling && d->B == 64;
}

// Streaming decode of a whole batch: every workspace runs its refill graph on its own stream,
// all drawing frames from one device-side queue (StreamJob::next).  Two stream-ordered parts:
// stream_setup writes the queue header (frames [0, avail) already on the device; the host path
// passes 0 and raises it with k_publish as its copies land), stream_launch starts the graphs.
metldpc_status stream_setup(metldpc_decoder d, int32_t batch, const float* llr, const uint32_t* synd, int N,
                            uint32_t* bits_out, int32_t* iters_out, uint8_t* conv_out, int32_t avail,
                            cudaStream_t s) {
    StreamJob h{};   // pageable source: cudaMemcpyAsync stages it before returning
    h.llr = llr;
    h.synd = synd;
    h.bits = bits_out;
    h.iters = iters_out;
    h.conv = conv_out;
    h.nframes = batch;
    h.next = 0;
    h.N = N;
    h.avail = avail;
    {
        // refill once 2 lanes have finished (headline config, r0.1de BIAWGN 0.161, 4096 frames per
        // call, same box: thresholds 1 / 2 / 4 / 8 -> 1855 / 1856 / 1844 / 1809 Mb/s with the
        // lane-list wave kernels; 8 was best while a wave cost 0.17 ms, profiles/r2_wave_parts.jsonl)
        const char* e = std::getenv("METLDPC_REFILL_MIN");
        h.wave_min = (e && std::atoi(e) > 0) ? std::atoi(e) : 2;
    }
    // hang guard only: a lane needs at most N + 1 passes per frame
    const int64_t guard = (int64_t(batch) + d->B) * (int64_t(N) + 2) + 1000;
    h.max_passes = int32_t(std::min<int64_t>(guard, INT32_MAX));
    CUDA_TRY(cudaMemcpyAsync(d->job, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    return METLDPC_OK;
}

metldpc_status stream_launch(metldpc_decoder d, int32_t batch, cudaStream_t s) {
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const int K = std::min(d->K, (batch + d->B - 1) / d->B);
    if (K > 1) {
        CUDA_TRY(cudaEventRecord(d->fork_ev[0], s));
        for (int k = 0; k < K; ++k) CUDA_TRY(cudaStreamWaitEvent(d->gs[size_t(k)], d->fork_ev[0], 0));
    }
    for (int k = 0; k < K; ++k) {
        cudaStream_t ks = K > 1 ? d->gs[size_t(k)] : s;
        const Group g = group_of(d, k);
        cudaGraphExec_t exec;
        metldpc_status st = stream_graph(d, k, &exec);
        if (st) return st;
        launch_stream_init(g, ks);
        launch_refill_wave(cd, g, d->job, ks);   // first fill
        CUDA_TRY(cudaGraphLaunch(exec, ks));
        d->prof.launches += 1;                   // + passes and waves, counted on the device
        d->stream_used = true;
        d->last_ws = k;
        d->last_streaming = true;
    }
    if (K > 1)
        for (int k = 0; k < K; ++k) {
            CUDA_TRY(cudaEventRecord(d->join_ev[size_t(k)], d->gs[size_t(k)]));
            CUDA_TRY(cudaStreamWaitEvent(s, d->join_ev[size_t(k)], 0));
        }
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

// Decodes up to K groups concurrently: forked from stream `s` onto the workspace streams,
// iterations interleaved group by group, joined back into `s`.
metldpc_status decode_round(metldpc_decoder d, std::vector<GroupJob>& jobs, int N, cudaStream_t s) {
    metldpc_status st;
    if (jobs.size() == 1) {
        jobs[0].s = s;
        if (jobs[0].ready) CUDA_TRY(cudaStreamWaitEvent(s, jobs[0].ready, 0));
        if ((st = group_begin(d, jobs[0], N))) return st;
        if ((st = group_loop(d, jobs[0], N))) return st;
        if ((st = group_end(d, jobs[0], N))) return st;
        if (jobs[0].done) CUDA_TRY(cudaEventRecord(jobs[0].done, s));
        return METLDPC_OK;
    }
    CUDA_TRY(cudaEventRecord(d->fork_ev[0], s));
    for (auto& j : jobs) {
        j.s = d->gs[size_t(j.k)];
        CUDA_TRY(cudaStreamWaitEvent(j.s, d->fork_ev[0], 0));
        if (j.ready) CUDA_TRY(cudaStreamWaitEvent(j.s, j.ready, 0));
        if ((st = group_begin(d, j, N))) return st;
    }
    if (d->use_graph && !d->profiling) {
        for (auto& j : jobs)
            if ((st = group_loop(d, j, N))) return st;
    } else {
        for (int l = 1; l <= N; ++l)
            for (auto& j : jobs) group_iter(d, j, l);
    }
    for (auto& j : jobs) {
        if ((st = group_end(d, j, N))) return st;
        if (j.done) CUDA_TRY(cudaEventRecord(j.done, j.s));
        CUDA_TRY(cudaEventRecord(d->join_ev[size_t(j.k)], j.s));
        CUDA_TRY(cudaStreamWaitEvent(s, d->join_ev[size_t(j.k)], 0));
    }
    return METLDPC_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ code

metldpc_status metldpc_code_create(int32_t device, int32_t n, int32_t m, int64_t num_edges, const int64_t* cn_ptr,
                                   const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                                   metldpc_code* out) {
    return metldpc_code_create_ex(device, n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge, 0u, out);
}

metldpc_status metldpc_code_create_ex(int32_t device, int32_t n, int32_t m, int64_t num_edges, const int64_t* cn_ptr,
                                      const int32_t* edge_vn, const int64_t* vn_ptr, const int64_t* vn_edge,
                                      uint32_t flags, metldpc_code* out) {
    if (!out) return fail(METLDPC_EINVAL, "out is NULL");
    *out = nullptr;
    if (flags & ~uint32_t(METLDPC_CODE_NO_SKIP)) return fail(METLDPC_EINVAL, "unknown code flags");
    metldpc_code c = new (std::nothrow) metldpc_code_s();
    if (!c) return fail(METLDPC_ENOMEM, "host allocation");
    metldpc_status s = build_layout(n, m, num_edges, cn_ptr, edge_vn, vn_ptr, vn_edge, &c->host, flags);
    if (s == METLDPC_OK) s = check_device(device, &c->num_sms);
    if (s) {
        delete c;
        return s;
    }
    c->device = device;
    cudaSetDevice(device);
    const HostLayout& L = c->host;
    const std::vector<float> te = phi_device_table(METLDPC_RULE_EXACT), tl = phi_device_table(METLDPC_RULE_PHI_LUT);
    if ((s = upload(&c->d_cn_aptr, L.cn_aptr)) || (s = upload(&c->d_cn_dptr, L.cn_dptr)) ||
        (s = upload(&c->d_a_vn, padded(L.a_vn))) || (s = upload(&c->d_vn_aptr, L.vn_aptr)) ||
        (s = upload(&c->d_vn_aedge, L.vn_aedge)) || (s = upload(&c->d_vmap, L.vmap)) ||
        (s = upload(&c->d_cn_new, L.cn_new)) || (s = upload(&c->d_csr_ptr, L.csr_ptr)) ||
        (s = upload(&c->d_csr_vn, L.csr_vn)) ||
        (s = upload(&c->d_phi_exact, te)) || (s = upload(&c->d_phi_lut, tl))) {
        metldpc_code_destroy(c);
        return s;
    }
    *out = c;
    return METLDPC_OK;
}

metldpc_status metldpc_code_load_alist(int32_t device, const char* path, metldpc_code* out) {
    if (!path || !out) return fail(METLDPC_EINVAL, "NULL argument");
    int32_t n = 0, m = 0;
    std::vector<int64_t> cn_ptr, vn_ptr, vn_edge;
    std::vector<int32_t> edge_vn;
    metldpc_status s = parse_alist(path, &n, &m, &cn_ptr, &edge_vn, &vn_ptr, &vn_edge);
    if (s) return s;
    return metldpc_code_create(device, n, m, int64_t(edge_vn.size()), cn_ptr.data(), edge_vn.data(), vn_ptr.data(),
                               vn_edge.data(), out);
}

metldpc_status metldpc_code_info(metldpc_code code, metldpc_code_info_t* out) {
    if (!code || !out) return fail(METLDPC_EINVAL, "NULL argument");
    fill_info(code->host, out);
    return METLDPC_OK;
}

void metldpc_code_destroy(metldpc_code c) {
    if (!c) return;
    cudaSetDevice(c->device);
    dfree(c->d_cn_aptr);
    dfree(c->d_cn_dptr);
    dfree(c->d_a_vn);
    dfree(c->d_vn_aptr);
    dfree(c->d_vn_aedge);
    dfree(c->d_vmap);
    dfree(c->d_cn_new);
    dfree(c->d_csr_ptr);
    dfree(c->d_csr_vn);
    dfree(c->d_phi_exact);
    dfree(c->d_phi_lut);
    delete c;
}

// ------------------------------------------------------------------ decoder

void metldpc_config_default(metldpc_config_t* cfg) {
    if (!cfg) return;
    cfg->rule = METLDPC_RULE_EXACT;
    cfg->max_iter = 100;
    cfg->early_term = 1;
    cfg->lanes_per_group = 64;
    cfg->groups_in_flight = 1;
    cfg->lane_refill = 1;
    cfg->msg_bits = 32;
}

metldpc_status metldpc_decoder_create(metldpc_code code, int32_t max_batch, const metldpc_config_t* cfg_in,
                                      metldpc_decoder* out) {
    if (!code || !out) return fail(METLDPC_EINVAL, "NULL argument");
    *out = nullptr;
    metldpc_config_t cfg;
    metldpc_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (cfg.rule != METLDPC_RULE_EXACT && cfg.rule != METLDPC_RULE_PHI_LUT) return fail(METLDPC_EINVAL, "unknown rule");
    if (cfg.max_iter < 1) return fail(METLDPC_EINVAL, "max_iter must be >= 1");
    if (cfg.lanes_per_group != 32 && cfg.lanes_per_group != 64 && cfg.lanes_per_group != 128)
        return fail(METLDPC_EINVAL, "lanes_per_group must be 32, 64 or 128");
    if (cfg.groups_in_flight < 1 || cfg.groups_in_flight > 8) return fail(METLDPC_EINVAL, "groups_in_flight must be 1..8");
    if (max_batch < 1) return fail(METLDPC_EINVAL, "max_batch must be >= 1");
    if (cfg.msg_bits != 32 && cfg.msg_bits != 16) return fail(METLDPC_EINVAL, "msg_bits must be 32 or 16");
    if (cfg.msg_bits == 16 && cfg.lanes_per_group != 64)
        return fail(METLDPC_EUNSUPPORTED, "msg_bits = 16 needs lanes_per_group = 64");
    if ((code->host.E_it + 1) * int64_t(cfg.lanes_per_group) >= (int64_t(1) << 31) ||
        (int64_t(code->host.n_a) + 1) * cfg.lanes_per_group >= (int64_t(1) << 31))
        return fail(METLDPC_EUNSUPPORTED, "edge-message array exceeds 2^31 elements per lane group");
    cudaSetDevice(code->device);
    metldpc_decoder d = new (std::nothrow) metldpc_decoder_s();
    if (!d) return fail(METLDPC_ENOMEM, "host allocation");
    d->code = code;
    d->cfg = cfg;
    d->max_batch = max_batch;
    d->B = cfg.lanes_per_group;
    d->C = d->B / 32;
    const HostLayout& L = code->host;
    const size_t B = size_t(d->B), C = size_t(d->C);
    metldpc_status s;
    // groups in flight: never more than the batch needs
    d->K = std::max(1, std::min(cfg.groups_in_flight, (max_batch + d->B - 1) / d->B));
    d->ws.resize(size_t(d->K));
    for (auto& w : d->ws) {
        if ((s = dalloc(&w.r, size_t(L.E_it) * B * size_t(cfg.msg_bits) / 32)) || (s = dalloc(&w.L, 2 * size_t(L.n_a) * B)) ||
            (s = dalloc(&w.lam_a, size_t(L.n_a) * B)) || (s = dalloc(&w.lam1, size_t((L.n_1 + 15) & ~7) * B)) ||
            (s = dalloc(&w.d1bits, 2 * size_t(L.n_1) * C + 8)) || (s = dalloc(&w.synd_t, size_t(L.m) * C + 8)) ||
            (s = dalloc(&w.ctl, 32)) || (s = dalloc(&w.iters, B)) || (s = dalloc(&w.conv, B)) ||
            (s = dalloc(&w.lane_l, B)) || (s = dalloc(&w.lane_frame, B)) || (s = dalloc(&w.lane_fbuf, B)) ||
            (s = dalloc(&w.done, 1))) {
            metldpc_decoder_destroy(d);
            return s;
        }
        cudaMemset(w.d1bits, 0, 2 * size_t(L.n_1) * C * sizeof(uint32_t));
        cudaMemset(w.ctl, 0, 32 * sizeof(uint32_t));
        // Lanes without a frame are computed too (unpredicated CN kernels).  Their lam1 entries
        // are the degree-1 inputs p of checks with D <= 5, whose output phi is evaluated without an
        // upper clamp on the premise p <= phi(2^-44) (k_cn_ring / k_cn_pipe / k_cn_tile): a lane that
        // has not yet held a frame in the streaming decode must therefore read a valid prior, not
        // whatever a previous allocation left (+0 is one: phi form of |lambda| = +inf).  L and
        // lambda_a are cleared for the same lanes' determinism.
        cudaMemset(w.lam1, 0, size_t((L.n_1 + 15) & ~7) * B * sizeof(float));
        cudaMemset(w.L, 0, 2 * size_t(L.n_a) * B * sizeof(float));
        cudaMemset(w.lam_a, 0, size_t(L.n_a) * B * sizeof(float));
    }
    // Persisting-L2 window over the workspace's L / accumulator rows (the CN gathers and
    // atomics hit them ~23 times per iteration per VN).  Measured (round 1, C3): +2 % with one
    // group in flight, strongly negative with 4 (the windows thrash the set-aside), so it is
    // on by default when groups_in_flight == 1 (METLDPC_L2PERSIST=0 disables it): measured
    // 1143 vs 1124 Mb/s at C3; with two groups in flight their rows no longer fit.
    d->l2w.assign(size_t(d->K), L2Window{});
    {
        const char* e = std::getenv("METLDPC_L2PERSIST");
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, code->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, code->device);
        const size_t rows = 2 * size_t(L.n_a) * B * sizeof(float);
        // Only when the rows fit the set-aside: a window larger than it (no-skip layouts, whose
        // rows are ~8x larger) keeps a fraction of the rows persisting and starves the streams
        // (measured: no-skip C3 CN phase 0.68 -> 1.51 ms).
        if (!(e && *e == '0') && d->K == 1 && max_persist > 0 && max_window > 0 && rows <= size_t(max_persist) &&
            rows <= size_t(max_window)) {
            const size_t want = std::min(size_t(max_persist), rows * size_t(d->K));
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            for (int k = 0; k < d->K; ++k) {
                L2Window& w = d->l2w[size_t(k)];
                w.base = d->ws[size_t(k)].L;
                w.bytes = std::min(rows, size_t(max_window));
                // share the persisting set-aside between the groups in flight
                w.hit_ratio = float(std::min(1.0, double(want) / double(d->K) / double(w.bytes)));
            }
        }
        cudaGetLastError();
    }
    d->loop_exec.assign(size_t(d->K), nullptr);
    d->stream_exec.assign(size_t(d->K), nullptr);
    if (cfg.lane_refill) {
        if (cudaMalloc(reinterpret_cast<void**>(&d->job), sizeof(StreamJob)) != cudaSuccess) {
            cudaGetLastError();
            metldpc_decoder_destroy(d);
            return fail(METLDPC_ENOMEM, "device allocation (stream job)");
        }
    }
    {
        const char* e = std::getenv("METLDPC_GRAPH");
        d->use_graph = (e && *e == '0') ? 0 : 1;
    }
    if (d->K > 1) {
        d->gs.resize(size_t(d->K));
        d->join_ev.resize(size_t(d->K));
        d->fork_ev.resize(1);
        for (auto& st : d->gs) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        for (auto& e : d->join_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&d->fork_ev[0], cudaEventDisableTiming);
    }
    const int sms = code->num_sms;
    for (const auto& k : L.classes) {
        // The tiled kernels are specialised for 64-lane groups; other group sizes and the
        // generic classes take the run-time-degree kernel.  Tile: up to cn_tile_max CNs per
        // warp, fewer for small classes so every SM still gets >= 16 warp units.
        const int D = (d->B == 64) ? k.D : -1;
        const int warps_per_cta = kCnThreadsHost / 32;
        int ts = 1;
        long units = long(k.count) * d->C;
        if (D >= 0) {
            const long want = long(k.count) / (long(sms) * 16);
            ts = int(std::max(1L, std::min(long(cn_tile_max(D, k.nd)), want)));
            units = ((long(k.count) + ts - 1) / ts) * cn_units_per_tile(D, k.nd);
        }
        const long full =
            long(sms) * std::max(1, cn_blocks_per_sm(cfg.rule, D, k.nd, cfg.msg_bits == 16) / grid_split(d->K));
        const long need = (units + warps_per_cta - 1) / warps_per_cta;
        d->cn_classes.push_back({D, k.nd, k.begin, k.count, ts, int(std::max(1L, std::min(full, need)))});
    }
    d->vn_grid = sms * std::max(1, finish_blocks_per_sm() / grid_split(d->K));
    d->chk_grid = sms * 4;
    *out = d;
    return METLDPC_OK;
}

void metldpc_decoder_destroy(metldpc_decoder d) {
    if (!d) return;
    cudaSetDevice(d->code->device);
    for (auto& w : d->ws) {
        dfree(w.r);
        dfree(w.L);
        dfree(w.lam_a);
        dfree(w.lam1);
        dfree(w.d1bits);
        dfree(w.synd_t);
        dfree(w.ctl);
        dfree(w.lane_l);
        dfree(w.lane_frame);
        dfree(w.lane_fbuf);
        dfree(w.iters);
        dfree(w.conv);
        dfree(w.done);
    }
    for (auto ex : d->loop_exec)
        if (ex) cudaGraphExecDestroy(ex);
    for (auto ex : d->stream_exec)
        if (ex) cudaGraphExecDestroy(ex);
    if (d->job) cudaFree(d->job);
    for (auto st : d->gs) cudaStreamDestroy(st);
    for (auto e : d->join_ev) cudaEventDestroy(e);
    for (auto e : d->fork_ev) cudaEventDestroy(e);
    for (auto& sl : d->st) {
        dfree(sl.llr);
        dfree(sl.synd);
        dfree(sl.bits);
        dfree(sl.iters);
        dfree(sl.conv);
        dfree(sl.xnorm);
    }
    dfree(d->hs.llr);
    dfree(d->hs.synd);
    dfree(d->hs.bits);
    dfree(d->hs.iters);
    dfree(d->hs.conv);
    dfree(d->hs.xnorm);
    if (d->s_h2d) cudaStreamDestroy(d->s_h2d);
    if (d->s_comp) cudaStreamDestroy(d->s_comp);
    if (d->s_d2h) cudaStreamDestroy(d->s_d2h);
    for (auto e : d->ev_pool) cudaEventDestroy(e);
    delete d;
}

// ------------------------------------------------------------------ LLR from MD output

metldpc_status metldpc_llr_from_md(metldpc_decoder d, int32_t batch, int32_t dim, float snr, const float* v,
                                   const float* xnorm, float* llr_out, uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    const int n = d->code->host.n;
    if (batch < 0 || batch > d->max_batch) return fail(METLDPC_EINVAL, "batch out of range");
    if (dim != 1 && dim != 2 && dim != 4 && dim != 8) return fail(METLDPC_EINVAL, "d must be 1, 2, 4 or 8");
    if (n % dim) return fail(METLDPC_EINVAL, "n must be divisible by d");
    if (!(snr > 0.0f) || !std::isfinite(snr)) return fail(METLDPC_EINVAL, "snr must be finite and > 0");
    if (batch == 0) return METLDPC_OK;
    if (!v || !llr_out) return fail(METLDPC_EINVAL, "NULL buffer");
    cudaSetDevice(d->code->device);
    const double sd = double(snr);
    const float c = float(2.0 * std::sqrt(sd * (1.0 + sd)));
    launch_md_llr(int64_t(batch) * n, n, dim, c, v, xnorm, llr_out, reinterpret_cast<cudaStream_t>(stream));
    d->prof.launches++;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

// ------------------------------------------------------------------ MD front end, syndrome

metldpc_status metldpc_md_alice_llr(metldpc_decoder d, int32_t batch, int32_t dim, float snr, const float* x,
                                    const float* alpha, float* llr_out, uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    const int n = d->code->host.n;
    if (batch < 0 || batch > d->max_batch) return fail(METLDPC_EINVAL, "batch out of range");
    if (dim != 1 && dim != 2 && dim != 4 && dim != 8) return fail(METLDPC_EINVAL, "d must be 1, 2, 4 or 8");
    if (n % dim) return fail(METLDPC_EINVAL, "n must be divisible by d");
    if (!(snr > 0.0f) || !std::isfinite(snr)) return fail(METLDPC_EINVAL, "snr must be finite and > 0");
    if (batch == 0) return METLDPC_OK;
    if (!x || !alpha || !llr_out) return fail(METLDPC_EINVAL, "NULL buffer");
    cudaSetDevice(d->code->device);
    MdTable t{};
    md_product_table(dim, t.kp, t.ks);
    const double sd = double(snr);
    const float c = float(2.0 * std::sqrt(sd * (1.0 + sd)));
    launch_md_alice(int64_t(batch) * (n / dim), dim, c, x, alpha, llr_out, t, reinterpret_cast<cudaStream_t>(stream));
    d->prof.launches++;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

metldpc_status metldpc_syndrome(metldpc_decoder d, int32_t batch, const uint32_t* bits, uint32_t* synd_out,
                                uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (batch < 0) return fail(METLDPC_EINVAL, "batch < 0");
    if (batch == 0) return METLDPC_OK;
    if (!bits || !synd_out) return fail(METLDPC_EINVAL, "NULL buffer");
    cudaSetDevice(d->code->device);
    const HostLayout& L = d->code->host;
    launch_syndrome(d->code->d_csr_ptr, d->code->d_csr_vn, L.n, L.m, batch, bits, synd_out,
                    reinterpret_cast<cudaStream_t>(stream));
    d->prof.launches++;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

// ------------------------------------------------------------------ decode

metldpc_status metldpc_decode(metldpc_decoder d, int32_t batch, const float* llr, const uint32_t* syndrome,
                              int32_t max_iter, uint32_t* bits_out, int32_t* iters_out, uint8_t* conv_out,
                              uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (batch < 0 || batch > d->max_batch) return fail(METLDPC_EINVAL, "batch out of range [0, max_batch]");
    if (max_iter < 0 || max_iter > d->cfg.max_iter) return fail(METLDPC_EINVAL, "max_iter out of range");
    if (batch == 0) return METLDPC_OK;
    if (!llr || !syndrome || !bits_out || !iters_out || !conv_out) return fail(METLDPC_EINVAL, "NULL buffer");
    const int N = max_iter ? max_iter : d->cfg.max_iter;
    cudaSetDevice(d->code->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const HostLayout& L = d->code->host;
    const size_t W = size_t(L.m + 31) / 32, NW = size_t(L.n + 31) / 32;
    const int groups = (batch + d->B - 1) / d->B;
    if (stream_mode(d)) {
        metldpc_status st = stream_setup(d, batch, llr, syndrome, N, bits_out, iters_out, conv_out, batch, s);
        return st ? st : stream_launch(d, batch, s);
    }
    if (d->K > 1 && d->use_graph && !d->profiling && groups > d->K) {
        // Group queue: workspace k decodes groups k, k + K, ... on its own stream with no
        // per-round join, so with early termination a workspace whose group finished early
        // starts its next group at once instead of waiting for the round's slowest group.
        CUDA_TRY(cudaEventRecord(d->fork_ev[0], s));
        for (int k = 0; k < d->K; ++k) CUDA_TRY(cudaStreamWaitEvent(d->gs[size_t(k)], d->fork_ev[0], 0));
        for (int gi = 0; gi < groups; ++gi) {
            const int k = gi % d->K, f0 = gi * d->B;
            GroupJob j{k, llr + size_t(f0) * L.n, syndrome + size_t(f0) * W, std::min(d->B, batch - f0),
                       bits_out + size_t(f0) * NW, iters_out + f0, conv_out + f0, d->gs[size_t(k)]};
            metldpc_status st;
            if ((st = group_begin(d, j, N)) || (st = group_loop(d, j, N)) || (st = group_end(d, j, N))) return st;
        }
        for (int k = 0; k < d->K; ++k) {
            CUDA_TRY(cudaEventRecord(d->join_ev[size_t(k)], d->gs[size_t(k)]));
            CUDA_TRY(cudaStreamWaitEvent(s, d->join_ev[size_t(k)], 0));
        }
        return METLDPC_OK;
    }
    for (int g0 = 0; g0 < groups; g0 += d->K) {
        std::vector<GroupJob> jobs;
        for (int k = 0; k < d->K && g0 + k < groups; ++k) {
            const int f0 = (g0 + k) * d->B;
            jobs.push_back({k, llr + size_t(f0) * L.n, syndrome + size_t(f0) * W, std::min(d->B, batch - f0),
                            bits_out + size_t(f0) * NW, iters_out + f0, conv_out + f0, s});
        }
        metldpc_status st = decode_round(d, jobs, N, s);
        if (st) return st;
    }
    return METLDPC_OK;
}

}  // extern "C"

namespace {

// Host-buffer paths (metldpc_decode_host: LLR input; metldpc_decode_md_host: MD output input).
//
// Streaming (lane refill, the default with early termination): the batch is copied to device
// staging in chunks on the copy stream -- each chunk's H2D, its LLR conversion, then k_publish
// raising the queue's `avail` -- while the streaming decode (stream_launch) already runs on the
// compute stream from the first chunk on; freed lanes take frames as they become available.
// Results go to device staging (k_finalize_lanes) and come back in one D2H per super-chunk.
// Batches larger than the staging capacity run as consecutive super-chunks.
//
// Group mode (lane_refill = 0, early_term = 0 or profiling): groups are decoded in rounds of K
// workspaces with staging double-buffered across rounds, so the H2D of round r+1 and the D2H of
// round r-1 run on their own streams while round r decodes.
//
// Every CUDA call's status is checked; the first failure stops the enqueueing, the streams are
// drained and ECUDA is returned.
#define HP(expr)                                                               \
    do {                                                                       \
        if (ce == cudaSuccess) {                                               \
            ce = (expr);                                                       \
            if (ce != cudaSuccess) what = #expr;                               \
        }                                                                      \
    } while (0)

constexpr int kHostStreamCap = 2048;   // frames staged at once by the streaming host path
constexpr int kHostChunk = 32;         // frames per H2D chunk (one k_publish each)

metldpc_status ensure_host_streams(metldpc_decoder d) {
    if (d->s_comp) return METLDPC_OK;
    CUDA_TRY(cudaStreamCreateWithFlags(&d->s_h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&d->s_comp, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&d->s_d2h, cudaStreamNonBlocking));
    return METLDPC_OK;
}

metldpc_status host_stream(metldpc_decoder d, int32_t batch, int md, int32_t dim, float snr, const float* in_h,
                           const float* xnorm_h, const uint32_t* synd_h, int N, uint32_t* bits_h, int32_t* iters_h,
                           uint8_t* conv_h) {
    const HostLayout& L = d->code->host;
    const size_t n = size_t(L.n), W = size_t(L.m + 31) / 32, NW = size_t(L.n + 31) / 32;
    const size_t nx = md ? n / size_t(dim) : 0;
    const int cap = std::min(d->max_batch, kHostStreamCap);
    metldpc_status st;
    if ((st = ensure_host_streams(d))) return st;
    auto& hs = d->hs;
    if (!hs.llr) {
        if ((st = dalloc(&hs.llr, size_t(cap) * n)) || (st = dalloc(&hs.synd, size_t(cap) * W)) ||
            (st = dalloc(&hs.bits, size_t(cap) * NW)) || (st = dalloc(&hs.iters, size_t(cap))) ||
            (st = dalloc(&hs.conv, size_t(cap))))
            return st;
    }
    if (md && xnorm_h && hs.xnorm_cap < size_t(cap) * nx) {
        dfree(hs.xnorm);
        hs.xnorm_cap = 0;
        if ((st = dalloc(&hs.xnorm, size_t(cap) * nx))) return st;
        hs.xnorm_cap = size_t(cap) * nx;
    }
    const float c_md = md ? float(2.0 * std::sqrt(double(snr) * (1.0 + double(snr)))) : 0.f;
    cudaError_t ce = cudaSuccess;
    const char* what = "";
    cudaEvent_t ev_job = nullptr, ev_first = nullptr, ev_free = nullptr;
    HP(cudaEventCreateWithFlags(&ev_job, cudaEventDisableTiming));
    HP(cudaEventCreateWithFlags(&ev_first, cudaEventDisableTiming));
    HP(cudaEventCreateWithFlags(&ev_free, cudaEventDisableTiming));
    for (int f0 = 0; f0 < batch && ce == cudaSuccess; f0 += cap) {
        const int nb = std::min(cap, batch - f0);
        // queue header first (avail = 0), then the copies may publish into it
        if ((st = stream_setup(d, nb, hs.llr, hs.synd, N, hs.bits, hs.iters, hs.conv, 0, d->s_comp))) break;
        HP(cudaEventRecord(ev_job, d->s_comp));
        HP(cudaStreamWaitEvent(d->s_h2d, ev_job, 0));
        for (int c0 = 0; c0 < nb && ce == cudaSuccess; c0 += kHostChunk) {
            const int k = std::min(kHostChunk, nb - c0);
            const size_t g0 = size_t(f0) + size_t(c0);
            HP(cudaMemcpyAsync(hs.llr + size_t(c0) * n, in_h + g0 * n, size_t(k) * n * sizeof(float),
                               cudaMemcpyHostToDevice, d->s_h2d));
            if (md && xnorm_h)
                HP(cudaMemcpyAsync(hs.xnorm + size_t(c0) * nx, xnorm_h + g0 * nx, size_t(k) * nx * sizeof(float),
                                   cudaMemcpyHostToDevice, d->s_h2d));
            HP(cudaMemcpyAsync(hs.synd + size_t(c0) * W, synd_h + g0 * W, size_t(k) * W * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, d->s_h2d));
            if (md && ce == cudaSuccess) {   // LLRs in place over the staged v (R13)
                launch_md_llr(int64_t(k) * int64_t(n), int(n), dim, c_md, hs.llr + size_t(c0) * n,
                              xnorm_h ? hs.xnorm + size_t(c0) * nx : nullptr, hs.llr + size_t(c0) * n, d->s_h2d);
                HP(cudaGetLastError());
                d->prof.launches++;
            }
            launch_publish(d->job, c0 + k, d->s_h2d);
            HP(cudaGetLastError());
            d->prof.launches++;
            if (c0 == 0) HP(cudaEventRecord(ev_first, d->s_h2d));
        }
        if (ce != cudaSuccess) {
            // never leave a launched queue waiting for frames that will not come
            launch_publish(d->job, nb, d->s_h2d);
            break;
        }
        HP(cudaStreamWaitEvent(d->s_comp, ev_first, 0));
        if (ce != cudaSuccess) break;
        if ((st = stream_launch(d, nb, d->s_comp))) break;
        HP(cudaMemcpyAsync(bits_h + size_t(f0) * NW, hs.bits, size_t(nb) * NW * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, d->s_comp));
        HP(cudaMemcpyAsync(iters_h + f0, hs.iters, size_t(nb) * sizeof(int32_t), cudaMemcpyDeviceToHost, d->s_comp));
        HP(cudaMemcpyAsync(conv_h + f0, hs.conv, size_t(nb), cudaMemcpyDeviceToHost, d->s_comp));
        // the next super-chunk's copies overwrite the staging: after this one's decode and D2H
        HP(cudaEventRecord(ev_free, d->s_comp));
        HP(cudaStreamWaitEvent(d->s_h2d, ev_free, 0));
    }
    cudaError_t e1 = cudaStreamSynchronize(d->s_h2d);
    cudaError_t e2 = cudaStreamSynchronize(d->s_comp);
    if (ev_job) cudaEventDestroy(ev_job);
    if (ev_first) cudaEventDestroy(ev_first);
    if (ev_free) cudaEventDestroy(ev_free);
    if (st) return st;
    if (ce != cudaSuccess) return fail(METLDPC_ECUDA, std::string("host path: ") + what + ": " + cudaGetErrorString(ce));
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(METLDPC_ECUDA, std::string("host path: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return METLDPC_OK;
}

metldpc_status host_pipeline(metldpc_decoder d, int32_t batch, int md, int32_t dim, float snr, const float* in_h,
                             const float* xnorm_h, const uint32_t* synd_h, int32_t max_iter, uint32_t* bits_h,
                             int32_t* iters_h, uint8_t* conv_h) {
    const int N = max_iter ? max_iter : d->cfg.max_iter;
    cudaSetDevice(d->code->device);
    if (stream_mode(d)) return host_stream(d, batch, md, dim, snr, in_h, xnorm_h, synd_h, N, bits_h, iters_h, conv_h);
    const HostLayout& L = d->code->host;
    const size_t n = size_t(L.n), W = size_t(L.m + 31) / 32, NW = size_t(L.n + 31) / 32, B = size_t(d->B);
    const size_t nx = md ? n / size_t(dim) : 0;
    const int K = d->K, S = 2 * K;
    metldpc_status st;
    if ((st = ensure_host_streams(d))) return st;
    if (d->st.empty()) {
        d->st.resize(size_t(S));
        for (auto& sl : d->st)
            if ((st = dalloc(&sl.llr, B * n)) || (st = dalloc(&sl.synd, B * W)) || (st = dalloc(&sl.bits, B * NW)) ||
                (st = dalloc(&sl.iters, B)) || (st = dalloc(&sl.conv, B)))
                return st;
    }
    if (md && xnorm_h && d->st_xnorm_cap < B * nx) {   // B * n / d floats per slot: sized for this call's d
        for (auto& sl : d->st) {
            dfree(sl.xnorm);
            if ((st = dalloc(&sl.xnorm, B * nx))) {
                d->st_xnorm_cap = 0;
                return st;
            }
        }
        d->st_xnorm_cap = B * nx;
    }
    const float c_md = md ? float(2.0 * std::sqrt(double(snr) * (1.0 + double(snr)))) : 0.f;
    cudaError_t ce = cudaSuccess;
    const char* what = "";
    const size_t nslots = static_cast<size_t>(S);
    std::vector<cudaEvent_t> in_ready(nslots, nullptr), slot_free(nslots, nullptr), out_ready(nslots, nullptr),
        out_free(nslots, nullptr);
    for (size_t k = 0; k < nslots; ++k) {
        HP(cudaEventCreateWithFlags(&in_ready[k], cudaEventDisableTiming));
        HP(cudaEventCreateWithFlags(&slot_free[k], cudaEventDisableTiming));
        HP(cudaEventCreateWithFlags(&out_ready[k], cudaEventDisableTiming));
        HP(cudaEventCreateWithFlags(&out_free[k], cudaEventDisableTiming));
        HP(cudaEventRecord(slot_free[k], d->s_comp));
        HP(cudaEventRecord(out_free[k], d->s_d2h));
    }
    const int groups = (batch + d->B - 1) / d->B;
    st = METLDPC_OK;
    auto stage_in = [&](int slot, int f0, int nb) {
        auto& sl = d->st[size_t(slot)];
        // the slot's previous decode and D2H must be done before new inputs overwrite it
        HP(cudaStreamWaitEvent(d->s_h2d, slot_free[size_t(slot)], 0));
        HP(cudaStreamWaitEvent(d->s_h2d, out_free[size_t(slot)], 0));
        HP(cudaMemcpyAsync(sl.llr, in_h + size_t(f0) * n, size_t(nb) * n * sizeof(float), cudaMemcpyHostToDevice,
                           d->s_h2d));
        if (md && xnorm_h)
            HP(cudaMemcpyAsync(sl.xnorm, xnorm_h + size_t(f0) * nx, size_t(nb) * nx * sizeof(float),
                               cudaMemcpyHostToDevice, d->s_h2d));
        HP(cudaMemcpyAsync(sl.synd, synd_h + size_t(f0) * W, size_t(nb) * W * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           d->s_h2d));
        if (md && ce == cudaSuccess) {   // LLRs in place over the staged v (metldpc_llr_from_md, R13)
            launch_md_llr(int64_t(nb) * int64_t(n), int(n), dim, c_md, sl.llr, xnorm_h ? sl.xnorm : nullptr, sl.llr,
                          d->s_h2d);
            HP(cudaGetLastError());
            d->prof.launches++;
        }
        HP(cudaEventRecord(in_ready[size_t(slot)], d->s_h2d));
    };
    auto stage_out = [&](int slot, int f0, int nb) {
        auto& sl = d->st[size_t(slot)];
        HP(cudaStreamWaitEvent(d->s_d2h, out_ready[size_t(slot)], 0));
        HP(cudaMemcpyAsync(bits_h + size_t(f0) * NW, sl.bits, size_t(nb) * NW * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           d->s_d2h));
        HP(cudaMemcpyAsync(iters_h + f0, sl.iters, size_t(nb) * sizeof(int32_t), cudaMemcpyDeviceToHost, d->s_d2h));
        HP(cudaMemcpyAsync(conv_h + f0, sl.conv, size_t(nb), cudaMemcpyDeviceToHost, d->s_d2h));
        HP(cudaEventRecord(out_free[size_t(slot)], d->s_d2h));
    };
    const bool queue = K > 1 && d->use_graph && !d->profiling;
    // Group queue (as in metldpc_decode): group gi uses staging slot gi mod 2K and workspace
    // gi mod K on that workspace's stream, ordered only by its own events (inputs staged,
    // previous occupant of the slot decoded and copied out) -- no per-round join.
    for (int gi = 0; queue && gi < groups && st == METLDPC_OK && ce == cudaSuccess; ++gi) {
        const int k = gi % K, slot = gi % S;
        auto& sl = d->st[size_t(slot)];
        const int f0 = gi * d->B, nb = std::min(d->B, batch - f0);
        cudaStream_t gs = d->gs[size_t(k)];
        stage_in(slot, f0, nb);
        HP(cudaStreamWaitEvent(gs, in_ready[size_t(slot)], 0));
        if (ce != cudaSuccess) break;
        GroupJob j{k, sl.llr, sl.synd, nb, sl.bits, sl.iters, sl.conv, gs};
        if ((st = group_begin(d, j, N)) || (st = group_loop(d, j, N)) || (st = group_end(d, j, N))) break;
        HP(cudaEventRecord(out_ready[size_t(slot)], gs));
        HP(cudaEventRecord(slot_free[size_t(slot)], gs));
        stage_out(slot, f0, nb);
    }
    for (int g0 = 0, round = 0; !queue && g0 < groups && st == METLDPC_OK && ce == cudaSuccess; g0 += K, ++round) {
        std::vector<GroupJob> jobs;
        std::vector<int> slots;
        for (int k = 0; k < K && g0 + k < groups; ++k) {
            const int slot = (round & 1) * K + k;
            auto& sl = d->st[size_t(slot)];
            const int f0 = (g0 + k) * d->B, nb = std::min(d->B, batch - f0);
            stage_in(slot, f0, nb);
            GroupJob j{k, sl.llr, sl.synd, nb, sl.bits, sl.iters, sl.conv, d->s_comp};
            j.ready = in_ready[size_t(slot)];
            j.done = out_ready[size_t(slot)];
            jobs.push_back(j);
            slots.push_back(slot);
        }
        if (ce != cudaSuccess) break;
        if ((st = decode_round(d, jobs, N, d->s_comp))) break;
        for (size_t q = 0; q < jobs.size(); ++q) {
            HP(cudaEventRecord(slot_free[size_t(slots[q])], d->s_comp));
            stage_out(slots[q], (g0 + int(q)) * d->B, jobs[q].nb);
        }
    }
    cudaError_t e = cudaStreamSynchronize(d->s_h2d);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->s_d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->s_comp);
    for (int k = 0; queue && k < K; ++k)
        if (e == cudaSuccess) e = cudaStreamSynchronize(d->gs[size_t(k)]);
    for (size_t k = 0; k < nslots; ++k) {
        if (in_ready[k]) cudaEventDestroy(in_ready[k]);
        if (slot_free[k]) cudaEventDestroy(slot_free[k]);
        if (out_ready[k]) cudaEventDestroy(out_ready[k]);
        if (out_free[k]) cudaEventDestroy(out_free[k]);
    }
    if (st) return st;
    if (ce != cudaSuccess) return fail(METLDPC_ECUDA, std::string("host pipeline: ") + what + ": " + cudaGetErrorString(ce));
    if (e != cudaSuccess) return fail(METLDPC_ECUDA, std::string("host pipeline: ") + cudaGetErrorString(e));
    return METLDPC_OK;
}

}  // namespace

extern "C" {

metldpc_status metldpc_decode_host(metldpc_decoder d, int32_t batch, const float* llr_h, const uint32_t* synd_h,
                                   int32_t max_iter, uint32_t* bits_h, int32_t* iters_h, uint8_t* conv_h) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (batch < 0 || batch > d->max_batch) return fail(METLDPC_EINVAL, "batch out of range [0, max_batch]");
    if (max_iter < 0 || max_iter > d->cfg.max_iter) return fail(METLDPC_EINVAL, "max_iter out of range");
    if (batch == 0) return METLDPC_OK;
    if (!llr_h || !synd_h || !bits_h || !iters_h || !conv_h) return fail(METLDPC_EINVAL, "NULL buffer");
    return host_pipeline(d, batch, 0, 1, 0.f, llr_h, nullptr, synd_h, max_iter, bits_h, iters_h, conv_h);
}

metldpc_status metldpc_decode_md_host(metldpc_decoder d, int32_t batch, int32_t dim, float snr, const float* v_h,
                                      const float* xnorm_h, const uint32_t* synd_h, int32_t max_iter,
                                      uint32_t* bits_h, int32_t* iters_h, uint8_t* conv_h) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (batch < 0 || batch > d->max_batch) return fail(METLDPC_EINVAL, "batch out of range [0, max_batch]");
    if (max_iter < 0 || max_iter > d->cfg.max_iter) return fail(METLDPC_EINVAL, "max_iter out of range");
    if (dim != 1 && dim != 2 && dim != 4 && dim != 8) return fail(METLDPC_EINVAL, "d must be 1, 2, 4 or 8");
    if (d->code->host.n % dim) return fail(METLDPC_EINVAL, "n must be divisible by d");
    if (!(snr > 0.0f) || !std::isfinite(snr)) return fail(METLDPC_EINVAL, "snr must be finite and > 0");
    if (batch == 0) return METLDPC_OK;
    if (!v_h || !synd_h || !bits_h || !iters_h || !conv_h) return fail(METLDPC_EINVAL, "NULL buffer");
    return host_pipeline(d, batch, 1, dim, snr, v_h, xnorm_h, synd_h, max_iter, bits_h, iters_h, conv_h);
}

metldpc_status metldpc_batch_counters(metldpc_decoder d, int32_t batch, const int32_t* iters, const uint8_t* conv,
                                      int64_t* counters_out, uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (batch < 0) return fail(METLDPC_EINVAL, "batch < 0");
    if (batch == 0) return METLDPC_OK;
    if (!iters || !conv || !counters_out) return fail(METLDPC_EINVAL, "NULL buffer");
    cudaSetDevice(d->code->device);
    launch_counters(batch, iters, conv, counters_out, reinterpret_cast<cudaStream_t>(stream));
    d->prof.launches++;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

// ------------------------------------------------------------------ debug / accounting

metldpc_status metldpc_debug_dump(metldpc_decoder d, int32_t lane, float* r_out, float* L_out) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (lane < 0 || lane >= d->B) return fail(METLDPC_EINVAL, "lane out of range");
    cudaSetDevice(d->code->device);
    CUDA_TRY(cudaDeviceSynchronize());
    const HostLayout& L = d->code->host;
    if (r_out && L.E_it && d->cfg.msg_bits == 16) {   // 16-bit rows (N7): half-word (lane & 31, lane >> 5)
        std::vector<uint16_t> tmp(size_t(L.E_it));
        const char* base = reinterpret_cast<const char*>(d->ws[size_t(d->last_ws)].r) + 4 * (lane & 31) + 2 * (lane >> 5);
        CUDA_TRY(cudaMemcpy2D(tmp.data(), 2, base, 128, 2, size_t(L.E_it), cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < L.E_it; ++t)
            r_out[L.perm_r[size_t(t)]] = float(int(tmp[size_t(t)]) - 0x8080) * (1.0f / 1024.0f);
    } else if (r_out && L.E_it) {   // device order (relabelled CNs) -> canonical active-edge CSR order
        std::vector<float> tmp(size_t(L.E_it));
        CUDA_TRY(cudaMemcpy2D(tmp.data(), sizeof(float), d->ws[size_t(d->last_ws)].r + lpos(lane, d->B), size_t(d->B) * sizeof(float), sizeof(float),
                              size_t(L.E_it), cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < L.E_it; ++t) r_out[L.perm_r[size_t(t)]] = tmp[size_t(t)];
    }
    if (L_out && L.n_a)
        CUDA_TRY(cudaMemcpy2D(L_out, sizeof(float), d->ws[size_t(d->last_ws)].L + lpos(lane, d->B), 2 * size_t(d->B) * sizeof(float), sizeof(float),
                              size_t(L.n_a), cudaMemcpyDeviceToHost));
    return METLDPC_OK;
}

metldpc_status metldpc_debug_step(metldpc_decoder d, int32_t k, uintptr_t stream) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    if (k < 1) return fail(METLDPC_EINVAL, "k must be >= 1");
    if (d->last_nb < 1 || d->last_streaming)
        return fail(METLDPC_EINVAL, "debug_step needs a preceding group-mode decode (lane_refill = 0 or early_term = 0)");
    cudaSetDevice(d->code->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const CodeDev cd = code_dev(d->code, d->cfg.rule);
    const Group g = group_of(d, d->last_ws);
    // re-activate the group's valid lanes (the final latch retired them), then k plain
    // iterations: CN classes (no syndrome test) + VN finish, exactly the decode's pass
    launch_init_ctl(g, d->last_nb, d->cfg.max_iter, s);
    for (int i = 1; i <= k; ++i) {
        launch_cn_classes(d, cd, g, i, false, s, d->l2w[size_t(d->last_ws)]);
        launch_finish(cd, g, d->vn_grid, s, d->l2w[size_t(d->last_ws)]);
        d->prof.launches += int64_t(d->cn_classes.size()) + 1;
    }
    d->prof.launches++;
    CUDA_TRY(cudaGetLastError());
    return METLDPC_OK;
}

metldpc_status metldpc_set_profiling(metldpc_decoder d, int32_t enable) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    d->profiling = enable ? 1 : 0;
    return METLDPC_OK;
}

metldpc_status metldpc_get_profile(metldpc_decoder d, metldpc_profile_t* out) {
    if (!d || !out) return fail(METLDPC_EINVAL, "NULL argument");
    ev_collect(d);
    *out = d->prof;
    if (d->stream_used) {   // streaming passes / waves are counted on the device
        CUDA_TRY(cudaDeviceSynchronize());
        size_t per_pass = 2;   // latch (+ loop control), finish
        for (const auto& c : d->cn_classes) per_pass += 1;
        for (const auto& w : d->ws) {
            uint32_t st[2] = {0, 0};
            CUDA_TRY(cudaMemcpy(st, w.ctl + 14, sizeof(st), cudaMemcpyDeviceToHost));
            out->launches += int64_t(st[0]) * int64_t(per_pass) + int64_t(st[1]) * 5;
            out->cn_launches += st[0];
            out->vn_launches += st[0];
            out->cn_lane_iters += int64_t(st[0]) * d->B;
        }
    }
    return METLDPC_OK;
}

metldpc_status metldpc_reset_profile(metldpc_decoder d) {
    if (!d) return fail(METLDPC_EINVAL, "NULL decoder");
    ev_collect(d);
    d->prof = metldpc_profile_t{};
    if (d->stream_used) {
        CUDA_TRY(cudaDeviceSynchronize());
        for (const auto& w : d->ws) CUDA_TRY(cudaMemset(w.ctl + 14, 0, 2 * sizeof(uint32_t)));
    }
    return METLDPC_OK;
}

}  // extern "C"
