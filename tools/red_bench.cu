// Micro-benchmark (tools only, not part of the library): throughput of warp-wide
// RED.ADD.S32 into an L2-resident [rows][64] int32 accumulator with random rows -- the
// access pattern a fused CN pass would use to accumulate VN sums.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>   // 0: RED.ADD, 1: plain store, 2: load (gather)
__global__ void k(int* acc, int rows, long edges, int* sink) {
    const int lane = threadIdx.x & 31;
    long w = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long nw = (long(gridDim.x) * blockDim.x) >> 5;
    int s = 0;
    for (long e = w; e < edges; e += nw) {
        const uint32_t row = hash32(uint32_t(e)) % uint32_t(rows);
        int* p = acc + size_t(row) * 64 + lane;
        if (MODE == 0) { atomicAdd(p, int(e & 7)); atomicAdd(p + 32, int(e & 5)); }
        else if (MODE == 1) { p[0] = int(e); p[32] = int(e); }
        else { s += __ldcg(p) + __ldcg(p + 32); }
    }
    if (MODE == 2 && s == 12345) sink[0] = s;
}

int main() {
    const int rows = 125000;
    const long edges = 2892500;
    int *acc, *sink;
    cudaMalloc(&acc, size_t(rows) * 64 * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(acc, 0, size_t(rows) * 64 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"RED.ADD.S32 x2 per warp-edge", "STG x2 per warp-edge", "LDG.CG x2 per warp-edge"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(acc, rows, edges, sink);
            if (mode == 1) k<1><<<148 * 8, 256>>>(acc, rows, edges, sink);
            if (mode == 2) k<2><<<148 * 8, 256>>>(acc, rows, edges, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 3)
                printf("%-32s %8.3f us  (%.1f G warp-ops/s, %.0f GB/s of 128-B rows)\n", names[mode], ms * 1e3,
                       2.0 * edges / (ms * 1e-3) / 1e9, 2.0 * edges * 128 / (ms * 1e-3) / 1e9);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
