// Microbenchmark: cost of computing "lanes with the same 8-bit digit" on sm_100a.
//   (a) __match_any_sync            (b) 8 ballots, lean combine   (c) 8 ballots, ternary combine
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const uint32_t* __restrict__ in, uint32_t* out, int iters) {
    uint32_t d[8];
    for (int j = 0; j < 8; ++j) d[j] = in[(blockIdx.x * blockDim.x + threadIdx.x) * 8 + j] & 0xff;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t x = (d[j] + it) & 0xff;
            uint32_t peers;
            if (MODE == 0) {
                peers = __match_any_sync(0xffffffffu, x);
            } else if (MODE == 1) {
                peers = 0xffffffffu;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    uint32_t bal = __ballot_sync(0xffffffffu, (x >> b) & 1u);
                    uint32_t m = (uint32_t)((int32_t)(x << (31 - b)) >> 31);
                    peers &= ~(bal ^ m);
                }
            } else {
                peers = 0xffffffffu;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    bool bit = (x >> b) & 1u;
                    uint32_t bal = __ballot_sync(0xffffffffu, bit);
                    peers &= bit ? bal : ~bal;
                }
            }
            acc += __popc(peers) ^ (peers >> 7);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int blocks = 148 * 4, threads = 512, iters = 200;
    size_t n = (size_t)blocks * threads;
    uint32_t *in, *out;
    cudaMalloc(&in, n * 8 * 4);
    cudaMalloc(&out, n * 4);
    uint32_t* h = new uint32_t[n * 8];
    uint64_t s = 88172645463325252ull;
    for (size_t i = 0; i < n * 8; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s; }
    cudaMemcpy(in, h, n * 32, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[3] = {"match_any", "ballot_lean", "ballot_ternary"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(in, out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(in, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)n * iters * 8;   // thread-level peer computations
            if (rep) printf("%-15s %8.3f ms  %7.2f G peer-ops/s  (%.2f ns per warp-op per SM)\n", names[mode], ms,
                            ops / ms / 1e6, ms * 1e6 / (ops / 32 / 148));
        }
    }
    return 0;
}
