// Bandwidth of the radix-pass memory pattern without the ranking: per
// 4096-key tile, read 8-byte keys + 1-byte payloads contiguously and write
// them as R runs (one per digit, 4096 / R keys each) into R output streams,
// consecutive tiles appending to each stream -- the best case of a radix
// scatter (equal, aligned runs).  R = 1 is a plain copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbench_scatter tools/mbench_scatter.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R>
__global__ __launch_bounds__(512) void k_scatter(const uint64_t* __restrict__ in, const uint8_t* __restrict__ ia,
                                                 uint64_t* __restrict__ out, uint8_t* __restrict__ oa, int64_t n) {
    constexpr int T = 4096, RUN = T / R;
    const int64_t tiles = n / T, stream_len = n / R;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int li = j * 512 + threadIdx.x;
            const int64_t i = tile * T + li;
            const int d = li / RUN, r = li % RUN;
            const int64_t o = (int64_t)d * stream_len + tile * RUN + r;
            out[o] = in[i];
            oa[o] = ia[i];
        }
    }
}

template <int R>
static void run(const uint64_t* in, const uint8_t* ia, uint64_t* out, uint8_t* oa, int64_t n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 4;
    for (int w = 0; w < 3; ++w) k_scatter<R><<<grid, 512>>>(in, ia, out, oa, n);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) k_scatter<R><<<grid, 512>>>(in, ia, out, oa, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= it;
    printf("streams %4d (runs of %4d keys): %.3f ms per 1e8 keys, %.0f GB/s (18 B/key)\n", R, 4096 / R, ms,
           18.0 * n / (ms * 1e6));
}

int main() {
    const int64_t n = 100000000 / 4096 * 4096;
    uint64_t *in, *out;
    uint8_t *ia, *oa;
    cudaMalloc(&in, n * 8);
    cudaMalloc(&out, n * 8);
    cudaMalloc(&ia, n);
    cudaMalloc(&oa, n);
    cudaMemset(in, 1, n * 8);
    cudaMemset(ia, 1, n);
    run<1>(in, ia, out, oa, n);
    run<16>(in, ia, out, oa, n);
    run<64>(in, ia, out, oa, n);
    run<256>(in, ia, out, oa, n);
    run<512>(in, ia, out, oa, n);
    return 0;
}
