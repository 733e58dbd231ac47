// Microbenchmark: scatter-add throughput of an A x A (count u32, sum u64)
// table for A = 256, placed (a) in global memory (RED.64 to L2), (b) split
// across the distributed shared memory of a thread-block cluster (each CTA owns
// 1/K of the edges; remote CTAs are reached with atomics on DSMEM addresses).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mbench_dsmem tools/mbench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int E = 65536;

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return (uint32_t)x;
}

__global__ void k_global(uint32_t* cnt, unsigned long long* sum, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = hsh(i);
        uint32_t e = h & (E - 1);
        atomicAdd(&cnt[e], 1u);
        atomicAdd(&sum[e], (unsigned long long)(h >> 8));
    }
}

__global__ void k_global64(unsigned long long* cnt, unsigned long long* sum, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = hsh(i);
        uint32_t e = h & (E - 1);
        atomicAdd(&cnt[e], 1ull);
        atomicAdd(&sum[e], (unsigned long long)(h >> 8));
    }
}

__global__ void k_sumonly(unsigned long long* sum, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = hsh(i);
        uint32_t e = h & (E - 1);
        atomicAdd(&sum[e], (unsigned long long)(h >> 8));
    }
}

// counts as u16 pairs in shared memory (128 KB for 65536 edges), sums to global
__global__ void k_smem16(uint32_t* gcnt, unsigned long long* sum, uint64_t n) {
    extern __shared__ uint32_t s_c[];
    for (int i = threadIdx.x; i < E / 2; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = hsh(i);
        uint32_t e = h & (E - 1);
        const uint32_t inc = (e & 1) ? 0x10000u : 1u;
        const uint32_t old = atomicAdd(&s_c[e >> 1], inc);
        if ((((e & 1) ? (old >> 16) : old) & 0xffffu) == 0x3fffu) {
            atomicSub(&s_c[e >> 1], inc * 0x4000u);
            atomicAdd(&gcnt[e], 0x4000u);
        }
        atomicAdd(&sum[e], (unsigned long long)(h >> 8));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E / 2; i += blockDim.x) {
        uint32_t v = s_c[i];
        if (v & 0xffff) atomicAdd(&gcnt[2 * i], v & 0xffff);
        if (v >> 16) atomicAdd(&gcnt[2 * i + 1], v >> 16);
    }
}

template <int K>
__global__ void k_cluster(uint32_t* gcnt, unsigned long long* gsum, uint64_t n) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int PER = E / K;
    unsigned long long* s_sum = (unsigned long long*)sm;
    uint32_t* s_cnt = (uint32_t*)(s_sum + PER);
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < PER; i += blockDim.x) { s_sum[i] = 0; s_cnt[i] = 0; }
    cl.sync();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = hsh(i);
        uint32_t e = h & (E - 1);
        uint32_t owner = e % K, idx = e / K;
        unsigned long long* rs = cl.map_shared_rank(s_sum, owner);
        uint32_t* rc = cl.map_shared_rank(s_cnt, owner);
        atomicAdd(&rc[idx], 1u);
        atomicAdd(&rs[idx], (unsigned long long)(h >> 8));
    }
    cl.sync();
    const uint32_t r = cl.block_rank();
    for (int i = threadIdx.x; i < PER; i += blockDim.x) {
        if (s_cnt[i]) {
            atomicAdd(&gcnt[i * K + r], s_cnt[i]);
            atomicAdd(&gsum[i * K + r], s_sum[i]);
        }
    }
}

template <int K>
float run_cluster(uint32_t* c, unsigned long long* s, uint64_t n, int blocks_per_sm) {
    size_t smem = (size_t)(E / K) * 12;
    cudaFuncSetAttribute(k_cluster<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (K > 8) cudaFuncSetAttribute(k_cluster<K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int grid = 148 / K * K * blocks_per_sm;
    if (grid < K) grid = K;
    grid = grid / K * K;
    cfg.gridDim = grid;
    cfg.blockDim = 512;
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k_cluster<K>, c, s, n);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&cfg, k_cluster<K>, c, s, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t err = cudaGetLastError();
    if (err) printf("K=%d err %s\n", K, cudaGetErrorString(err));
    return ms / 5;
}

int main() {
    uint64_t n = 100000000ull;
    uint32_t* c; unsigned long long* s;
    cudaMalloc(&c, E * 4); cudaMalloc(&s, E * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k_global<<<148 * 8, 256>>>(c, s, n);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_global<<<148 * 8, 256>>>(c, s, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("global RED  : %.3f ms per 1e8 pairs\n", ms / 5);
    unsigned long long* c64; cudaMalloc(&c64, E * 8);
    for (int g : {148 * 2, 148 * 4, 148 * 8, 148 * 16}) {
        k_global64<<<g, 256>>>(c64, s, n);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_global64<<<g, 256>>>(c64, s, n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("global RED u64 cnt grid %d: %.3f ms\n", g, ms / 5);
        k_global<<<g, 256>>>(c, s, n);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_global<<<g, 256>>>(c, s, n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("global RED u32 cnt grid %d: %.3f ms\n", g, ms / 5);
    }
    k_sumonly<<<148 * 8, 256>>>(s, n);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_sumonly<<<148 * 8, 256>>>(s, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("global sum only: %.3f ms\n", ms / 5);
    cudaFuncSetAttribute(k_smem16, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int t : {256, 512, 1024}) {
        k_smem16<<<148, t, 131072>>>(c, s, n);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_smem16<<<148, t, 131072>>>(c, s, n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("smem16 cnt + global sum, %d thr: %.3f ms (%s)\n", t, ms / 5, cudaGetErrorString(cudaGetLastError()));
    }
    for (int bps = 2; bps <= 1; ++bps) {
        printf("cluster 4  bps=%d: %.3f ms\n", bps, run_cluster<4>(c, s, n, bps));
        printf("cluster 8  bps=%d: %.3f ms\n", bps, run_cluster<8>(c, s, n, bps));
        printf("cluster 16 bps=%d: %.3f ms\n", bps, run_cluster<16>(c, s, n, bps));
    }
    return 0;
}
