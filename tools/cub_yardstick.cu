// Yardstick only (not product code): CUB DeviceRadixSort::SortPairs on the same
// problem the pm4g case passes solve -- 100M (u64 key, u8 act) pairs, sorted
// stably on the 24 case bits above bit 36 -- to compare per-pass throughput.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

int main() {
    const size_t n = 100000000;
    std::vector<uint64_t> hk(n);
    std::vector<uint8_t> hv(n);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (size_t i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        uint64_t cs = (s >> 40) % 10000000ull, t = s & ((1ull << 36) - 1);
        hk[i] = (cs << 36) | t;
        hv[i] = (uint8_t)(s >> 8);
    }
    uint64_t *k0, *k1; uint8_t *v0, *v1;
    cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n); cudaMalloc(&v1, n);
    cudaMemcpy(k0, hk.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), n, cudaMemcpyHostToDevice);
    size_t tmp = 0;   // the full-key sort needs the most temporary storage
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, (int)n, 0, 60);
    void* t; cudaMalloc(&t, tmp);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bits : {24, 60}) {
        int begin = bits == 24 ? 36 : 0;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, (int)n, begin, 60);
            cudaEventRecord(b); cudaEventSynchronize(b);
            if (cudaGetLastError() != cudaSuccess) { printf("CUB sort failed\n"); return 1; }
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r == 2) printf("CUB SortPairs u64+u8, %zu items, bits [%d,60): %.3f ms (%.2f G items/s)\n", n, begin, ms, n / ms / 1e6);
        }
    }
    return 0;
}
