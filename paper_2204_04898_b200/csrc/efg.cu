// NEXT-3: eventually-follows graph and temporal profile ("EFG retrieval /
// Temporal Profile (efg.py): discovers the eventually-follows graphs or the
// temporal profile"; reading R22).
//
// For every case of the formatted log and every ordered row pair i < j inside
// it: edge (a_i, a_j) gets count += 1, sum += d, sumsq += d^2, d = key_j - key_i
// (= ts_j - ts_i, u64).  The work is O(sum m^2) -- 45 pairs per event at m = 10
// -- and bound by shared-memory atomics, not HBM.
//
// k_efg: persistent CTAs over tiles of consecutive cases (tile edges are case
// edges).  A tile whose rows fit is staged in shared memory with each row's
// case end; thread t takes rows i = e0 + t, e0 + t + 512, ... and walks its
// case's later rows.  Tiles too large to stage (long cases) are walked case by
// case from global memory.  Accumulation is privatised per CTA: EFG_FULL (A <=
// 71) a dense table, EFG_HASH a 4096-slot hash table keyed by edge id (global
// fallback after 16 probes).  Per edge: u32 count, u32 lo / hi sum with exact
// carry, and d^2 (d < 2^32) as two u32 limbs whose carry out of 64 bits goes
// to the global high word; d >= 2^32 goes straight to the global 128-bit sum.
// Flushed once per CTA with 64-bit global atomics (128-bit adds carry through
// the returned low word).
#include <cuda_runtime.h>

#include <algorithm>

#include "pm4g_internal.cuh"

namespace pm4g {

constexpr int EFG_THREADS = 512;
constexpr int EFG_STAGE = 2048;          // rows of a staged tile (2048: the dense table + stage fit 2 CTAs per SM)
constexpr int EFG_MAX_CPT = 1024;        // cases per tile
constexpr uint32_t EFG_HS = 4096;        // hash slots
constexpr int EFG_PROBES = 16;
constexpr uint32_t EFG_EMPTY = 0xffffffffu;
constexpr size_t EFG_FULL_MAX = 100 * 1024;
enum { EFG_FULL = 0, EFG_HASH = 1 };

struct EfgTab {
    uint64_t* cnt;     // [AA]
    uint64_t* sum;     // [AA]
    uint64_t* sq_lo;   // [AA]
    uint64_t* sq_hi;   // [AA]
};

// 128-bit global add of (lo, hi): the carry out of the low word decides the high add
__device__ __forceinline__ void g_add128(uint64_t* lo_p, uint64_t* hi_p, uint64_t lo, uint64_t hi) {
    const unsigned long long old = atomicAdd((unsigned long long*)lo_p, (unsigned long long)lo);
    hi += (old + lo < old) ? 1ull : 0ull;
    if (hi) atomicAdd((unsigned long long*)hi_p, (unsigned long long)hi);
}

template <class P, int MODE>
__global__ __launch_bounds__(EFG_THREADS) void k_efg(const uint64_t* __restrict__ key, const P* __restrict__ act,
                                                     const uint32_t* __restrict__ off,
                                                     const uint64_t* __restrict__ d_n_cases, uint32_t A,
                                                     uint32_t cpt, EfgTab g) {
    extern __shared__ __align__(16) unsigned char efg_sm[];
    const uint32_t AA = A * A;
    const uint32_t TW = MODE == EFG_FULL ? AA : EFG_HS;
    uint32_t* s_cnt = (uint32_t*)efg_sm;
    uint32_t* s_slo = s_cnt + TW;
    uint32_t* s_shi = s_slo + TW;
    uint32_t* s_q0 = s_shi + TW;
    uint32_t* s_q1 = s_q0 + TW;
    uint32_t* s_key = s_q1 + TW;                                   // HASH only
    const uint32_t tw_words = (MODE == EFG_FULL ? 5 : 6) * TW;
    uint64_t* st_key = (uint64_t*)(efg_sm + (((size_t)tw_words * 4 + 15) & ~(size_t)15));   // [EFG_STAGE]
    uint16_t* st_end = (uint16_t*)(st_key + EFG_STAGE);              // [EFG_STAGE] case end (tile-relative)
    uint32_t* st_off = (uint32_t*)(st_end + EFG_STAGE);              // [EFG_MAX_CPT + 1]
    P* st_act = (P*)(st_off + EFG_MAX_CPT + 2);                      // [EFG_STAGE]
    __shared__ int s_staged;
    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < tw_words; i += EFG_THREADS)
        s_cnt[i] = (MODE == EFG_HASH && i >= 5 * TW) ? EFG_EMPTY : 0u;
    __syncthreads();

    // accumulate pair (e, d) into the CTA table
    auto acc = [&](uint32_t e, uint64_t d) {
        uint32_t x = e;
        if (MODE == EFG_HASH) {
            uint32_t h = (e * 0x9E3779B1u) >> (32 - 12);
            x = EFG_EMPTY;
            for (int p = 0; p < EFG_PROBES; ++p, h = (h + 1) & (EFG_HS - 1)) {
                uint32_t k = s_key[h];
                if (k == EFG_EMPTY) k = atomicCAS(&s_key[h], EFG_EMPTY, e);
                if (k == EFG_EMPTY || k == e) {
                    x = h;
                    break;
                }
            }
            if (x == EFG_EMPTY) {   // no slot near: straight to the global table
                atomicAdd((unsigned long long*)&g.cnt[e], 1ull);
                atomicAdd((unsigned long long*)&g.sum[e], (unsigned long long)d);
                g_add128(&g.sq_lo[e], &g.sq_hi[e], d * d, __umul64hi(d, d));
                return;
            }
        }
        atomicAdd(&s_cnt[x], 1u);
        {
            const uint32_t l = (uint32_t)d;
            uint32_t hi = (uint32_t)(d >> 32);
            const uint32_t old = atomicAdd(&s_slo[x], l);
            hi += (old + l < old) ? 1u : 0u;
            if (hi) atomicAdd(&s_shi[x], hi);   // wraps modulo 2^64 with the sum (R8)
        }
        if ((d >> 32) == 0) {
            const uint64_t q = d * d;            // < 2^64
            const uint32_t q0 = (uint32_t)q;
            uint32_t q1 = (uint32_t)(q >> 32);    // <= 0xfffffffe
            const uint32_t o0 = atomicAdd(&s_q0[x], q0);
            q1 += (o0 + q0 < o0) ? 1u : 0u;
            if (q1) {
                const uint32_t o1 = atomicAdd(&s_q1[x], q1);
                if (o1 + q1 < o1) atomicAdd((unsigned long long*)&g.sq_hi[e], 1ull);   // carry out of 64 bits
            }
        } else {
            g_add128(&g.sq_lo[e], &g.sq_hi[e], d * d, __umul64hi(d, d));
        }
    };

    const uint64_t C = *d_n_cases;
    const uint64_t tiles = (C + cpt - 1) / cpt;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const uint64_t c0 = t * cpt;
        const uint32_t nc = (uint32_t)min((uint64_t)cpt, C - c0);
        for (uint32_t j = tid; j <= nc; j += EFG_THREADS) st_off[j] = off[c0 + j];
        __syncthreads();
        const uint32_t e0 = st_off[0], e1 = st_off[nc];
        if (tid == 0) s_staged = (e1 - e0) <= (uint32_t)EFG_STAGE;
        __syncthreads();
        if (s_staged) {
            for (uint32_t r = tid; r < e1 - e0; r += EFG_THREADS) {
                st_key[r] = key[e0 + r];
                st_act[r] = act[e0 + r];
            }
            for (uint32_t c = tid; c < nc; c += EFG_THREADS)
                for (uint32_t r = st_off[c]; r < st_off[c + 1]; ++r) st_end[r - e0] = (uint16_t)(st_off[c + 1] - e0);
            __syncthreads();
            for (uint32_t r = tid; r < e1 - e0; r += EFG_THREADS) {
                const uint32_t end = st_end[r];
                const uint64_t ki = st_key[r];
                const uint32_t ai = (uint32_t)st_act[r] * A;
                for (uint32_t j = r + 1; j < end; ++j) acc(ai + (uint32_t)st_act[j], st_key[j] - ki);
            }
        } else {
            for (uint32_t c = 0; c < nc; ++c) {          // long cases: case by case from global memory
                const uint32_t f = st_off[c], l = st_off[c + 1];
                for (uint32_t r = f + tid; r < l; r += EFG_THREADS) {
                    const uint64_t ki = key[r];
                    const uint32_t ai = (uint32_t)act[r] * A;
                    for (uint32_t j = r + 1; j < l; ++j) acc(ai + (uint32_t)act[j], key[j] - ki);
                }
            }
        }
        __syncthreads();
    }
    // flush
    for (uint32_t x = tid; x < TW; x += EFG_THREADS) {
        const uint32_t cn = s_cnt[x];
        if (!cn) continue;
        const uint32_t e = MODE == EFG_FULL ? x : s_key[x];
        atomicAdd((unsigned long long*)&g.cnt[e], (unsigned long long)cn);
        const uint64_t sm = ((uint64_t)s_shi[x] << 32) | s_slo[x];
        if (sm) atomicAdd((unsigned long long*)&g.sum[e], (unsigned long long)sm);
        const uint64_t q = ((uint64_t)s_q1[x] << 32) | s_q0[x];
        if (q) g_add128(&g.sq_lo[e], &g.sq_hi[e], q, 0);
    }
}

// cross-rank sum of the 128-bit words: split into four 32-bit limbs (as u64,
// so a sum over ranks cannot overflow), allreduce, recombine with carries
__global__ void k_efg_limbs(const uint64_t* lo, const uint64_t* hi, size_t AA, uint64_t* limbs) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < AA; e += (size_t)gridDim.x * blockDim.x) {
        limbs[e] = (uint32_t)lo[e];
        limbs[AA + e] = lo[e] >> 32;
        limbs[2 * AA + e] = (uint32_t)hi[e];
        limbs[3 * AA + e] = hi[e] >> 32;
    }
}
__global__ void k_efg_unlimb(const uint64_t* limbs, size_t AA, uint64_t* lo, uint64_t* hi) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < AA; e += (size_t)gridDim.x * blockDim.x) {
        unsigned __int128 v = (unsigned __int128)limbs[e] + ((unsigned __int128)limbs[AA + e] << 32) +
                              ((unsigned __int128)limbs[2 * AA + e] << 64) + ((unsigned __int128)limbs[3 * AA + e] << 96);
        lo[e] = (uint64_t)v;
        hi[e] = (uint64_t)(v >> 64);
    }
}

// R22: mean = sum / m; s2 = hi * 2^64 + lo; V = (s2 - sum * mean) / m;
// stdev = V > 0 ? sqrt(V) : 0 (explicit RN intrinsics: no contraction)
__global__ void k_efg_finalize(EfgTab g, size_t AA, uint64_t* cnt, uint64_t* sum, uint64_t* sq, double* mean,
                               double* stdev) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < AA; e += (size_t)gridDim.x * blockDim.x) {
        const uint64_t c = g.cnt[e], s = g.sum[e], lo = g.sq_lo[e], hi = g.sq_hi[e];
        if (cnt) cnt[e] = c;
        if (sum) sum[e] = s;
        if (sq) {
            sq[e] = lo;
            sq[AA + e] = hi;
        }
        double mu = 0.0, sd = 0.0;
        if (c) {
            const double m = __ull2double_rn(c);
            mu = __ddiv_rn(__ull2double_rn(s), m);
            const double s2 = __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
            const double V = __ddiv_rn(__dsub_rn(s2, __dmul_rn(__ull2double_rn(s), mu)), m);
            sd = V > 0.0 ? __dsqrt_rn(V) : 0.0;
        }
        if (mean) mean[e] = mu;
        if (stdev) stdev[e] = sd;
    }
}

template <class P, int MODE>
static pm4g_status launch_efg(const pm4g_log* L, const EfgTab& g, cudaStream_t s) {
    const uint32_t A = L->A;
    const uint32_t TW = MODE == EFG_FULL ? A * A : EFG_HS;
    const size_t tab = (((size_t)(MODE == EFG_FULL ? 5 : 6) * TW * 4) + 15) & ~(size_t)15;
    const size_t smem = tab + (size_t)EFG_STAGE * (8 + 2 + sizeof(P)) + (EFG_MAX_CPT + 2) * 4 + 16;
    PM4G_MAX_SMEM(k_efg<P, MODE>);
    const uint64_t cap = std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1);
    const double mean_len = (double)L->n / (double)std::max<uint64_t>(cap, 1);
    const uint32_t cpt = (uint32_t)std::max(16.0, std::min((double)EFG_MAX_CPT, 0.7 * EFG_STAGE / std::max(mean_len, 1.0)));
    const uint64_t tiles = std::max<uint64_t>(1, (cap + cpt - 1) / cpt);
    const int per_sm = std::max(1, (int)std::min<size_t>(4, (226 * 1024) / (smem + 1024)));
    const uint64_t grid = std::min<uint64_t>(tiles, (uint64_t)num_sms() * per_sm);
    PM4G_LAUNCH("k_efg", (double)L->n * (8 + sizeof(P)), s,
                (k_efg<P, MODE><<<(unsigned)grid, EFG_THREADS, smem, s>>>(L->key, (const P*)L->s_act, L->off,
                                                                        L->d_n_cases, A, cpt, g)));
    return PM4G_OK;
}

template <class P>
static pm4g_status launch_efg_p(const pm4g_log* L, const EfgTab& g, cudaStream_t s) {
    if ((size_t)5 * L->A * L->A * 4 <= EFG_FULL_MAX) return launch_efg<P, EFG_FULL>(L, g, s);
    return launch_efg<P, EFG_HASH>(L, g, s);
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_efg(const pm4g_log* L, uint64_t* cnt, uint64_t* dur_sum, uint64_t* dur_sumsq, double* mean,
                     double* stdev, pm4g_comm* comm, pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_efg");
    PM4G_TRY(check_log(L));
    if (!L->sorted) return fail(PM4G_EINVAL, "log is not sorted (call pm4g_sort first)");
    if (!cnt && !dur_sum && !dur_sumsq && !mean && !stdev) return fail(PM4G_EINVAL, "no output requested");
    if ((uint64_t)L->A * L->A > 0xffffffffull) return fail(PM4G_EINVAL, "n_activities too large for an A x A table");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t AA = (size_t)L->A * L->A;
    Scratch tb(s), lb(s);
    PM4G_TRY(tb.alloc(4 * AA * 8));
    PM4G_CK(cudaMemsetAsync(tb.p, 0, 4 * AA * 8, s));
    EfgTab g{tb.as<uint64_t>(), tb.as<uint64_t>() + AA, tb.as<uint64_t>() + 2 * AA, tb.as<uint64_t>() + 3 * AA};
    if (L->n > 0) {
        switch (L->act_bytes) {
            case 1: PM4G_TRY(launch_efg_p<uint8_t>(L, g, s)); break;
            case 2: PM4G_TRY(launch_efg_p<uint16_t>(L, g, s)); break;
            default: PM4G_TRY(launch_efg_p<uint32_t>(L, g, s)); break;
        }
    }
    const int gsz = (int)std::max<size_t>(1, std::min<size_t>((AA + 255) / 256, (size_t)num_sms() * 4));
    if (comm) {
        PM4G_TRY(comm_allreduce_u64(comm, g.cnt, 2 * AA, s));   // counts and sums
        PM4G_TRY(lb.alloc(4 * AA * 8));
        PM4G_LAUNCH("k_efg_limbs", AA * 48.0, s, (k_efg_limbs<<<gsz, 256, 0, s>>>(g.sq_lo, g.sq_hi, AA, lb.as<uint64_t>())));
        PM4G_TRY(comm_allreduce_u64(comm, lb.as<uint64_t>(), 4 * AA, s));
        PM4G_LAUNCH("k_efg_unlimb", AA * 48.0, s, (k_efg_unlimb<<<gsz, 256, 0, s>>>(lb.as<uint64_t>(), AA, g.sq_lo, g.sq_hi)));
    }
    PM4G_LAUNCH("k_efg_finalize", AA * 72.0, s,
                (k_efg_finalize<<<gsz, 256, 0, s>>>(g, AA, cnt, dur_sum, dur_sumsq, mean, stdev)));
    return PM4G_OK;
}

}  // extern "C"
