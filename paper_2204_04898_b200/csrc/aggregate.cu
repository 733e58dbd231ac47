// A5-A8: the fused aggregate pass over the formatted log (K6) and the table
// finaliser (K11).
//
//  A5  DFG ("calculating the frequency/performance directly-follows
//      graph"; P:110 previous-event columns): for consecutive rows
//      i, i+1 of one case, cnt[a_i][a_{i+1}] += 1, sum += ts_{i+1} - ts_i.  On
//      the composite key the duration is key_{i+1} - key_i (the case bits
//      cancel), so timestamps are never decoded.
//  A6  start/end activities.
//  A7  events per case and throughput time = last ts - first ts (P:101,
//      P:112-114).
//  A8  per-case variant key ("numerical features that uniquely identify
//      the case's variant"): two 64-bit polynomial hashes of the
//      (act + 1) sequence plus the length, verified exactly later (A9).
//
// Work split: a CTA owns tiles of up to 256 consecutive CASES (tile edges are
// case edges, so no directly-follows pair straddles two CTAs); the host sizes
// tiles from the mean case length so a tile's rows fit one TMA stage.  Pairs
// are processed event-parallel (coalesced), per-case work case-parallel.  The
// A x A table lives where it fits:
//   TAB_FULL  (3 A^2 words <= 100 KB, A <= 91): privatised per CTA in shared
//             memory (u32 counts; u32 lo/hi duration sums with exact carry
//             propagation, because 64-bit shared atomics are CAS loops on
//             sm_100a), flushed once per CTA with 64-bit global atomics;
//   TAB_HASH  (larger A): a per-CTA shared-memory hash table keyed by edge id
//             (key, count, lo, hi) -- process DFGs are sparse (a handful of
//             successors per activity), so the edges a CTA sees fit; an edge
//             that finds no slot within HASH_PROBES goes straight to the
//             global table.  Global atomics alone serialise on the hot edges
//             of a skewed DFG (measured 2.4 ms per 1e8 events at A = 256), and
//             a DSMEM-distributed dense table is slower than L2 atomics
//             (tools/mbench_dsmem.cu).
#include <cuda_runtime.h>

#include <algorithm>

#include "pm4g_internal.cuh"

namespace pm4g {

constexpr int AGG_THREADS = 256;
constexpr int AGG_CASES = 256;   // cases per tile
constexpr size_t AGG_SMEM_MAX = 100 * 1024;     // TAB_FULL table budget

#ifndef PM4G_AGG_PMIN   // fewest pair threads left when the case-holding warps skip the pairs
#define PM4G_AGG_PMIN 512
#endif
#ifndef PM4G_AGG_FCONS
#define PM4G_AGG_FCONS 992
#endif
#ifndef PM4G_AGG_HCONS
#define PM4G_AGG_HCONS 992
#endif

enum { TAB_FULL = 1, TAB_HASH = 2 };

// Geometry per table mode (measured on one B200; the kernel is latency-bound,
// so the number of warps in flight decides).  TAB_FULL: 31 consumer warps,
// 3 stages of 4096 rows, one CTA per SM (100M, A = 64: 0.478 ms; two CTAs per
// SM of 3 x 2048-row stages with 8 / 12 / 16 / 24 consumer warps 0.516 /
// 0.498 / 0.498 / 0.572 ms; 31 warps with 2048-row stages 0.73, 2 x 4096
// 0.487).  TAB_HASH: 31 consumer warps, 8192 slots, 2 stages of 4096 rows, one
// CTA per SM (1B/8 shard, A = 256, ~1,000 distinct edges: 0.597 ms; the same
// with 23 warps 0.603; 16 warps + 4096 slots + 2 x 2048 rows at two CTAs per
// SM 0.667, with 8 warps 0.796; 3 stages or 1024-row stages slower).  The
// PM4G_AGG_* macros are the sweep's knobs.
#ifndef PM4G_AGG_HROWS
#define PM4G_AGG_HROWS 4096
#endif
#ifndef PM4G_AGG_HSTAGES
#define PM4G_AGG_HSTAGES 2
#endif
#ifndef PM4G_AGG_HSLOTS
#define PM4G_AGG_HSLOTS 8192
#endif
#ifndef PM4G_AGG_FROWS
#define PM4G_AGG_FROWS 4096
#endif
#ifndef PM4G_AGG_FSTAGES
#define PM4G_AGG_FSTAGES 3
#endif
template <class P, int MODE>
struct AggGeom {
    // rows of a staged case tile (wider activity codes: half the TAB_FULL stage, so
    // a 100 KB dense table and three stages still fit one CTA's shared memory)
    static constexpr uint32_t ROWS = MODE == TAB_FULL ? (sizeof(P) == 1 ? PM4G_AGG_FROWS : PM4G_AGG_FROWS / 2)
                                                      : PM4G_AGG_HROWS;
    static constexpr int STAGES = MODE == TAB_FULL ? PM4G_AGG_FSTAGES : PM4G_AGG_HSTAGES;
    static constexpr int CONS = MODE == TAB_FULL ? PM4G_AGG_FCONS : PM4G_AGG_HCONS;       // consumer threads
    static constexpr int BLOCK = CONS + 32;                                                 // + 1 producer warp
    static_assert(CONS >= AGG_CASES, "one consumer thread per case of a tile");
};

// One pipeline stage: the tile's case offsets and its rows (keys, activities).
template <class P, uint32_t ROWS>
struct alignas(128) AggStage {
    uint32_t off[AGG_CASES + 4];
    uint64_t key[ROWS + 16];
    P act[ROWS + 32];
    uint32_t nc, ka, aa, staged;
    uint64_t c0;
};

constexpr int HASH_PROBES = 16;
constexpr uint32_t HASH_EMPTY = 0xffffffffu;

// shared-memory hash slots: 4096 (two CTAs per SM next to two 2048-row stages)
template <class P, bool MM>
__host__ __device__ constexpr uint32_t hash_slots() { return (sizeof(P) == 1 && !MM) ? (uint32_t)PM4G_AGG_HSLOTS : 4096u; }

// start/end counters are privatised when A is small enough
constexpr uint32_t SE_SMEM_MAX_A = 2048;
__host__ __device__ constexpr uint32_t se_words(uint32_t A) { return A <= SE_SMEM_MAX_A ? 2 * A : 0u; }

// table layout (u32 words): FULL [cnt | lo | hi](A^2 each) [start | end](A) [min | max](A^2 each, MM);
// HASH [cnt | lo | hi | key](HS each) [start | end] [min | max](HS each, MM)
template <class P, bool MM>
__host__ __device__ constexpr uint32_t tab_words_for(int mode, uint32_t A) {
    return mode == TAB_FULL ? (((3 + (MM ? 2 : 0)) * A * A + 2 * A + 31) & ~31u)
                            : ((4 + (MM ? 2 : 0)) * hash_slots<P, MM>() + se_words(A) + 31) & ~31u;
}

// per-pair min / max of the u64 duration (R20): u32 shared tables for
// durations below 2^32, the global u64 table otherwise
__device__ __forceinline__ void smem_minmax(uint32_t* mn, uint32_t* mx, unsigned long long* gmn,
                                            unsigned long long* gmx, uint64_t d) {
    if ((d >> 32) == 0) {
        atomicMin(mn, (uint32_t)d);
        atomicMax(mx, (uint32_t)d);
    } else {
        atomicMin(gmn, (unsigned long long)d);
        atomicMax(gmx, (unsigned long long)d);
    }
}

// per-pair accumulation into a (count, lo, hi) triple in shared memory; the
// carry out of the low word is exact because the returned old value decides it
__device__ __forceinline__ void smem_acc(uint32_t* cnt, uint32_t* lo, uint32_t* hi, uint64_t d) {
    atomicAdd(cnt, 1u);
    const uint32_t l = (uint32_t)d;
    uint32_t h = (uint32_t)(d >> 32);
    const uint32_t old = atomicAdd(lo, l);
    h += (old + l < old) ? 1u : 0u;
    if (h) atomicAdd(hi, h);
}

// WIDE: the log's key is ts - ts_min alone; a row's case is rcase[row]
template <class P, int MODE, bool MM, bool WIDE = false>
__global__ __launch_bounds__(AggGeom<P, MODE>::BLOCK) void k_aggregate(
    const uint64_t* __restrict__ key, const P* __restrict__ act, const uint32_t* __restrict__ off,
    const uint64_t* __restrict__ d_n_cases, int ts_bits, uint32_t A, uint32_t cpt,
    uint64_t* __restrict__ packed, uint64_t* __restrict__ mm, uint32_t* __restrict__ n_events,
    int64_t* __restrict__ dur, uint64_t* __restrict__ k1o, uint64_t* __restrict__ k2o, int weak,
    uint32_t* __restrict__ cco, uint32_t case_min, const uint32_t* __restrict__ rcase) {
    constexpr uint32_t AGG_STAGE = AggGeom<P, MODE>::ROWS;
    constexpr int AGG_STAGES = AggGeom<P, MODE>::STAGES;
    constexpr int AGG_CONSUMERS = AggGeom<P, MODE>::CONS, AGG_BLOCK = AggGeom<P, MODE>::BLOCK;
    using Stage = AggStage<P, AGG_STAGE>;
    extern __shared__ __align__(128) unsigned char agg_sm[];
    __shared__ __align__(8) uint64_t s_full[AGG_STAGES], s_empty[AGG_STAGES];
    const bool tables = packed != nullptr;
    const uint32_t AA = A * A;
    const uint32_t tab_words = tables ? tab_words_for<P, MM>(MODE, A) : 0;
    constexpr uint32_t HS = hash_slots<P, MM>();
    const uint32_t TW = MODE == TAB_FULL ? AA : HS;         // table entries
    uint32_t* sm = (uint32_t*)agg_sm;
    uint32_t* s_cnt = sm;
    uint32_t* s_lo = sm + TW;
    uint32_t* s_hi = sm + 2 * TW;
    uint32_t* s_key = sm + 3 * TW;                          // HASH: edge id or HASH_EMPTY
    uint32_t* s_st = sm + (MODE == TAB_FULL ? 3 * AA : 4 * HS);
    uint32_t* s_en = s_st + A;
    uint32_t* s_mn = s_st + (MODE == TAB_FULL ? 2 * A : se_words(A));   // MM: [TW]
    uint32_t* s_mx = s_mn + TW;
    unsigned long long* g_mn = (unsigned long long*)mm;
    unsigned long long* g_mx = g_mn + AA;
    Stage* stage = (Stage*)(agg_sm + (size_t)tab_words * 4);
    uint64_t* g_cnt = packed;
    uint64_t* g_sum = packed + AA;
    uint64_t* g_st = packed + 2 * (size_t)AA;
    uint64_t* g_en = g_st + A;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (uint32_t i = tid; i < tab_words; i += AGG_BLOCK) {
        const bool empty_key = MODE == TAB_HASH && i >= 3 * HS && i < 4 * HS;
        const bool min_init = MM && sm + i >= s_mn && sm + i < s_mx;
        sm[i] = (empty_key || min_init) ? 0xffffffffu : 0u;
    }
    if (tid == 0) {
        for (int s = 0; s < AGG_STAGES; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], AGG_CONSUMERS);
        }
    }
    __syncthreads();
    const uint64_t C = *d_n_cases;
    const uint64_t tiles = (C + cpt - 1) / cpt;

    if (warp == 0) {
        // ---------------- producer warp: stream tiles into the ring with TMA.
        // The case offsets of the NEXT tile are loaded into registers right after
        // this tile's rows are requested, so their latency hides behind the wait
        // for a free stage instead of delaying the row transfer.
        constexpr int OPL = (AGG_CASES + 1 + 31) / 32;   // offsets per lane
        uint32_t ro[OPL];
        auto load_off = [&](uint64_t t) {
            const uint64_t c0 = t * cpt;
            const uint32_t nc = t < tiles ? (uint32_t)min((uint64_t)cpt, C - c0) : 0u;
#pragma unroll
            for (int q = 0; q < OPL; ++q) {
                const uint32_t j = lane + 32 * q;
                ro[q] = (t < tiles && j <= nc) ? off[c0 + j] : 0u;
            }
        };
#ifndef PM4G_AGG_NOPF
        load_off(blockIdx.x);
#endif
        uint32_t i = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            const int s = i % AGG_STAGES;
            if (i >= AGG_STAGES) mbar_wait(&s_empty[s], ((i / AGG_STAGES) - 1) & 1);
            Stage& st = stage[s];
            const uint64_t c0 = t * cpt;
            const uint32_t nc = (uint32_t)min((uint64_t)cpt, C - c0);
#ifdef PM4G_AGG_NOPF
            for (uint32_t j = lane; j <= nc; j += 32) st.off[j] = off[c0 + j];
#else
#pragma unroll
            for (int q = 0; q < OPL; ++q) {
                const uint32_t j = lane + 32 * q;
                if (j <= nc) st.off[j] = ro[q];
            }
#endif
            __syncwarp();
            if (lane == 0) {
                const uint32_t e0 = st.off[0], e1 = st.off[nc];
                const uint32_t ka = e0 & ~1u, kb = (e1 + 1) & ~1u;                  // keys: 2 per 16 B
                const uint32_t ea = (uint32_t)(16 / sizeof(P));
                const uint32_t aa = e0 & ~(ea - 1), ab = (e1 + ea - 1) & ~(ea - 1);
                const bool fit = kb - ka <= AGG_STAGE + 16 && ab - aa <= AGG_STAGE + 32;
                st.nc = nc;
                st.c0 = c0;
                st.ka = ka;
                st.aa = aa;
                st.staged = fit ? 1u : 0u;
                if (fit) {
                    mbar_expect_tx(&s_full[s], (kb - ka) * 8 + (ab - aa) * (uint32_t)sizeof(P));
                    tma_load_1d(st.key, key + ka, (kb - ka) * 8, &s_full[s]);
                    tma_load_1d(st.act, act + aa, (ab - aa) * (uint32_t)sizeof(P), &s_full[s]);
                } else {
                    mbar_arrive(&s_full[s]);     // oversized tile: consumers read global memory
                }
            }
            __syncwarp();
#ifndef PM4G_AGG_NOPF
            load_off(t + gridDim.x);
#endif
        }
    } else {
        // ---------------- consumer warps
        const int ct = tid - 32;
        uint32_t i = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            const int s = i % AGG_STAGES;
            mbar_wait(&s_full[s], (i / AGG_STAGES) & 1);
            const Stage& st = stage[s];
            const uint32_t nc = st.nc, ka = st.ka, aa = st.aa;
            const bool staged = st.staged != 0;
            const uint64_t c0 = st.c0;
            const uint32_t e0 = st.off[0], e1 = st.off[nc];
            auto K_at = [&](uint32_t r) -> uint64_t { return staged ? st.key[r - ka] : key[r]; };
            auto A_at = [&](uint32_t r) -> uint32_t { return staged ? (uint32_t)st.act[r - aa] : (uint32_t)act[r]; };
            if (tables) {
                // directly-follows pairs (r, r+1) of one case
                // the warps holding the tile's cases (threads < nc, one serial
                // per-case loop each, below) take no pairs when enough other
                // warps remain, so they do not hold the stage's release (ncu:
                // 39% of the stall samples were consumers waiting for a full
                // stage, i.e. for the case-holding warps to free one; 1B/8 shard
                // 0.60 -> 0.46 ms, 100M 0.48 -> 0.41 ms; a team-parallel Horner
                // hash instead cost 7x the instructions and was 2-3x slower)
                const uint32_t pw = (nc + 31) & ~31u;
                const uint32_t p0 = AGG_CONSUMERS - pw >= PM4G_AGG_PMIN ? pw : 0u;
                const uint32_t r0 = (uint32_t)ct >= p0 ? e0 + (ct - p0) : e1;   // e1: no pairs
                for (uint32_t r = r0; r + 1 < e1; r += AGG_CONSUMERS - p0) {
                    const uint64_t kk = K_at(r), kn = K_at(r + 1);
                    if (WIDE ? rcase[r] != rcase[r + 1] : !same_case(kk, kn, ts_bits)) continue;
                    const uint32_t e = A_at(r) * A + A_at(r + 1);
                    const uint64_t d = kn - kk;
                    if (MODE == TAB_FULL) {
                        smem_acc(&s_cnt[e], &s_lo[e], &s_hi[e], d);
                        if (MM) smem_minmax(&s_mn[e], &s_mx[e], &g_mn[e], &g_mx[e], d);
                        continue;
                    }
                    // probe sequence h1, h2, h2 + 1, ... (two independent hashes, then
                    // linear): a key already in the table is found by the two
                    // unconditional reads (no loop, so one lane's collision does not
                    // serialise its warp -- with one linear sequence 3/4 of the warps
                    // took a second probe at the 1B/8 shard); inserts and the rare
                    // third-or-later positions take the loop, which walks the same
                    // sequence, so every lane agrees on a key's slot.
                    const uint32_t h1 = (e * 0x9E3779B1u) >> (32 - __builtin_ctz(HS));
                    const uint32_t h2 = ((e ^ 0x5bd1e995u) * 0x85EBCA77u) >> (32 - __builtin_ctz(HS));
                    const uint32_t k1 = s_key[h1], k2 = s_key[h2];
                    uint32_t hs = k1 == e ? h1 : (k2 == e ? h2 : HASH_EMPTY);
                    if (hs == HASH_EMPTY) {
                        uint32_t h = h1;
                        for (int p = 0; p < HASH_PROBES; ++p) {
                            uint32_t k = s_key[h];
                            if (k == HASH_EMPTY) k = atomicCAS(&s_key[h], HASH_EMPTY, e);
                            if (k == HASH_EMPTY || k == e) {
                                hs = h;
                                break;
                            }
                            h = p == 0 ? h2 : (h + 1) & (HS - 1);
                        }
                    }
                    const bool done = hs != HASH_EMPTY;
                    if (done) {
                        smem_acc(&s_cnt[hs], &s_lo[hs], &s_hi[hs], d);
                        if (MM) smem_minmax(&s_mn[hs], &s_mx[hs], &g_mn[e], &g_mx[e], d);
                    }
                    if (!done) {   // no slot near: straight to the global table
                        atomicAdd((unsigned long long*)&g_cnt[e], 1ull);
                        atomicAdd((unsigned long long*)&g_sum[e], (unsigned long long)d);
                        if (MM) {
                            atomicMin(&g_mn[e], (unsigned long long)d);
                            atomicMax(&g_mx[e], (unsigned long long)d);
                        }
                    }
                }
            }
            if ((uint32_t)ct < nc) {
                const uint64_t c = c0 + ct;
                const uint32_t f = st.off[ct], l = st.off[ct + 1] - 1;
                if (tables) {
                    const uint32_t as = A_at(f), ae = A_at(l);
                    if (se_words(A)) {
                        atomicAdd(&s_st[as], 1u);
                        atomicAdd(&s_en[ae], 1u);
                    } else {
                        atomicAdd((unsigned long long*)&g_st[as], 1ull);
                        atomicAdd((unsigned long long*)&g_en[ae], 1ull);
                    }
                }
                if (n_events) n_events[c] = l - f + 1;
                if (cco) cco[c] = case_min + (WIDE ? rcase[f] : case32(K_at(f), ts_bits));
                if (dur) dur[c] = (int64_t)(K_at(l) - K_at(f));
                if (k1o) {
                    uint64_t h1 = 0, h2 = 0;
                    for (uint32_t r = f; r <= l; ++r) {
                        const uint64_t a = (uint64_t)A_at(r) + 1;
                        h1 = h1 * HB1 + a;
                        h2 = h2 * HB2 + a;
                    }
                    uint64_t x1, x2;
                    finish_key(h1, h2, l - f + 1, weak != 0, x1, x2);
                    k1o[c] = x1;
                    k2o[c] = x2;
                }
            }
            mbar_arrive(&s_empty[s]);   // this thread is done reading the stage
        }
    }
    __syncthreads();
    if (tables) {
        for (uint32_t a = tid; a < (se_words(A) ? A : 0u); a += AGG_BLOCK) {
            if (s_st[a]) atomicAdd((unsigned long long*)&g_st[a], (unsigned long long)s_st[a]);
            if (s_en[a]) atomicAdd((unsigned long long*)&g_en[a], (unsigned long long)s_en[a]);
        }
        for (uint32_t j = tid; j < TW; j += AGG_BLOCK) {
            const uint32_t cn = s_cnt[j];
            if (!cn) continue;
            const uint32_t e = MODE == TAB_FULL ? j : s_key[j];
            atomicAdd((unsigned long long*)&g_cnt[e], (unsigned long long)cn);
            const uint64_t sm64 = ((uint64_t)s_hi[j] << 32) | s_lo[j];
            if (sm64) atomicAdd((unsigned long long*)&g_sum[e], (unsigned long long)sm64);
            if (MM) {
                if (s_mn[j] != 0xffffffffu) atomicMin(&g_mn[e], (unsigned long long)s_mn[j]);
                if (s_mx[j]) atomicMax(&g_mx[e], (unsigned long long)s_mx[j]);
            }
        }
    }
}

template <class P, int MODE, bool MM, bool WIDE>
static pm4g_status launch_agg_w(const pm4g_log* L, const AggOut& o, cudaStream_t s) {
    const uint32_t A = L->A;
    const size_t tab = o.tables ? (size_t)tab_words_for<P, MM>(MODE, A) * 4 : 0;
    constexpr uint32_t AGG_STAGE = AggGeom<P, MODE>::ROWS;
    const size_t smem = tab + AggGeom<P, MODE>::STAGES * sizeof(AggStage<P, AGG_STAGE>);
    PM4G_MAX_SMEM(k_aggregate<P, MODE, MM, WIDE>);
    const uint64_t cap = std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1);
    // cases per tile: a tile's rows should fit one stage (mean length from the
    // case-code range, exact when codes are dense; a rare oversized tile is
    // read from global memory instead)
    const double mean_len = (double)L->n / (double)std::max<uint64_t>(cap, 1);
    const uint32_t cpt = (uint32_t)std::max(32.0, std::min((double)AGG_CASES, 0.7 * AGG_STAGE / std::max(mean_len, 1.0)));
    const uint64_t tiles = std::max<uint64_t>(1, (cap + cpt - 1) / cpt);
    static int per_sm_c[2] = {-1, -1};   // smem depends only on whether tables are requested
    int& per_sm = per_sm_c[o.tables ? 1 : 0];
    if (per_sm < 0)
        PM4G_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_aggregate<P, MODE, MM, WIDE>,
                                                              AggGeom<P, MODE>::BLOCK, smem));
    per_sm = std::max(per_sm, 1);
    const uint64_t grid = std::min<uint64_t>(tiles, (uint64_t)num_sms() * per_sm);
    // algorithmic bytes: read key + act once per event, + per-case offsets and outputs
    const double bytes = (double)L->n * (8 + sizeof(P) + (WIDE ? 4 : 0)) + (double)cap * 4 + (o.n_events ? cap * 4.0 : 0) +
                         (o.dur ? cap * 8.0 : 0) + (o.k1 ? cap * 16.0 : 0) + (o.case_code ? cap * 4.0 : 0);
    PM4G_LAUNCH("k_aggregate", bytes, s,
                (k_aggregate<P, MODE, MM, WIDE><<<(unsigned)grid, AggGeom<P, MODE>::BLOCK, smem, s>>>(
                    L->key, (const P*)L->s_act, L->off, L->d_n_cases, L->ts_bits, A, cpt,
                    o.tables ? o.packed : nullptr, o.mm, o.n_events, o.dur, o.k1, o.k2,
                    debug_weak_hash() ? 1 : 0, o.case_code, L->case_min, L->rcase)));
    return PM4G_OK;
}

template <class P, int MODE, bool MM>
static pm4g_status launch_agg(const pm4g_log* L, const AggOut& o, cudaStream_t s) {
    return L->wide ? launch_agg_w<P, MODE, MM, true>(L, o, s) : launch_agg_w<P, MODE, MM, false>(L, o, s);
}

template <class P>
static pm4g_status launch_agg_p(const pm4g_log* L, const AggOut& o, cudaStream_t s) {
    const uint32_t A = L->A;
    const bool mm = o.tables && o.mm;
    if (mm) {
        if ((size_t)tab_words_for<P, true>(TAB_FULL, A) * 4 <= AGG_SMEM_MAX) return launch_agg<P, TAB_FULL, true>(L, o, s);
        return launch_agg<P, TAB_HASH, true>(L, o, s);
    }
    if ((size_t)tab_words_for<P, false>(TAB_FULL, A) * 4 <= AGG_SMEM_MAX) return launch_agg<P, TAB_FULL, false>(L, o, s);
    return launch_agg<P, TAB_HASH, false>(L, o, s);
}

pm4g_status aggregate(const pm4g_log* L, const AggOut& o, cudaStream_t s) {
    if (L->n == 0) return PM4G_OK;
    switch (L->act_bytes) {
        case 1: return launch_agg_p<uint8_t>(L, o, s);
        case 2: return launch_agg_p<uint16_t>(L, o, s);
        default: return launch_agg_p<uint32_t>(L, o, s);
    }
}

// ------------------------------------------------------------------ K11 finalise
// R6: mean = (double)sum / (double)cnt for cnt > 0 (IEEE round-to-nearest), else 0.
__global__ void k_finalize(const uint64_t* __restrict__ packed, uint32_t A, uint64_t* cnt,
                           int64_t* sum, double* mean, uint64_t* st, uint64_t* en) {
    const size_t AA = (size_t)A * A;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < AA + A;
         e += (size_t)gridDim.x * blockDim.x) {
        if (e < AA) {
            uint64_t c = packed[e];
            int64_t sm = (int64_t)packed[AA + e];
            if (cnt) cnt[e] = c;
            if (sum) sum[e] = sm;
            if (mean) mean[e] = c ? __ddiv_rn((double)sm, (double)c) : 0.0;
        } else {
            size_t a = e - AA;
            if (st) st[a] = packed[2 * AA + a];
            if (en) en[a] = packed[2 * AA + A + a];
        }
    }
}

pm4g_status finalize_tables(const uint64_t* packed, uint32_t A, uint64_t* cnt, int64_t* sum,
                            double* mean, uint64_t* st, uint64_t* en, cudaStream_t s) {
    size_t total = (size_t)A * A + A;
    int g = (int)std::min<size_t>((total + 255) / 256, (size_t)num_sms() * 4);
    PM4G_LAUNCH("k_finalize", total * 8.0 * 2, s,
                k_finalize<<<std::max(g, 1), 256, 0, s>>>(packed, A, cnt, sum, mean, st, en));
    return PM4G_OK;
}

// R20: per-edge min / max of the pair duration, 0 where the edge never occurs
__global__ void k_finalize_minmax(const uint64_t* __restrict__ packed, const uint64_t* __restrict__ mm,
                                  uint32_t A, uint64_t* dmin, uint64_t* dmax) {
    const size_t AA = (size_t)A * A;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < AA; e += (size_t)gridDim.x * blockDim.x) {
        const bool any = packed[e] != 0;
        if (dmin) dmin[e] = any ? mm[e] : 0;
        if (dmax) dmax[e] = any ? mm[AA + e] : 0;
    }
}

static pm4g_status finalize_minmax(const uint64_t* packed, const uint64_t* mm, uint32_t A, uint64_t* dmin,
                                   uint64_t* dmax, cudaStream_t s) {
    const size_t AA = (size_t)A * A;
    const int g = (int)std::min<size_t>((AA + 255) / 256, (size_t)num_sms() * 4);
    PM4G_LAUNCH("k_finalize_minmax", AA * 8.0 * 5, s,
                k_finalize_minmax<<<std::max(g, 1), 256, 0, s>>>(packed, mm, A, dmin, dmax));
    return PM4G_OK;
}

// [min A2 | max A2] initial values: min = ~0, max = 0
static pm4g_status init_minmax(uint64_t* mm, uint32_t A, cudaStream_t s) {
    const size_t AA = (size_t)A * A;
    PM4G_CK(cudaMemsetAsync(mm, 0xff, AA * 8, s));
    PM4G_CK(cudaMemsetAsync(mm + AA, 0, AA * 8, s));
    return PM4G_OK;
}

static pm4g_status reduce_minmax(pm4g_comm* comm, uint64_t* mm, uint32_t A, cudaStream_t s) {
    const size_t AA = (size_t)A * A;
    PM4G_TRY(comm_allreduce_u64_op(comm, mm, AA, COMM_MIN, s));
    return comm_allreduce_u64_op(comm, mm + AA, AA, COMM_MAX, s);
}

static pm4g_status require_sorted(const pm4g_log* L) {
    PM4G_TRY(check_log(L));
    if (!L->sorted) return fail(PM4G_EINVAL, "log is not sorted (call pm4g_sort first)");
    return PM4G_OK;
}

static size_t packed_len(uint32_t A) { return 2 * (size_t)A * A + 2 * (size_t)A; }

// edge ids a * A + b are 32-bit on the device
static pm4g_status check_table_size(const pm4g_log* L) {
    if ((uint64_t)L->A * L->A > 0xffffffffull)
        return fail(PM4G_EINVAL, "n_activities too large for an A x A table (A^2 must fit 32 bits)");
    return PM4G_OK;
}

static pm4g_status tables_into(const pm4g_log* L, uint64_t* packed, cudaStream_t s) {
    PM4G_TRY(check_table_size(L));
    PM4G_CK(cudaMemsetAsync(packed, 0, packed_len(L->A) * 8, s));
    AggOut o;
    o.packed = packed;
    o.tables = true;
    return aggregate(L, o, s);
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_tables_partial(const pm4g_log* L, uint64_t* packed, pm4g_stream_t stream) {
    PM4G_TRY(require_sorted(L));
    if (!packed) return fail(PM4G_EINVAL, "null packed buffer");
    return tables_into(L, packed, (cudaStream_t)stream);
}

pm4g_status pm4g_tables_finalize(const uint64_t* packed, uint32_t A, uint64_t* cnt,
                                 int64_t* dur_sum, double* mean, uint64_t* start, uint64_t* end,
                                 pm4g_stream_t stream) {
    if (!packed || A == 0) return fail(PM4G_EINVAL, "bad arguments");
    return finalize_tables(packed, A, cnt, dur_sum, mean, start, end, (cudaStream_t)stream);
}

pm4g_status pm4g_dfg(const pm4g_log* L, uint64_t* cnt, int64_t* dur_sum, double* mean,
                     pm4g_comm* comm, pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_dfg");
    PM4G_TRY(require_sorted(L));
    if (!cnt || !dur_sum) return fail(PM4G_EINVAL, "cnt and dur_sum are required");
    cudaStream_t s = (cudaStream_t)stream;
    PM4G_TRY(check_table_size(L));
    Scratch pk(s);
    PM4G_TRY(pk.alloc(packed_len(L->A) * 8));
    PM4G_TRY(tables_into(L, pk.as<uint64_t>(), s));
    if (comm) PM4G_TRY(comm_allreduce_u64(comm, pk.as<uint64_t>(), packed_len(L->A), s));
    return finalize_tables(pk.as<uint64_t>(), L->A, cnt, dur_sum, mean, nullptr, nullptr, s);
}

pm4g_status pm4g_case_capacity(const pm4g_log* L, uint64_t* capacity) {
    if (!L || !capacity) return fail(PM4G_EINVAL, "null argument");
    *capacity = L->n > 0 ? std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1) : 0;
    return PM4G_OK;
}

pm4g_status pm4g_dfg_minmax(const pm4g_log* L, uint64_t* dur_min, uint64_t* dur_max, pm4g_comm* comm,
                            pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_dfg_minmax");
    PM4G_TRY(require_sorted(L));
    if (!dur_min && !dur_max) return fail(PM4G_EINVAL, "dur_min or dur_max is required");
    PM4G_TRY(check_table_size(L));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t AA = (size_t)L->A * L->A;
    Scratch pk(s), mm(s);
    PM4G_TRY(pk.alloc(packed_len(L->A) * 8));
    PM4G_TRY(mm.alloc(2 * AA * 8));
    PM4G_CK(cudaMemsetAsync(pk.p, 0, packed_len(L->A) * 8, s));
    PM4G_TRY(init_minmax(mm.as<uint64_t>(), L->A, s));
    AggOut o;
    o.packed = pk.as<uint64_t>();
    o.mm = mm.as<uint64_t>();
    o.tables = true;
    PM4G_TRY(aggregate(L, o, s));
    if (comm) {
        PM4G_TRY(comm_allreduce_u64(comm, pk.as<uint64_t>(), AA, s));   // counts decide empty edges
        PM4G_TRY(reduce_minmax(comm, mm.as<uint64_t>(), L->A, s));
    }
    return finalize_minmax(pk.as<uint64_t>(), mm.as<uint64_t>(), L->A, dur_min, dur_max, s);
}

pm4g_status pm4g_start_end(const pm4g_log* L, uint64_t* start, uint64_t* end, pm4g_comm* comm,
                           pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_start_end");
    PM4G_TRY(require_sorted(L));
    if (!start || !end) return fail(PM4G_EINVAL, "start and end are required");
    cudaStream_t s = (cudaStream_t)stream;
    PM4G_TRY(check_table_size(L));
    Scratch pk(s);
    PM4G_TRY(pk.alloc(packed_len(L->A) * 8));
    PM4G_TRY(tables_into(L, pk.as<uint64_t>(), s));
    if (comm) PM4G_TRY(comm_allreduce_u64(comm, pk.as<uint64_t>(), packed_len(L->A), s));
    return finalize_tables(pk.as<uint64_t>(), L->A, nullptr, nullptr, nullptr, start, end, s);
}

pm4g_status pm4g_case_durations(const pm4g_log* L, uint32_t* case_code, uint32_t* n_events,
                                int64_t* dur, uint64_t capacity, uint64_t* n_cases_out,
                                pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_case_durations");
    PM4G_TRY(require_sorted(L));
    cudaStream_t s = (cudaStream_t)stream;
    PM4G_TRY(fetch_n_cases(L, s));
    if (n_cases_out) *n_cases_out = (uint64_t)L->n_cases;
    if ((case_code || n_events || dur) && capacity < (uint64_t)L->n_cases)
        return fail(PM4G_EINVAL, "capacity < n_cases");
    if (L->n_cases == 0) return PM4G_OK;
    if (case_code)
        PM4G_CK(cudaMemcpyAsync(case_code, L->s_case_code, L->n_cases * 4, cudaMemcpyDeviceToDevice, s));
    if (n_events || dur) {
        AggOut o;
        o.n_events = n_events;
        o.dur = dur;
        PM4G_TRY(aggregate(L, o, s));
    }
    return PM4G_OK;
}

pm4g_status pm4g_variants(const pm4g_log* L, pm4g_comm* comm, pm4g_stream_t stream,
                          pm4g_variant_table** out) {
    PM4G_NVTX("pm4g_variants");
    PM4G_TRY(require_sorted(L));
    if (!out) return fail(PM4G_EINVAL, "null out");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t cap = std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1);
    Scratch keys(s);
    PM4G_TRY(keys.alloc(std::max<uint64_t>(cap, 1) * 16));
    AggOut o;
    o.k1 = keys.as<uint64_t>();
    o.k2 = o.k1 + std::max<uint64_t>(cap, 1);
    PM4G_TRY(aggregate(L, o, s));
    pm4g_variant_table* local = nullptr;
    PM4G_TRY(variants_from_keys(L, o.k1, o.k2, s, &local));
    if (!comm) {
        *out = local;
        return PM4G_OK;
    }
    pm4g_status st = comm_variants_allgather_merge(comm, local, s, out);
    free_variants(local);
    return st;
}

pm4g_status pm4g_analyze(const pm4g_log* L, const pm4g_outputs* out, pm4g_comm* comm,
                         pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_analyze");
    PM4G_TRY(require_sorted(L));
    if (!out) return fail(PM4G_EINVAL, "null outputs");
    cudaStream_t s = (cudaStream_t)stream;
    const bool want_tables = out->cnt || out->dur_sum || out->mean || out->start || out->end;
    const bool want_cases = out->case_code || out->n_events || out->dur;
    uint64_t cap = std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1);
    // capacity >= the host-known bound on n_cases: no need to wait for the count
    if (want_cases && out->capacity < cap) {
        PM4G_TRY(fetch_n_cases(L, s));
        if (out->capacity < (uint64_t)L->n_cases) return fail(PM4G_EINVAL, "capacity < n_cases");
    }
    Scratch pk(s), keys(s), mm(s);
    AggOut o;
    const bool want_mm = out->dur_min || out->dur_max;
    if (want_tables || want_mm) {
        PM4G_TRY(check_table_size(L));
        PM4G_TRY(pk.alloc(packed_len(L->A) * 8));
        PM4G_CK(cudaMemsetAsync(pk.p, 0, packed_len(L->A) * 8, s));
        o.packed = pk.as<uint64_t>();
        o.tables = true;
    }
    if (want_mm) {
        PM4G_TRY(mm.alloc(2 * (size_t)L->A * L->A * 8));
        PM4G_TRY(init_minmax(mm.as<uint64_t>(), L->A, s));
        o.mm = mm.as<uint64_t>();
    }
    o.n_events = out->n_events;
    o.dur = out->dur;
    o.case_code = out->case_code;
    if (out->variants) {
        PM4G_TRY(keys.alloc(std::max<uint64_t>(cap, 1) * 16));
        o.k1 = keys.as<uint64_t>();
        o.k2 = o.k1 + std::max<uint64_t>(cap, 1);
    }
    PM4G_TRY(aggregate(L, o, s));
    if (t_pending_format) {   // pm4g_sort_analyze: the format's fallback count, now past the aggregate
        PM4G_TRY(sort_defer_copy(t_pending_format, s));
        t_pending_format = nullptr;
    }
    if (want_tables || want_mm) {
        if (comm) PM4G_TRY(comm_allreduce_u64(comm, o.packed, packed_len(L->A), s));
        PM4G_TRY(finalize_tables(o.packed, L->A, out->cnt, out->dur_sum, out->mean, out->start,
                                 out->end, s));
    }
    if (want_mm) {
        if (comm) PM4G_TRY(reduce_minmax(comm, o.mm, L->A, s));
        PM4G_TRY(finalize_minmax(o.packed, o.mm, L->A, out->dur_min, out->dur_max, s));
    }
    if (out->variants) {
        *out->variants = nullptr;
        pm4g_variant_table* local = nullptr;
        PM4G_TRY(variants_from_keys(L, o.k1, o.k2, s, &local));
        if (!comm) {
            *out->variants = local;
        } else {
            pm4g_status st = comm_variants_allgather_merge(comm, local, s, out->variants);
            free_variants(local);
            PM4G_TRY(st);
        }
    }
    return PM4G_OK;
}

}  // extern "C"
