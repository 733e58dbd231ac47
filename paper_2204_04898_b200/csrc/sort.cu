// A2-A4: composite-key build, stable LSD radix sort (onesweep), case segments.
//
// P:108 "The dataframe is ordered based on three criteria (in order, case
// identifier, the timestamp, and the absolute index of the event in the
// dataframe)".  Reading R1/R2: case order = dictionary code, ties = ingest index.
// We sort the composite key  key = ((case - case_min) << ts_bits) | (ts - ts_min)
// with a STABLE least-significant-digit radix sort, so equal keys keep
// ingest order: stability realises the third criterion without storing it.
//
// Design (B200): 8-bit digits; one up-front kernel reads (case, ts) once and
// builds the histograms of every digit; each pass is one "onesweep" kernel
// (tiles of 4096 keys, tile ids from an atomic counter, per-digit decoupled
// look-back over the tile status array, local ranking with __match_any_sync
// warp aggregation, smem staging so the scatter writes runs of equal digits).
// The first pass reads the raw columns and builds the key on the fly, so the
// key is never written unsorted.  HBM bytes per event (act u8, P passes):
// hist 12 + pass0 (13 read + 9 write) + (P-1) * 18.
#include <cuda_runtime.h>

#include <algorithm>

#include "pm4g_internal.cuh"

namespace pm4g {

constexpr int RADIX = 256;
constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int SORT_IPT = 16;
constexpr int SORT_TILE = SORT_THREADS * SORT_IPT;  // 4096
constexpr int MAX_PASSES = 8;

struct KeyParams {
    uint32_t case_min;
    int64_t ts_min;
    int ts_bits;
};

__device__ __forceinline__ uint64_t make_key(uint32_t c, int64_t t, const KeyParams& kp) {
    uint64_t cr = (uint64_t)(c - kp.case_min);
    uint64_t tr = (uint64_t)t - (uint64_t)kp.ts_min;
    return (kp.ts_bits >= 64 ? 0 : (cr << kp.ts_bits)) | tr;
}

// ------------------------------------------------------------------ histograms
template <bool FROM_COLS>
__global__ __launch_bounds__(256) void k_hist(const uint64_t* __restrict__ keys,
                                              const uint32_t* __restrict__ cs,
                                              const int64_t* __restrict__ ts, int64_t n,
                                              KeyParams kp, int passes, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[MAX_PASSES][RADIX];
    for (int i = threadIdx.x; i < MAX_PASSES * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = FROM_COLS ? make_key(cs[i], ts[i], kp) : keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * RADIX; i += blockDim.x) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// exclusive scan of each pass's 256 bins (one block of 256 threads)
__global__ void k_hist_scan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ off,
                            int passes) {
    __shared__ uint32_t sw[SORT_WARPS + 1];
    for (int p = 0; p < passes; ++p) {
        uint32_t v = hist[p * RADIX + threadIdx.x];
        uint32_t e = block_excl_scan<RADIX>(v, sw, nullptr);
        off[p * RADIX + threadIdx.x] = e;
        __syncthreads();
    }
}

// ------------------------------------------------------------------ one onesweep pass
template <class P, bool FROM_COLS, bool WITH_IDX>
struct PassArgs {
    const uint64_t* in_key;
    const uint32_t* in_case;
    const int64_t* in_ts;
    const P* in_act;
    const uint32_t* in_idx;
    uint64_t* out_key;
    P* out_act;
    uint32_t* out_idx;
    int64_t n;
    int shift;
    const uint32_t* bucket_off;  // [256]
    uint32_t* status;            // [tiles * 256]
    uint32_t* tile_counter;
    KeyParams kp;
};

template <class P, bool FROM_COLS, bool WITH_IDX>
__global__ __launch_bounds__(SORT_THREADS) void k_onesweep(PassArgs<P, FROM_COLS, WITH_IDX> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* s_key = (uint64_t*)smem;
    P* s_act = (P*)(smem + SORT_TILE * 8);
    uint32_t* s_idx = (uint32_t*)(smem + SORT_TILE * 8 + SORT_TILE * sizeof(P));
    __shared__ uint32_t s_whist[SORT_WARPS][RADIX];
    __shared__ uint32_t s_start[RADIX];
    __shared__ long long s_gbase[RADIX];
    __shared__ uint32_t s_scan[SORT_WARPS + 1];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    for (int i = tid; i < SORT_WARPS * RADIX; i += SORT_THREADS) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * SORT_TILE;
    const int64_t wbase = base + warp * (32 * SORT_IPT);

    uint64_t k[SORT_IPT];
    P v[SORT_IPT];
    uint32_t ix[SORT_IPT];
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        int64_t i = wbase + j * 32 + lane;
        bool ok = i < a.n;
        if (FROM_COLS) {
            k[j] = ok ? make_key(a.in_case[i], a.in_ts[i], a.kp) : ~0ull;
            if (WITH_IDX) ix[j] = (uint32_t)i;
        } else {
            k[j] = ok ? a.in_key[i] : ~0ull;
            if (WITH_IDX) ix[j] = ok ? a.in_idx[i] : 0u;
        }
        v[j] = ok ? a.in_act[i] : (P)0;
    }

    // ---- stable local rank: warp-striped order (warp, j, lane) == index order.
    // Peers (lanes holding the same digit) come from 8 ballots, one per digit
    // bit: cheaper than MATCH.ANY, whose latency serialised the first version.
    uint32_t rank[SORT_IPT];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        uint32_t d = (uint32_t)(k[j] >> a.shift) & 0xffu;
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const bool bit = (d >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
        int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (lane == leader) {
            b = s_whist[warp][d];
            s_whist[warp][d] = b + __popc(peers);
        }
        b = __shfl_sync(0xffffffffu, b, leader);
        rank[j] = b + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // ---- per-digit totals, warp-exclusive prefixes (thread == digit)
    const int d = tid;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < SORT_WARPS; ++w) {
        uint32_t c = s_whist[w][d];
        s_whist[w][d] = tot;
        tot += c;
    }
    // invalid items (past n, only in the last tile) carry digit 255 of ~0 and
    // rank last; they are not part of the published counts.
    int64_t nvalid64 = a.n - base;
    const uint32_t nvalid = (uint32_t)(nvalid64 < SORT_TILE ? nvalid64 : SORT_TILE);
    uint32_t pub = tot;
    if (d == (int)((~0ull >> a.shift) & 0xffu)) pub -= (SORT_TILE - nvalid);
    uint32_t* st = a.status + (size_t)tile * RADIX + d;
    if (tile == 0) st_volatile(st, ST_INC | pub);
    else st_volatile(st, ST_AGG | pub);

    uint32_t start = block_excl_scan<SORT_THREADS>(tot, s_scan, nullptr);
    s_start[d] = start;

    // ---- decoupled look-back for this digit
    // batched: 4 predecessors per round trip (tile 0 is always inclusive)
    uint32_t prefix = 0;
    if (tile > 0) {
        int64_t p = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = (p - q >= 0) ? ld_volatile(a.status + (size_t)(p - q) * RADIX + d) : ST_INC;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (done) break;
                while ((w[q] >> 30) == 0) w[q] = ld_volatile(a.status + (size_t)(p - q) * RADIX + d);
                prefix += w[q] & ST_VAL;
                if ((w[q] >> 30) == 2) done = true;
            }
            p -= 4;
        }
        st_volatile(st, ST_INC | (prefix + pub));
    }
    s_gbase[d] = (long long)a.bucket_off[d] + prefix - start;
    __syncthreads();

    // ---- scatter into smem in digit order
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        uint32_t dd = (uint32_t)(k[j] >> a.shift) & 0xffu;
        uint32_t pos = s_start[dd] + s_whist[warp][dd] + rank[j];
        s_key[pos] = k[j];
        s_act[pos] = v[j];
        if (WITH_IDX) s_idx[pos] = ix[j];
    }
    __syncthreads();

    // ---- coalesced write-out: consecutive threads, consecutive positions
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        uint32_t sidx = j * SORT_THREADS + tid;
        if (sidx < nvalid) {
            uint64_t kk = s_key[sidx];
            uint32_t dd = (uint32_t)(kk >> a.shift) & 0xffu;
            long long g = s_gbase[dd] + sidx;
            a.out_key[g] = kk;
            a.out_act[g] = s_act[sidx];
            if (WITH_IDX) a.out_idx[g] = s_idx[sidx];
        }
    }
}

template <class P, bool FC, bool WI>
static pm4g_status launch_pass(const PassArgs<P, FC, WI>& args, int64_t tiles, cudaStream_t s,
                               const char* name, double bytes) {
    size_t smem = (size_t)SORT_TILE * (8 + sizeof(P) + (WI ? 4 : 0));
    static bool attr = false;
    if (!attr) {
        PM4G_CK(cudaFuncSetAttribute(k_onesweep<P, FC, WI>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    PM4G_LAUNCH(name, bytes, s, k_onesweep<P, FC, WI><<<(unsigned)tiles, SORT_THREADS, smem, s>>>(args));
    return PM4G_OK;
}

// LSD sort of (key, act[, idx]).  FROM_COLS first pass builds keys from (case, ts).
template <class P, bool WI>
static pm4g_status lsd_sort(const uint32_t* cs, const int64_t* ts, const uint64_t* keys_in,
                            const P* act_in, const uint32_t* idx_in, uint64_t* key_out,
                            P* act_out, uint32_t* idx_out, int64_t n, int passes, KeyParams kp,
                            cudaStream_t s) {
    const bool from_cols = (keys_in == nullptr);
    passes = std::max(1, std::min(passes, MAX_PASSES));
    const int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
    Scratch aux(s), tmp(s);
    size_t status_words = (size_t)tiles * RADIX * passes;
    size_t aux_bytes = (status_words + passes /*counters*/ + 2 * MAX_PASSES * RADIX) * 4;
    PM4G_TRY(aux.alloc(aux_bytes));
    uint32_t* status = aux.as<uint32_t>();
    uint32_t* counters = status + status_words;
    uint32_t* hist = counters + passes;
    uint32_t* off = hist + MAX_PASSES * RADIX;
    PM4G_CK(cudaMemsetAsync(status, 0, (status_words + passes + MAX_PASSES * RADIX) * 4, s));
    {
        int g = std::max(1, std::min<int>((int)((n + 255) / 256), num_sms() * 4));
        double bytes = (double)n * (from_cols ? 12 : 8);
        if (from_cols)
            PM4G_LAUNCH("k_hist", bytes, s, k_hist<true><<<g, 256, 0, s>>>(nullptr, cs, ts, n, kp, passes, hist));
        else
            PM4G_LAUNCH("k_hist", bytes, s, k_hist<false><<<g, 256, 0, s>>>(keys_in, nullptr, nullptr, n, kp, passes, hist));
        PM4G_LAUNCH("k_hist_scan", 0, s, k_hist_scan<<<1, RADIX, 0, s>>>(hist, off, passes));
    }
    // ping-pong so that the last pass lands in the output buffers
    const size_t per = (size_t)n * (8 + sizeof(P) + (WI ? 4 : 0));
    PM4G_TRY(tmp.alloc(per));
    // layout keeps every array naturally aligned: keys (8n) | idx (4n) | act
    uint64_t* tkey = tmp.as<uint64_t>();
    uint32_t* tidx = (uint32_t*)((char*)tmp.p + (size_t)n * 8);
    P* tact = (P*)((char*)tmp.p + (size_t)n * (8 + (WI ? 4 : 0)));
    const uint64_t* ck = keys_in;
    const P* ca = act_in;
    const uint32_t* ci = idx_in;
    for (int p = 0; p < passes; ++p) {
        bool to_out = ((passes - 1 - p) % 2) == 0;
        uint64_t* ok = to_out ? key_out : tkey;
        P* oa = to_out ? act_out : tact;
        uint32_t* oi = to_out ? idx_out : tidx;
        double rd = (p == 0 && from_cols) ? 12.0 + sizeof(P) : 8.0 + sizeof(P) + (WI ? 4 : 0);
        double bytes = (double)n * (rd + 8 + sizeof(P) + (WI ? 4 : 0));
        if (p == 0 && from_cols) {
            PassArgs<P, true, WI> a{nullptr, cs, ts, act_in, nullptr, ok, oa, oi, n, 0,
                                    off, status, counters, kp};
            PM4G_TRY(launch_pass(a, tiles, s, "k_onesweep", bytes));
        } else {
            PassArgs<P, false, WI> a{ck, nullptr, nullptr, ca, ci, ok, oa, oi, n, 8 * p,
                                     off + p * RADIX, status + (size_t)p * tiles * RADIX,
                                     counters + p, kp};
            PM4G_TRY(launch_pass(a, tiles, s, "k_onesweep", bytes));
        }
        ck = ok;
        ca = oa;
        ci = oi;
    }
    return PM4G_OK;
}

// ------------------------------------------------------------------ A4 segments
// flag[i] = (i == 0) || case(i) != case(i-1) ("the different groups are
// identified ... as the set of rows indices"); heads compacted in order give
// the CSR offsets of the cases dataframe.
constexpr int SEG_THREADS = 256, SEG_IPT = 16, SEG_TILE = SEG_THREADS * SEG_IPT;

__global__ __launch_bounds__(SEG_THREADS) void k_segments(const uint64_t* __restrict__ key,
                                                          int64_t n, int ts_bits, uint32_t case_min,
                                                          uint32_t* __restrict__ off,
                                                          uint32_t* __restrict__ case_code,
                                                          uint64_t* __restrict__ n_cases,
                                                          uint32_t* status, uint32_t* counter) {
    __shared__ uint32_t s_tile, s_warp_tot[SEG_THREADS / 32], s_scan[SEG_THREADS / 32 + 1];
    __shared__ uint32_t s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wbase = (int64_t)tile * SEG_TILE + warp * (32 * SEG_IPT);
    const uint32_t lt = lanemask_lt();
    uint32_t ballots[SEG_IPT];
    uint64_t cs[SEG_IPT];
    uint64_t prev_last = 0;
    {
        int64_t pi = wbase - 1;
        if (pi >= 0 && pi < n) prev_last = shr64(key[pi], ts_bits);
    }
    uint32_t wcount = 0;
#pragma unroll
    for (int j = 0; j < SEG_IPT; ++j) {
        int64_t i = wbase + j * 32 + lane;
        bool ok = i < n;
        uint64_t c = ok ? shr64(key[i], ts_bits) : 0;
        uint64_t pc = __shfl_up_sync(0xffffffffu, c, 1);
        if (lane == 0) pc = prev_last;
        prev_last = __shfl_sync(0xffffffffu, c, 31);
        bool head = ok && (i == 0 || c != pc);
        uint32_t b = __ballot_sync(0xffffffffu, head);
        ballots[j] = b;
        cs[j] = c;
        wcount += __popc(b);
    }
    if (lane == 0) s_warp_tot[warp] = wcount;
    __syncthreads();
    uint32_t wt = tid < SEG_THREADS / 32 ? s_warp_tot[tid] : 0;
    uint32_t total;
    uint32_t wex = block_excl_scan<SEG_THREADS>(wt, s_scan, &total);
    if (tid < SEG_THREADS / 32) s_warp_tot[tid] = wex;
    if (warp == 0) {
        uint32_t pf = lookback_warp(status, tile, total);
        if (lane == 0) s_prefix = pf;
    }
    __syncthreads();
    uint32_t r = s_prefix + s_warp_tot[warp];
#pragma unroll
    for (int j = 0; j < SEG_IPT; ++j) {
        int64_t i = wbase + j * 32 + lane;
        uint32_t b = ballots[j];
        if (b & (1u << lane)) {
            uint32_t rk = r + __popc(b & lt);
            off[rk] = (uint32_t)i;
            case_code[rk] = case_min + (uint32_t)cs[j];
        }
        r += __popc(b);
    }
    // the last tile closes the CSR and publishes n_cases
    if (tid == 0 && (int64_t)(tile + 1) * SEG_TILE >= n) {
        off[s_prefix + total] = (uint32_t)n;
        *n_cases = s_prefix + total;
    }
}

__global__ void k_zero_cases(uint32_t* off, uint64_t* n_cases) {
    off[0] = 0;
    *n_cases = 0;
}

pm4g_status segments(pm4g_log* L, cudaStream_t s) {
    const int64_t n = L->n;
    dfree(L->off, s);
    dfree(L->s_case_code, s);
    L->off = nullptr;
    L->s_case_code = nullptr;
    L->n_cases = -1;
    // number of cases <= min(n, case range)
    uint64_t cap = std::min<uint64_t>((uint64_t)n, (uint64_t)(L->case_max - L->case_min) + 1);
    PM4G_TRY(dalloc_t(&L->off, cap + 1, s));
    PM4G_TRY(dalloc_t(&L->s_case_code, std::max<uint64_t>(cap, 1), s));
    if (n == 0) {
        PM4G_LAUNCH("k_zero_cases", 0, s, k_zero_cases<<<1, 1, 0, s>>>(L->off, L->d_n_cases));
        L->n_cases = 0;
        return PM4G_OK;
    }
    const int64_t tiles = (n + SEG_TILE - 1) / SEG_TILE;
    Scratch st(s);
    PM4G_TRY(st.alloc((tiles + 1) * 4));
    PM4G_CK(cudaMemsetAsync(st.p, 0, (tiles + 1) * 4, s));
    uint32_t* status = st.as<uint32_t>();
    PM4G_LAUNCH("k_segments", n * 8.0, s,
                k_segments<<<(unsigned)tiles, SEG_THREADS, 0, s>>>(L->key, n, L->ts_bits, L->case_min,
                                                                  L->off, L->s_case_code,
                                                                  L->d_n_cases, status + 1, status));
    return PM4G_OK;
}

// ------------------------------------------------------------------ extra-column gather
template <class T>
__global__ void k_gather(const T* __restrict__ in, const uint32_t* __restrict__ perm, T* __restrict__ out,
                         int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}

static pm4g_status gather_extras(pm4g_log* L, cudaStream_t s) {
    const int64_t n = L->n;
    int g = std::max(1, std::min<int>((int)((n + 255) / 256), num_sms() * 8));
    for (auto& x : L->extra) {
        void* nd = nullptr;
        uint8_t* nv = nullptr;
        PM4G_TRY(dalloc(&nd, n * x.elem, s));
        if (n) {
            if (x.elem == 4)
                PM4G_LAUNCH("k_gather", n * 12.0, s, k_gather<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)x.data, L->perm, (uint32_t*)nd, n));
            else
                PM4G_LAUNCH("k_gather", n * 20.0, s, k_gather<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)x.data, L->perm, (uint64_t*)nd, n));
        }
        if (x.valid) {
            PM4G_TRY(dalloc((void**)&nv, n, s));
            if (n) PM4G_LAUNCH("k_gather", n * 9.0, s, k_gather<uint8_t><<<g, 256, 0, s>>>(x.valid, L->perm, nv, n));
        }
        if (x.owned) {
            dfree(x.data, s);
            dfree(x.valid, s);
        }
        x.data = nd;
        x.valid = nv;
        x.owned = true;
    }
    return PM4G_OK;
}

pm4g_status sort_log(pm4g_log* L, cudaStream_t s) {
    const int64_t n = L->n;
    const bool wi = !L->extra.empty();
    PM4G_TRY(dalloc_t(&L->key, std::max<int64_t>(n, 1), s));
    PM4G_TRY(dalloc(&L->s_act, std::max<int64_t>(n, 1) * L->act_bytes, s));
    if (wi) PM4G_TRY(dalloc_t(&L->perm, std::max<int64_t>(n, 1), s));
    if (n == 0) return PM4G_OK;
    KeyParams kp{L->case_min, L->ts_min, L->ts_bits};
    int passes = std::max(1, L->passes);
#define PM4G_SORT_CASE(P)                                                                  \
    if (wi)                                                                                \
        PM4G_TRY((lsd_sort<P, true>(L->case_, L->ts, nullptr, (const P*)L->act, nullptr,   \
                                    L->key, (P*)L->s_act, L->perm, n, passes, kp, s)));    \
    else                                                                                   \
        PM4G_TRY((lsd_sort<P, false>(L->case_, L->ts, nullptr, (const P*)L->act, nullptr,  \
                                     L->key, (P*)L->s_act, nullptr, n, passes, kp, s)));
    switch (L->act_bytes) {
        case 1: PM4G_SORT_CASE(uint8_t) break;
        case 2: PM4G_SORT_CASE(uint16_t) break;
        default: PM4G_SORT_CASE(uint32_t) break;
    }
#undef PM4G_SORT_CASE
    if (wi) PM4G_TRY(gather_extras(L, s));
    return PM4G_OK;
}

// generic (u64 key, u32 value) sort on `bits` low key bits, result in place
pm4g_status radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits, cudaStream_t s) {
    if (n <= 1) return PM4G_OK;
    int passes = std::max(1, (std::min(bits, 64) + 7) / 8);
    Scratch out(s);
    PM4G_TRY(out.alloc((size_t)n * 12));
    uint64_t* ok = out.as<uint64_t>();
    uint32_t* ov = (uint32_t*)((char*)out.p + (size_t)n * 8);
    KeyParams kp{0, 0, 0};
    PM4G_TRY((lsd_sort<uint32_t, false>(nullptr, nullptr, keys, vals, nullptr, ok, ov, nullptr, n,
                                        passes, kp, s)));
    PM4G_CK(cudaMemcpyAsync(keys, ok, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    PM4G_CK(cudaMemcpyAsync(vals, ov, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    return PM4G_OK;
}

// ------------------------------------------------------------------ decode (formatted log view)
template <class P>
__global__ void k_decode(const uint64_t* __restrict__ key, const P* __restrict__ sact, int64_t n,
                         int ts_bits, uint32_t case_min, int64_t ts_min, uint32_t* __restrict__ oc,
                         uint32_t* __restrict__ oa, int64_t* __restrict__ ot) {
    const uint64_t m = low_mask(ts_bits);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[i];
        if (oc) oc[i] = case_min + (uint32_t)shr64(k, ts_bits);
        if (oa) oa[i] = (uint32_t)sact[i];
        if (ot) ot[i] = (int64_t)((uint64_t)ts_min + (k & m));
    }
}

}  // namespace pm4g

using namespace pm4g;

extern "C" pm4g_status pm4g_sorted_columns(const pm4g_log* L, uint32_t* case_code, uint32_t* act,
                                           int64_t* ts, pm4g_stream_t stream) {
    if (!L) return fail(PM4G_EINVAL, "null log");
    if (!L->sorted) return fail(PM4G_EINVAL, "log is not sorted (call pm4g_sort)");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = L->n;
    if (n == 0) return PM4G_OK;
    int g = std::max(1, std::min<int>((int)((n + 255) / 256), num_sms() * 8));
    switch (L->act_bytes) {
        case 1: PM4G_LAUNCH("k_decode", n * 25.0, s, k_decode<uint8_t><<<g, 256, 0, s>>>(L->key, (const uint8_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
        case 2: PM4G_LAUNCH("k_decode", n * 26.0, s, k_decode<uint16_t><<<g, 256, 0, s>>>(L->key, (const uint16_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
        default: PM4G_LAUNCH("k_decode", n * 28.0, s, k_decode<uint32_t><<<g, 256, 0, s>>>(L->key, (const uint32_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
    }
    return PM4G_OK;
}
