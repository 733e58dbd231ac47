// A1 / A10: filters as stream compaction.
//
// P:126 (timestamp.py) "three different types of timestamp filtering (events,
// cases contained, cases intersecting)"; P:96-97, P:101, P:128 (attributes.py)
// event-level and case-level attribute filters.  Readings R12-R15.
//
// Each filter = (1) a predicate kernel writing a u8 keep mask (case-level
// predicates first reduce a per-case flag over a dense case-code range with
// global atomics -- no sort needed, so filters work on ingested and formatted
// logs alike), then (2) one stable compaction kernel (single pass, decoupled
// look-back, warp-striped so each warp's kept rows are written contiguously)
// that moves every column of the log.  Relative row order is preserved
// (S:483), so a formatted input stays formatted and only its case offsets are
// rebuilt.  On an ingested log the compaction of the core columns is one
// column-typed kernel that also evaluates the events-mode time predicate
// itself (no mask pass) and produces the output log's metadata and radix
// histograms (no second validation pass: the rows were validated when the
// parent log was created).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

// row accessor for both log states
struct RowView {
    const uint32_t* cs;      // ingested
    const int64_t* ts;       // ingested
    const uint64_t* key;     // formatted
    const uint32_t* rcase;   // formatted wide log: case - case_min per row
    int ts_bits;
    uint32_t case_min;
    int64_t ts_min;
    __device__ __forceinline__ uint32_t case_of(int64_t i) const {
        if (rcase) return case_min + rcase[i];
        return key ? case_min + (uint32_t)shr64(key[i], ts_bits) : cs[i];
    }
    __device__ __forceinline__ int64_t ts_of(int64_t i) const {
        return key ? (int64_t)((uint64_t)ts_min + (key[i] & low_mask(ts_bits))) : ts[i];
    }
};

static RowView view_of(const pm4g_log* L) {
    RowView v;
    v.cs = L->sorted ? nullptr : L->case_;
    v.ts = L->sorted ? nullptr : L->ts;
    v.key = L->sorted ? L->key : nullptr;
    v.rcase = L->sorted ? L->rcase : nullptr;
    v.ts_bits = L->ts_bits;
    v.case_min = L->case_min;
    v.ts_min = L->ts_min;
    return v;
}

static int gsz(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
}

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ predicates
__global__ void k_time_events(RowView v, int64_t n, int64_t t1, int64_t t2, uint8_t* keep) {
    GRID_LOOP(i, n) {
        int64_t t = v.ts_of(i);
        keep[i] = (t >= t1 && t <= t2) ? 1 : 0;
    }
}

__global__ void k_init_span(long long* lo, long long* hi, int64_t R) {
    GRID_LOOP(i, R) {
        lo[i] = LLONG_MAX;
        hi[i] = LLONG_MIN;
    }
}

__global__ void k_case_span(RowView v, int64_t n, long long* lo, long long* hi) {
    GRID_LOOP(i, n) {
        uint32_t c = v.case_of(i) - v.case_min;
        long long t = v.ts_of(i);
        atomicMin(&lo[c], t);
        atomicMax(&hi[c], t);
    }
}

// mode 1 contained: first >= t1 && last <= t2; mode 2 intersecting: first <= t2 && last >= t1
__global__ void k_time_cases(RowView v, int64_t n, const long long* lo, const long long* hi,
                             int64_t t1, int64_t t2, int mode, uint8_t* keep) {
    GRID_LOOP(i, n) {
        uint32_t c = v.case_of(i) - v.case_min;
        long long a = lo[c], b = hi[c];
        bool k = mode == 1 ? (a >= t1 && b <= t2) : (a <= t2 && b >= t1);
        keep[i] = k ? 1 : 0;
    }
}

// attribute match: codes in a sorted device set / i64 range / f64 range; nulls never match
struct AttrPred {
    int kind;
    const void* col;
    int col_bytes;              // for codes: element width (1, 2, 4)
    const uint8_t* valid;
    const uint32_t* set;
    int64_t nset;
    int64_t lo_i, hi_i;
    double lo_f, hi_f;
    __device__ __forceinline__ bool match(int64_t i) const {
        if (valid && !valid[i]) return false;
        if (kind == PM4G_PRED_IN_SET) {
            uint32_t x = col_bytes == 1 ? ((const uint8_t*)col)[i]
                       : col_bytes == 2 ? ((const uint16_t*)col)[i] : ((const uint32_t*)col)[i];
            int64_t a = 0, b = nset;
            while (a < b) {
                int64_t m = (a + b) >> 1;
                if (set[m] < x) a = m + 1; else b = m;
            }
            return a < nset && set[a] == x;
        }
        if (kind == PM4G_PRED_RANGE_I64) {
            int64_t x = ((const int64_t*)col)[i];
            return x >= lo_i && x <= hi_i;
        }
        double x = ((const double*)col)[i];
        return x >= lo_f && x <= hi_f;
    }
};

__global__ void k_attr_events(AttrPred p, int64_t n, int keep_match, uint8_t* keep) {
    GRID_LOOP(i, n) keep[i] = (p.match(i) == (keep_match != 0)) ? 1 : 0;
}
__global__ void k_attr_any(AttrPred p, RowView v, int64_t n, uint8_t* any) {
    GRID_LOOP(i, n) if (p.match(i)) any[v.case_of(i) - v.case_min] = 1;
}
__global__ void k_attr_cases(RowView v, int64_t n, const uint8_t* any, int keep_match, uint8_t* keep) {
    GRID_LOOP(i, n) keep[i] = ((any[v.case_of(i) - v.case_min] != 0) == (keep_match != 0)) ? 1 : 0;
}

// ------------------------------------------------------------------ stable compaction
// Two passes over tiles of CMP_TILE rows, no look-back: (1) count the kept
// rows of every tile (the keep mask, or the events-mode time predicate on the
// ts column), (2) exclusive scan of the tile counts, (3) scatter: each tile
// re-reads its rows and writes the kept ones at tile_off[t] + their in-tile
// rank (warp-striped, so each warp's kept rows land contiguously).  Every
// pass is embarrassingly parallel.  A single-pass decoupled-look-back
// compaction was measured latency-bound here (1.5 TB/s: each CTA serialises
// load -> look-back -> store), and prefetching tiles into a per-CTA ring
// makes the look-back chain convoy (a tile's aggregate waits for the tiles
// queued before it in its owner's ring).
constexpr int CMP_THREADS = 256, CMP_IPT = 8, CMP_TILE = CMP_THREADS * CMP_IPT, CMP_MAXCOL = 12;

struct ColSet {
    const void* in[CMP_MAXCOL];
    void* out[CMP_MAXCOL];
    int elem[CMP_MAXCOL];
    int ncol;
};

// keep predicate of row i: mask[i] != 0, or (TIME) t1 <= ts[i] <= t2
template <bool TIME>
__device__ __forceinline__ bool keep_row(const uint8_t* mask, const int64_t* ts, int64_t i, int64_t t1, int64_t t2) {
    if (TIME) {
        const int64_t t = ts[i];
        return t >= t1 && t <= t2;
    }
    return mask[i] != 0;
}

template <bool TIME>
__global__ __launch_bounds__(CMP_THREADS) void k_count_tiles(const uint8_t* __restrict__ mask,
                                                             const int64_t* __restrict__ ts, int64_t n,
                                                             int64_t t1, int64_t t2, uint32_t* __restrict__ cnt) {
    __shared__ uint32_t s_w[CMP_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * CMP_TILE;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < CMP_IPT; ++j) {
        const int64_t i = base + j * CMP_THREADS + threadIdx.x;
        c += (i < n && keep_row<TIME>(mask, ts, i, t1, t2)) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < CMP_THREADS / 32; ++w) t += s_w[w];
        cnt[blockIdx.x] = t;
    }
}

// In-tile ranks: ballots of the warp-striped rows and the warp's exclusive
// offset within the tile.  Rows: warp w, item j, lane l -> w*256 + j*32 + l.
template <bool TIME>
__device__ __forceinline__ uint32_t tile_ballots(const uint8_t* mask, const int64_t* ts, int64_t n, int64_t wbase,
                                                 int64_t t1, int64_t t2, uint32_t (&ball)[CMP_IPT],
                                                 uint32_t* s_wt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t wc = 0;
#pragma unroll
    for (int j = 0; j < CMP_IPT; ++j) {
        const int64_t i = wbase + j * 32 + lane;
        ball[j] = __ballot_sync(0xffffffffu, i < n && keep_row<TIME>(mask, ts, i, t1, t2));
        wc += __popc(ball[j]);
    }
    if (lane == 0) s_wt[warp] = wc;
    __syncthreads();
    uint32_t wex = 0;
#pragma unroll
    for (int w = 0; w < CMP_THREADS / 32; ++w) wex += w < warp ? s_wt[w] : 0u;
    return wex;
}

// generic columns (formatted logs, extra columns): per column all loads of the
// thread's rows first, then the stores
__global__ __launch_bounds__(CMP_THREADS) void k_compact_rows(const uint8_t* __restrict__ keep, int64_t n,
                                                              ColSet cols, const uint64_t* __restrict__ tile_off) {
    __shared__ uint32_t s_wt[CMP_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wbase = (int64_t)blockIdx.x * CMP_TILE + warp * (32 * CMP_IPT);
    uint32_t ball[CMP_IPT];
    const uint32_t wex = tile_ballots<false>(keep, nullptr, n, wbase, 0, 0, ball, s_wt);
    const uint32_t lt = lanemask_lt();
    uint64_t o[CMP_IPT];
    {
        uint64_t r = tile_off[blockIdx.x] + wex;
#pragma unroll
        for (int j = 0; j < CMP_IPT; ++j) {
            o[j] = r + __popc(ball[j] & lt);
            r += __popc(ball[j]);
        }
    }
    for (int c = 0; c < cols.ncol; ++c) {
        const int el = cols.elem[c];
        const void* in = cols.in[c];
        void* out = cols.out[c];
        uint64_t v[CMP_IPT];
#pragma unroll
        for (int j = 0; j < CMP_IPT; ++j) {
            const int64_t i = wbase + j * 32 + lane;
            v[j] = 0;
            if (ball[j] & (1u << lane)) {
                v[j] = el == 1 ? ((const uint8_t*)in)[i]
                     : el == 2 ? ((const uint16_t*)in)[i]
                     : el == 4 ? ((const uint32_t*)in)[i] : ((const uint64_t*)in)[i];
            }
        }
#pragma unroll
        for (int j = 0; j < CMP_IPT; ++j) {
            if (!(ball[j] & (1u << lane))) continue;
            if (el == 1) ((uint8_t*)out)[o[j]] = (uint8_t)v[j];
            else if (el == 2) ((uint16_t*)out)[o[j]] = (uint16_t)v[j];
            else if (el == 4) ((uint32_t*)out)[o[j]] = (uint32_t)v[j];
            else ((uint64_t*)out)[o[j]] = v[j];
        }
    }
}

struct FilterMeta {
    long long ts_min, ts_max;
    unsigned int case_min, case_max;
};

// Ingested log: scatter of (case, act, ts) plus the output log's metadata (ts /
// case ranges) and case-digit histograms of the kept rows, in the layout
// validate_and_meta uses (hist_layout) -- no second validation pass: the rows
// were validated when the parent log was created.  omask (optional) receives
// the keep mask for the extra columns' compaction.
//
// Persistent and warp-specialised: a producer warp streams the CTA's tiles
// (t = blockIdx.x + k gridDim.x) into a ring of FS_STAGES shared-memory stages
// with TMA bulk copies while 8 consumer warps rank and store the previous
// ones; output offsets come from the count pass (tile_off), so tiles are
// independent.  Without the ring each CTA serialises load -> rank -> store
// and the scatter is load-latency bound (~2 TB/s measured).
constexpr int FS_CONSUMERS = CMP_THREADS, FS_BLOCK = FS_CONSUMERS + 32, FS_STAGES = 3;

template <class P>
struct alignas(128) FsStage {
    int64_t ts[CMP_TILE];
    uint32_t cs[CMP_TILE];
    P act[CMP_TILE];
};

template <class P, bool TIME>
__global__ __launch_bounds__(FS_BLOCK) void k_filter_cols(
    const uint8_t* __restrict__ mask, const uint32_t* __restrict__ cs, const P* __restrict__ act,
    const int64_t* __restrict__ ts, int64_t n, int64_t t1, int64_t t2, const uint64_t* __restrict__ tile_off,
    uint32_t* __restrict__ ocs, P* __restrict__ oact, int64_t* __restrict__ ots, uint8_t* __restrict__ omask,
    FilterMeta* m, uint32_t case_lo, int hpasses, int hbits, uint32_t* __restrict__ hist, int tma_ok) {
    extern __shared__ __align__(128) unsigned char fs_sm[];
    FsStage<P>* stage = (FsStage<P>*)fs_sm;
    __shared__ __align__(8) uint64_t s_full[FS_STAGES], s_empty[FS_STAGES];
    __shared__ uint32_t sh[4][256];
    __shared__ uint32_t s_wt[2][FS_CONSUMERS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 4 * 256; i += FS_BLOCK) (&sh[0][0])[i] = 0;
    if (tid == 0) {
        for (int s = 0; s < FS_STAGES; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], FS_CONSUMERS);
        }
    }
    __syncthreads();
    const int64_t tiles = (n + CMP_TILE - 1) / CMP_TILE;
    // a tile is staged by TMA when it is whole and the columns are 16-byte aligned
    auto staged_tile = [&](int64_t t) { return tma_ok && (t + 1) * CMP_TILE <= n; };
    if (warp == 0) {
        if (lane == 0) {
            uint32_t i = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
                const int s = i % FS_STAGES;
                if (i >= FS_STAGES) mbar_wait(&s_empty[s], ((i / FS_STAGES) - 1) & 1);
                if (staged_tile(t)) {
                    FsStage<P>& st = stage[s];
                    const int64_t r0 = t * CMP_TILE;
                    mbar_expect_tx(&s_full[s], CMP_TILE * (8 + 4 + (uint32_t)sizeof(P)));
                    tma_load_1d(st.ts, ts + r0, CMP_TILE * 8, &s_full[s]);
                    tma_load_1d(st.cs, cs + r0, CMP_TILE * 4, &s_full[s]);
                    tma_load_1d(st.act, act + r0, CMP_TILE * (uint32_t)sizeof(P), &s_full[s]);
                } else {
                    mbar_arrive(&s_full[s]);   // tail tile: consumers read global memory
                }
            }
        }
    } else {
        const int ct = tid - 32, cw = ct >> 5;
        long long tmin = LLONG_MAX, tmax = LLONG_MIN;
        uint32_t cmin = 0xffffffffu, cmax = 0;
        const uint32_t hmask = (1u << hbits) - 1;
        const uint32_t lt = lanemask_lt();
        uint32_t i = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
            const int s = i % FS_STAGES;
            mbar_wait(&s_full[s], (i / FS_STAGES) & 1);
            const FsStage<P>& st = stage[s];
            const bool staged = staged_tile(t);
            const int64_t wbase = t * CMP_TILE + cw * (32 * CMP_IPT);
            uint32_t c[CMP_IPT], ball[CMP_IPT], wc = 0;
            int64_t tv[CMP_IPT];
            P a[CMP_IPT];
#pragma unroll
            for (int j = 0; j < CMP_IPT; ++j) {
                const int li = cw * (32 * CMP_IPT) + j * 32 + lane;
                const int64_t row = wbase + j * 32 + lane;
                const bool in = row < n;
                if (staged) {
                    c[j] = st.cs[li];
                    tv[j] = st.ts[li];
                    a[j] = st.act[li];
                } else {
                    c[j] = in ? cs[row] : 0u;
                    tv[j] = in ? ts[row] : 0;
                    a[j] = in ? act[row] : (P)0;
                }
            }
            mbar_arrive(&s_empty[s]);   // the stage is in registers now
#pragma unroll
            for (int j = 0; j < CMP_IPT; ++j) {
                const int64_t row = wbase + j * 32 + lane;
                const bool in = row < n;
                const bool k = in && (TIME ? (tv[j] >= t1 && tv[j] <= t2) : mask[row] != 0);
                if (omask && in) omask[row] = k ? 1 : 0;
                ball[j] = __ballot_sync(0xffffffffu, k);
                wc += __popc(ball[j]);
            }
            if (lane == 0) s_wt[i & 1][cw] = wc;
            asm volatile("bar.sync 1, %0;" ::"n"(FS_CONSUMERS) : "memory");
            uint32_t wex = 0;
#pragma unroll
            for (int w = 0; w < FS_CONSUMERS / 32; ++w) wex += w < cw ? s_wt[i & 1][w] : 0u;
            uint64_t r = tile_off[t] + wex;
#pragma unroll
            for (int j = 0; j < CMP_IPT; ++j) {
                if (ball[j] & (1u << lane)) {
                    const uint64_t o = r + __popc(ball[j] & lt);
                    ocs[o] = c[j];
                    oact[o] = a[j];
                    ots[o] = tv[j];
                    tmin = min(tmin, (long long)tv[j]);
                    tmax = max(tmax, (long long)tv[j]);
                    cmin = min(cmin, c[j]);
                    cmax = max(cmax, c[j]);
                    const uint32_t f = c[j] - case_lo;
                    for (int p = 0; p < hpasses; ++p) atomicAdd(&sh[p][(f >> (p * hbits)) & hmask], 1u);
                }
                r += __popc(ball[j]);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            tmin = min(tmin, __shfl_xor_sync(~0u, tmin, o));
            tmax = max(tmax, __shfl_xor_sync(~0u, tmax, o));
            cmin = min(cmin, __shfl_xor_sync(~0u, cmin, o));
            cmax = max(cmax, __shfl_xor_sync(~0u, cmax, o));
        }
        if (lane == 0 && tmin <= tmax) {
            atomicMin(&m->ts_min, tmin);
            atomicMax(&m->ts_max, tmax);
            atomicMin(&m->case_min, cmin);
            atomicMax(&m->case_max, cmax);
        }
    }
    __syncthreads();
    for (int i = tid; i < hpasses * 256; i += FS_BLOCK) {
        const uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// Time predicate for the fused path (events mode on an ingested log).
struct TimePred {
    int64_t t1, t2;
};

// Build the output log from the keep mask (or, with tp, from the events-mode
// time predicate on an ingested log's ts column).
static pm4g_status compact_log(const pm4g_log* in, const uint8_t* keep, cudaStream_t s,
                               pm4g_log** out, const TimePred* tp = nullptr) {
    const int64_t n = in->n;
    pm4g_log* L = new pm4g_log();
    L->A = in->A;
    L->act_bytes = in->act_bytes;
    L->n_case_codes = in->n_case_codes;
    L->case_lo = in->case_lo;
    L->case_hi = in->case_hi;
    L->stream = s;
    LogGuard guard(L);
    auto bail = [&](pm4g_status st) { return st; };   // the guard destroys L
    pm4g_status st;
    if ((st = dalloc((void**)&L->d_n_cases, 8, s))) return bail(st);
    const int64_t N = std::max<int64_t>(n, 1);
    ColSet cs{};
    auto add = [&](const void* i, void* o, int e) {
        cs.in[cs.ncol] = i;
        cs.out[cs.ncol] = o;
        cs.elem[cs.ncol] = e;
        cs.ncol++;
    };
    const bool fused = !in->sorted;
    if (!fused) {
        if ((st = dalloc((void**)&L->key, (N + 32) * 8, s))) return bail(st);
        if ((st = dalloc(&L->s_act, (N + 32) * in->act_bytes, s))) return bail(st);
        add(in->key, L->key, 8);
        add(in->s_act, L->s_act, in->act_bytes);
        if (in->perm) {
            if ((st = dalloc((void**)&L->perm, N * 4, s))) return bail(st);
            add(in->perm, L->perm, 4);
        }
        if (in->rcase) {
            if ((st = dalloc((void**)&L->rcase, (N + 32) * 4, s))) return bail(st);
            add(in->rcase, L->rcase, 4);
        }
    } else {
        L->owns_cols = true;
        if ((st = dalloc((void**)&L->case_, N * 4, s))) return bail(st);
        if ((st = dalloc(&L->act, N * in->act_bytes, s))) return bail(st);
        if ((st = dalloc((void**)&L->ts, N * 8, s))) return bail(st);
    }
    for (auto& x : in->extra) {
        ExtraCol y = x;
        y.owned = true;
        y.data = nullptr;
        y.valid = nullptr;
        if ((st = dalloc(&y.data, N * x.elem, s))) return bail(st);
        if (x.valid && (st = dalloc((void**)&y.valid, N, s))) return bail(st);
        L->extra.push_back(y);
        if (cs.ncol + 2 > CMP_MAXCOL) return bail(fail(PM4G_EINVAL, "too many extra columns for a filter"));
        add(x.data, y.data, x.elem);
        if (x.valid) add(x.valid, y.valid, 1);
    }
    uint64_t kept = 0;
    FilterMeta fm{LLONG_MAX, LLONG_MIN, 0xffffffffu, 0u};
    int hpasses = 0, hbits = 0;
    Scratch wk(s), om(s);
    if (fused) {
        hist_layout(L, &hpasses, &hbits);
        if ((st = dalloc_t(&L->hist, 4 * 256, s))) return bail(st);
        if (cudaMemsetAsync(L->hist, 0, 4 * 256 * 4, s) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "memset"));
    }
    if (n > 0) {
        const int64_t tiles = (n + CMP_TILE - 1) / CMP_TILE;
        // [tile counts u32: tiles] [tile offsets u64: tiles + 1] [meta]
        const size_t cnt_bytes = ((size_t)tiles * 4 + 15) & ~(size_t)15;
        if ((st = wk.alloc(cnt_bytes + (tiles + 1) * 8 + sizeof(FilterMeta) + 16))) return bail(st);
        uint32_t* tcnt = wk.as<uint32_t>();
        uint64_t* toff = (uint64_t*)((char*)wk.p + cnt_bytes);
        FilterMeta* d_meta = (FilterMeta*)(toff + tiles + 1);
        const int64_t t1 = tp ? tp->t1 : 0, t2 = tp ? tp->t2 : 0;
        if (tp)
            PM4G_LAUNCH("k_count_tiles", n * 8.0, s,
                        (k_count_tiles<true><<<(unsigned)tiles, CMP_THREADS, 0, s>>>(nullptr, in->ts, n, t1, t2, tcnt)));
        else
            PM4G_LAUNCH("k_count_tiles", n * 1.0, s,
                        (k_count_tiles<false><<<(unsigned)tiles, CMP_THREADS, 0, s>>>(keep, nullptr, n, 0, 0, tcnt)));
        if ((st = excl_scan_u32_to_u64(tcnt, toff, tiles, s))) return bail(st);
        if (fused) {
            uint8_t* omask = nullptr;
            if (!in->extra.empty()) {
                if ((st = om.alloc(N))) return bail(st);
                omask = om.as<uint8_t>();
            }
            if (cudaMemcpyAsync(d_meta, &fm, sizeof(fm), cudaMemcpyHostToDevice, s) != cudaSuccess)
                return bail(cuda_fail(cudaGetLastError(), "filter setup"));
            const int tma_ok = (((uintptr_t)in->case_ | (uintptr_t)in->act | (uintptr_t)in->ts) & 15) == 0;
            // reads (+ mask in / out); the kept rows' writes are added below
            const double rb = n * (12.0 + in->act_bytes + (tp ? 0 : 1) + (omask ? 1 : 0));
#define PM4G_FILTER_COLS(P)                                                                                     \
    {                                                                                                           \
        const size_t smem = FS_STAGES * sizeof(FsStage<P>);                                                     \
        PM4G_MAX_SMEM(k_filter_cols<P, true>);                                                                  \
        PM4G_MAX_SMEM(k_filter_cols<P, false>);                                                                 \
        const int per_sm = std::max(1, std::min(3, (int)((220 * 1024) / (smem + 6 * 1024))));                  \
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * per_sm)); \
        if (tp)                                                                                                 \
            PM4G_LAUNCH("k_filter_cols", rb, s,                                                                 \
                        (k_filter_cols<P, true><<<grid, FS_BLOCK, smem, s>>>(                                   \
                            keep, in->case_, (const P*)in->act, in->ts, n, t1, t2, toff, L->case_, (P*)L->act,  \
                            L->ts, omask, d_meta, L->case_lo, hpasses, hbits, L->hist, tma_ok)));               \
        else                                                                                                    \
            PM4G_LAUNCH("k_filter_cols", rb, s,                                                                 \
                        (k_filter_cols<P, false><<<grid, FS_BLOCK, smem, s>>>(                                  \
                            keep, in->case_, (const P*)in->act, in->ts, n, t1, t2, toff, L->case_, (P*)L->act,  \
                            L->ts, omask, d_meta, L->case_lo, hpasses, hbits, L->hist, tma_ok)));               \
    }
            switch (in->act_bytes) {
                case 1: PM4G_FILTER_COLS(uint8_t); break;
                case 2: PM4G_FILTER_COLS(uint16_t); break;
                default: PM4G_FILTER_COLS(uint32_t); break;
            }
#undef PM4G_FILTER_COLS
            keep = omask;   // the extra columns follow the same mask
        }
        double row_bytes = 0;
        for (int c = 0; c < cs.ncol; ++c) row_bytes += cs.elem[c];
        if (cs.ncol > 0)
            PM4G_LAUNCH("k_compact_rows", n * (1.0 + row_bytes), s,
                        (k_compact_rows<<<(unsigned)tiles, CMP_THREADS, 0, s>>>(keep, n, cs, toff)));
        if (cudaMemcpyAsync(&kept, toff + tiles, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            (fused && cudaMemcpyAsync(&fm, d_meta, sizeof(fm), cudaMemcpyDeviceToHost, s) != cudaSuccess) ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return bail(cuda_fail(cudaGetLastError(), "filter count"));
        if (fused) prof_add_bytes("k_filter_cols", (double)kept * (12.0 + in->act_bytes));
        if (cs.ncol > 0) prof_add_bytes("k_compact_rows", (double)kept * row_bytes);
    }
    L->n = (int64_t)kept;
    if (!fused) {
        L->sorted = true;
        L->ts_min = in->ts_min;
        L->ts_max = in->ts_max;
        L->case_min = in->case_min;
        L->case_max = in->case_max;
        L->case_bits = in->case_bits;
        L->ts_bits = in->ts_bits;
        L->key_bits = in->key_bits;
        L->wide = in->wide;
        L->passes = in->passes;
        if ((st = segments(L, s))) return bail(st);
    } else {
        apply_meta(L, fm.ts_min, fm.ts_max, fm.case_min, fm.case_max, hpasses, hbits);
    }
    *out = guard.release();
    return PM4G_OK;
}

// ------------------------------------------------------------------ whole-case filters (NEXT-1)
// On a formatted log: one thread per case evaluates the case predicate on its
// rows [off[c], off[c+1]) and writes the case's keep bytes; compact_log then
// moves the kept rows and rebuilds the case offsets (R21).
struct CasePred {
    int kind;
    const uint32_t* bitmap;   // START_IN / END_IN: A-bit activity set
    const uint64_t* pairs;    // PATHS: sorted unique edge ids a * A + b
    int64_t npairs;
    int64_t lo, hi;
    int keep;
};

__device__ __forceinline__ bool in_sorted(const uint64_t* v, int64_t n, uint64_t x) {
    int64_t a = 0, b = n;
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (v[m] < x) a = m + 1; else b = m;
    }
    return a < n && v[a] == x;
}

template <class P>
__global__ void k_case_filter(const uint64_t* __restrict__ key, const P* __restrict__ act,
                              const uint32_t* __restrict__ off, const uint64_t* __restrict__ d_n_cases,
                              uint32_t A, CasePred p, uint8_t* __restrict__ mask) {
    const uint64_t C = *d_n_cases;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < C; c += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t f = off[c], e = off[c + 1];
        bool m = false;
        if (p.kind == PM4G_CASE_START_IN || p.kind == PM4G_CASE_END_IN) {
            const uint32_t a = (uint32_t)act[p.kind == PM4G_CASE_START_IN ? f : e - 1];
            m = (p.bitmap[a >> 5] >> (a & 31)) & 1u;
        } else if (p.kind == PM4G_CASE_SIZE) {
            const int64_t len = (int64_t)(e - f);
            m = len >= p.lo && len <= p.hi;
        } else if (p.kind == PM4G_CASE_THROUGHPUT) {
            const int64_t d = (int64_t)(key[e - 1] - key[f]);   // last ts - first ts (R9)
            m = d >= p.lo && d <= p.hi;
        } else {   // PATHS
            for (uint32_t r = f; r + 1 < e && !m; ++r)
                m = in_sorted(p.pairs, p.npairs, (uint64_t)act[r] * A + (uint64_t)act[r + 1]);
        }
        const uint8_t k = (m == (p.keep != 0)) ? 1 : 0;
        for (uint32_t r = f; r < e; ++r) mask[r] = k;
    }
}

// filter_by_variants: the case's variant key (same hash as A8) is looked up
// among the query keys (sorted, host-hashed); every equal key is verified by
// comparing the sequences exactly.
struct VarQuery {
    const uint64_t* k1;       // sorted by (k1, k2)
    const uint64_t* k2;
    const uint32_t* qi;       // query sequence of each key
    int64_t nq;
    const uint64_t* qoff;     // query CSR
    const uint32_t* qact;
    int keep;
};

template <class P>
__global__ void k_variant_filter(const P* __restrict__ act, const uint32_t* __restrict__ off,
                                 const uint64_t* __restrict__ d_n_cases, const uint64_t* __restrict__ ck1,
                                 const uint64_t* __restrict__ ck2, VarQuery q, uint8_t* __restrict__ mask) {
    const uint64_t C = *d_n_cases;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < C; c += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t f = off[c], e = off[c + 1];
        const uint64_t a1 = ck1[c], a2 = ck2[c];
        int64_t lo = 0, hi = q.nq;   // first key >= (a1, a2)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (q.k1[mid] < a1 || (q.k1[mid] == a1 && q.k2[mid] < a2)) lo = mid + 1; else hi = mid;
        }
        bool m = false;
        for (int64_t j = lo; j < q.nq && q.k1[j] == a1 && q.k2[j] == a2 && !m; ++j) {
            const uint32_t s = q.qi[j];
            const uint64_t s0 = q.qoff[s], s1 = q.qoff[s + 1];
            if (s1 - s0 != (uint64_t)(e - f)) continue;
            bool eq = true;
            for (uint64_t t = 0; t < s1 - s0 && eq; ++t) eq = (uint32_t)act[f + t] == q.qact[s0 + t];
            m = eq;
        }
        const uint8_t k = (m == (q.keep != 0)) ? 1 : 0;
        for (uint32_t r = f; r < e; ++r) mask[r] = k;
    }
}

static int case_grid(uint64_t C) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((C + 255) / 256, (uint64_t)num_sms() * 8));
}

// ------------------------------------------------------------------ A1 fused into the sort
// Events-mode time filter on an ingested log (the usual filter -> sort step,
// P:126): the filtered log is created lazily.  One scan of the case and ts
// columns (12 B/row) counts the kept rows and builds their metadata and
// case-digit histograms; the rows themselves are not copied -- the sort's
// first radix pass reads the shared raw columns and ranks only the kept rows
// (sort.cu, PassArgs::tf).  Saves the compaction's 13 B/row read + 13 B/kept
// row write + the sort's 13 B/kept row re-read.
__global__ __launch_bounds__(256) void k_tf_scan(const uint32_t* __restrict__ cs, const int64_t* __restrict__ ts,
                                                 int64_t n, int64_t t1, int64_t t2, uint32_t lo, FilterMeta* m,
                                                 unsigned long long* kept, int hpasses, int hbits,
                                                 uint32_t* __restrict__ hist) {
    __shared__ uint32_t shw[8][4][256];   // per-warp digit histograms
    for (int i = threadIdx.x; i < 8 * 4 * 256; i += blockDim.x) (&shw[0][0][0])[i] = 0;
    __syncthreads();
    uint32_t (*sh)[256] = shw[threadIdx.x >> 5];
    long long tmin = LLONG_MAX, tmax = LLONG_MIN;
    unsigned cmin = 0xffffffffu, cmax = 0, cnt = 0;
    const uint32_t hmask = (1u << hbits) - 1;
    auto row = [&](uint32_t c, long long t) {
        if (t < t1 || t > t2) return;
        ++cnt;
        tmin = min(tmin, t);
        tmax = max(tmax, t);
        cmin = min(cmin, c);
        cmax = max(cmax, c);
        const uint32_t f = c - lo;
        for (int p = 0; p < hpasses; ++p) atomicAdd(&sh[p][(f >> (p * hbits)) & hmask], 1u);
    };
    const bool vec = (((uintptr_t)cs | (uintptr_t)ts) & 15) == 0;
    const int64_t nq = vec ? n / 4 : 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 c4 = ((const uint4*)cs)[q];
        const longlong2 t01 = ((const longlong2*)ts)[2 * q], t23 = ((const longlong2*)ts)[2 * q + 1];
        row(c4.x, t01.x);
        row(c4.y, t01.y);
        row(c4.z, t23.x);
        row(c4.w, t23.y);
    }
    for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        row(cs[i], ts[i]);
    for (int o = 16; o; o >>= 1) {
        tmin = min(tmin, __shfl_xor_sync(~0u, tmin, o));
        tmax = max(tmax, __shfl_xor_sync(~0u, tmax, o));
        cmin = min(cmin, __shfl_xor_sync(~0u, cmin, o));
        cmax = max(cmax, __shfl_xor_sync(~0u, cmax, o));
        cnt += __shfl_xor_sync(~0u, cnt, o);
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicMin(&m->ts_min, tmin);
        atomicMax(&m->ts_max, tmax);
        atomicMin(&m->case_min, cmin);
        atomicMax(&m->case_max, cmax);
        atomicAdd(kept, (unsigned long long)cnt);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < hpasses * 256; i += blockDim.x) {
        uint32_t v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += (&shw[w][0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// an ingested log's header (no columns, no state) for a derived log on stream s
static pm4g_log* derived_header(const pm4g_log* in, cudaStream_t s) {
    pm4g_log* L = new pm4g_log();
    L->A = in->A;
    L->act_bytes = in->act_bytes;
    L->n_case_codes = in->n_case_codes;
    L->case_lo = in->case_lo;
    L->case_hi = in->case_hi;
    L->stream = s;
    return L;
}

// The lazily filtered log over `in`'s columns (in is unsorted, has no extra
// columns; a lazy `in` is filtered on its own parent rows with the
// intersected time range).
static pm4g_status filter_time_lazy(const pm4g_log* in, int64_t t1, int64_t t2, cudaStream_t s, pm4g_log** out) {
    pm4g_log* L = derived_header(in, s);
    LogGuard guard(L);
    PM4G_TRY(dalloc((void**)&L->d_n_cases, 8, s));
    pm4g_log* P = const_cast<pm4g_log*>(in);   // the parent's observable state does not change
    if (P->owns_cols) {                        // its columns become shared
        P->hold = std::make_shared<ColHold>();
        P->hold->case_ = P->case_;
        P->hold->act = P->act;
        P->hold->ts = P->ts;
        P->owns_cols = false;
    }
    L->hold = P->hold;
    L->case_ = P->case_;
    L->act = P->act;
    L->ts = P->ts;
    L->tf_n = in->tf_n >= 0 ? in->tf_n : in->n;
    L->tf_t1 = in->tf_n >= 0 ? std::max(t1, in->tf_t1) : t1;
    L->tf_t2 = in->tf_n >= 0 ? std::min(t2, in->tf_t2) : t2;
    int hpasses = 0, hbits = 0;
    hist_layout(L, &hpasses, &hbits);
    PM4G_TRY(dalloc_t(&L->hist, 4 * 256, s));
    PM4G_CK(cudaMemsetAsync(L->hist, 0, 4 * 256 * 4, s));
    struct Stage {
        FilterMeta fm;
        unsigned long long kept;
    };
    static thread_local Stage* hp = nullptr;   // pinned: one async init copy, one result copy
    if (!hp) PM4G_CK(cudaHostAlloc((void**)&hp, sizeof(Stage), cudaHostAllocDefault));
    hp->fm = FilterMeta{LLONG_MAX, LLONG_MIN, 0xffffffffu, 0u};
    hp->kept = 0;
    Scratch md(s);
    PM4G_TRY(md.alloc(sizeof(Stage)));
    Stage* dm = md.as<Stage>();
    PM4G_CK(cudaMemcpyAsync(dm, hp, sizeof(Stage), cudaMemcpyHostToDevice, s));
    const int64_t n = L->tf_n;
    if (n > 0) {
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, (int64_t)num_sms() * 4));
        PM4G_LAUNCH("k_tf_scan", n * 12.0, s,
                    (k_tf_scan<<<g, 256, 0, s>>>(L->case_, L->ts, n, L->tf_t1, L->tf_t2, L->case_lo, &dm->fm,
                                                 &dm->kept, hpasses, hbits, L->hist)));
    }
    PM4G_CK(cudaMemcpyAsync(hp, dm, sizeof(Stage), cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    L->n = (int64_t)hp->kept;
    apply_meta(L, hp->fm.ts_min, hp->fm.ts_max, hp->fm.case_min, hp->fm.case_max, hpasses, hbits);
    // only the narrow first pass of a non-empty log keeps rows on the fly
    if (L->n == 0 || L->wide) PM4G_TRY(materialize(L, s));
    *out = guard.release();
    return PM4G_OK;
}

pm4g_status materialize(pm4g_log* L, cudaStream_t s) {
    if (L->tf_n < 0) return PM4G_OK;
    pm4g_log view;   // the parent rows the lazy log filters (columns borrowed)
    view.n = L->tf_n;
    view.A = L->A;
    view.act_bytes = L->act_bytes;
    view.n_case_codes = L->n_case_codes;
    view.case_lo = L->case_lo;
    view.case_hi = L->case_hi;
    view.case_ = L->case_;
    view.act = L->act;
    view.ts = L->ts;
    view.stream = s;
    pm4g_log* M = nullptr;
    const TimePred tp{L->tf_t1, L->tf_t2};
    PM4G_TRY(compact_log(&view, nullptr, s, &M, &tp));
    free_log_cols(L, s);   // drops the shared columns (and clears tf_n)
    L->case_ = M->case_;
    L->act = M->act;
    L->ts = M->ts;
    L->owns_cols = true;
    M->case_ = nullptr;
    M->act = nullptr;
    M->ts = nullptr;
    M->owns_cols = false;
    std::swap(L->hist, M->hist);
    L->n = M->n;
    L->ts_min = M->ts_min;
    L->ts_max = M->ts_max;
    L->case_min = M->case_min;
    L->case_max = M->case_max;
    L->case_bits = M->case_bits;
    L->ts_bits = M->ts_bits;
    L->key_bits = M->key_bits;
    L->wide = M->wide;
    L->passes = M->passes;
    L->hist_passes = M->hist_passes;
    L->hist_bits = M->hist_bits;
    pm4g_log_destroy(M);
    return PM4G_OK;
}

static bool lazy_filter_off() {
    const char* e = getenv("PM4G_NO_LAZY_FILTER");
    return e && e[0] == '1';
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_filter_time(const pm4g_log* in, int64_t t1, int64_t t2, int32_t mode,
                             pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_filter_time");
    if (!in || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    PM4G_TRY(check_log(in));
    if (t1 > t2) return fail(PM4G_EINVAL, "t1 > t2 (S:414)");
    if (mode < 0 || mode > 2) return fail(PM4G_EINVAL, "bad time-filter mode");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = in->n;
    if (mode == PM4G_TIME_EVENTS && !in->sorted && in->extra.empty() && !lazy_filter_off())
        return filter_time_lazy(in, t1, t2, s, out);
    PM4G_TRY(materialize(const_cast<pm4g_log*>(in), s));
    Scratch mask(s), span(s);
    RowView v = view_of(in);
    if (mode == PM4G_TIME_EVENTS && !in->sorted) {
        const TimePred tp{t1, t2};
        return compact_log(in, nullptr, s, out, &tp);
    }
    PM4G_TRY(mask.alloc(std::max<int64_t>(n, 1)));
    if (n > 0) {
        if (mode == PM4G_TIME_EVENTS) {
            PM4G_LAUNCH("k_time_events", n * 9.0, s, k_time_events<<<gsz(n), 256, 0, s>>>(v, n, t1, t2, mask.as<uint8_t>()));
        } else {
            const int64_t R = (int64_t)(in->case_max - in->case_min) + 1;
            PM4G_TRY(span.alloc(R * 16));
            long long* lo = span.as<long long>();
            long long* hi = lo + R;
            PM4G_LAUNCH("k_init_span", R * 16.0, s, k_init_span<<<gsz(R), 256, 0, s>>>(lo, hi, R));
            PM4G_LAUNCH("k_case_span", n * 12.0, s, k_case_span<<<gsz(n), 256, 0, s>>>(v, n, lo, hi));
            PM4G_LAUNCH("k_time_cases", n * 13.0, s, k_time_cases<<<gsz(n), 256, 0, s>>>(v, n, lo, hi, t1, t2, mode, mask.as<uint8_t>()));
        }
    }
    return compact_log(in, mask.as<uint8_t>(), s, out);
}

pm4g_status pm4g_filter_cases(const pm4g_log* in, const pm4g_case_pred* pred, int32_t keep,
                              pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_filter_cases");
    if (!in || !pred || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    PM4G_TRY(check_log(in));
    if (!in->sorted) return fail(PM4G_EINVAL, "case-level filters need a formatted log (call pm4g_sort first)");
    const int kind = pred->kind;
    if (kind < PM4G_CASE_START_IN || kind > PM4G_CASE_PATHS) return fail(PM4G_EINVAL, "bad case predicate kind");
    if ((kind == PM4G_CASE_SIZE || kind == PM4G_CASE_THROUGHPUT) && pred->lo > pred->hi)
        return fail(PM4G_EINVAL, "lo > hi (S:459)");
    if (pred->n_codes < 0 || (pred->n_codes > 0 && !pred->codes)) return fail(PM4G_EINVAL, "bad code list");
    if (kind == PM4G_CASE_PATHS && (pred->n_codes % 2) != 0) return fail(PM4G_EINVAL, "paths need (a, b) pairs");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t A = in->A;
    CasePred p{};
    p.kind = kind;
    p.lo = pred->lo;
    p.hi = pred->hi;
    p.keep = keep ? 1 : 0;
    Scratch aux(s), mask(s);
    if (kind == PM4G_CASE_START_IN || kind == PM4G_CASE_END_IN) {
        std::vector<uint32_t> bm((A + 31) / 32, 0u);
        for (int64_t i = 0; i < pred->n_codes; ++i)
            if (pred->codes[i] < A) bm[pred->codes[i] >> 5] |= 1u << (pred->codes[i] & 31);
        PM4G_TRY(aux.alloc(bm.size() * 4));
        PM4G_CK(cudaMemcpyAsync(aux.p, bm.data(), bm.size() * 4, cudaMemcpyHostToDevice, s));
        p.bitmap = aux.as<uint32_t>();
    } else if (kind == PM4G_CASE_PATHS) {
        std::vector<uint64_t> pr;
        for (int64_t i = 0; i + 1 < pred->n_codes; i += 2)
            if (pred->codes[i] < A && pred->codes[i + 1] < A)
                pr.push_back((uint64_t)pred->codes[i] * A + pred->codes[i + 1]);
        std::sort(pr.begin(), pr.end());
        pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
        PM4G_TRY(aux.alloc(std::max<size_t>(pr.size(), 1) * 8));
        if (!pr.empty()) PM4G_CK(cudaMemcpyAsync(aux.p, pr.data(), pr.size() * 8, cudaMemcpyHostToDevice, s));
        p.pairs = aux.as<uint64_t>();
        p.npairs = (int64_t)pr.size();
    }
    const int64_t n = in->n;
    PM4G_TRY(mask.alloc(std::max<int64_t>(n, 1)));
    if (n > 0) {
        const uint64_t cap = std::min<uint64_t>((uint64_t)n, (uint64_t)(in->case_max - in->case_min) + 1);
        const int g = case_grid(cap);
        switch (in->act_bytes) {
            case 1: PM4G_LAUNCH("k_case_filter", n * 1.0 + cap * 8.0, s, (k_case_filter<uint8_t><<<g, 256, 0, s>>>(in->key, (const uint8_t*)in->s_act, in->off, in->d_n_cases, A, p, mask.as<uint8_t>()))); break;
            case 2: PM4G_LAUNCH("k_case_filter", n * 1.0 + cap * 8.0, s, (k_case_filter<uint16_t><<<g, 256, 0, s>>>(in->key, (const uint16_t*)in->s_act, in->off, in->d_n_cases, A, p, mask.as<uint8_t>()))); break;
            default: PM4G_LAUNCH("k_case_filter", n * 1.0 + cap * 8.0, s, (k_case_filter<uint32_t><<<g, 256, 0, s>>>(in->key, (const uint32_t*)in->s_act, in->off, in->d_n_cases, A, p, mask.as<uint8_t>()))); break;
        }
    }
    return compact_log(in, mask.as<uint8_t>(), s, out);
}

pm4g_status pm4g_filter_variants(const pm4g_log* in, const uint64_t* seq_off, const uint32_t* seq_act,
                                 int64_t n_seqs, int32_t keep, pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_filter_variants");
    if (!in || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    PM4G_TRY(check_log(in));
    if (!in->sorted) return fail(PM4G_EINVAL, "case-level filters need a formatted log (call pm4g_sort first)");
    if (n_seqs < 0 || (n_seqs > 0 && (!seq_off || !seq_act))) return fail(PM4G_EINVAL, "bad sequence list");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t A = in->A;
    // host: hash every query sequence like A8 (sequences with codes >= A cannot match)
    const bool weak = debug_weak_hash();
    struct QK {
        uint64_t k1, k2;
        uint32_t qi;
    };
    std::vector<QK> keys;
    std::vector<uint64_t> qoff(1, 0);
    std::vector<uint32_t> qact;
    for (int64_t i = 0; i < n_seqs; ++i) {
        const uint64_t b = seq_off[i], e = seq_off[i + 1];
        if (e < b) return fail(PM4G_EINVAL, "seq_off not ascending");
        if (e == b) continue;   // the empty sequence is no case's variant
        bool ok = true;
        uint64_t h1 = 0, h2 = 0;
        for (uint64_t t = b; t < e; ++t) {
            ok = ok && seq_act[t] < A;
            h1 = h1 * HB1 + ((uint64_t)seq_act[t] + 1);
            h2 = h2 * HB2 + ((uint64_t)seq_act[t] + 1);
        }
        if (!ok || e - b > 0xffffffffull) continue;
        QK k;
        finish_key(h1, h2, (uint32_t)(e - b), weak, k.k1, k.k2);
        k.qi = (uint32_t)(qoff.size() - 1);
        keys.push_back(k);
        qact.insert(qact.end(), seq_act + b, seq_act + e);
        qoff.push_back(qact.size());
    }
    std::sort(keys.begin(), keys.end(), [](const QK& x, const QK& y) {
        return x.k1 != y.k1 ? x.k1 < y.k1 : (x.k2 != y.k2 ? x.k2 < y.k2 : x.qi < y.qi);
    });
    const size_t nq = keys.size();
    std::vector<uint64_t> hk1(nq), hk2(nq);
    std::vector<uint32_t> hqi(nq);
    for (size_t i = 0; i < nq; ++i) {
        hk1[i] = keys[i].k1;
        hk2[i] = keys[i].k2;
        hqi[i] = keys[i].qi;
    }
    Scratch qb(s), ck(s), mask(s);
    const size_t n1 = std::max<size_t>(nq, 1), no = qoff.size(), na = std::max<size_t>(qact.size(), 1);
    PM4G_TRY(qb.alloc(n1 * 20 + no * 8 + na * 4 + 64));
    uint64_t* d_k1 = qb.as<uint64_t>();
    uint64_t* d_k2 = d_k1 + n1;
    uint64_t* d_off = d_k2 + n1;
    uint32_t* d_qi = (uint32_t*)(d_off + no);
    uint32_t* d_act = d_qi + n1;
    if (nq) {
        PM4G_CK(cudaMemcpyAsync(d_k1, hk1.data(), nq * 8, cudaMemcpyHostToDevice, s));
        PM4G_CK(cudaMemcpyAsync(d_k2, hk2.data(), nq * 8, cudaMemcpyHostToDevice, s));
        PM4G_CK(cudaMemcpyAsync(d_qi, hqi.data(), nq * 4, cudaMemcpyHostToDevice, s));
        PM4G_CK(cudaMemcpyAsync(d_act, qact.data(), qact.size() * 4, cudaMemcpyHostToDevice, s));
    }
    PM4G_CK(cudaMemcpyAsync(d_off, qoff.data(), no * 8, cudaMemcpyHostToDevice, s));
    // per-case keys: the same A8 pass the variant pipeline uses
    const int64_t n = in->n;
    const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)n, (uint64_t)(in->case_max - in->case_min) + 1));
    PM4G_TRY(ck.alloc(cap * 16));
    PM4G_TRY(mask.alloc(std::max<int64_t>(n, 1)));
    if (n > 0) {
        AggOut o;
        o.k1 = ck.as<uint64_t>();
        o.k2 = o.k1 + cap;
        PM4G_TRY(aggregate(in, o, s));
        VarQuery q{d_k1, d_k2, d_qi, (int64_t)nq, d_off, d_act, keep ? 1 : 0};
        const int g = case_grid(cap);
        switch (in->act_bytes) {
            case 1: PM4G_LAUNCH("k_variant_filter", n * 2.0 + cap * 24.0, s, (k_variant_filter<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in->s_act, in->off, in->d_n_cases, o.k1, o.k2, q, mask.as<uint8_t>()))); break;
            case 2: PM4G_LAUNCH("k_variant_filter", n * 3.0 + cap * 24.0, s, (k_variant_filter<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in->s_act, in->off, in->d_n_cases, o.k1, o.k2, q, mask.as<uint8_t>()))); break;
            default: PM4G_LAUNCH("k_variant_filter", n * 5.0 + cap * 24.0, s, (k_variant_filter<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)in->s_act, in->off, in->d_n_cases, o.k1, o.k2, q, mask.as<uint8_t>()))); break;
        }
    }
    return compact_log(in, mask.as<uint8_t>(), s, out);
}

pm4g_status pm4g_filter_attr(const pm4g_log* in, int32_t column, const pm4g_pred* pred,
                             int32_t level, int32_t keep, pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_filter_attr");
    if (!in || !pred || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    PM4G_TRY(check_log(in));
    if (level != PM4G_LEVEL_EVENTS && level != PM4G_LEVEL_CASES) return fail(PM4G_EINVAL, "bad level");
    cudaStream_t s = (cudaStream_t)stream;
    PM4G_TRY(materialize(const_cast<pm4g_log*>(in), s));
    AttrPred p{};
    p.kind = pred->kind;
    int col_kind;
    if (column == PM4G_COL_ACTIVITY) {
        col_kind = PM4G_KIND_CODES;
        p.col = in->sorted ? in->s_act : in->act;
        p.col_bytes = in->act_bytes;
        p.valid = nullptr;
    } else {
        if (column < 0 || column >= (int32_t)in->extra.size()) return fail(PM4G_EINVAL, "unknown column (S:440)");
        const ExtraCol& x = in->extra[column];
        col_kind = x.kind;
        p.col = x.data;
        p.col_bytes = 4;
        p.valid = x.valid;
    }
    const int want = col_kind == PM4G_KIND_CODES ? PM4G_PRED_IN_SET
                   : col_kind == PM4G_KIND_I64 ? PM4G_PRED_RANGE_I64 : PM4G_PRED_RANGE_F64;
    if (pred->kind != want) return fail(PM4G_EINVAL, "predicate kind does not match column kind (S:449)");
    p.lo_i = pred->lo_i;
    p.hi_i = pred->hi_i;
    p.lo_f = pred->lo_f;
    p.hi_f = pred->hi_f;
    if (pred->kind == PM4G_PRED_RANGE_I64 && pred->lo_i > pred->hi_i) return fail(PM4G_EINVAL, "lo > hi");
    if (pred->kind == PM4G_PRED_RANGE_F64 && !(pred->lo_f <= pred->hi_f)) return fail(PM4G_EINVAL, "lo > hi");
    const int64_t n = in->n;
    Scratch setb(s), mask(s), any(s);
    if (pred->kind == PM4G_PRED_IN_SET) {
        if (pred->n_codes < 0 || (pred->n_codes > 0 && !pred->codes)) return fail(PM4G_EINVAL, "bad code set");
        std::vector<uint32_t> codes(pred->codes, pred->codes + pred->n_codes);
        std::sort(codes.begin(), codes.end());
        codes.erase(std::unique(codes.begin(), codes.end()), codes.end());
        PM4G_TRY(setb.alloc(std::max<size_t>(codes.size(), 1) * 4));
        if (!codes.empty())
            PM4G_CK(cudaMemcpyAsync(setb.p, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice, s));
        p.set = setb.as<uint32_t>();
        p.nset = (int64_t)codes.size();
    }
    PM4G_TRY(mask.alloc(std::max<int64_t>(n, 1)));
    if (n > 0) {
        RowView v = view_of(in);
        if (level == PM4G_LEVEL_EVENTS) {
            PM4G_LAUNCH("k_attr_events", n * 6.0, s, k_attr_events<<<gsz(n), 256, 0, s>>>(p, n, keep, mask.as<uint8_t>()));
        } else {
            const int64_t R = (int64_t)(in->case_max - in->case_min) + 1;
            PM4G_TRY(any.alloc(R));
            PM4G_CK(cudaMemsetAsync(any.p, 0, R, s));
            PM4G_LAUNCH("k_attr_any", n * 9.0, s, k_attr_any<<<gsz(n), 256, 0, s>>>(p, v, n, any.as<uint8_t>()));
            PM4G_LAUNCH("k_attr_cases", n * 10.0, s, k_attr_cases<<<gsz(n), 256, 0, s>>>(v, n, any.as<uint8_t>(), keep, mask.as<uint8_t>()));
        }
    }
    return compact_log(in, mask.as<uint8_t>(), s, out);
}

}  // extern "C"
