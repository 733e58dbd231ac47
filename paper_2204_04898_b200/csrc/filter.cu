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
// rebuilt.
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
    int ts_bits;
    uint32_t case_min;
    int64_t ts_min;
    __device__ __forceinline__ uint32_t case_of(int64_t i) const {
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
constexpr int CMP_THREADS = 256, CMP_IPT = 8, CMP_TILE = CMP_THREADS * CMP_IPT, CMP_MAXCOL = 12;

struct ColSet {
    const void* in[CMP_MAXCOL];
    void* out[CMP_MAXCOL];
    int elem[CMP_MAXCOL];
    int ncol;
};

__global__ __launch_bounds__(CMP_THREADS) void k_compact_rows(const uint8_t* __restrict__ keep,
                                                              int64_t n, ColSet cols,
                                                              uint32_t* status, uint32_t* counter,
                                                              uint64_t* n_out) {
    __shared__ uint32_t s_tile, s_wt[CMP_THREADS / 32], s_scan[CMP_THREADS / 32 + 1], s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wbase = (int64_t)tile * CMP_TILE + warp * (32 * CMP_IPT);
    uint32_t ball[CMP_IPT], wc = 0;
#pragma unroll
    for (int j = 0; j < CMP_IPT; ++j) {
        int64_t i = wbase + j * 32 + lane;
        bool k = i < n && keep[i];
        ball[j] = __ballot_sync(0xffffffffu, k);
        wc += __popc(ball[j]);
    }
    if (lane == 0) s_wt[warp] = wc;
    __syncthreads();
    uint32_t total;
    uint32_t wex = block_excl_scan<CMP_THREADS>(tid < CMP_THREADS / 32 ? s_wt[tid] : 0u, s_scan, &total);
    if (tid < CMP_THREADS / 32) s_wt[tid] = wex;
    if (warp == 0) {
        uint32_t pf = lookback_warp(status, tile, total);
        if (lane == 0) s_prefix = pf;
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    uint64_t r = (uint64_t)s_prefix + s_wt[warp];
#pragma unroll
    for (int j = 0; j < CMP_IPT; ++j) {
        if (ball[j] & (1u << lane)) {
            int64_t i = wbase + j * 32 + lane;
            uint64_t o = r + __popc(ball[j] & lt);
            for (int c = 0; c < cols.ncol; ++c) {
                switch (cols.elem[c]) {
                    case 1: ((uint8_t*)cols.out[c])[o] = ((const uint8_t*)cols.in[c])[i]; break;
                    case 2: ((uint16_t*)cols.out[c])[o] = ((const uint16_t*)cols.in[c])[i]; break;
                    case 4: ((uint32_t*)cols.out[c])[o] = ((const uint32_t*)cols.in[c])[i]; break;
                    default: ((uint64_t*)cols.out[c])[o] = ((const uint64_t*)cols.in[c])[i]; break;
                }
            }
        }
        r += __popc(ball[j]);
    }
    if (tid == 0 && (int64_t)(tile + 1) * CMP_TILE >= n) *n_out = (uint64_t)s_prefix + total;
}

// Build the output log from the keep mask.
static pm4g_status compact_log(const pm4g_log* in, const uint8_t* keep, cudaStream_t s,
                               pm4g_log** out) {
    const int64_t n = in->n;
    pm4g_log* L = new pm4g_log();
    L->A = in->A;
    L->act_bytes = in->act_bytes;
    L->n_case_codes = in->n_case_codes;
    L->case_lo = in->case_lo;
    L->case_hi = in->case_hi;
    L->stream = s;
    auto bail = [&](pm4g_status st) {
        pm4g_log_destroy(L);
        return st;
    };
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
    if (in->sorted) {
        if ((st = dalloc((void**)&L->key, (N + 32) * 8, s))) return bail(st);
        if ((st = dalloc(&L->s_act, (N + 32) * in->act_bytes, s))) return bail(st);
        add(in->key, L->key, 8);
        add(in->s_act, L->s_act, in->act_bytes);
        if (in->perm) {
            if ((st = dalloc((void**)&L->perm, N * 4, s))) return bail(st);
            add(in->perm, L->perm, 4);
        }
    } else {
        L->owns_cols = true;
        if ((st = dalloc((void**)&L->case_, N * 4, s))) return bail(st);
        if ((st = dalloc(&L->act, N * in->act_bytes, s))) return bail(st);
        if ((st = dalloc((void**)&L->ts, N * 8, s))) return bail(st);
        add(in->case_, L->case_, 4);
        add(in->act, L->act, in->act_bytes);
        add(in->ts, L->ts, 8);
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
    if (n > 0) {
        const int64_t tiles = (n + CMP_TILE - 1) / CMP_TILE;
        Scratch stt(s);
        if ((st = stt.alloc((tiles + 1) * 4 + 16))) return bail(st);
        uint32_t* status = stt.as<uint32_t>();
        uint64_t* d_kept = (uint64_t*)(((uintptr_t)(status + tiles + 1) + 7) & ~(uintptr_t)7);
        if (cudaMemsetAsync(stt.p, 0, (tiles + 1) * 4, s) != cudaSuccess)
            return bail(cuda_fail(cudaGetLastError(), "memset"));
        double row_bytes = 0;
        for (int c = 0; c < cs.ncol; ++c) row_bytes += cs.elem[c];
        cudaError_t e;
        prof_begin("k_compact_rows", n * (1.0 + row_bytes), s);
        k_compact_rows<<<(unsigned)tiles, CMP_THREADS, 0, s>>>(keep, n, cs, status + 1, status, d_kept);
        e = cudaGetLastError();
        prof_end(s);
        count_launch();
        if (e != cudaSuccess) return bail(cuda_fail(e, "k_compact_rows"));
        if (cudaMemcpyAsync(&kept, d_kept, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return bail(cuda_fail(cudaGetLastError(), "filter count"));
    }
    L->n = (int64_t)kept;
    if (in->sorted) {
        L->sorted = true;
        L->ts_min = in->ts_min;
        L->ts_max = in->ts_max;
        L->case_min = in->case_min;
        L->case_max = in->case_max;
        L->case_bits = in->case_bits;
        L->ts_bits = in->ts_bits;
        L->key_bits = in->key_bits;
        L->passes = in->passes;
        if ((st = segments(L, s))) return bail(st);
    } else {
        if ((st = validate_and_meta(L, s))) return bail(st);
    }
    *out = L;
    return PM4G_OK;
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_filter_time(const pm4g_log* in, int64_t t1, int64_t t2, int32_t mode,
                             pm4g_stream_t stream, pm4g_log** out) {
    if (!in || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    if (t1 > t2) return fail(PM4G_EINVAL, "t1 > t2 (S:414)");
    if (mode < 0 || mode > 2) return fail(PM4G_EINVAL, "bad time-filter mode");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = in->n;
    Scratch mask(s), span(s);
    PM4G_TRY(mask.alloc(std::max<int64_t>(n, 1)));
    RowView v = view_of(in);
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

pm4g_status pm4g_filter_attr(const pm4g_log* in, int32_t column, const pm4g_pred* pred,
                             int32_t level, int32_t keep, pm4g_stream_t stream, pm4g_log** out) {
    if (!in || !pred || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    if (level != PM4G_LEVEL_EVENTS && level != PM4G_LEVEL_CASES) return fail(PM4G_EINVAL, "bad level");
    cudaStream_t s = (cudaStream_t)stream;
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
