// libpm4g: handles, status/error machinery, profiling, log creation (K1) and
// the thin C-ABI dispatch layer.  See include/pm4g.h for the contract.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
pm4g_status fail(pm4g_status st, const std::string& m) {
    g_err = m;
    return st;
}
pm4g_status cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? PM4G_ENOMEM : PM4G_ECUDA;
}

// ------------------------------------------------------------------ launches / profiling
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct ProfRec {
    const char* name;
    double bytes;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_event_pool;
struct ProfAgg {
    std::string name;
    uint64_t launches;
    double ms, bytes;
};
static std::vector<ProfAgg> g_prof_aggs;
struct ProfLine {
    std::string name;
    double start_ms, dur_ms;
};
static std::vector<ProfLine> g_prof_lines;

static cudaEvent_t get_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(const char* name, double bytes, cudaStream_t s) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r{name, bytes, get_event(), get_event()};
    // inside a captured graph segment the events become external event-record
    // nodes, recorded each time the graph runs
    if (gseg_active()) cudaEventRecordWithFlags(r.a, s, cudaEventRecordExternal);
    else cudaEventRecord(r.a, s);
    g_prof_recs.push_back(r);
}
// add bytes known only after the launch (e.g. a compaction's kept rows) to
// the most recent record of that kernel
void prof_add_bytes(const char* name, double bytes) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (size_t i = g_prof_recs.size(); i-- > 0;)
        if (!strcmp(g_prof_recs[i].name, name)) {
            g_prof_recs[i].bytes += bytes;
            return;
        }
}
void prof_end(cudaStream_t s) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_recs.empty()) {
        if (gseg_active()) cudaEventRecordWithFlags(g_prof_recs.back().b, s, cudaEventRecordExternal);
        else cudaEventRecord(g_prof_recs.back().b, s);
    }
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

int max_smem_optin() {
    static const int v = [] {
        int dev = 0, m = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&m, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || m <= 0)
            m = 227 * 1024;
        return m;
    }();
    return v;
}

cudaError_t set_max_dynamic_smem(const void* func) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, func);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem_optin() - (int)fa.sharedSizeBytes);
}

bool debug_weak_hash() {
    const char* e = getenv("PM4G_DEBUG_WEAK_HASH");
    return e && e[0] == '1';
}

uint64_t debug_variant_cap() {
    const char* e = getenv("PM4G_DEBUG_VARIANT_CAP");
    return e ? strtoull(e, nullptr, 10) : 0;
}

// ------------------------------------------------------------------ memory
static void setup_pool() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}
// Stream-aware block cache over cudaMallocAsync: a freed block is kept and
// handed back to the next request of the same size class on the same stream
// (stream order makes the reuse safe).  The hot path allocates the same
// buffers every call, so after the first call no allocator work remains on
// the host between kernel launches.
struct CachedBlock {
    void* p;
    cudaStream_t s;
};
static std::mutex g_alloc_mu;
static std::vector<std::pair<size_t, CachedBlock>> g_free_blocks;
static std::vector<std::pair<void*, size_t>> g_live_blocks;
static size_t g_cached_bytes = 0;
static const size_t kCacheCap = 48ull << 30;

static size_t size_class(size_t b) {
    if (b <= 4096) return 4096;
    size_t p = 1;
    while (p < b) p <<= 1;
    size_t q = p >> 3;  // eighth-of-power-of-two steps (<= 12.5% waste)
    return (b + q - 1) / q * q;
}

pm4g_status dalloc(void** p, size_t bytes, cudaStream_t s) {
    setup_pool();
    const size_t cls = size_class(bytes ? bytes : 16);
    {
        std::lock_guard<std::mutex> lk(g_alloc_mu);
        for (size_t i = g_free_blocks.size(); i-- > 0;) {
            if (g_free_blocks[i].first == cls && g_free_blocks[i].second.s == s) {
                *p = g_free_blocks[i].second.p;
                g_cached_bytes -= cls;
                g_free_blocks.erase(g_free_blocks.begin() + i);
                g_live_blocks.push_back({*p, cls});
                return PM4G_OK;
            }
        }
    }
    cudaError_t e = cudaMallocAsync(p, cls, s);
    if (e == cudaErrorMemoryAllocation) {  // drop the cache and retry once
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(g_alloc_mu);
        for (auto& fb : g_free_blocks) cudaFreeAsync(fb.second.p, fb.second.s);
        g_free_blocks.clear();
        g_cached_bytes = 0;
        e = cudaMallocAsync(p, cls, s);
    }
    if (e != cudaSuccess) {
        *p = nullptr;
        return cuda_fail(e, "cudaMallocAsync");
    }
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_live_blocks.push_back({*p, cls});
    return PM4G_OK;
}
void dfree(void* p, cudaStream_t s) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    size_t cls = 0;
    for (size_t i = g_live_blocks.size(); i-- > 0;) {
        if (g_live_blocks[i].first == p) {
            cls = g_live_blocks[i].second;
            g_live_blocks.erase(g_live_blocks.begin() + i);
            break;
        }
    }
    if (!cls || g_cached_bytes + cls > kCacheCap) {
        cudaFreeAsync(p, s);
        return;
    }
    g_free_blocks.push_back({cls, {p, s}});
    g_cached_bytes += cls;
}

// ------------------------------------------------------------------ K1: validate + metadata
struct Meta {
    long long ts_min, ts_max;
    unsigned int case_min, case_max;
    unsigned long long bad_case, bad_act, bad_extra;
    unsigned long long kept;   // rows with t1 <= ts <= t2 (pm4g_log_create_filtered)
};

// One pass over the ingested columns: metadata (ts / case ranges), the first
// invalid row, and -- since the case column is being read anyway -- the
// histograms of the case digits the sort's LSD passes will use (digit p of
// case - case_lo, `bits` per digit, layout derived from [case_lo, case_hi)).
// Vectorised: 4 rows per thread per iteration (16-byte loads of case and ts).
// With tf, every row is still validated but the metadata, the kept count and
// the histograms cover only the rows with t1 <= ts <= t2 (the events-mode
// time filter of pm4g_log_create_filtered, fused into this pass).
template <class P, bool TF>
__global__ __launch_bounds__(256) void k_validate(const uint32_t* __restrict__ cs, const P* __restrict__ act,
                                                  const int64_t* __restrict__ ts, int64_t n, uint32_t lo,
                                                  uint32_t hi, uint32_t A, Meta* m, int hpasses, int hbits,
                                                  uint32_t* __restrict__ hist, int64_t t1, int64_t t2) {
    // per-warp digit histograms (same-address atomics only within a warp)
    __shared__ uint32_t shw[8][4][256];
    for (int i = threadIdx.x; i < 8 * 4 * 256; i += blockDim.x) (&shw[0][0][0])[i] = 0;
    __syncthreads();
    uint32_t (*sh)[256] = shw[threadIdx.x >> 5];
    long long tmin = LLONG_MAX, tmax = LLONG_MIN;
    unsigned cmin = 0xffffffffu, cmax = 0;
    unsigned long long bc = ~0ull, ba = ~0ull;
    unsigned kept = 0;
    const uint32_t hmask = (1u << hbits) - 1;
    auto row = [&](int64_t i, uint32_t c, long long t, uint32_t a) {
        if ((c < lo || c >= hi) && (unsigned long long)i < bc) bc = i;
        if (a >= A && (unsigned long long)i < ba) ba = i;
        if (TF) {
            if (t < t1 || t > t2) return;
            ++kept;
        }
        tmin = min(tmin, t);
        tmax = max(tmax, t);
        cmin = min(cmin, c);
        cmax = max(cmax, c);
        const uint32_t f = c - lo;
        for (int p = 0; p < hpasses; ++p) atomicAdd(&sh[p][(f >> (p * hbits)) & hmask], 1u);
    };
    const bool vec = (((uintptr_t)cs | (uintptr_t)ts) & 15) == 0 && ((uintptr_t)act & (4 * sizeof(P) - 1)) == 0;
    const int64_t nq = vec ? n / 4 : 0;
    auto quad = [&](int64_t q, const uint4& c4, const longlong2& t01, const longlong2& t23, const uint4& aw) {
        const int64_t i = 4 * q;
        uint32_t a[4];
        if constexpr (sizeof(P) == 1) {   // the four activities in one 4-byte load
#pragma unroll
            for (int k = 0; k < 4; ++k) a[k] = (aw.x >> (8 * k)) & 0xffu;
        } else if constexpr (sizeof(P) == 2) {
            a[0] = aw.x & 0xffffu;
            a[1] = aw.x >> 16;
            a[2] = aw.y & 0xffffu;
            a[3] = aw.y >> 16;
        } else {
            a[0] = aw.x;
            a[1] = aw.y;
            a[2] = aw.z;
            a[3] = aw.w;
        }
        row(i, c4.x, t01.x, a[0]);
        row(i + 1, c4.y, t01.y, a[1]);
        row(i + 2, c4.z, t23.x, a[2]);
        row(i + 3, c4.w, t23.y, a[3]);
    };
    auto load_act = [&](int64_t q) -> uint4 {
        if constexpr (sizeof(P) == 1) return make_uint4(((const uint32_t*)act)[q], 0, 0, 0);
        else if constexpr (sizeof(P) == 2) {
            const uint2 w = ((const uint2*)act)[q];
            return make_uint4(w.x, w.y, 0, 0);
        } else return ((const uint4*)act)[q];
    };
    // two quads per thread per trip, every load issued before any row is processed
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; q + stride < nq; q += 2 * stride) {
        const int64_t r = q + stride;
        const uint4 c4 = ((const uint4*)cs)[q], d4 = ((const uint4*)cs)[r];
        const longlong2 t01 = ((const longlong2*)ts)[2 * q], t23 = ((const longlong2*)ts)[2 * q + 1];
        const longlong2 u01 = ((const longlong2*)ts)[2 * r], u23 = ((const longlong2*)ts)[2 * r + 1];
        const uint4 aq = load_act(q), ar = load_act(r);
        quad(q, c4, t01, t23, aq);
        quad(r, d4, u01, u23, ar);
    }
    for (; q < nq; q += stride)
        quad(q, ((const uint4*)cs)[q], ((const longlong2*)ts)[2 * q], ((const longlong2*)ts)[2 * q + 1], load_act(q));
    for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        row(i, cs[i], ts[i], (uint32_t)act[i]);
    for (int o = 16; o; o >>= 1) {
        tmin = min(tmin, __shfl_xor_sync(~0u, tmin, o));
        tmax = max(tmax, __shfl_xor_sync(~0u, tmax, o));
        cmin = min(cmin, __shfl_xor_sync(~0u, cmin, o));
        cmax = max(cmax, __shfl_xor_sync(~0u, cmax, o));
        bc = min(bc, __shfl_xor_sync(~0u, bc, o));
        ba = min(ba, __shfl_xor_sync(~0u, ba, o));
        if (TF) kept += __shfl_xor_sync(~0u, kept, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (TF && kept) atomicAdd(&m->kept, (unsigned long long)kept);
        atomicMin(&m->ts_min, tmin);
        atomicMax(&m->ts_max, tmax);
        atomicMin(&m->case_min, cmin);
        atomicMax(&m->case_max, cmax);
        if (bc != ~0ull) atomicMin(&m->bad_case, bc);
        if (ba != ~0ull) atomicMin(&m->bad_act, ba);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < hpasses * 256; i += blockDim.x) {
        uint32_t v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += (&shw[w][0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

__global__ void k_validate_codes(const uint32_t* __restrict__ col, const uint8_t* __restrict__ valid,
                                 int64_t n, uint64_t dict, Meta* m) {
    unsigned long long b = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (valid && !valid[i]) continue;
        if ((uint64_t)col[i] >= dict && (unsigned long long)i < b) b = i;
    }
    for (int o = 16; o; o >>= 1) b = min(b, __shfl_xor_sync(~0u, b, o));
    if ((threadIdx.x & 31) == 0 && b != ~0ull) atomicMin(&m->bad_extra, b);
}

static int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)num_sms() * 8;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

// Case-digit histogram layout for the range [case_lo, case_hi): the sort can
// reuse histograms built in this layout when its own digit layout matches.
void hist_layout(const pm4g_log* L, int* hpasses, int* hbits) {
    const uint32_t hi = L->case_hi;
    const int rbits = bit_width_u64((uint64_t)(hi > L->case_lo ? hi - 1 - L->case_lo : 0));
    *hpasses = std::max(1, std::min(4, (std::max(rbits, 1) + 7) / 8));
    *hbits = (std::max(rbits, 1) + *hpasses - 1) / *hpasses;
}

// Log metadata from the observed ranges (n > 0) and the key layout derived
// from it; marks the prebuilt histograms reusable iff the layouts agree.
void apply_meta(pm4g_log* L, int64_t ts_min, int64_t ts_max, uint32_t case_min, uint32_t case_max,
                int hpasses, int hbits) {
    const int64_t n = L->n;
    if (n == 0) {
        L->ts_min = 0;
        L->ts_max = -1;
        L->case_min = L->case_max = L->case_lo;
    } else {
        L->ts_min = ts_min;
        L->ts_max = ts_max;
        L->case_min = case_min;
        L->case_max = case_max;
    }
    uint64_t ts_span = n ? (uint64_t)L->ts_max - (uint64_t)L->ts_min : 0;
    L->case_bits = bit_width_u64((uint64_t)(L->case_max - L->case_min));
    L->ts_bits = bit_width_u64(ts_span);
    L->key_bits = L->case_bits + L->ts_bits;
    L->wide = L->key_bits > 64;
    L->passes = L->wide ? (L->case_bits + 7) / 8 : (std::min(L->key_bits, 64) + 7) / 8;
    L->hist_passes = 0;
    const int cb = std::max(L->case_bits, 1);
    const int sp = (cb + 7) / 8, sb = (cb + sp - 1) / sp;
    if (n > 0 && L->case_min == L->case_lo && sp == hpasses && sb == hbits) {
        L->hist_passes = hpasses;
        L->hist_bits = hbits;
    }
}

pm4g_status validate_and_meta(pm4g_log* L, cudaStream_t s, const int64_t* tfilt) {
    Meta h{LLONG_MAX, LLONG_MIN, 0xffffffffu, 0u, ~0ull, ~0ull, ~0ull, 0ull};
    const int tf = tfilt ? 1 : 0;
    const int64_t t1 = tfilt ? tfilt[0] : 0, t2 = tfilt ? tfilt[1] : 0;
    Scratch md(s);
    PM4G_TRY(md.alloc(sizeof(Meta)));
    Meta* dm = md.as<Meta>();
    // pinned staging: the init copy is a true async DMA, the result one copy + one wait
    static thread_local Meta* hp = nullptr;
    if (!hp) PM4G_CK(cudaHostAlloc((void**)&hp, sizeof(Meta), cudaHostAllocDefault));
    *hp = h;
    PM4G_CK(cudaMemcpyAsync(dm, hp, sizeof(Meta), cudaMemcpyHostToDevice, s));
    const int64_t n = L->n;
    uint32_t hi = L->case_hi;
    int hpasses, hbits;
    hist_layout(L, &hpasses, &hbits);
    L->hist_passes = 0;
    if (!L->hist) PM4G_TRY(dalloc_t(&L->hist, 4 * 256, s));
    PM4G_CK(cudaMemsetAsync(L->hist, 0, 4 * 256 * 4, s));
    if (n > 0) {
        int g = grid_for((n + 3) / 4, 256);
        double bytes = (double)n * (12 + L->act_bytes);
        switch (L->act_bytes) {
            case 1: PM4G_LAUNCH("k_validate", bytes, s, (tf ? k_validate<uint8_t, true> : k_validate<uint8_t, false>)<<<g, 256, 0, s>>>(L->case_, (const uint8_t*)L->act, L->ts, n, L->case_lo, hi, L->A, dm, hpasses, hbits, L->hist, t1, t2)); break;
            case 2: PM4G_LAUNCH("k_validate", bytes, s, (tf ? k_validate<uint16_t, true> : k_validate<uint16_t, false>)<<<g, 256, 0, s>>>(L->case_, (const uint16_t*)L->act, L->ts, n, L->case_lo, hi, L->A, dm, hpasses, hbits, L->hist, t1, t2)); break;
            default: PM4G_LAUNCH("k_validate", bytes, s, (tf ? k_validate<uint32_t, true> : k_validate<uint32_t, false>)<<<g, 256, 0, s>>>(L->case_, (const uint32_t*)L->act, L->ts, n, L->case_lo, hi, L->A, dm, hpasses, hbits, L->hist, t1, t2)); break;
        }
        for (auto& c : L->extra)
            if (c.kind == PM4G_KIND_CODES)
                PM4G_LAUNCH("k_validate_codes", n * 4.0, s, k_validate_codes<<<g, 256, 0, s>>>((const uint32_t*)c.data, c.valid, n, c.dict_size, dm));
    }
    PM4G_CK(cudaMemcpyAsync(hp, dm, sizeof(Meta), cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    h = *hp;
    if (h.bad_case != ~0ull)
        return fail(PM4G_EDATA, "case code out of range [case_lo, case_hi) at row " + std::to_string(h.bad_case));
    if (h.bad_act != ~0ull)
        return fail(PM4G_EDATA, "activity code out of range (>= n_activities) at row " + std::to_string(h.bad_act));
    if (h.bad_extra != ~0ull)
        return fail(PM4G_EDATA, "extra-column code out of range at row " + std::to_string(h.bad_extra));
    if (tf) {   // the log is the lazily time-filtered one (A1 fused into the sort's first pass)
        L->tf_n = L->n;
        L->tf_t1 = t1;
        L->tf_t2 = t2;
        L->n = (int64_t)h.kept;
    }
    apply_meta(L, h.ts_min, h.ts_max, h.case_min, h.case_max, hpasses, hbits);
    return PM4G_OK;
}

pm4g_status fetch_n_cases(const pm4g_log* Lc, cudaStream_t s) {
    pm4g_log* L = const_cast<pm4g_log*>(Lc);
    if (L->n_cases >= 0) return PM4G_OK;
    uint64_t v = 0;
    pm4g_status gs;
    const bool seg = gseg_suspend(s, &gs);   // (a pageable copy cannot sit in a graph segment)
    PM4G_TRY(gs);
    PM4G_CK(cudaMemcpyAsync(&v, L->d_n_cases, sizeof(v), cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    L->n_cases = (int64_t)v;
    if (seg) PM4G_TRY(gseg_resume());
    return PM4G_OK;
}

pm4g_status check_log(const pm4g_log* L) {
    if (!L) return fail(PM4G_EINVAL, "null log");
    if (L->broken)
        return fail(PM4G_EINVAL, "log unusable: formatting it failed in an earlier pm4g_sort_analyze call");
    return PM4G_OK;
}

void free_log_cols(pm4g_log* L, cudaStream_t s) {
    if (L->owns_cols) {
        dfree(L->case_, s);
        dfree(L->act, s);
        dfree(L->ts, s);
    }
    if (L->hold) {   // shared with a parent / child log: the last holder frees them
        if (L->hold.use_count() == 1) {
            dfree(L->hold->case_, s);
            dfree(L->hold->act, s);
            dfree(L->hold->ts, s);
        }
        L->hold.reset();
    }
    L->tf_n = -1;
    L->case_ = nullptr;
    L->act = nullptr;
    L->ts = nullptr;
    L->owns_cols = false;
}

}  // namespace pm4g

using namespace pm4g;

// ====================================================================== C ABI
extern "C" {

const char* pm4g_last_error(void) { return g_err.c_str(); }
const char* pm4g_version(void) { return "pm4g 0.1 (sm_100a)"; }
uint64_t pm4g_launch_count(void) { return g_launches.load(); }

pm4g_status pm4g_mem_stats(uint64_t* live_blocks, uint64_t* live_bytes, uint64_t* cached_bytes) {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    uint64_t b = 0;
    for (auto& x : g_live_blocks) b += x.second;
    if (live_blocks) *live_blocks = g_live_blocks.size();
    if (live_bytes) *live_bytes = b;
    if (cached_bytes) *cached_bytes = g_cached_bytes;
    return PM4G_OK;
}

pm4g_status pm4g_mem_release(void) {
    PM4G_CK(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    for (auto& fb : g_free_blocks) cudaFreeAsync(fb.second.p, fb.second.s);
    g_free_blocks.clear();
    g_cached_bytes = 0;
    PM4G_CK(cudaDeviceSynchronize());
    return PM4G_OK;
}

pm4g_status pm4g_prof_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    return PM4G_OK;
}
pm4g_status pm4g_prof_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof_recs) {
        g_event_pool.push_back(r.a);
        g_event_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    g_prof_aggs.clear();
    return PM4G_OK;
}
pm4g_status pm4g_prof_collect(int32_t* n_names) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_aggs.clear();
    g_prof_lines.clear();
    for (auto& r : g_prof_recs) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0, t0 = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        cudaEventElapsedTime(&t0, g_prof_recs.front().a, r.a);
        g_prof_lines.push_back({r.name, (double)t0, (double)ms});
        auto it = std::find_if(g_prof_aggs.begin(), g_prof_aggs.end(),
                               [&](const ProfAgg& a) { return a.name == r.name; });
        if (it == g_prof_aggs.end()) {
            g_prof_aggs.push_back({r.name, 0, 0.0, 0.0});
            it = g_prof_aggs.end() - 1;
        }
        it->launches += 1;
        it->ms += ms;
        it->bytes += r.bytes;
    }
    if (n_names) *n_names = (int32_t)g_prof_aggs.size();
    return PM4G_OK;
}
pm4g_status pm4g_prof_entry(int32_t i, const char** name, uint64_t* launches, double* total_ms,
                            double* bytes) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (i < 0 || i >= (int32_t)g_prof_aggs.size()) return fail(PM4G_EINVAL, "prof entry out of range");
    if (name) *name = g_prof_aggs[i].name.c_str();
    if (launches) *launches = g_prof_aggs[i].launches;
    if (total_ms) *total_ms = g_prof_aggs[i].ms;
    if (bytes) *bytes = g_prof_aggs[i].bytes;
    return PM4G_OK;
}

int32_t pm4g_prof_n_records(void) { return (int32_t)g_prof_lines.size(); }
pm4g_status pm4g_prof_record(int32_t i, const char** name, double* start_ms, double* dur_ms) {
    if (i < 0 || i >= (int32_t)g_prof_lines.size()) return fail(PM4G_EINVAL, "record out of range");
    if (name) *name = g_prof_lines[i].name.c_str();
    if (start_ms) *start_ms = g_prof_lines[i].start_ms;
    if (dur_ms) *dur_ms = g_prof_lines[i].dur_ms;
    return PM4G_OK;
}

static pm4g_status log_create_impl(const pm4g_log_desc* d, cudaStream_t s, pm4g_log** out, const int64_t* tfilt);

pm4g_status pm4g_log_create(const pm4g_log_desc* d, pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_log_create");
    return log_create_impl(d, (cudaStream_t)stream, out, nullptr);
}

pm4g_status pm4g_log_create_filtered(const pm4g_log_desc* d, int64_t t1, int64_t t2, pm4g_stream_t stream,
                                     pm4g_log** out) {
    PM4G_NVTX("pm4g_log_create_filtered");
    if (!d || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    if (t1 > t2) return fail(PM4G_EINVAL, "t1 > t2 (S:414)");
    cudaStream_t s = (cudaStream_t)stream;
    if (d->n_extra > 0 || getenv("PM4G_NO_LAZY_FILTER")) {   // create, then the compacting filter
        pm4g_log* P = nullptr;
        PM4G_TRY(log_create_impl(d, s, &P, nullptr));
        const pm4g_status st = pm4g_filter_time(P, t1, t2, PM4G_TIME_EVENTS, (pm4g_stream_t)s, out);
        pm4g_log_destroy(P);
        return st;
    }
    const int64_t tf[2] = {t1, t2};
    pm4g_log* L = nullptr;
    PM4G_TRY(log_create_impl(d, s, &L, tf));
    if (L->n == 0 || L->wide) {   // only the narrow first pass of a non-empty log keeps rows on the fly
        const pm4g_status st = materialize(L, s);
        if (st) {
            pm4g_log_destroy(L);
            return st;
        }
    }
    *out = L;
    return PM4G_OK;
}

static pm4g_status log_create_impl(const pm4g_log_desc* d, cudaStream_t s, pm4g_log** out, const int64_t* tfilt) {
    if (!d || !out) return fail(PM4G_EINVAL, "null argument");
    *out = nullptr;
    if (d->n_events < 0) return fail(PM4G_EINVAL, "n_events < 0");
    if (d->n_events > MAX_SHARD_EVENTS)
        return fail(PM4G_EINVAL, "n_events exceeds 2^31-2 per shard; shard the log across ranks");
    if (d->act_bytes != 1 && d->act_bytes != 2 && d->act_bytes != 4)
        return fail(PM4G_EINVAL, "act_bytes must be 1, 2 or 4");
    if (d->n_activities == 0) return fail(PM4G_EINVAL, "n_activities must be >= 1");
    if (d->act_bytes == 1 && d->n_activities > 256) return fail(PM4G_EINVAL, "n_activities > 256 needs act_bytes >= 2");
    if (d->act_bytes == 2 && d->n_activities > 65536) return fail(PM4G_EINVAL, "n_activities > 65536 needs act_bytes = 4");
    if (d->n_events > 0 && (!d->case_code || !d->act || !d->ts)) return fail(PM4G_EINVAL, "null column");
    if (d->n_extra < 0 || (d->n_extra > 0 && !d->extra)) return fail(PM4G_EINVAL, "bad extra columns");
    uint64_t hi = d->case_hi ? d->case_hi : d->n_case_codes;
    if (hi > d->n_case_codes || d->case_lo > hi || hi > 0xffffffffull)
        return fail(PM4G_EINVAL, "bad case range");
    const bool host = d->flags & PM4G_HOST_INPUT;
    const bool borrow = (d->flags & PM4G_BORROW) && !host;

    pm4g_log* L = new pm4g_log();
    L->n = d->n_events;
    L->A = d->n_activities;
    L->act_bytes = d->act_bytes;
    L->n_case_codes = d->n_case_codes;
    L->case_lo = d->case_lo;
    L->case_hi = (uint32_t)hi;
    L->stream = s;
    const int64_t n = L->n;
    auto bail = [&](pm4g_status st) {
        pm4g_log_destroy(L);
        return st;
    };
    pm4g_status st;
    if (borrow) {
        L->case_ = (uint32_t*)d->case_code;
        L->act = (void*)d->act;
        L->ts = (int64_t*)d->ts;
        L->owns_cols = false;
    } else {
        L->owns_cols = true;
        if ((st = dalloc((void**)&L->case_, n * 4, s)) != PM4G_OK) return bail(st);
        if ((st = dalloc(&L->act, n * L->act_bytes, s)) != PM4G_OK) return bail(st);
        if ((st = dalloc((void**)&L->ts, n * 8, s)) != PM4G_OK) return bail(st);
        cudaMemcpyKind k = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        if (n > 0) {
            cudaError_t e = cudaMemcpyAsync(L->case_, d->case_code, n * 4, k, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(L->act, d->act, n * L->act_bytes, k, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(L->ts, d->ts, n * 8, k, s);
            if (e != cudaSuccess) return bail(cuda_fail(e, "column copy"));
        }
    }
    for (int i = 0; i < d->n_extra; ++i) {
        const pm4g_column& c = d->extra[i];
        if (c.kind < 0 || c.kind > 2 || (n > 0 && !c.data)) {
            fail(PM4G_EINVAL, "bad extra column descriptor");
            return bail(PM4G_EINVAL);
        }
        ExtraCol x;
        x.kind = c.kind;
        x.elem = c.kind == PM4G_KIND_CODES ? 4 : 8;
        x.dict_size = c.dict_size;
        if (borrow) {
            x.data = (void*)c.data;
            x.valid = (uint8_t*)c.valid;
        } else {
            x.owned = true;
            if ((st = dalloc(&x.data, n * x.elem, s)) != PM4G_OK) return bail(st);
            cudaMemcpyKind k = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
            if (n > 0) {
                cudaError_t e = cudaMemcpyAsync(x.data, c.data, n * x.elem, k, s);
                if (e != cudaSuccess) return bail(cuda_fail(e, "extra copy"));
            }
            if (c.valid) {
                if ((st = dalloc((void**)&x.valid, n, s)) != PM4G_OK) return bail(st);
                if (n > 0) {
                    cudaError_t e = cudaMemcpyAsync(x.valid, c.valid, n, k, s);
                    if (e != cudaSuccess) return bail(cuda_fail(e, "valid copy"));
                }
            }
        }
        L->extra.push_back(x);
    }
    if ((st = dalloc((void**)&L->d_n_cases, 8, s)) != PM4G_OK) return bail(st);
    if ((st = validate_and_meta(L, s, tfilt)) != PM4G_OK) return bail(st);
    *out = L;
    return PM4G_OK;
}

pm4g_status pm4g_log_destroy(pm4g_log* L) {
    if (!L) return PM4G_OK;
    cudaStream_t s = L->stream;
    free_log_cols(L, s);
    dfree(L->key, s);
    dfree(L->s_act, s);
    dfree(L->perm, s);
    dfree(L->rcase, s);
    dfree(L->off, s);
    dfree(L->s_case_code, s);
    dfree(L->d_n_cases, s);
    dfree(L->hist, s);
    for (auto& x : L->extra)
        if (x.owned) {
            dfree(x.data, s);
            dfree(x.valid, s);
        }
    delete L;
    return PM4G_OK;
}

pm4g_status pm4g_log_info_get(const pm4g_log* L, pm4g_log_info* info) {
    if (!L || !info) return fail(PM4G_EINVAL, "null argument");
    if (L->sorted) PM4G_TRY(fetch_n_cases(L, L->stream));
    info->n_events = L->n;
    info->n_cases = L->sorted ? L->n_cases : -1;
    info->sorted = L->sorted ? 1 : 0;
    info->act_bytes = L->act_bytes;
    info->n_activities = L->A;
    info->case_lo = L->case_lo;
    info->case_hi = L->case_hi;
    info->ts_min = L->ts_min;
    info->ts_max = L->ts_max;
    info->case_bits = L->case_bits;
    info->ts_bits = L->ts_bits;
    info->key_bits = L->key_bits;
    info->radix_passes = L->passes;
    return PM4G_OK;
}

}  // extern "C" (the graph segment helpers are C++)

// ------------------------------------------------------------------ graph segments
namespace pm4g {
namespace {
struct GraphSeg {
    bool on = false, capturing = false;
    int slot = 0;
    cudaStream_t s = nullptr;
};
thread_local GraphSeg t_gseg;
std::mutex g_exec_mu;
std::map<std::tuple<int, cudaStream_t, int>, cudaGraphExec_t> g_execs;   // (device, stream, segment slot) -> executable graph

pm4g_status gseg_begin() {
    if (!t_gseg.on) return PM4G_OK;
    PM4G_CK(cudaStreamBeginCapture(t_gseg.s, cudaStreamCaptureModeRelaxed));
    t_gseg.capturing = true;
    return PM4G_OK;
}
}  // namespace

bool graph_mode() {
    static const bool on = getenv("PM4G_GRAPH") && atoi(getenv("PM4G_GRAPH")) != 0;
    return on;
}

bool gseg_active() { return t_gseg.capturing; }

pm4g_status gseg_open(cudaStream_t s) {
    t_gseg.on = true;
    t_gseg.slot = 0;
    t_gseg.s = s;
    return gseg_begin();
}

pm4g_status gseg_close(bool discard) {
    if (!t_gseg.capturing) return PM4G_OK;
    t_gseg.capturing = false;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(t_gseg.s, &g);
    if (e != cudaSuccess || !g) {
        cudaGetLastError();
        return discard ? PM4G_OK : cuda_fail(e != cudaSuccess ? e : cudaErrorStreamCaptureInvalidated, "stream capture");
    }
    if (discard) {
        cudaGraphDestroy(g);
        return PM4G_OK;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaGraphExec_t ex = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_exec_mu);
        const auto key = std::make_tuple(dev, t_gseg.s, t_gseg.slot++);
        auto it = g_execs.find(key);
        if (it != g_execs.end()) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(it->second, g, &info) == cudaSuccess) {
                ex = it->second;
            } else {   // another topology: instantiate anew
                if (getenv("PM4G_GRAPH_TRACE")) {
                    cudaGraphNodeType nt = cudaGraphNodeTypeCount;
                    if (info.errorNode) cudaGraphNodeGetType(info.errorNode, &nt);
                    const char* fn = "";
                    if (nt == cudaGraphNodeTypeKernel) {
                        cudaKernelNodeParams kp;
                        if (cudaGraphKernelNodeGetParams(info.errorNode, &kp) == cudaSuccess) {
                            cudaFuncAttributes fa;
                            (void)fa;
                        }
                    }
                    if (nt == cudaGraphNodeTypeMemset) {
                        cudaMemsetParams mp;
                        if (cudaGraphMemsetNodeGetParams(info.errorNode, &mp) == cudaSuccess)
                            fprintf(stderr, "  memset node: elem %u width %zu height %zu value %u\n", mp.elementSize, mp.width,
                                    mp.height, mp.value);
                    }
                    if (nt == cudaGraphNodeTypeMemcpy) {
                        cudaMemcpy3DParms cp;
                        if (cudaGraphMemcpyNodeGetParams(info.errorNode, &cp) == cudaSuccess)
                            fprintf(stderr, "  memcpy node: kind %d extent %zu\n", (int)cp.kind, cp.extent.width);
                    }
                    fprintf(stderr, "pm4g graph slot %d: update refused (result %d, node type %d)%s\n", std::get<2>(key),
                            (int)info.result, (int)nt, fn);
                }
                cudaGetLastError();
                cudaGraphExecDestroy(it->second);
                g_execs.erase(it);
            }
        }
        if (!ex) {
            e = cudaGraphInstantiate(&ex, g, 0);
            if (e != cudaSuccess) {
                cudaGraphDestroy(g);
                return cuda_fail(e, "cudaGraphInstantiate");
            }
            g_execs[key] = ex;
        }
    }
    e = cudaGraphLaunch(ex, t_gseg.s);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
    return PM4G_OK;
}

__global__ void k_copy_words(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
}

pm4g_status copy_words_to_host(void* h, const void* d, size_t bytes, cudaStream_t s) {
    if (!t_gseg.capturing || (bytes & 3)) {
        PM4G_CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
        return PM4G_OK;
    }
    void* hd = nullptr;
    PM4G_CK(cudaHostGetDevicePointer(&hd, h, 0));
    PM4G_LAUNCH("k_copy_words", (double)bytes, s,
                (k_copy_words<<<1, 32, 0, s>>>((uint32_t*)hd, (const uint32_t*)d, (uint32_t)(bytes / 4))));
    return PM4G_OK;
}

bool gseg_suspend(cudaStream_t s, pm4g_status* st) {
    *st = PM4G_OK;
    if (!(t_gseg.capturing && t_gseg.s == s)) return false;
    *st = gseg_close(false);
    return true;
}

pm4g_status gseg_resume() { return gseg_begin(); }

pm4g_status stream_sync(cudaStream_t s) {
    const bool seg = t_gseg.capturing && t_gseg.s == s;
    if (seg) PM4G_TRY(gseg_close(false));
    PM4G_CK(cudaStreamSynchronize(s));
    if (seg) PM4G_TRY(gseg_begin());
    return PM4G_OK;
}

}  // namespace pm4g

extern "C" {

static pm4g_status sort_impl(pm4g_log* L, cudaStream_t s, FmtDeferred* d) {
    PM4G_TRY(sort_log(L, s, d));   // sort + case offsets (format kernel)
    free_log_cols(L, s);
    L->sorted = true;
    L->stream = s;
    return PM4G_OK;
}

pm4g_status pm4g_sort(pm4g_log* L, pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_sort");
    PM4G_TRY(check_log(L));
    if (L->sorted) return PM4G_OK;
    return sort_impl(L, (cudaStream_t)stream, nullptr);
}

pm4g_status pm4g_sort_analyze(pm4g_log* L, const pm4g_outputs* out, pm4g_comm* comm, pm4g_stream_t stream) {
    PM4G_NVTX("pm4g_sort_analyze");
    PM4G_TRY(check_log(L));
    if (!out) return fail(PM4G_EINVAL, "null outputs");
    if (L->sorted) return pm4g_analyze(L, out, comm, stream);
    if (comm || !out->variants) {
        PM4G_TRY(pm4g_sort(L, stream));
        return pm4g_analyze(L, out, comm, stream);
    }
    cudaStream_t s = (cudaStream_t)stream;
    FmtDeferred d(s);
    // (the legacy default stream cannot be captured: such calls run eagerly)
    const bool graphs = graph_mode() && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread;
    if (graphs) PM4G_TRY(gseg_open(s));
    pm4g_status st = sort_impl(L, s, &d);
    if (st != PM4G_OK) {
        gseg_close(true);
        return st;
    }
    // the analysis synchronises (variant counters); the deferred format check
    // then costs no extra wait (its count is copied right after the aggregate launch)
    t_pending_format = &d;
    st = pm4g_analyze(L, out, comm, stream);
    t_pending_format = nullptr;
    if (graphs) {   // the last segment; on an error the captured work never ran
        const pm4g_status gs = gseg_close(st != PM4G_OK);
        if (st == PM4G_OK) st = gs;
    }
    bool fixed = false;
    const pm4g_status fs = sort_finish(&d, s, &fixed);
    if (fs != PM4G_OK) {   // the input columns are gone and the order is provisional
        L->broken = true;
        if (st == PM4G_OK && *out->variants) pm4g_variants_destroy(*out->variants);
        *out->variants = nullptr;
        return fs;
    }
    if (fixed) {   // some cases were re-sorted exactly: recompute from the final order
        if (st == PM4G_OK && *out->variants) pm4g_variants_destroy(*out->variants);
        *out->variants = nullptr;
        st = pm4g_analyze(L, out, comm, stream);
    }
    return st;
}

}  // extern "C"
