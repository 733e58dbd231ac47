// Internal declarations shared by the libpm4g translation units.
// Product code: sm_100a only, no CPU fallback, no dependency on oracle/.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <memory>
#include <vector>

#include "../../include/pm4g.h"

namespace pm4g {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
pm4g_status fail(pm4g_status st, const std::string& msg);
pm4g_status cuda_fail(cudaError_t e, const char* what);

#define PM4G_CK(call)                                          \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return ::pm4g::cuda_fail(_e, #call); \
    } while (0)

// Opt a kernel into the device's full dynamic shared memory once (thread-safe
// static initialisation; occupancy still follows each launch's actual size).
// The cap is the device's opt-in limit minus the kernel's static shared memory.
int max_smem_optin();
cudaError_t set_max_dynamic_smem(const void* func);
#define PM4G_MAX_SMEM(...)                                                                          \
    do {                                                                                            \
        static const cudaError_t _se = ::pm4g::set_max_dynamic_smem((const void*)(__VA_ARGS__));    \
        if (_se != cudaSuccess) return ::pm4g::cuda_fail(_se, "cudaFuncSetAttribute");              \
    } while (0)

#define PM4G_TRY(call)                          \
    do {                                        \
        pm4g_status _s = (call);                \
        if (_s != PM4G_OK) return _s;           \
    } while (0)

// ------------------------------------------------------------------ launches
// Every kernel launch goes through PM4G_LAUNCH: it counts the launch and, when
// profiling is on, brackets it with CUDA events on the launching stream.
void prof_begin(const char* name, double bytes, cudaStream_t s);
void prof_end(cudaStream_t s);
void prof_add_bytes(const char* name, double bytes);
void count_launch();

// NVTX range around a C-ABI entry point (visible in nsys / ncu timelines; a
// push / pop costs tens of nanoseconds when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define PM4G_NVTX(name) ::pm4g::NvtxRange _pm4g_nvtx_range(name)

#define PM4G_LAUNCH(name, bytes, stream, ...)                                  \
    do {                                                                       \
        ::pm4g::prof_begin(name, (double)(bytes), stream);                     \
        __VA_ARGS__;                                                           \
        cudaError_t _le = cudaGetLastError();                                  \
        ::pm4g::prof_end(stream);                                              \
        ::pm4g::count_launch();                                                \
        if (_le != cudaSuccess) return ::pm4g::cuda_fail(_le, name);           \
    } while (0)

int num_sms();
bool debug_weak_hash();
// test hook: first-try variant table size (PM4G_DEBUG_VARIANT_CAP, 0 = automatic),
// forcing the load-limit regrowth path on small inputs
uint64_t debug_variant_cap();

// ------------------------------------------------------------------ memory
// Stream-ordered allocations from the device's default pool (kept cached).
pm4g_status dalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);

template <class T>
pm4g_status dalloc_t(T** p, size_t count, cudaStream_t s) {
    return dalloc((void**)p, count * sizeof(T), s);
}

// RAII scratch buffer freed (stream-ordered) at scope exit.
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    explicit Scratch(cudaStream_t st) : s(st) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() { if (p) dfree(p, s); }
    pm4g_status alloc(size_t bytes) { return dalloc(&p, bytes ? bytes : 16, s); }
    template <class T> T* as() const { return (T*)p; }
    void take(Scratch& o) {   // ownership moves here
        if (p) dfree(p, s);
        p = o.p;
        s = o.s;
        o.p = nullptr;
    }
};

// ------------------------------------------------------------------ the log
struct ExtraCol {
    int32_t kind = 0;
    int elem = 4;               // bytes per element (4 codes, 8 i64 / f64)
    void* data = nullptr;       // device [n]
    uint8_t* valid = nullptr;   // device [n] or nullptr
    uint64_t dict_size = 0;
    bool owned = false;
};

// Ingested columns shared by a parent log and its lazily time-filtered child
// (pm4g_filter_time, events mode): freed by whichever log releases them last.
struct ColHold {
    uint32_t* case_ = nullptr;
    void* act = nullptr;
    int64_t* ts = nullptr;
};

}  // namespace pm4g

struct pm4g_log {
    int64_t n = 0;
    uint32_t A = 1;
    int act_bytes = 1;          // internal activity width (1, 2, 4)
    uint64_t n_case_codes = 0;
    uint32_t case_lo = 0, case_hi = 0;
    int64_t ts_min = 0, ts_max = -1;
    uint32_t case_min = 0, case_max = 0;   // present range
    // composite key ((case - case_min) << ts_bits) | (ts - ts_min); a WIDE log
    // (case_bits + ts_bits > 64) keys on ts - ts_min alone and carries the case
    // per formatted row in rcase (SURVEY.md 8(a) A2 "otherwise the wide path")
    int case_bits = 0, ts_bits = 0, key_bits = 0, passes = 0;
    bool wide = false;
    bool sorted = false;
    bool broken = false;        // a deferred format step failed: every call on the log fails
    // ingested state
    uint32_t* case_ = nullptr;
    void* act = nullptr;
    int64_t* ts = nullptr;
    bool owns_cols = false;
    std::shared_ptr<pm4g::ColHold> hold;   // shared ownership of case_ / act / ts (then owns_cols = false)
    // lazily time-filtered log (A1 fused into the sort's first pass): its rows
    // are the tf_n rows of case_ / act / ts with tf_t1 <= ts <= tf_t2, in
    // order; n, the metadata and the histograms describe the kept rows.  Only
    // pm4g_sort reads it in this form; every other consumer materialises it.
    int64_t tf_n = -1, tf_t1 = 0, tf_t2 = 0;
    // formatted state
    uint64_t* key = nullptr;    // [n] sorted composite keys
    void* s_act = nullptr;      // [n] sorted activities
    uint32_t* perm = nullptr;   // [n] ingest row of each formatted row (only with extras)
    uint32_t* rcase = nullptr;  // [n] case - case_min of each formatted row (wide logs only)
    uint32_t* off = nullptr;    // [n_cases + 1] case row offsets (CSR)
    uint32_t* s_case_code = nullptr;  // [n_cases] case code of each case
    uint64_t* d_n_cases = nullptr;    // device scalar
    int64_t n_cases = -1;             // host copy (-1 until fetched)
    // case-digit histograms computed during validation (reused by the sort
    // when hist_passes > 0: digit p of case - case_lo, hist_bits per digit)
    uint32_t* hist = nullptr;         // [4][256]
    int hist_passes = 0, hist_bits = 0;
    std::vector<pm4g::ExtraCol> extra;
    cudaStream_t stream = nullptr;
};

struct pm4g_variant_table {
    uint64_t V = 0, total_len = 0, n_cases = 0;
    uint64_t* count = nullptr;     // [V]
    uint32_t* len = nullptr;       // [V]
    uint32_t* rep_case = nullptr;  // [V] case code
    uint64_t* seq_off = nullptr;   // [V+1]
    uint32_t* seq_act = nullptr;   // [total_len]
    uint64_t* k1 = nullptr;        // [V] variant key (for cross-rank merge)
    uint64_t* k2 = nullptr;        // [V]
    uint32_t* case_variant = nullptr;  // [n_cases]
    cudaStream_t stream = nullptr;
};

namespace pm4g {

// A log whose deferred format step failed (pm4g_sort_analyze) has neither its
// ingested columns nor a correct formatted order: every call on it fails.
pm4g_status check_log(const pm4g_log* L);
// release a log's ingested columns (owned, shared or borrowed) on stream s
void free_log_cols(pm4g_log* L, cudaStream_t s);
// a lazily time-filtered log -> an ordinary ingested log (its kept rows compacted)
pm4g_status materialize(pm4g_log* L, cudaStream_t s);

// ------------------------------------------------------------------ helpers
__host__ __device__ inline int bit_width_u64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return x ? 64 - __clzll((long long)x) : 0;
#else
    return x ? 64 - __builtin_clzll(x) : 0;
#endif
}
__host__ __device__ inline uint64_t shr64(uint64_t x, int s) { return s >= 64 ? 0 : (x >> s); }
// the case part of a composite key (case - case_min < 2^32) as one 32-bit word
__host__ __device__ __forceinline__ uint32_t case32(uint64_t key, int ts_bits) {
    return ts_bits >= 64 ? 0u : (uint32_t)(key >> ts_bits);
}
// two composite keys of the same case
__host__ __device__ __forceinline__ bool same_case(uint64_t a, uint64_t b, int ts_bits) {
    return ts_bits >= 64 || ((a ^ b) >> ts_bits) == 0;
}
__host__ __device__ inline uint64_t low_mask(int bits) {
    return bits >= 64 ? ~0ull : ((1ull << bits) - 1);
}

template <class T>
__device__ __forceinline__ T ld_volatile(const T* p) { return *(const volatile T*)p; }
template <class T>
__device__ __forceinline__ void st_volatile(T* p, T v) { *(volatile T*)p = v; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- TMA bulk copies (cp.async.bulk, 1-D) completing on an mbarrier (sm_90+/sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// bytes and both addresses must be multiples of 16
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Decoupled look-back status word (32 bits): 0 = not ready, 2 v + 2 = the
// tile's own aggregate v, 2 v + 3 = its inclusive prefix v.  Values up to
// 2^31 - 2 fit, which bounds the events of one log shard (MAX_SHARD_EVENTS).
// (A 64-bit word costs a radix pass ~6%: twice the look-back traffic.)
typedef uint32_t st_t;
__host__ __device__ __forceinline__ st_t st_agg(uint32_t v) { return 2u * v + 2u; }
__host__ __device__ __forceinline__ st_t st_inc(uint32_t v) { return 2u * v + 3u; }
__host__ __device__ __forceinline__ bool st_is_inc(st_t w) { return (w & 1u) != 0; }
__host__ __device__ __forceinline__ uint32_t st_val(st_t w) { return (w - 2u) >> 1; }
constexpr int64_t MAX_SHARD_EVENTS = (1ll << 31) - 2;

// Decoupled look-back (one value per tile),
// warp-cooperative, reading K predecessors per lane (32 K per L2 round trip:
// with T tiles in flight the newest tile's walk spans ~T predecessors, so the
// window width bounds a single-pass kernel's steady state).  Called by all 32
// lanes of one warp; publishes the tile's aggregate, walks back to the nearest
// inclusive prefix, publishes its own.  Lane l covers predecessors
// end - (l K + j), j = 0..K-1, nearest first.  Returns the exclusive prefix.
template <int K>
__device__ __forceinline__ uint32_t lookback_warp_k(st_t* status, uint32_t tile, uint32_t aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], st_inc(aggregate));
        return 0;
    }
    if (lane == 0) st_volatile(&status[tile], st_agg(aggregate));
    uint32_t prefix = 0;
    int64_t end = (int64_t)tile - 1;
    while (true) {
        st_t v[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int64_t idx = end - (lane * K + j);
            v[j] = idx >= 0 ? ld_volatile(&status[idx]) : st_inc(0);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int64_t idx = end - (lane * K + j);
            while (v[j] == 0) v[j] = ld_volatile(&status[idx]);
        }
        int fj = K;   // this lane's nearest inclusive entry
#pragma unroll
        for (int j = K - 1; j >= 0; --j)
            if (st_is_inc(v[j])) fj = j;
        const uint32_t inc = __ballot_sync(0xffffffffu, fj < K);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        uint32_t x = 0;
        if (lane <= stop) {
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (lane < stop || j <= fj) x += st_val(v[j]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        prefix += x;
        if (inc) break;
        end -= 32 * K;
    }
    if (lane == 0) st_volatile(&status[tile], st_inc(prefix + aggregate));
    return prefix;
}

// Block-wide exclusive scan of one u32 per thread (BLOCK threads, multiple of 32).
template <int BLOCK>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
    constexpr int W = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < W ? s_warp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < W) s_warp[lane] = wi - w;
        if (lane == W - 1) s_warp[W] = wi;
    }
    __syncthreads();
    uint32_t r = s_warp[warp] + inc - x;
    if (total) *total = s_warp[W];
    return r;
}

// ------------------------------------------------------------------ entry points
// (implemented across the .cu files)
// K1; tfilt = {t1, t2}: the log becomes the lazily events-filtered one (pm4g_log_create_filtered)
pm4g_status validate_and_meta(pm4g_log* L, cudaStream_t s, const int64_t* tfilt = nullptr);
void hist_layout(const pm4g_log* L, int* hpasses, int* hbits);
void apply_meta(pm4g_log* L, int64_t ts_min, int64_t ts_max, uint32_t case_min, uint32_t case_max,
                int hpasses, int hbits);
// A sort whose format fallback (cases k_format cannot sort in shared memory) is
// deferred to the caller's next host synchronisation: sort_log(L, s, &d) returns
// without waiting; sort_finish(&d, s, &fixed) then waits, runs the fallback if
// any case needs it and says so (the caller recomputes what it derived from
// the log meanwhile).
struct FmtDeferred {
    Scratch grp, st;                        // grouped keys (fallback input), format scratch
    alignas(16) unsigned char fa_raw[256];  // the format arguments (type-erased FmtArgs<P>)
    int act_bytes = 1;
    bool active = false;
    uint32_t* h_nbig = nullptr;             // pinned: fallback count, copied after k_format
    cudaEvent_t ev = nullptr;               // recorded after that copy
    const uint32_t* d_nbig = nullptr;       // the device count, until the copy is enqueued
    explicit FmtDeferred(cudaStream_t s) : grp(s), st(s) {}
};
// Enqueue the fallback count's copy to pinned memory (+ its event): deferred
// past the aggregate launch, so no copy sits between k_format and k_aggregate.
pm4g_status sort_defer_copy(FmtDeferred* d, cudaStream_t s);
// set by pm4g_sort_analyze for the pm4g_analyze call it makes (this thread)
extern thread_local FmtDeferred* t_pending_format;
pm4g_status sort_log(pm4g_log* L, cudaStream_t s, FmtDeferred* d = nullptr);   // A2-A4
pm4g_status sort_finish(FmtDeferred* d, cudaStream_t s, bool* fixed);
pm4g_status segments(pm4g_log* L, cudaStream_t s);            // A4
pm4g_status fetch_n_cases(const pm4g_log* L, cudaStream_t s);

// CUDA-graph segments of pm4g_sort_analyze (opt-in, PM4G_GRAPH=1): the launches
// between the call's host round trips are captured from the stream and run as
// one graph each (an executable graph per segment slot is kept and updated in
// place when the next call captures the same topology).  stream_sync() is the
// round trip: it ends and launches the open segment, synchronises, and opens
// the next one.
bool graph_mode();
pm4g_status gseg_open(cudaStream_t s);    // start capturing a sort_analyze call's first segment
pm4g_status gseg_close(bool discard);     // end and launch (or discard) the open segment
bool gseg_active();
pm4g_status stream_sync(cudaStream_t s);
// for a host round trip through pageable memory (not capturable): end and launch
// the open segment on s (returns whether one was open), then gseg_resume()
bool gseg_suspend(cudaStream_t s, pm4g_status* st);
pm4g_status gseg_resume();
// a few words device -> pinned host (the host reads them after stream_sync): a
// cudaMemcpyAsync normally; inside a graph segment a one-warp kernel storing
// into the mapped pinned words (a kernel node updates in place when the device
// pointer changes between calls, a device-to-host memcpy node does not)
pm4g_status copy_words_to_host(void* h, const void* d, size_t bytes, cudaStream_t s);
pm4g_status radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                           cudaStream_t s);  // generic: (key, u32 payload), in place
pm4g_status radix_sort_u64_to(const uint64_t* keys, const uint32_t* vals, uint32_t* vals_out, int64_t n,
                              int bits, cudaStream_t s);  // payload only, to vals_out != vals
pm4g_status excl_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s);

// Variant-key hash (internal, verified): Horner polynomial mod 2^64 over
// act + 1, two bases, finished with the length.  Host and device: the variant
// filter hashes its query sequences on the host the same way.
constexpr uint64_t HB1 = 0x00000100000001B3ull;
constexpr uint64_t HB2 = 0xC2B2AE3D27D4EB4Full;

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

__host__ __device__ __forceinline__ void finish_key(uint64_t h1, uint64_t h2, uint32_t len, bool weak,
                                                    uint64_t& k1, uint64_t& k2) {
    if (weak) {  // debug: 4-bit key, forces collisions (exercises the exact fallback)
        k1 = 1ull | ((fmix64(h1) & 0xFull) << 1);
        k2 = 0;
        return;
    }
    k1 = fmix64(h1 ^ ((uint64_t)len * 0x9E3779B97F4A7C15ull)) | 1ull;
    k2 = fmix64(h2 + (uint64_t)len * 0xff51afd7ed558ccdull);
}

struct AggOut {
    uint64_t* packed = nullptr;   // [cnt A2 | sum A2 | start A | end A] (zeroed by caller)
    uint64_t* mm = nullptr;       // [min A2 | max A2] (caller sets min = ~0, max = 0); with packed only
    uint32_t* n_events = nullptr; // [n_cases]
    uint32_t* case_code = nullptr; // [n_cases] (case_min + case part of the first key)
    int64_t* dur = nullptr;       // [n_cases]
    uint64_t* k1 = nullptr;       // [n_cases] variant keys
    uint64_t* k2 = nullptr;
    bool tables = false;
};
pm4g_status aggregate(const pm4g_log* L, const AggOut& o, cudaStream_t s);   // K6
pm4g_status finalize_tables(const uint64_t* packed, uint32_t A, uint64_t* cnt, int64_t* sum,
                            double* mean, uint64_t* start, uint64_t* end, cudaStream_t s);
pm4g_status variants_from_keys(const pm4g_log* L, const uint64_t* k1, const uint64_t* k2,
                               cudaStream_t s, pm4g_variant_table** out);
pm4g_status comm_allreduce_u64(pm4g_comm* c, uint64_t* buf, size_t count, cudaStream_t s);
enum { COMM_SUM = 0, COMM_MAX = 2, COMM_MIN = 3 };   // ncclRedOp_t values
pm4g_status comm_allreduce_u64_op(pm4g_comm* c, uint64_t* buf, size_t count, int op, cudaStream_t s);
pm4g_status comm_variants_allgather_merge(pm4g_comm* c, pm4g_variant_table* local, cudaStream_t s,
                                          pm4g_variant_table** out);
// Owns a log under construction: destroyed on every early return (the
// PM4G_CK / PM4G_TRY / PM4G_LAUNCH macros return directly), released on success.
struct LogGuard {
    pm4g_log* L;
    explicit LogGuard(pm4g_log* l) : L(l) {}
    LogGuard(const LogGuard&) = delete;
    LogGuard& operator=(const LogGuard&) = delete;
    ~LogGuard() {
        if (L) pm4g_log_destroy(L);
    }
    pm4g_log* release() {
        pm4g_log* t = L;
        L = nullptr;
        return t;
    }
};

// NEXT-4 repartition (repartition.cu): rows of an ingested log grouped by
// destination rank, every column gathered into one buffer (dest-major)
struct PartitionedRows {
    Scratch buf;
    std::vector<void*> cols;          // per column: [n] rows, destination-major
    std::vector<int> elems;           // bytes per element
    std::vector<uint64_t> counts;     // rows per destination
    explicit PartitionedRows(cudaStream_t s) : buf(s) {}
};
void log_columns(const pm4g_log* L, std::vector<const void*>* cols, std::vector<int>* elems);
pm4g_status partition_rows(const pm4g_log* in, const uint32_t* bounds, int R, cudaStream_t s, PartitionedRows* out);
pm4g_status make_ingested_log(const pm4g_log* like, int64_t n, uint32_t case_lo, uint32_t case_hi,
                              const std::function<pm4g_status(const std::vector<void*>&)>& fill, cudaStream_t s,
                              pm4g_log** out);

pm4g_status merge_variant_tables(const pm4g_variant_table* const* parts, int n_parts, cudaStream_t s,
                                 pm4g_variant_table** out, int local_part);
// the merge's items, flat (entries of every part, part-major; see merge_flat)
struct MergeItems {
    uint64_t V = 0, T = 0;
    uint64_t* k1 = nullptr;
    uint64_t* k2 = nullptr;
    uint64_t* w = nullptr;     // [V] entry counts
    uint32_t* ord = nullptr;   // [V] entry representative cases
    uint32_t* so = nullptr;    // [V + 1] sequence offsets into sa
    uint32_t* sa = nullptr;    // [T]
};
pm4g_status merge_items_alloc(uint64_t V, uint64_t T, Scratch& buf, MergeItems* m);
pm4g_status merge_flat(const MergeItems& in, const pm4g_variant_table* lp, uint64_t lp_first, cudaStream_t s,
                       pm4g_variant_table** out);
void free_variants(pm4g_variant_table* v);

}  // namespace pm4g
