// A2-A4: stable sort of the log by (case, ts, ingest index) and case segments.
//
// P:108 "The dataframe is ordered based on three criteria (in order, case
// identifier, the timestamp, and the absolute index of the event in the
// dataframe)".  Readings R1/R2: case order = dictionary code, ties = ingest
// index.  Output (the "formatted log"): the composite key
//     key = ((case - case_min) << ts_bits) | (ts - ts_min)
// in sorted order, the activity (and, with extra columns, the ingest row)
// alongside, and the case offsets (CSR) of the cases dataframe.
//
// B200 design.  A radix pass on B200 is instruction-issue bound
// (6.5 TB/s over 148 SMs is 23 B per SM clock), so the number of passes and
// the number of arrays each pass moves are what matter:
//   1. the composite key is built once, on the fly, by the first pass;
//   2. a stable LSD "onesweep" radix sort runs over the CASE bits of the key
//      only (digit shift = ts_bits + p * bits, ceil(case_bits / 8) passes):
//      events end up grouped by case, in ingest order inside each case.  Each
//      pass moves 8 B of key + the activity; tiles are fetched with TMA bulk
//      copies (cp.async.bulk + mbarrier), ranked with ballots, published with
//      a decoupled look-back, and written out in digit runs;
//   3. one fused "format" kernel finds case heads, ranks them (look-back ->
//      case offsets), and sorts every case by timestamp in shared memory
//      (rank = #smaller-or-equal-earlier, so ties keep ingest order).  Cases
//      longer than FMT_WARP_MAX (or running too far past a tile) go to an
//      exact fallback: a stable radix sort of that case's keys.
// HBM bytes per event (u8 act, P case passes): hist 4 + (13 + 9) + (P-1) * 18
// + format 18 (+ 8 per case).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

constexpr int RADIX = 256;
#ifndef PM4G_SORT_THREADS   // sweep knobs (PM4G_NVCC_EXTRA): radix-pass CTA geometry
#define PM4G_SORT_THREADS 512
#endif
#ifndef PM4G_SORT_IPT
#define PM4G_SORT_IPT 8
#endif
#ifndef PM4G_RANK_OR   // radix ranking peers: 1 = shared-memory atomicOr masks, 0 = 8 ballots
#define PM4G_RANK_OR 1
#endif
#ifndef PM4G_LB            // look-back predecessors per L2 round trip
#define PM4G_LB 4
#endif
#ifndef PM4G_SORT_MINB
#define PM4G_SORT_MINB 2
#endif
#ifndef PM4G_FMT_THREADS       // format-kernel CTA geometry
#define PM4G_FMT_THREADS 512
#endif
#ifndef PM4G_FMT_IPT
#define PM4G_FMT_IPT 8
#endif
constexpr int SORT_THREADS = PM4G_SORT_THREADS;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int SORT_IPT = PM4G_SORT_IPT;
constexpr int SORT_TILE = SORT_THREADS * SORT_IPT;  // 4096
constexpr int MAX_PASSES = 8;

struct KeyParams {
    uint32_t case_min;
    int64_t ts_min;
    int ts_bits;
};

// A1 fused into the sort: pass 0 reads n_scan raw rows, keeps t1 <= ts <= t2
struct TimeFilt {
    int64_t n_scan, t1, t2;
};

__host__ __device__ inline uint64_t make_key(uint64_t case_rel, int64_t t, int64_t ts_min, int ts_bits) {
    return (ts_bits >= 64 ? 0 : (case_rel << ts_bits)) | ((uint64_t)t - (uint64_t)ts_min);
}

// ------------------------------------------------------------------ histograms
// digit p of an item = (field >> (p * bits)) & mask, where field = case - case_min
// (FROM_COLS: read from the case column) or key >> shift0.
template <bool FROM_COLS>
__global__ __launch_bounds__(256) void k_hist(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ cs,
                                              int64_t n, uint32_t case_min, int shift0, int bits,
                                              int passes, uint32_t* __restrict__ hist,
                                              const int64_t* __restrict__ tf_ts = nullptr, int64_t t1 = 0, int64_t t2 = 0) {
    __shared__ uint32_t sh[MAX_PASSES][RADIX];
    for (int i = threadIdx.x; i < MAX_PASSES * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const uint32_t mask = (1u << bits) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (FROM_COLS && tf_ts && (tf_ts[i] < t1 || tf_ts[i] > t2)) continue;   // dropped by a fused time filter
        const uint64_t f = FROM_COLS ? (uint64_t)(cs[i] - case_min) : shr64(keys[i], shift0);
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(uint32_t)(f >> (p * bits)) & mask], 1u);
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
// Stable scatter of (u64 key, payload P [, u32 ingest row]) by one digit of
// the key.  FROM_COLS: the key is built from the raw (case, ts) columns.
template <class P, bool FROM_COLS, bool WITH_IDX>
struct PassArgs {
    const uint64_t* in_key;
    const uint32_t* in_case;
    const int64_t* in_ts;
    const P* in_act;
    const uint32_t* in_idx;   // nullptr with WITH_IDX: generate the ingest row
    uint64_t* out_key;
    P* out_act;
    uint32_t* out_idx;
    int64_t n;
    int shift, bits;
    KeyParams kp;
    const uint32_t* bucket_off;  // [256]
    st_t* status;                // [tiles * 256]
    uint32_t* tile_counter;
    bool aligned;                // every input array 16-byte aligned (TMA bulk path)
    st_t* next_status;           // the next pass's look-back words (zeroed here, row per tile), or nullptr
    // wide logs (case_bits + ts_bits > 64): the key is ts - ts_min only, the
    // payload row is the ingest row, and a pass's digit is digit `wshift` of
    // case_col[ingest row] - case_min (pass 0 reads the case column directly)
    const uint32_t* case_col;
    int wshift;
    // pass 0 of a lazily time-filtered log (A1 fused into the key build): only
    // raw rows with tf_t1 <= ts <= tf_t2 are ranked and written (tf != 0)
    int tf = 0;
    int64_t tf_t1 = 0, tf_t2 = 0;
};

// Shared-memory layout of one tile (all offsets multiples of 16):
//   u_case[T] u_ts[T] (FROM_COLS) | u_key[T];  u_idx[T];  u_act[T]  -- as loaded
//   v_act[T], v_idx[T] (WITH_IDX)  -- payloads in digit order
// After ranking every key is in registers, so the keys are permuted IN PLACE
// (u_key holds them in digit order for the write-out); payloads are copied to
// v_*.  (FROM_COLS builds the keys over the consumed u_ts.)
template <class P, bool FROM_COLS, bool WITH_IDX, bool WIDE = false>
struct OsLayout {
    static constexpr size_t T = SORT_TILE;
    static constexpr size_t o_in = 0;                                   // u_key or u_ts
    static constexpr size_t o_case = o_in + T * 8;                      // FROM_COLS only
    static constexpr size_t o_idx = o_case + (FROM_COLS ? T * 4 : 0);
    static constexpr size_t o_act = o_idx + (WITH_IDX ? T * 4 : 0);
    static constexpr size_t o_vidx = (o_act + T * sizeof(P) + 15) / 16 * 16;
    static constexpr size_t o_vact = o_vidx + (WITH_IDX ? T * 4 : 0);
    static constexpr size_t o_vdig = (o_vact + T * sizeof(P) + 15) / 16 * 16;   // WIDE: digits in digit order
    static constexpr size_t bytes = (o_vdig + (WIDE ? T : 0) + 15) / 16 * 16;
};

#ifdef PM4G_OS_PROF
__device__ unsigned long long g_osprof[8];
extern "C" void pm4g_debug_osprof(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_osprof, 8 * 8);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_osprof, z, 8 * 8);
}
#endif
struct NoHook {
    __device__ void operator()() const {}
};

// One tile's stable rank / publish / permute / look-back / write-out.  The
// tile's rows are in u_key (FROM_COLS: u_case, u_ts) and u_act; s_whist must
// be zero on entry.  after_rank() runs (every thread) once the tile's inputs
// other than u_act / u_key are no longer read (after the ranking barrier).
template <class P, bool FROM_COLS, bool WITH_IDX, bool HI, bool TF, class Hook = NoHook, bool WIDE = false>
__device__ __forceinline__ void os_tile(const PassArgs<P, FROM_COLS, WITH_IDX>& a, const uint32_t tile,
                                        const uint32_t nvalid, uint64_t* u_key, const int64_t* u_ts,
                                        const uint32_t* u_case, const uint32_t* u_idx, const P* u_act,
                                        uint32_t* v_idx, P* v_act, uint32_t (*s_whist)[RADIX],
                                        long long* s_gbase, uint32_t* s_scan, Hook after_rank = Hook(),
                                        uint8_t* v_dig = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)tile * SORT_TILE;
    const uint32_t dmask = (1u << a.bits) - 1;
    // the next pass runs after this kernel: clear its status row for this tile
    // here instead of a host memset of every pass's status up front
    if (a.next_status && tid < RADIX) a.next_status[(size_t)tile * RADIX + tid] = 0;
    const bool gen_idx = WITH_IDX && a.in_idx == nullptr;
    // digit of a key: shift < 64 except for a single-case log (no case bits)
    const int sh = a.shift;
    const bool sh_ok = sh < 64;
    const uint32_t shh = (uint32_t)(sh - 32);
    auto digit = [&](uint64_t k) -> uint32_t {
        if (HI) return ((uint32_t)(k >> 32) >> shh) & dmask;
        return sh_ok ? (uint32_t)(k >> sh) & dmask : 0u;
    };

#ifdef PM4G_OS_PROF
    const long long pt0 = clock64();
    long long pt1 = 0, pt2 = 0, pt3 = 0;
    uint32_t ptrips = 0;
#endif
    // ---- stable local rank: warp-striped order (warp, j, lane) == index order.
    // dp[j] = digit << 16 | rank of the key among its warp's keys of that digit.
    uint64_t k[SORT_IPT];
    uint32_t dp[SORT_IPT];   // the digit, then digit << 16 | rank; 0xffffffff: a row dropped by the time filter (tf)
    const uint32_t lt = lanemask_lt();
    constexpr bool tf = FROM_COLS && TF;   // a time-filtered pass 0 (a separate instantiation)
    uint32_t okm = 0;                      // bit j: row j is kept (tf)
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {   // the warp's rows -> registers
        const uint32_t li = warp * (32 * SORT_IPT) + j * 32 + lane;
        uint32_t d = dmask;
        k[j] = ~0ull;
        bool ok = li < nvalid;
        if (ok) {
            if (FROM_COLS && WIDE) {   // wide pass 0: key = ts - ts_min, digit from the case column
                k[j] = (uint64_t)u_ts[li] - (uint64_t)a.kp.ts_min;
                d = (u_case[li] - a.kp.case_min) & dmask;
            } else if (WIDE) {         // wide pass p: digit of the ingest row's case
                k[j] = u_key[li];
                d = ((a.case_col[u_idx[li]] - a.kp.case_min) >> a.wshift) & dmask;
            } else if (FROM_COLS) {   // pass 0: its digit is the low bits of case - case_min (shift == ts_bits)
                const int64_t t = u_ts[li];
                if (tf) ok = t >= a.tf_t1 && t <= a.tf_t2;
                const uint32_t crel = u_case[li] - a.kp.case_min;
                k[j] = make_key(crel, t, a.kp.ts_min, a.kp.ts_bits);
                d = crel & dmask;
            } else {
                k[j] = u_key[li];
                d = digit(k[j]);
            }
        }
        dp[j] = d;
        if (!tf || ok) okm |= 1u << j;
    }
#if PM4G_RANK_OR
    // Peers (lanes holding the same digit) from one shared-memory atomicOr of
    // the lane's bit into its digit's word of a warp-private mask table, read
    // back after the warp's ORs; the group's leader clears the word for the
    // next key.  The table (RADIX words) overlays the warp's own key rows
    // (2 KB), whose values are in registers now and which are next written by
    // the permutation after the block barrier.  (8 ballots per key cost ~30
    // more instructions; MATCH.ANY is slower still, tools/mbench_peers.cu.)
    static_assert(SORT_IPT * 32 * 8 >= RADIX * 4, "the mask table must fit the warp's key rows");
    uint32_t* wmask = (uint32_t*)(u_key + warp * (32 * SORT_IPT));
    __syncwarp();
#pragma unroll
    for (int q = 0; q < RADIX / 128; ++q) ((uint4*)wmask)[lane + 32 * q] = make_uint4(0, 0, 0, 0);
    __syncwarp();
#endif
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        const uint32_t d = dp[j];
        const bool ok = (okm >> j) & 1u;
        uint32_t peers;
#if PM4G_RANK_OR
        if (ok) atomicOr(&wmask[d], 1u << lane);
        __syncwarp();
        peers = ok ? wmask[d] : 0u;
        __syncwarp();
#else
        // peers = AND over digit bits of (ballot of lanes with the bit == my bit):
        // the bit tested against a constant mask is the ballot predicate, and
        // its sign-extended copy (0 or ~0) folds the choice into one 3-input op
        peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {   // bits above a.bits are 0 in every lane: no-ops
            uint32_t bal, m;   // ballot of the bit, and the bit as 0 / ~0, from one predicate
            asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
                "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\tselp.b32 %1, -1, 0, p;\n}"
                : "=r"(bal), "=r"(m)
                : "r"(d), "r"(1u << b));
            peers &= ~(bal ^ m);
        }
        if (tf) peers &= __ballot_sync(0xffffffffu, ok);   // dropped rows are nobody's peers
#endif
        const int leader = (__ffs(peers) - 1) & 31;   // (a dropped lane has no peers)
        uint32_t bse = 0;
        if (lane == leader && ok) {
            bse = s_whist[warp][d];
            s_whist[warp][d] = bse + __popc(peers);
#if PM4G_RANK_OR
            wmask[d] = 0u;
#endif
        }
        bse = __shfl_sync(0xffffffffu, bse, leader);
        dp[j] = !ok ? 0xffffffffu : (d << 16) | (bse + __popc(peers & lt));
        __syncwarp();
    }
    __syncthreads();   // every key is in registers: u_key may be overwritten
#ifdef PM4G_OS_PROF
    pt1 = clock64();
#endif
    after_rank();

    // ---- per-digit totals; warp bases = tile-exclusive start + warp-exclusive prefix
    const int d = tid;
    const bool dig = tid < RADIX && d <= (int)dmask;
    uint32_t tot = 0;
    st_t* st = a.status + (size_t)tile * RADIX + d;
    uint32_t pub = 0;
    if (tid < RADIX) {
#pragma unroll
        for (int w = 0; w < SORT_WARPS; ++w) {
            uint32_t c = s_whist[w][d];
            s_whist[w][d] = tot;
            tot += c;
        }
        // invalid items (only in the last tile) carry the all-ones digit and
        // rank last; they are not part of the published counts
        pub = tot;
        if (!tf && d == (int)dmask) pub -= (SORT_TILE - nvalid);
        if (dig) {
            if (tile == 0) st_volatile(st, st_inc(pub));
            else st_volatile(st, st_agg(pub));
        }
    }
    uint32_t ranked = 0;   // rows placed: nvalid, or the kept rows of a filtered pass 0
    // exclusive scan of the RADIX digit totals (held by threads < RADIX) with one
    // barrier: warp-inclusive scans, then each thread adds the totals of the
    // warps before it (a two-level block scan costs a second barrier)
    uint32_t start;
    {
        constexpr int DW = RADIX / 32;
        static_assert(RADIX % 32 == 0 && RADIX <= SORT_THREADS && DW <= SORT_WARPS + 1, "digit scan layout");
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31 && warp < DW) s_scan[warp] = inc;
        __syncthreads();
        start = inc - tot;
        uint32_t all = 0;
#pragma unroll
        for (int w = 0; w < DW; ++w) {
            const uint32_t x = s_scan[w];
            if (w < warp) start += x;
            all += x;
        }
        ranked = all;
    }
    const uint32_t nout = tf ? ranked : nvalid;
    if (tid < RADIX) {
#pragma unroll
        for (int w = 0; w < SORT_WARPS; ++w) s_whist[w][d] += start;
    }
    __syncthreads();

    // ---- keys in place, payloads to v_*, all in digit order
#pragma unroll
    for (int j = 0; j < SORT_IPT; ++j) {
        const uint32_t li = warp * (32 * SORT_IPT) + j * 32 + lane;
        if (tf && dp[j] == 0xffffffffu) continue;
        const uint32_t p = (dp[j] & 0xffffu) + s_whist[warp][dp[j] >> 16];
        u_key[p] = k[j];
        v_act[p] = u_act[li];
        if (WITH_IDX) v_idx[p] = gen_idx ? (uint32_t)(base + li) : u_idx[li];
        if (WIDE) v_dig[p] = (uint8_t)(dp[j] >> 16);
    }

#ifdef PM4G_OS_PROF
    pt2 = clock64();
#endif
    // ---- decoupled look-back for this digit, PM4G_LB predecessors per round trip
    // (4, 8 or 16 per trip, with or without requesting the first batch right
    // after the publish, measured equal or slower: the wait is for predecessors
    // still ranking, not the walk -- PM4G_OS_PROF phase counters)
    if (dig) {
        uint32_t prefix = 0;
        if (tile > 0) {
            int64_t p = (int64_t)tile - 1;
            bool done = false;
            while (!done) {
                st_t w[PM4G_LB];
#pragma unroll
                for (int q = 0; q < PM4G_LB; ++q)
                    w[q] = (p - q >= 0) ? ld_volatile(a.status + (size_t)(p - q) * RADIX + d) : st_inc(0);
#pragma unroll
                for (int q = 0; q < PM4G_LB; ++q) {
                    if (done) break;
                    while (w[q] == 0) w[q] = ld_volatile(a.status + (size_t)(p - q) * RADIX + d);
                    prefix += st_val(w[q]);
                    if (st_is_inc(w[q])) done = true;
                }
                p -= PM4G_LB;
#ifdef PM4G_OS_PROF
                ++ptrips;
#endif
            }
            st_volatile(st, st_inc(prefix + pub));
        }
        s_gbase[d] = (long long)a.bucket_off[d] + prefix - start;
    }
    __syncthreads();
#ifdef PM4G_OS_PROF
    pt3 = clock64();
#endif

    // ---- coalesced write-out: consecutive threads, consecutive positions
#pragma unroll 4
    for (int j = 0; j < SORT_IPT; ++j) {
        const uint32_t sidx = j * SORT_THREADS + tid;
        if (sidx < nout) {
            const uint64_t kk = u_key[sidx];
            const long long g = s_gbase[WIDE ? (uint32_t)v_dig[sidx] : digit(kk)] + sidx;
            a.out_key[g] = kk;
            a.out_act[g] = v_act[sidx];
            if (WITH_IDX) a.out_idx[g] = v_idx[sidx];
        }
    }
#ifdef PM4G_OS_PROF
    if (tid == 0) {
        const long long pt4 = clock64();
        atomicAdd(&g_osprof[0], (unsigned long long)(pt1 - pt0));
        atomicAdd(&g_osprof[1], (unsigned long long)(pt2 - pt1));
        atomicAdd(&g_osprof[2], (unsigned long long)(pt3 - pt2));
        atomicAdd(&g_osprof[3], (unsigned long long)(pt4 - pt3));
        atomicAdd(&g_osprof[4], (unsigned long long)ptrips);
        atomicAdd(&g_osprof[5], 1ull);
    }
#endif
}

// HI: the digit lies in the key's high word (32 <= shift < 64, the usual case:
// the digits sit above ts_bits >= 32), extracted with one 32-bit shift
template <class P, bool FROM_COLS, bool WITH_IDX, bool HI, bool WIDE = false, bool TF = false>
__global__ __launch_bounds__(SORT_THREADS, PM4G_SORT_MINB) void k_onesweep(PassArgs<P, FROM_COLS, WITH_IDX> a) {
    using Lay = OsLayout<P, FROM_COLS, WITH_IDX, WIDE>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* u_key = (uint64_t*)(smem + Lay::o_in);
    int64_t* u_ts = (int64_t*)(smem + Lay::o_in);
    uint32_t* u_case = (uint32_t*)(smem + Lay::o_case);
    uint32_t* u_idx = (uint32_t*)(smem + Lay::o_idx);
    P* u_act = (P*)(smem + Lay::o_act);
    uint32_t* v_idx = (uint32_t*)(smem + Lay::o_vidx);
    P* v_act = (P*)(smem + Lay::o_vact);
    __shared__ uint32_t s_whist[SORT_WARPS][RADIX];
    __shared__ long long s_gbase[RADIX];
    __shared__ uint32_t s_scan[SORT_WARPS + 1];
    __shared__ uint32_t s_tile;
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x;
    if (tid == 0) {
        s_tile = atomicAdd(a.tile_counter, 1u);
        mbar_init(&s_bar, 1);
    }
    for (int i = tid; i < SORT_WARPS * RADIX; i += SORT_THREADS) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * SORT_TILE;
    const int64_t nv64 = a.n - base;
    const uint32_t nvalid = (uint32_t)(nv64 < SORT_TILE ? nv64 : SORT_TILE);
    const bool gen_idx = WITH_IDX && a.in_idx == nullptr;

    // ---- tile load: TMA bulk copies for full aligned tiles, plain loads otherwise
    if (nvalid == SORT_TILE && a.aligned) {
        if (tid == 0) {
            const uint32_t bytes = SORT_TILE * (uint32_t)(8 + sizeof(P) + (FROM_COLS ? 4 : 0) +
                                                          ((WITH_IDX && !gen_idx) ? 4 : 0));
            mbar_expect_tx(&s_bar, bytes);
            if (FROM_COLS) {
                tma_load_1d(u_ts, a.in_ts + base, SORT_TILE * 8, &s_bar);
                tma_load_1d(u_case, a.in_case + base, SORT_TILE * 4, &s_bar);
            } else {
                tma_load_1d(u_key, a.in_key + base, SORT_TILE * 8, &s_bar);
            }
            if (WITH_IDX && !gen_idx) tma_load_1d(u_idx, a.in_idx + base, SORT_TILE * 4, &s_bar);
            tma_load_1d(u_act, a.in_act + base, SORT_TILE * sizeof(P), &s_bar);
        }
        mbar_wait(&s_bar, 0);
    } else {
        for (uint32_t i = tid; i < nvalid; i += SORT_THREADS) {
            if (FROM_COLS) {
                u_ts[i] = a.in_ts[base + i];
                u_case[i] = a.in_case[base + i];
            } else {
                u_key[i] = a.in_key[base + i];
            }
            if (WITH_IDX && !gen_idx) u_idx[i] = a.in_idx[base + i];
            u_act[i] = a.in_act[base + i];
        }
        __syncthreads();
    }

    os_tile<P, FROM_COLS, WITH_IDX, HI, TF, NoHook, WIDE>(a, tile, nvalid, u_key, u_ts, u_case, u_idx, u_act, v_idx,
                                                      v_act, s_whist, s_gbase, s_scan, NoHook(),
                                                      (uint8_t*)(smem + Lay::o_vdig));
}

// Persistent form of a key pass (keys + a u8/u16 activity, no ingest row):
// each CTA claims tiles in order and prefetches its NEXT tile with TMA into
// the second of two smem buffers while it ranks and writes out the current
// one, so the load latency (13% of the stall samples of the one-tile-per-CTA
// kernel, ncu source view) hides behind the previous tile's work.  Look-back
// safety: a CTA holds at most two claimed tiles and finishes the older first,
// so the oldest unfinished tile is always being processed.
template <class P>
struct OsPfLayout {
    static constexpr size_t T = SORT_TILE;
    static constexpr size_t o_act = T * 8;
    static constexpr size_t buf = (T * 8 + T * sizeof(P) + 15) / 16 * 16;
    static constexpr size_t o_vact = 2 * buf;
    static constexpr size_t bytes = (o_vact + T * sizeof(P) + 15) / 16 * 16;
};

template <class P, bool HI>
__global__ __launch_bounds__(SORT_THREADS, PM4G_SORT_MINB) void k_onesweep_pf(PassArgs<P, false, false> a, uint32_t n_tiles) {
    using Lay = OsPfLayout<P>;
    extern __shared__ __align__(128) unsigned char smem[];
    P* v_act = (P*)(smem + Lay::o_vact);
    __shared__ uint32_t s_whist[SORT_WARPS][RADIX];
    __shared__ long long s_gbase[RADIX];
    __shared__ uint32_t s_scan[SORT_WARPS + 1];
    __shared__ uint32_t s_tile[2];
    __shared__ __align__(8) uint64_t s_bar[2];

    const int tid = threadIdx.x;
    // full tiles of 16-byte aligned inputs come by TMA; the ragged last tile by plain loads
    auto bulk = [&](uint32_t t) { return a.aligned && (int64_t)(t + 1) * SORT_TILE <= a.n; };
    auto issue = [&](uint32_t t, int b) {   // thread 0
        if (t < n_tiles && bulk(t)) {
            unsigned char* buf = smem + b * Lay::buf;
            mbar_expect_tx(&s_bar[b], SORT_TILE * (uint32_t)(8 + sizeof(P)));
            tma_load_1d(buf, a.in_key + (int64_t)t * SORT_TILE, SORT_TILE * 8, &s_bar[b]);
            tma_load_1d(buf + Lay::o_act, a.in_act + (int64_t)t * SORT_TILE, SORT_TILE * sizeof(P), &s_bar[b]);
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        const uint32_t t = atomicAdd(a.tile_counter, 1u);
        s_tile[0] = t;
        issue(t, 0);
    }
    uint32_t ph = 0;   // mbarrier parity of each buffer (bit b)
    for (int b = 0;; b ^= 1) {
        for (int i = tid; i < SORT_WARPS * RADIX; i += SORT_THREADS) (&s_whist[0][0])[i] = 0;
        // the other buffer was written through the generic proxy (in-place
        // permutation) by the previous tile: order that before the TMA refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const uint32_t tile = s_tile[b];
        if (tile >= n_tiles) break;
        if (tid == 0) {
            const uint32_t t = atomicAdd(a.tile_counter, 1u);
            s_tile[b ^ 1] = t;   // read after the next iteration's barrier
            issue(t, b ^ 1);
        }
        uint64_t* u_key = (uint64_t*)(smem + b * Lay::buf);
        P* u_act = (P*)(smem + b * Lay::buf + Lay::o_act);
        const int64_t base = (int64_t)tile * SORT_TILE;
        const int64_t nv64 = a.n - base;
        const uint32_t nvalid = (uint32_t)(nv64 < SORT_TILE ? nv64 : SORT_TILE);
        if (bulk(tile)) {
            mbar_wait(&s_bar[b], (ph >> b) & 1u);
            ph ^= 1u << b;
        } else {
            for (uint32_t i = tid; i < nvalid; i += SORT_THREADS) {
                u_key[i] = a.in_key[base + i];
                u_act[i] = a.in_act[base + i];
            }
            __syncthreads();
        }
        os_tile<P, false, false, HI, false>(a, tile, nvalid, u_key, nullptr, nullptr, nullptr, u_act, nullptr, v_act,
                                     s_whist, s_gbase, s_scan);
    }
}

// Persistent form of pass 0 (raw columns in, u8/u16 activity, no ingest row):
// the next tile's timestamps + activities are TMA-prefetched into the second of
// two buffers at tile start, and its case codes into the single case buffer as
// soon as the current tile's ranking has consumed it (after_rank), so neither
// load is exposed; 13 B/row of double buffering would not fit two CTAs per SM.
template <class P>
struct Os0Layout {
    static constexpr size_t T = SORT_TILE;
    static constexpr size_t o_act = T * 8;
    static constexpr size_t buf = (T * 8 + T * sizeof(P) + 15) / 16 * 16;   // ts (-> keys) | act
    static constexpr size_t o_case = 2 * buf;
    static constexpr size_t o_vact = o_case + T * 4;
    static constexpr size_t bytes = (o_vact + T * sizeof(P) + 15) / 16 * 16;
};

template <class P, bool HI, bool TF>
__global__ __launch_bounds__(SORT_THREADS, PM4G_SORT_MINB) void k_onesweep_pf0(PassArgs<P, true, false> a, uint32_t n_tiles) {
    using Lay = Os0Layout<P>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* u_case = (uint32_t*)(smem + Lay::o_case);
    P* v_act = (P*)(smem + Lay::o_vact);
    __shared__ uint32_t s_whist[SORT_WARPS][RADIX];
    __shared__ long long s_gbase[RADIX];
    __shared__ uint32_t s_scan[SORT_WARPS + 1];
    __shared__ uint32_t s_tile[2];
    __shared__ __align__(8) uint64_t s_bar[2], s_cbar;

    const int tid = threadIdx.x;
    auto bulk = [&](uint32_t t) { return t < n_tiles && a.aligned && (int64_t)(t + 1) * SORT_TILE <= a.n; };
    auto issue_ta = [&](uint32_t t, int b) {   // thread 0: timestamps + activities of tile t
        unsigned char* buf = smem + b * Lay::buf;
        mbar_expect_tx(&s_bar[b], SORT_TILE * (uint32_t)(8 + sizeof(P)));
        tma_load_1d(buf, a.in_ts + (int64_t)t * SORT_TILE, SORT_TILE * 8, &s_bar[b]);
        tma_load_1d(buf + Lay::o_act, a.in_act + (int64_t)t * SORT_TILE, SORT_TILE * sizeof(P), &s_bar[b]);
    };
    auto issue_case = [&](uint32_t t) {       // thread 0: case codes of tile t
        mbar_expect_tx(&s_cbar, SORT_TILE * 4);
        tma_load_1d(u_case, a.in_case + (int64_t)t * SORT_TILE, SORT_TILE * 4, &s_cbar);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_init(&s_cbar, 1);
        const uint32_t t = atomicAdd(a.tile_counter, 1u);
        s_tile[0] = t;
        if (bulk(t)) {
            issue_ta(t, 0);
            issue_case(t);
        }
    }
    uint32_t ph = 0, pc = 0;   // mbarrier parities: ts/act buffers (bit b), case buffer
    for (int b = 0;; b ^= 1) {
        for (int i = tid; i < SORT_WARPS * RADIX; i += SORT_THREADS) (&s_whist[0][0])[i] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const uint32_t tile = s_tile[b];
        if (tile >= n_tiles) break;
        uint32_t next = 0;
        if (tid == 0) {
            next = atomicAdd(a.tile_counter, 1u);
            s_tile[b ^ 1] = next;   // read after the next iteration's barrier
            if (bulk(next)) issue_ta(next, b ^ 1);
        }
        uint64_t* u_key = (uint64_t*)(smem + b * Lay::buf);
        int64_t* u_ts = (int64_t*)u_key;
        P* u_act = (P*)(smem + b * Lay::buf + Lay::o_act);
        const int64_t base = (int64_t)tile * SORT_TILE;
        const int64_t nv64 = a.n - base;
        const uint32_t nvalid = (uint32_t)(nv64 < SORT_TILE ? nv64 : SORT_TILE);
        if (bulk(tile)) {
            mbar_wait(&s_bar[b], (ph >> b) & 1u);
            ph ^= 1u << b;
            mbar_wait(&s_cbar, pc);
            pc ^= 1u;
        } else {   // the ragged last tile
            for (uint32_t i = tid; i < nvalid; i += SORT_THREADS) {
                u_ts[i] = a.in_ts[base + i];
                u_case[i] = a.in_case[base + i];
                u_act[i] = a.in_act[base + i];
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before any TMA refill
            __syncthreads();
        }
        // the case buffer is free once the ranking has read it: fetch the next tile's
        auto hook = [&]() {
            if (tid == 0 && bulk(next)) issue_case(next);
        };
        os_tile<P, true, false, HI, TF>(a, tile, nvalid, u_key, u_ts, u_case, nullptr, u_act, nullptr, v_act,
                                    s_whist, s_gbase, s_scan, hook);
    }
}

template <class P, bool HI, bool TF>
static pm4g_status launch_pf0(const PassArgs<P, true, false>& args, int64_t tiles, cudaStream_t s,
                              const char* name, double bytes) {
    const size_t smem = Os0Layout<P>::bytes;
    PM4G_MAX_SMEM((k_onesweep_pf0<P, HI, TF>));
    static int per_sm = -1;
    if (per_sm < 0)
        PM4G_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep_pf0<P, HI, TF>, SORT_THREADS, smem));
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)std::max(per_sm, 1) * num_sms());
    PM4G_LAUNCH(name, bytes, s, (k_onesweep_pf0<P, HI, TF><<<grid, SORT_THREADS, smem, s>>>(args, (uint32_t)tiles)));
    return PM4G_OK;
}

template <class P, bool FC, bool WI, bool HI>
static pm4g_status launch_pass_t(const PassArgs<P, FC, WI>& args, int64_t tiles, cudaStream_t s,
                                 const char* name, double bytes) {
    if constexpr (FC && !WI && sizeof(P) == 1) {    // pass 0: persistent, prefetching form (2 CTAs/SM)
        if (tiles > 2 * num_sms() && !getenv("PM4G_NO_OS_PF"))
            return args.tf ? launch_pf0<P, HI, true>(args, tiles, s, name, bytes)
                           : launch_pf0<P, HI, false>(args, tiles, s, name, bytes);
    }
    if constexpr (FC && !WI) {   // a time-filtered pass 0, one tile per CTA
        if (args.tf) {
            const size_t smem = OsLayout<P, FC, WI>::bytes;
            PM4G_MAX_SMEM((k_onesweep<P, FC, WI, HI, false, true>));
            PM4G_LAUNCH(name, bytes, s,
                        (k_onesweep<P, FC, WI, HI, false, true><<<(unsigned)tiles, SORT_THREADS, smem, s>>>(args)));
            return PM4G_OK;
        }
    }
    if constexpr (!FC && !WI && sizeof(P) <= 2) {   // persistent, prefetching form (2 CTAs per SM)
        if (tiles > 2 * num_sms() && !getenv("PM4G_NO_OS_PF")) {
            const size_t smem = OsPfLayout<P>::bytes;
            PM4G_MAX_SMEM(k_onesweep_pf<P, HI>);
            static int per_sm = -1;
            if (per_sm < 0)
                PM4G_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep_pf<P, HI>,
                                                                      SORT_THREADS, smem));
            if (per_sm >= 2) {
                const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)per_sm * num_sms());
                PM4G_LAUNCH(name, bytes, s,
                            (k_onesweep_pf<P, HI><<<grid, SORT_THREADS, smem, s>>>(args, (uint32_t)tiles)));
                return PM4G_OK;
            }
        }
    }
    const size_t smem = OsLayout<P, FC, WI>::bytes;
    PM4G_MAX_SMEM(k_onesweep<P, FC, WI, HI>);
    PM4G_LAUNCH(name, bytes, s, (k_onesweep<P, FC, WI, HI><<<(unsigned)tiles, SORT_THREADS, smem, s>>>(args)));
    return PM4G_OK;
}

template <class P, bool FC, bool WI>
static pm4g_status launch_pass(const PassArgs<P, FC, WI>& args, int64_t tiles, cudaStream_t s,
                               const char* name, double bytes) {
    if constexpr (WI) {
        if (args.case_col) {   // wide log: one-tile-per-CTA kernel, digits from the case column
            const size_t smem = OsLayout<P, FC, WI, true>::bytes;
            PM4G_MAX_SMEM(k_onesweep<P, FC, WI, false, true>);
            PM4G_LAUNCH(name, bytes, s, (k_onesweep<P, FC, WI, false, true><<<(unsigned)tiles, SORT_THREADS, smem, s>>>(args)));
            return PM4G_OK;
        }
    }
    if (args.shift >= 32 && args.shift < 64) return launch_pass_t<P, FC, WI, true>(args, tiles, s, name, bytes);
    return launch_pass_t<P, FC, WI, false>(args, tiles, s, name, bytes);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// Stable LSD sort on `bits_total` bits of the key starting at bit `shift0`.
// Input: either raw columns (in_case/in_ts, key built on the fly) or keys.
// Result lands in the *_out buffers.
template <class P, bool WI>
static pm4g_status lsd_sort(const uint32_t* in_case, const int64_t* in_ts, const uint64_t* in_key,
                            const P* in_act, const uint32_t* in_idx, uint64_t* key_out, P* act_out,
                            uint32_t* idx_out, int64_t n, int shift0, int bits_total, KeyParams kp,
                            cudaStream_t s, const char* pass_name = "k_onesweep",
                            const uint32_t* pre_hist = nullptr, const uint32_t* wide_case = nullptr,
                            const TimeFilt* tfilt = nullptr) {
    const bool from_cols = in_case != nullptr;
    bits_total = std::max(1, bits_total);
    const int passes = std::max(1, std::min(MAX_PASSES, (bits_total + 7) / 8));
    const int bits = (bits_total + passes - 1) / passes;
    // a time-filtered pass 0 scans tfilt->n_scan raw rows and writes the n kept ones
    const int64_t n0 = tfilt ? tfilt->n_scan : n;
    const int64_t tiles0 = (n0 + SORT_TILE - 1) / SORT_TILE;
    const int64_t tiles = std::max<int64_t>((n + SORT_TILE - 1) / SORT_TILE, tiles0);   // look-back rows per pass
    Scratch aux(s), tmp(s);
    const size_t status_words = (size_t)tiles * RADIX * passes;
    PM4G_TRY(aux.alloc(status_words * sizeof(st_t) + (passes + 2 * MAX_PASSES * RADIX) * 4));
    st_t* status = aux.as<st_t>();
    uint32_t* counters = (uint32_t*)(status + status_words);
    uint32_t* hist = counters + passes;
    uint32_t* off = hist + MAX_PASSES * RADIX;
    // pass 0's look-back words, the tile counters and histograms; pass p zeroes pass p+1's words
    PM4G_CK(cudaMemsetAsync(status, 0, (size_t)tiles * RADIX * sizeof(st_t), s));
    PM4G_CK(cudaMemsetAsync(counters, 0, (passes + MAX_PASSES * RADIX) * 4, s));
    if (pre_hist) {   // histograms already built (by the validation pass)
        PM4G_LAUNCH("k_hist_scan", 0, s, k_hist_scan<<<1, RADIX, 0, s>>>(pre_hist, off, passes));
    } else {
        const int g = std::max(1, std::min<int>((int)((n + 255) / 256), num_sms() * 4));
        if (from_cols)
            PM4G_LAUNCH("k_hist", n0 * (tfilt ? 12.0 : 4.0), s,
                        (k_hist<true><<<g, 256, 0, s>>>(nullptr, in_case, n0, kp.case_min, 0, bits, passes, hist,
                                                        tfilt ? in_ts : nullptr, tfilt ? tfilt->t1 : 0,
                                                        tfilt ? tfilt->t2 : 0)));
        else
            PM4G_LAUNCH("k_hist", n * 8.0, s,
                        (k_hist<false><<<g, 256, 0, s>>>(in_key, nullptr, n, 0, shift0, bits, passes, hist)));
        PM4G_LAUNCH("k_hist_scan", 0, s, k_hist_scan<<<1, RADIX, 0, s>>>(hist, off, passes));
    }
    // ping-pong buffer: key (8n) | idx (4n) | act
    auto up16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
    const size_t o_idx = up16((size_t)n * 8), o_act = up16(o_idx + (WI ? (size_t)n * 4 : 0));
    PM4G_TRY(tmp.alloc(o_act + ((size_t)n + 32) * sizeof(P) + 64));
    uint64_t* tkey = tmp.as<uint64_t>();
    uint32_t* tidx = (uint32_t*)((char*)tmp.p + o_idx);
    P* tact = (P*)((char*)tmp.p + o_act);
    const uint64_t* ck = in_key;
    const P* ca = in_act;
    const uint32_t* ci = in_idx;
    for (int p = 0; p < passes; ++p) {
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        uint64_t* ok = to_out ? key_out : tkey;
        P* oa = to_out ? act_out : tact;
        uint32_t* oi = to_out ? idx_out : tidx;
        const int shift = shift0 + p * bits;
        const double wr = 8.0 + sizeof(P) + (WI ? 4 : 0);
        if (p == 0 && from_cols) {
            PassArgs<P, true, WI> a{nullptr, in_case, in_ts, ca, ci, ok, oa, oi, n0, shift, bits, kp,
                                    off, status, counters,
                                    aligned16(in_case) && aligned16(in_ts) && aligned16(ca) &&
                                        (!ci || aligned16(ci)),
                                    p + 1 < passes ? status + (size_t)(p + 1) * tiles * RADIX : nullptr};
            a.case_col = wide_case;
            a.wshift = 0;
            if (tfilt) {
                a.tf = 1;
                a.tf_t1 = tfilt->t1;
                a.tf_t2 = tfilt->t2;
            }
            PM4G_TRY(launch_pass(a, tiles0, s, pass_name, n0 * (12.0 + sizeof(P) + (ci ? 4 : 0)) + n * wr));
        } else {
            PassArgs<P, false, WI> a{ck, nullptr, nullptr, ca, ci, ok, oa, oi, n, shift, bits, kp,
                                     off + p * RADIX, status + (size_t)p * tiles * RADIX, counters + p,
                                     aligned16(ck) && aligned16(ca) && (!ci || aligned16(ci)),
                                     p + 1 < passes ? status + (size_t)(p + 1) * tiles * RADIX : nullptr};
            a.case_col = wide_case;
            a.wshift = p * bits;
            PM4G_TRY(launch_pass(a, (n + SORT_TILE - 1) / SORT_TILE, s, pass_name,
                                 n * ((ci ? wr : wr - (WI ? 4 : 0)) + wr + (wide_case ? 4.0 : 0.0))));
        }
        ck = ok;
        ca = oa;
        ci = oi;
    }
    return PM4G_OK;
}

// ------------------------------------------------------------------ A4 + format
// Input: composite keys grouped by case (stable), activity (+ ingest row).
// Per tile of 4096 positions: heads (case starts) -> ranks via look-back ->
// case offsets; each case owned by this tile (head inside it) is sorted by key
// in shared memory.  A case may run up to FMT_EXT positions past the tile end;
// longer ones (and cases over FMT_WARP_MAX rows) go to the exact fallback.
constexpr int FMT_THREADS = PM4G_FMT_THREADS, FMT_IPT = PM4G_FMT_IPT, FMT_TILE = FMT_THREADS * FMT_IPT;
constexpr int FMT_EXT = 512, FMT_BUF = FMT_TILE + FMT_EXT;
constexpr int FMT_WARP_MAX = 1024;  // longer cases: exact fallback (stable radix sort)
constexpr int FMT_TIES = 512;       // tie groups listed per tile (more: laid out in place)

template <class P>
struct FmtArgs {
    const uint64_t* gkey;
    const P* gact;
    const uint32_t* gidx;
    int64_t n;
    int ts_bits;
    uint32_t case_min;
    uint64_t* key_out;
    P* act_out;
    uint32_t* perm_out;        // nullptr: no extra columns
    uint32_t* off;
    uint32_t* case_code;
    uint64_t* n_cases;
    st_t* status;
    uint32_t* counter;
    uint32_t* big;             // ranks of fallback cases
    uint32_t* big_count;
    bool aligned;              // gkey / gact / gidx 16-byte aligned (TMA bulk path)
    // wide logs: gkey = ts - ts_min, gidx = ingest row; the case of a row is
    // case_col[gidx] - case_min, written to rcase_out alongside the formatted row
    const uint32_t* case_col;
    uint32_t* rcase_out;
};

// the TMA targets (s_key at 0, s_act, s_idx) must stay 16-byte aligned
static_assert(((FMT_BUF * 8 + FMT_BUF * 2 * 2 + (FMT_TILE + 8) * 2 + (FMT_TILE + 16)) % 16) == 0, "s_act alignment");

template <class P, bool WI, bool WIDE = false>
__global__ __launch_bounds__(FMT_THREADS) void k_format(FmtArgs<P> a) {
    static_assert(!WIDE || WI, "the wide format reads the ingest-row payload");
    extern __shared__ __align__(16) unsigned char fsm[];
    uint64_t* s_key = (uint64_t*)fsm;                              // [FMT_BUF]
    uint16_t* s_perm = (uint16_t*)(s_key + FMT_BUF);               // [FMT_BUF] slot -> row
    uint16_t* s_ci = s_perm + FMT_BUF;                              // [FMT_BUF] case of each row
    uint16_t* s_head = s_ci + FMT_BUF;                             // [FMT_TILE + 8]
    uint8_t* s_wide = (uint8_t*)(s_head + FMT_TILE + 8);           // [FMT_TILE + 16] case needs 64-bit ranks
    P* s_act = (P*)(s_wide + FMT_TILE + 16);                       // [FMT_BUF] (16-byte aligned: TMA target)
    uint32_t* s_idx = (uint32_t*)(((uintptr_t)(s_act + FMT_BUF) + 15) & ~(uintptr_t)15);  // WI only
    uint32_t* s_c = s_idx + FMT_BUF;                                                      // WIDE: case of each row
    __shared__ uint32_t s_tile, s_wt[FMT_THREADS / 32], s_scan[FMT_THREADS / 32 + 1];
    __shared__ uint32_t s_prefix, s_nbig, s_bigh[16], s_ntie, s_anywide;
    __shared__ uint16_t s_tie[FMT_TIES];   // slots starting a group of equal keys
    __shared__ int s_ext, s_wlast[FMT_THREADS / 32];
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(a.counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * FMT_TILE;
    const int tn = (int)min((int64_t)FMT_TILE, a.n - base);
    const int tb = a.ts_bits;
    const uint32_t lt = lanemask_lt();

    // ---- 1. the tile's rows -> smem (TMA bulk copies for full tiles), head ballots
    const bool bulk = tn == FMT_TILE && a.aligned;
    // the FMT_EXT rows after the tile come in the same transfer when they exist
    // (the tile's last case may run into them): the extension scan and rows then
    // read shared memory instead of waiting on global loads (11% of a tile's time)
    const bool xbulk = !WIDE && bulk && base + FMT_BUF <= a.n;
    if (bulk) {
        if (tid == 0) {
            const uint32_t rows = xbulk ? FMT_BUF : FMT_TILE;
            mbar_init(&s_bar, 1);
            mbar_expect_tx(&s_bar, rows * (uint32_t)(8 + sizeof(P) + (WI ? 4 : 0)));
            tma_load_1d(s_key, a.gkey + base, rows * 8, &s_bar);
            tma_load_1d(s_act, a.gact + base, rows * (uint32_t)sizeof(P), &s_bar);
            if (WI) tma_load_1d(s_idx, a.gidx + base, rows * 4, &s_bar);
        }
    } else {
        for (int p = tid; p < tn; p += FMT_THREADS) {
            s_key[p] = a.gkey[base + p];
            s_act[p] = a.gact[base + p];
            if (WI) s_idx[p] = a.gidx[base + p];
        }
    }
    // the case of global row i (case - case_min)
    auto gcase = [&](int64_t i) -> uint32_t {
        return WIDE ? a.case_col[a.gidx[i]] - a.case_min : case32(a.gkey[i], tb);
    };
    uint32_t prev_case = 0;
    {
        const int64_t pi = base + warp * (32 * FMT_IPT) - 1;
        if (pi >= 0 && pi < a.n) prev_case = gcase(pi);
    }
    __syncthreads();
    if (bulk) mbar_wait(&s_bar, 0);
    if (WIDE) {
        for (int p = tid; p < tn; p += FMT_THREADS) s_c[p] = a.case_col[s_idx[p]] - a.case_min;
        __syncthreads();
    }
    uint32_t ball[FMT_IPT], wc = 0;
    {
        uint32_t prev = prev_case;
#pragma unroll
        for (int j = 0; j < FMT_IPT; ++j) {
            const int li = warp * (32 * FMT_IPT) + j * 32 + lane;
            const int64_t i = base + li;
            const bool ok = li < tn;
            const uint32_t c = ok ? (WIDE ? s_c[li] : case32(s_key[li], tb)) : 0u;
            uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
            if (lane == 0) pc = prev;
            prev = __shfl_sync(0xffffffffu, c, 31);
            ball[j] = __ballot_sync(0xffffffffu, ok && (i == 0 || c != pc));
            wc += __popc(ball[j]);
        }
    }
    // last head of this warp (for the tile-extension scan)
    int lasth = -1;
#pragma unroll
    for (int j = 0; j < FMT_IPT; ++j)
        if (ball[j]) lasth = warp * (32 * FMT_IPT) + j * 32 + (31 - __clz(ball[j]));
    if (lane == 0) {
        s_wt[warp] = wc;
        s_wlast[warp] = lasth;
    }
    __syncthreads();
    // warp-exclusive head count, total heads H and the tile's last head, by
    // lane-parallel scans over the 16 warp entries (every warp computes them)
    uint32_t H, wex;
    int lastp;
    {
        constexpr int NWF = FMT_THREADS / 32;
        const uint32_t cw = lane < NWF ? s_wt[lane] : 0u;
        int lw = lane < NWF ? s_wlast[lane] : -1;
        uint32_t inc = cw;
#pragma unroll
        for (int o = 1; o < NWF; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
            lw = max(lw, __shfl_xor_sync(0xffffffffu, lw, o));
        }
        H = __shfl_sync(0xffffffffu, inc, NWF - 1);
        wex = __shfl_sync(0xffffffffu, inc - cw, warp);
        lastp = __shfl_sync(0xffffffffu, lw, 0);   // the max over lanes 0..15
    }

    // ---- 2. concurrently: every warp writes its heads and row->case indices;
    // warp 0 then runs the case-rank look-back, warp 1 finds how far the last
    // case runs past the tile end
    {
        uint32_t r = wex;
#pragma unroll
        for (int j = 0; j < FMT_IPT; ++j) {
            const int li = warp * (32 * FMT_IPT) + j * 32 + lane;
            const uint32_t b = ball[j];
            const uint32_t incl = r + __popc(b & (lt | (1u << lane)));   // heads at positions <= li
            if (b & (1u << lane)) s_head[incl - 1] = (uint16_t)li;
            if (li < tn) {
                s_ci[li] = incl ? (uint16_t)(incl - 1) : (uint16_t)0xffff;  // 0xffff: previous tile's case
                s_perm[li] = (uint16_t)0xffff;                                // slots start empty
            }
            r += __popc(b);
        }
    }
    if (tid < 16) s_bigh[tid] = 0;
    if (tid == 0) {
        s_nbig = 0;
        s_anywide = 0;
        s_ntie = 0;
    }
    for (uint32_t h = tid; h < H; h += FMT_THREADS) s_wide[h] = 0;
    __syncthreads();

    // ---- 3. warp 0 resolves the case ranks (decoupled look-back) while warps
    // 1..7 sort the tile; the workers synchronise on named barrier 1
    if (warp == 0) {
        const uint32_t pf = lookback_warp_k<8>(a.status, tile, H);
        if (lane == 0) s_prefix = pf;
    } else if (H > 0) {
        constexpr int NW = FMT_THREADS - 32;
        const int wt = tid - 32;
        auto wsync = [] { asm volatile("bar.sync 1, %0;" ::"n"(FMT_THREADS - 32) : "memory"); };
        if (warp == 1) {   // how far the last case runs past the tile end
            int ext = 0;
            if (base + tn < a.n) {
                const uint64_t last = s_key[lastp];
                const uint32_t lastc = WIDE ? s_c[lastp] : 0u;
                ext = -1;
                for (int o = 0; o <= FMT_EXT; o += 32) {
                    const int64_t i = base + tn + o + lane;
                    const bool stop = i >= a.n || (WIDE ? gcase(i) != lastc
                                                        : !same_case(xbulk && o + lane < FMT_EXT ? s_key[tn + o + lane] : a.gkey[i],
                                                                     last, tb));
                    const uint32_t bb = __ballot_sync(0xffffffffu, stop);
                    if (bb) {
                        const int e = o + __ffs(bb) - 1;
                        ext = e <= FMT_EXT ? e : -1;
                        break;
                    }
                }
            }
            if (lane == 0) s_ext = ext;
        }
        wsync();
        int ext = s_ext;
        int Hown = (int)H;
        if (ext < 0) {   // the last case runs far past the tile: exact fallback, not owned here
            Hown = (int)H - 1;
            ext = 0;
            if (wt == 0) s_bigh[atomicAdd(&s_nbig, 1u) & 15] = H - 1;
        }
        const int h0 = s_head[0];
        const int oend = Hown == (int)H ? tn + ext : (int)s_head[H - 1];   // owned rows [h0, oend)
        for (int p = tn + wt; p < oend; p += NW) {                          // extension rows
            const int64_t i = base + p;
            if (!xbulk) {
                s_key[p] = a.gkey[i];
                s_act[p] = a.gact[i];
                if (WI) s_idx[p] = a.gidx[i];
            }
            if (WIDE) s_c[p] = a.case_col[s_idx[p]] - a.case_min;
            s_ci[p] = (uint16_t)(H - 1);
            s_perm[p] = (uint16_t)0xffff;
        }
        wsync();

        // ---- 4. rank each row inside its case and claim slot s0 + rank (slots
        // = output positions, the case's own row range; they start empty).
        // Narrow cases (every key within +-2^30 of the case's first key, so any
        // two keys differ by < 2^31): rank = #(key_j < key_p), the sign of the
        // 32-bit low-word difference (exact, modular), one subtract + sign per
        // element; rows with equal keys (ties) claim the same slot, leaving
        // empty slots behind it, and phase 5 lays the tied rows out in ingest
        // order.  Every case is ranked narrow first while each row checks its
        // own key against the case's first; a case found wide (rare: a case
        // spanning > 2^30 key units) is re-ranked below with the exact stable
        // rank.  Rows of a fallback case (> FMT_WARP_MAX rows) mark their own
        // slot 0xfffe.  Event-parallel with one loop per case (a warp mostly
        // reads one case -> broadcast smem reads).
        for (int p = h0 + wt; p < oend; p += NW) {
            const uint32_t h = s_ci[p];
            const int s0 = s_head[h], e0 = ((int)h + 1 < Hown) ? s_head[h + 1] : oend;
            if (e0 - s0 > FMT_WARP_MAX) {   // long case: exact fallback
                s_perm[p] = (uint16_t)0xfffe;
                if (p == s0) s_bigh[atomicAdd(&s_nbig, 1u) & 15] = h;
                continue;
            }
            int r = 0;
            const uint64_t ki = s_key[p];
            const int64_t d = (int64_t)(ki - s_key[s0]);
            if (d < -(1ll << 30) || d >= (1ll << 30)) {
                s_wide[h] = 1;
                s_anywide = 1;
            }
            const uint32_t* lo = (const uint32_t*)(s_key + s0);   // low word of key s0 + j at lo[2 j]
            const uint32_t ti = (uint32_t)ki;
            const int m = e0 - s0;
            // four elements per trip, the < 4 left over predicated (no
            // remainder loops: lanes of one warp have different m)
            int j = 0;
#pragma unroll 1
            for (; j + 4 <= m; j += 4)
                r += (int)(((lo[2 * j] - ti) >> 31) + ((lo[2 * j + 2] - ti) >> 31) +
                           ((lo[2 * j + 4] - ti) >> 31) + ((lo[2 * j + 6] - ti) >> 31));
            if (j < m) r += (int)((lo[2 * j] - ti) >> 31);
            if (j + 1 < m) r += (int)((lo[2 * j + 2] - ti) >> 31);
            if (j + 2 < m) r += (int)((lo[2 * j + 4] - ti) >> 31);
            s_perm[s0 + r] = (uint16_t)p;   // (a wide case's claims stay inside its own slots)
        }
        wsync();
        if (s_anywide) {   // wide cases: clear their slots, then the exact stable rank (unique slots)
            for (int p = h0 + wt; p < oend; p += NW)
                if (s_wide[s_ci[p]]) s_perm[p] = (uint16_t)0xffff;
            wsync();
            for (int p = h0 + wt; p < oend; p += NW) {
                const uint32_t h = s_ci[p];
                if (!s_wide[h]) continue;
                const int s0 = s_head[h], e0 = ((int)h + 1 < Hown) ? s_head[h + 1] : oend;
                const uint64_t ki = s_key[p], ki1 = ki + 1;
                int r = 0;
                if (ki1 != 0) {   // the all-ones key (key_bits = 64) has no successor
                    for (int j = s0; j < e0; ++j) r += s_key[j] < (j < p ? ki1 : ki);
                } else {
                    for (int j = s0; j < e0; ++j) r += (s_key[j] < ki) | ((s_key[j] == ki) & (j < p));
                }
                s_perm[s0 + r] = (uint16_t)p;
            }
            wsync();
        }

        // ---- 5. write the formatted rows of the owned range, slot by slot
        // (consecutive threads, consecutive output rows).  A slot followed by
        // an empty one starts a group of equal keys: those are listed and laid
        // out in ingest order after the loop.
        auto put = [&](int src, int slot) {
            const int64_t g = base + slot;
            a.key_out[g] = s_key[src];
            a.act_out[g] = s_act[src];
            if (WI && a.perm_out) a.perm_out[g] = s_idx[src];
            if (WIDE) a.rcase_out[g] = s_c[src];
        };
        auto ties = [&](int q) {   // slots q, q+1, ... <- the rows of key(s_perm[q]), ascending row
            const int p = s_perm[q];
            const uint32_t h = s_ci[p];
            const int s0 = s_head[h], e0 = ((int)h + 1 < Hown) ? s_head[h + 1] : oend;
            const uint64_t kq = s_key[p];
            for (int j = s0, o = q; j < e0; ++j)
                if (s_key[j] == kq) put(j, o++);
        };
        for (int q = h0 + wt; q < oend; q += NW) {
            const uint32_t p = s_perm[q];
            if (p >= 0xfffe) continue;   // a fallback case's row, or an empty slot after a tie
            if (q + 1 < oend && s_perm[q + 1] == 0xffff) {
                const uint32_t t = atomicAdd(&s_ntie, 1u);
                if (t < FMT_TIES) s_tie[t] = (uint16_t)q;
                else ties(q);
                continue;
            }
            put((int)p, q);
        }
        wsync();
        for (uint32_t t = wt; t < min(s_ntie, (uint32_t)FMT_TIES); t += NW) ties(s_tie[t]);
    }
    __syncthreads();

    // ---- 6. case offsets and codes (ranks known now)
    const uint32_t R0 = s_prefix;
    for (uint32_t h = tid; h < H; h += FMT_THREADS) {
        const int hp = s_head[h];
        a.off[R0 + h] = (uint32_t)(base + hp);
        a.case_code[R0 + h] = a.case_min + (WIDE ? s_c[hp] : case32(s_key[hp], tb));
    }
    if (tid < min(s_nbig, 16u)) a.big[atomicAdd(a.big_count, 1u)] = R0 + s_bigh[tid];
    if (tid == 0 && base + tn >= a.n) {
        a.off[R0 + H] = (uint32_t)a.n;
        *a.n_cases = R0 + H;
    }
}

// ---- the exact fallback, batched over every listed case (one segmented sort):
// the rows of all listed cases are concatenated (segments ordered by start
// row), sorted stably by key, then stably by segment, and scattered back to
// their case's rows -- ties keep the grouped (= ingest) order inside a case.
// seg_start[j] / seg_pre[j]: start row / concatenation offset of segment j.
__device__ __forceinline__ uint32_t seg_of(const uint64_t* __restrict__ seg_pre, uint32_t nseg, uint64_t q) {
    uint32_t lo = 0, hi = nseg;   // last j with seg_pre[j] <= q
    while (hi - lo > 1) {
        const uint32_t m = (lo + hi) >> 1;
        if (seg_pre[m] <= q) lo = m; else hi = m;
    }
    return lo;
}
__global__ void k_big_bounds(const uint32_t* __restrict__ big, uint32_t nbig, const uint32_t* __restrict__ off,
                             uint32_t* __restrict__ se) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nbig; j += gridDim.x * blockDim.x) {
        se[2 * j] = off[big[j]];
        se[2 * j + 1] = off[big[j] + 1];
    }
}
__global__ void k_big_keys(const uint64_t* __restrict__ gkey, const uint64_t* __restrict__ seg_start,
                           const uint64_t* __restrict__ seg_pre, uint32_t nseg, uint64_t T,
                           uint64_t* __restrict__ k, uint32_t* __restrict__ v) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < T; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = seg_of(seg_pre, nseg, q);
        const uint64_t row = seg_start[j] + (q - seg_pre[j]);
        k[q] = gkey[row];
        v[q] = (uint32_t)row;
    }
}
__global__ void k_big_segkeys(const uint32_t* __restrict__ v, const uint64_t* __restrict__ seg_start, uint32_t nseg,
                              uint64_t T, uint64_t* __restrict__ k) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < T; q += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nseg;   // segment holding row v[q]
        while (hi - lo > 1) {
            const uint32_t m = (lo + hi) >> 1;
            if (seg_start[m] <= v[q]) lo = m; else hi = m;
        }
        k[q] = lo;
    }
}
template <class P>
__global__ void k_big_gather(FmtArgs<P> a, const uint64_t* __restrict__ seg_start, const uint64_t* __restrict__ seg_pre,
                             uint32_t nseg, uint64_t T, const uint32_t* __restrict__ v) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < T; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = seg_of(seg_pre, nseg, q);
        const uint64_t dst = seg_start[j] + (q - seg_pre[j]);
        const uint32_t src = v[q];
        a.key_out[dst] = a.gkey[src];
        a.act_out[dst] = a.gact[src];
        if (a.perm_out) a.perm_out[dst] = a.gidx[src];
        if (a.rcase_out) a.rcase_out[dst] = a.case_col[a.gidx[src]] - a.case_min;
    }
}

// Rows of the cases k_format listed for the exact fallback are not written by
// k_format.  Before the (deferred) fallback runs, the provisional order must
// still hold valid codes for every row: copy those cases' grouped rows through
// unchanged (same case, ingest order), so anything derived from the provisional
// order stays in bounds; the fallback then overwrites them with the exact order.
template <class P>
__global__ void k_big_identity(const uint32_t* __restrict__ big, const uint32_t* __restrict__ big_count,
                               const uint32_t* __restrict__ off, const uint64_t* __restrict__ gkey,
                               const P* __restrict__ gact, uint64_t* __restrict__ key_out, P* __restrict__ act_out) {
    const uint32_t nb = *big_count;
    for (uint32_t e = blockIdx.x; e < nb; e += gridDim.x) {
        const uint32_t r = big[e];
        const uint32_t a = off[r], b = off[r + 1];
        for (uint32_t i = a + threadIdx.x; i < b; i += blockDim.x) {
            key_out[i] = gkey[i];
            act_out[i] = gact[i];
        }
    }
}

// launch k_format; st holds its scratch (tile status, fallback list + count)
template <class P>
static pm4g_status format_launch(FmtArgs<P>& fa, Scratch& st, cudaStream_t s) {
    const int64_t n = fa.n;
    const int64_t tiles = (n + FMT_TILE - 1) / FMT_TILE;
    // [status st_t: tiles] [counter, big_count] [big list]
    const size_t words = 2 + ((size_t)n / FMT_WARP_MAX + tiles + 2);
    PM4G_TRY(st.alloc((size_t)tiles * sizeof(st_t) + words * 4));
    PM4G_CK(cudaMemsetAsync(st.p, 0, (size_t)tiles * sizeof(st_t) + 8, s));
    fa.status = st.as<st_t>();
    fa.counter = (uint32_t*)(fa.status + tiles);
    fa.big_count = fa.counter + 1;
    fa.big = fa.counter + 2;
    const bool wide = fa.rcase_out != nullptr;
    const bool wi = fa.gidx != nullptr;
    fa.aligned = aligned16(fa.gkey) && aligned16(fa.gact) && (!wi || aligned16(fa.gidx));
    const size_t smem_base = (size_t)FMT_BUF * (8 + 2 + 2 + sizeof(P)) + (FMT_TILE + 8) * 2 + (FMT_TILE + 16) + 16;
    const size_t smem = smem_base + (wi ? (size_t)FMT_BUF * 4 : 0) + (wide ? (size_t)FMT_BUF * 4 : 0);
    PM4G_MAX_SMEM(k_format<P, false>);
    PM4G_MAX_SMEM(k_format<P, true>);
    PM4G_MAX_SMEM(k_format<P, true, true>);
    const double bytes = (double)n * (2.0 * (8 + sizeof(P) + (wi ? 4 : 0)) + (wide ? 8.0 : 0.0));
    if (wide)
        PM4G_LAUNCH("k_format", bytes, s, (k_format<P, true, true><<<(unsigned)tiles, FMT_THREADS, smem, s>>>(fa)));
    else if (wi)
        PM4G_LAUNCH("k_format", bytes, s, (k_format<P, true><<<(unsigned)tiles, FMT_THREADS, smem, s>>>(fa)));
    else
        PM4G_LAUNCH("k_format", bytes, s, (k_format<P, false><<<(unsigned)tiles, FMT_THREADS, smem, s>>>(fa)));
    return PM4G_OK;
}

// the exact fallback for the nbig cases k_format listed (too long, or running
// too far past a tile): one batched segmented sort of all their rows (two host
// round trips in all: the list size, then the segment bounds)
template <class P>
static pm4g_status format_fallback(const FmtArgs<P>& fa, uint32_t nbig, cudaStream_t s) {
    Scratch se(s);
    PM4G_TRY(se.alloc((size_t)nbig * 8));
    const int gb = std::max(1, std::min<int>((int)((nbig + 255) / 256), num_sms()));
    PM4G_LAUNCH("k_big_bounds", nbig * 12.0, s, (k_big_bounds<<<gb, 256, 0, s>>>(fa.big, nbig, fa.off, se.as<uint32_t>())));
    std::vector<uint32_t> h(2 * (size_t)nbig);
    pm4g_status gs;
    const bool seg = gseg_suspend(s, &gs);   // (a pageable copy cannot sit in a graph segment)
    PM4G_TRY(gs);
    PM4G_CK(cudaMemcpyAsync(h.data(), se.p, (size_t)nbig * 8, cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    if (seg) PM4G_TRY(gseg_resume());
    std::vector<std::pair<uint64_t, uint64_t>> segs;   // (start, len), ascending start
    for (uint32_t j = 0; j < nbig; ++j)
        if (h[2 * j + 1] > h[2 * j]) segs.push_back({h[2 * j], (uint64_t)h[2 * j + 1] - h[2 * j]});
    std::sort(segs.begin(), segs.end());
    const uint32_t nseg = (uint32_t)segs.size();
    if (!nseg) return PM4G_OK;
    std::vector<uint64_t> meta(2 * (size_t)nseg + 1);   // seg_start[nseg] | seg_pre[nseg + 1]
    uint64_t T = 0;
    for (uint32_t j = 0; j < nseg; ++j) {
        meta[j] = segs[j].first;
        meta[nseg + j] = T;
        T += segs[j].second;
    }
    meta[2 * nseg] = T;
    Scratch md(s), kv(s);
    PM4G_TRY(md.alloc(meta.size() * 8));
    PM4G_CK(cudaMemcpyAsync(md.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, s));
    const uint64_t* seg_start = md.as<uint64_t>();
    const uint64_t* seg_pre = seg_start + nseg;
    PM4G_TRY(kv.alloc((size_t)T * 12 + 16));
    uint64_t* k = kv.as<uint64_t>();
    uint32_t* v = (uint32_t*)(k + T);
    const int g = std::max(1, std::min<int>((int)((T + 255) / 256), num_sms() * 4));
    PM4G_LAUNCH("k_big_keys", T * 20.0, s, (k_big_keys<<<g, 256, 0, s>>>(fa.gkey, seg_start, seg_pre, nseg, T, k, v)));
    // by key (the case bits are equal inside a segment), then stably by segment
    PM4G_TRY(radix_sort_u64(k, v, (int64_t)T, std::min(64, std::max(1, fa.ts_bits)), s));
    if (nseg > 1) {
        PM4G_LAUNCH("k_big_segkeys", T * 12.0, s, (k_big_segkeys<<<g, 256, 0, s>>>(v, seg_start, nseg, T, k)));
        PM4G_TRY(radix_sort_u64(k, v, (int64_t)T, std::max(1, bit_width_u64(nseg - 1)), s));
    }
    PM4G_LAUNCH("k_big_gather", T * 30.0, s, (k_big_gather<P><<<g, 256, 0, s>>>(fa, seg_start, seg_pre, nseg, T, v)));
    return PM4G_OK;
}

template <class P>
static pm4g_status format_log(const FmtArgs<P>& fa0, cudaStream_t s) {
    FmtArgs<P> fa = fa0;
    Scratch st(s);
    PM4G_TRY(format_launch<P>(fa, st, s));
    uint32_t nbig = 0;
    pm4g_status gs;
    const bool seg = gseg_suspend(s, &gs);   // (a pageable copy cannot sit in a graph segment)
    PM4G_TRY(gs);
    PM4G_CK(cudaMemcpyAsync(&nbig, fa.big_count, 4, cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    if (seg) PM4G_TRY(gseg_resume());
    return nbig ? format_fallback<P>(fa, nbig, s) : PM4G_OK;
}

// (test hook) flag any activity code >= A in the formatted columns
template <class P>
__global__ void k_check_acts(const P* __restrict__ act, int64_t n, uint32_t A, uint32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if ((uint32_t)act[i] >= A) atomicExch(bad, 1u);
}

template <class P>
static pm4g_status sort_log_t(pm4g_log* L, cudaStream_t s, FmtDeferred* d) {
    const int64_t n = L->n;
    // the ingest row travels with every row when extra columns must follow the
    // order (perm) or when the log is wide (the row's case is looked up by it)
    const bool wide = L->wide;
    const bool extras = !L->extra.empty();
    const bool wi = extras || wide;
    if (wi && L->tf_n >= 0) PM4G_TRY(materialize(L, s));   // (the lazy filter never leaves these)
    KeyParams kp{L->case_min, L->ts_min, L->ts_bits};
    // 1. stable LSD passes over the case bits of the composite key (built on the fly)
    Scratch grp(s);
    auto up16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
    const size_t o_idx = up16((size_t)n * 8), o_act = up16(o_idx + (wi ? (size_t)n * 4 : 0));
    PM4G_TRY(grp.alloc(o_act + ((size_t)n + 32) * sizeof(P) + 64));
    uint64_t* gkey = grp.as<uint64_t>();
    uint32_t* gidx = (uint32_t*)((char*)grp.p + o_idx);
    P* gact = (P*)((char*)grp.p + o_act);
    const uint32_t* pre = L->hist_passes > 0 ? L->hist : nullptr;
    if (wi)
        PM4G_TRY((lsd_sort<P, true>(L->case_, L->ts, nullptr, (const P*)L->act, nullptr, gkey, gact, gidx, n,
                                    wide ? 0 : L->ts_bits, L->case_bits, kp, s, "k_onesweep", pre,
                                    wide ? L->case_ : nullptr)));
    else {
        // a lazily time-filtered log: pass 0 scans the shared raw rows and keeps the filter's
        const TimeFilt tfv{L->tf_n, L->tf_t1, L->tf_t2};
        PM4G_TRY((lsd_sort<P, false>(L->case_, L->ts, nullptr, (const P*)L->act, nullptr, gkey, gact, nullptr,
                                     n, L->ts_bits, L->case_bits, kp, s, "k_onesweep", pre, nullptr,
                                     L->tf_n >= 0 ? &tfv : nullptr)));
    }
    // 2. per-case timestamp order + case offsets
    FmtArgs<P> fa{};
    fa.gkey = gkey;
    fa.gact = gact;
    fa.gidx = wi ? gidx : nullptr;
    fa.n = n;
    fa.ts_bits = L->ts_bits;
    fa.case_min = L->case_min;
    fa.key_out = L->key;
    fa.act_out = (P*)L->s_act;
    fa.perm_out = extras ? L->perm : nullptr;
    fa.case_col = wide ? L->case_ : nullptr;
    fa.rcase_out = wide ? L->rcase : nullptr;
    fa.off = L->off;
    fa.case_code = L->s_case_code;
    fa.n_cases = L->d_n_cases;
    if (!d) return format_log<P>(fa, s);
    // deferred: no host wait here; the caller runs sort_finish at its next
    // synchronisation (the grouped keys stay alive for the fallback)
    d->st.s = s;
    // test hook: every formatted row must hold a valid code before the deferred
    // fallback (the analysis reads the provisional order first)
    static const bool poison = getenv("PM4G_DEBUG_POISON_FORMAT") != nullptr;
    if (poison && n) PM4G_CK(cudaMemsetAsync(fa.act_out, 0xff, (size_t)n * sizeof(P), s));
    PM4G_TRY(format_launch<P>(fa, d->st, s));
    // fallback cases hold their grouped rows until the fallback runs (no stale bytes);
    // writing them inside k_format instead cost that kernel 2% at 100M
    PM4G_LAUNCH("k_big_identity", 0, s,
                (k_big_identity<P><<<num_sms(), 256, 0, s>>>(fa.big, fa.big_count, fa.off, fa.gkey, fa.gact,
                                                              fa.key_out, fa.act_out)));
    if (poison && n) {
        Scratch fl(s);
        PM4G_TRY(fl.alloc(16));
        PM4G_CK(cudaMemsetAsync(fl.p, 0, 4, s));
        PM4G_LAUNCH("k_check_acts", n * (double)sizeof(P), s,
                    (k_check_acts<P><<<num_sms() * 4, 256, 0, s>>>(fa.act_out, n, L->A, fl.as<uint32_t>())));
        uint32_t bad = 0;
        PM4G_CK(cudaMemcpyAsync(&bad, fl.p, 4, cudaMemcpyDeviceToHost, s));
        PM4G_CK(cudaStreamSynchronize(s));
        if (bad) return fail(PM4G_ECUDA, "formatted rows left unwritten before the deferred fallback");
    }
    // the fallback count goes to pinned host memory now (stream order); the
    // caller's own synchronisation later makes it readable without a wait.
    // Events belong to the device current at creation: one per device.
    constexpr int MAXDEV = 64;
    static thread_local uint32_t* h_nbig = nullptr;
    static thread_local cudaEvent_t evs[MAXDEV] = {};
    int dev = 0;
    PM4G_CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= MAXDEV) return fail(PM4G_EINVAL, "device ordinal out of range");
    if (!h_nbig) PM4G_CK(cudaHostAlloc((void**)&h_nbig, 4, cudaHostAllocPortable));
    if (!evs[dev]) PM4G_CK(cudaEventCreateWithFlags(&evs[dev], cudaEventDisableTiming));
    cudaEvent_t ev = evs[dev];
    d->h_nbig = h_nbig;
    d->ev = ev;
    d->d_nbig = fa.big_count;   // copied by sort_defer_copy (after the aggregate launch)
    d->grp.take(grp);
    static_assert(sizeof(FmtArgs<P>) <= sizeof(d->fa_raw), "type-erased FmtArgs");
    memcpy(d->fa_raw, &fa, sizeof(fa));
    d->act_bytes = (int)sizeof(P);
    d->active = true;
    return PM4G_OK;
}

// ------------------------------------------------------------------ A4 segments
// flag[i] = (i == 0) || case(i) != case(i-1) ("the different groups are
// identified ... as the set of rows indices"); heads compacted in order give
// the CSR offsets of the cases dataframe.
constexpr int SEG_THREADS = 256, SEG_IPT = 16, SEG_TILE = SEG_THREADS * SEG_IPT;

__global__ __launch_bounds__(SEG_THREADS) void k_segments(const uint64_t* __restrict__ key,
                                                          const uint32_t* __restrict__ rcase,
                                                          int64_t n, int ts_bits, uint32_t case_min,
                                                          uint32_t* __restrict__ off,
                                                          uint32_t* __restrict__ case_code,
                                                          uint64_t* __restrict__ n_cases,
                                                          st_t* status, uint32_t* counter) {
    __shared__ uint32_t s_tile, s_warp_tot[SEG_THREADS / 32], s_scan[SEG_THREADS / 32 + 1];
    __shared__ uint32_t s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wbase = (int64_t)tile * SEG_TILE + warp * (32 * SEG_IPT);
    const uint32_t lt = lanemask_lt();
    uint32_t ballots[SEG_IPT];
    uint32_t cs[SEG_IPT];
    uint32_t prev_last = 0;
    {
        int64_t pi = wbase - 1;
        if (pi >= 0 && pi < n) prev_last = rcase ? rcase[pi] : case32(key[pi], ts_bits);
    }
    uint32_t wcount = 0;
#pragma unroll
    for (int j = 0; j < SEG_IPT; ++j) {
        int64_t i = wbase + j * 32 + lane;
        bool ok = i < n;
        uint32_t c = ok ? (rcase ? rcase[i] : case32(key[i], ts_bits)) : 0u;
        uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
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
        uint32_t pf = lookback_warp_k<8>(status, tile, total);
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
            case_code[rk] = case_min + cs[j];
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
    PM4G_TRY(st.alloc((tiles + 1) * sizeof(st_t)));
    PM4G_CK(cudaMemsetAsync(st.p, 0, (tiles + 1) * sizeof(st_t), s));
    st_t* status = st.as<st_t>();
    PM4G_LAUNCH("k_segments", n * 8.0, s,
                k_segments<<<(unsigned)tiles, SEG_THREADS, 0, s>>>(L->key, L->rcase, n, L->ts_bits, L->case_min,
                                                                  L->off, L->s_case_code,
                                                                  L->d_n_cases, status + 1, (uint32_t*)status));
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

template <class P>
static pm4g_status finish_t(FmtDeferred* d, cudaStream_t s, bool* fixed) {
    FmtArgs<P> fa;
    memcpy(&fa, d->fa_raw, sizeof(fa));
    PM4G_CK(cudaEventSynchronize(d->ev));   // normally complete already: no wait
    const uint32_t nbig = *d->h_nbig;
    if (nbig == 0) return PM4G_OK;
    *fixed = true;
    return format_fallback<P>(fa, nbig, s);
}

thread_local FmtDeferred* t_pending_format = nullptr;

pm4g_status sort_defer_copy(FmtDeferred* d, cudaStream_t s) {
    if (!d || !d->d_nbig) return PM4G_OK;
    PM4G_TRY(copy_words_to_host(d->h_nbig, d->d_nbig, 4, s));
    // (inside a captured graph segment the copy completes before the segment's
    // closing synchronisation, which sort_finish's read follows)
    if (!gseg_active()) PM4G_CK(cudaEventRecord(d->ev, s));
    d->d_nbig = nullptr;
    return PM4G_OK;
}

pm4g_status sort_finish(FmtDeferred* d, cudaStream_t s, bool* fixed) {
    *fixed = false;
    if (!d->active) return PM4G_OK;
    PM4G_TRY(sort_defer_copy(d, s));
    d->active = false;
    switch (d->act_bytes) {
        case 1: return finish_t<uint8_t>(d, s, fixed);
        case 2: return finish_t<uint16_t>(d, s, fixed);
        default: return finish_t<uint32_t>(d, s, fixed);
    }
}

pm4g_status sort_log(pm4g_log* L, cudaStream_t s, FmtDeferred* d) {
    // extra columns are gathered by the final order, and a wide log's format reads
    // the ingest columns: no deferral
    if (d && (!L->extra.empty() || L->wide)) d = nullptr;
    const int64_t n = L->n;
    const bool wi = !L->extra.empty();
    // +32 rows: 16-byte aligned TMA reads of the formatted log may run one vector past n
    PM4G_TRY(dalloc_t(&L->key, (size_t)n + 32, s));
    PM4G_TRY(dalloc(&L->s_act, ((size_t)n + 32) * L->act_bytes, s));
    if (wi) PM4G_TRY(dalloc_t(&L->perm, std::max<int64_t>(n, 1), s));
    if (L->wide) PM4G_TRY(dalloc_t(&L->rcase, (size_t)n + 32, s));
    // offsets: number of cases <= min(n, case range)
    dfree(L->off, s);
    dfree(L->s_case_code, s);
    const uint64_t cap = std::min<uint64_t>((uint64_t)n, (uint64_t)(L->case_max - L->case_min) + 1);
    PM4G_TRY(dalloc_t(&L->off, cap + 1, s));
    PM4G_TRY(dalloc_t(&L->s_case_code, std::max<uint64_t>(cap, 1), s));
    L->n_cases = -1;
    if (n == 0) {
        PM4G_LAUNCH("k_zero_cases", 0, s, k_zero_cases<<<1, 1, 0, s>>>(L->off, L->d_n_cases));
        L->n_cases = 0;
        return PM4G_OK;
    }
    switch (L->act_bytes) {
        case 1: PM4G_TRY(sort_log_t<uint8_t>(L, s, d)); break;
        case 2: PM4G_TRY(sort_log_t<uint16_t>(L, s, d)); break;
        default: PM4G_TRY(sort_log_t<uint32_t>(L, s, d)); break;
    }
    if (wi) PM4G_TRY(gather_extras(L, s));
    return PM4G_OK;
}

// generic (u64 key, u32 value) stable sort on `bits` low key bits, in place
pm4g_status radix_sort_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits, cudaStream_t s) {
    if (n <= 1) return PM4G_OK;
    Scratch out(s);
    PM4G_TRY(out.alloc((size_t)n * 12 + 16));
    uint64_t* ok = out.as<uint64_t>();
    uint32_t* ov = (uint32_t*)(ok + n);
    KeyParams kp{0, 0, 0};
    PM4G_TRY((lsd_sort<uint32_t, false>(nullptr, nullptr, keys, vals, nullptr, ok, ov, nullptr, n, 0,
                                        std::max(1, std::min(bits, 64)), kp, s, "k_onesweep_small")));
    PM4G_CK(cudaMemcpyAsync(keys, ok, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    PM4G_CK(cudaMemcpyAsync(vals, ov, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    return PM4G_OK;
}

// (key, u32 payload) sorted by key; only the payload is kept, written straight
// to vals_out (distinct from vals): no copy-back of the result
pm4g_status radix_sort_u64_to(const uint64_t* keys, const uint32_t* vals, uint32_t* vals_out, int64_t n,
                              int bits, cudaStream_t s) {
    if (n <= 0) return PM4G_OK;
    if (n == 1) {
        PM4G_CK(cudaMemcpyAsync(vals_out, vals, 4, cudaMemcpyDeviceToDevice, s));
        return PM4G_OK;
    }
    Scratch ko(s);
    PM4G_TRY(ko.alloc((size_t)n * 8 + 16));
    KeyParams kp{0, 0, 0};
    return lsd_sort<uint32_t, false>(nullptr, nullptr, keys, vals, nullptr, ko.as<uint64_t>(), vals_out, nullptr, n, 0,
                                     std::max(1, std::min(bits, 64)), kp, s, "k_onesweep_small");
}

// ------------------------------------------------------------------ decode (formatted log view)
template <class P>
__global__ void k_decode(const uint64_t* __restrict__ key, const uint32_t* __restrict__ rcase,
                         const P* __restrict__ sact, int64_t n,
                         int ts_bits, uint32_t case_min, int64_t ts_min, uint32_t* __restrict__ oc,
                         uint32_t* __restrict__ oa, int64_t* __restrict__ ot) {
    const uint64_t m = low_mask(ts_bits);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[i];
        if (oc) oc[i] = case_min + (rcase ? rcase[i] : (uint32_t)shr64(k, ts_bits));
        if (oa) oa[i] = (uint32_t)sact[i];
        if (ot) ot[i] = (int64_t)((uint64_t)ts_min + (k & m));
    }
}

}  // namespace pm4g

using namespace pm4g;

extern "C" pm4g_status pm4g_sorted_columns(const pm4g_log* L, uint32_t* case_code, uint32_t* act,
                                           int64_t* ts, pm4g_stream_t stream) {
    PM4G_TRY(check_log(L));
    if (!L->sorted) return fail(PM4G_EINVAL, "log is not sorted (call pm4g_sort)");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = L->n;
    if (n == 0) return PM4G_OK;
    int g = std::max(1, std::min<int>((int)((n + 255) / 256), num_sms() * 8));
    switch (L->act_bytes) {
        case 1: PM4G_LAUNCH("k_decode", n * 25.0, s, k_decode<uint8_t><<<g, 256, 0, s>>>(L->key, L->rcase, (const uint8_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
        case 2: PM4G_LAUNCH("k_decode", n * 26.0, s, k_decode<uint16_t><<<g, 256, 0, s>>>(L->key, L->rcase, (const uint16_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
        default: PM4G_LAUNCH("k_decode", n * 28.0, s, k_decode<uint32_t><<<g, 256, 0, s>>>(L->key, L->rcase, (const uint32_t*)L->s_act, n, L->ts_bits, L->case_min, L->ts_min, case_code, act, ts)); break;
    }
    return PM4G_OK;
}
