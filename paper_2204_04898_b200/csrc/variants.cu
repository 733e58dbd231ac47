// A9: variants -- group-count of cases by exact activity sequence.
//
// P:102-103 "This requires a double aggregation: first, the events need to be
// grouped in cases. Then this grouping is used to aggregate the cases into the
// variants."  P:113: the cases dataframe carries "numerical features that
// uniquely identify the case's variant" -- here a 128-bit key (two 64-bit
// polynomial hashes + length, computed in the fused pass A8).  Identity is the
// exact sequence (R10), so hashing is only an accelerator:
//
//   round r:  every unresolved item inserts its (salted) key into a device
//             open-addressing table (one 128-bit CAS claims a slot), adds its
//             weight, and atomicMin's its order key (-> the group's
//             representative = smallest case code, R11);
//             every item compares its sequence with its representative's;
//             mismatches (hash collisions) are taken back out of the group and
//             retried in round r+1 with a fresh salt.  Each round resolves at
//             least the representative's sequence of every slot, so the loop
//             terminates even with a degenerate hash (PM4G_DEBUG_WEAK_HASH=1
//             uses a 4-bit key to exercise exactly this path).
//
// The same engine merges per-shard variant tables (items = table entries,
// weight = count, order = representative case code) for the multi-GPU path.
// Output order: count desc, then representative case code asc (R11), via the
// library's radix sort on ((~count) << 32 | order).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

struct alignas(16) Slot {
    unsigned long long k1, k2;
    unsigned long long weight;
    unsigned int rep;   // min order key
    unsigned int len;
};
struct alignas(16) K128 {
    unsigned long long a, b;
};

__device__ __forceinline__ K128 ld_k128(const void* p) {
    K128 r;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.a), "=l"(r.b) : "l"(p));
    return r;
}

__device__ __forceinline__ uint64_t vmix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

__global__ void k_init_table(Slot* table, uint64_t cap) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x) {
        Slot z;
        z.k1 = 0;
        z.k2 = 0;
        z.weight = 0;
        z.rep = 0xffffffffu;
        z.len = 0;
        table[i] = z;
    }
}

// Find or claim the global slot of key (a, b): linear probing, one 128-bit CAS
// claims an empty slot (*claimed = true).  Returns the slot, or ~0 when the
// table is full or abandoned (ctl[0] = overflow flag, raised here or by the
// load-limit check in claim_count).
__device__ __forceinline__ uint64_t table_slot(Slot* table, uint64_t mask, uint64_t a, uint64_t b,
                                               uint32_t* ctl, bool* claimed) {
    uint64_t h = (a ^ (a >> 29) ^ (b * 0x9E3779B97F4A7C15ull)) & mask;
    for (uint64_t probes = 0; probes <= mask; ++probes) {
        Slot* sp = &table[h];
        K128 cur = ld_k128(sp);
        if (cur.a == a && cur.b == b) return h;
        if (cur.a == 0 && cur.b == 0) {
            K128 exp{0, 0}, des{a, b};
            K128 old = atomicCAS((K128*)sp, exp, des);
            if (old.a == 0 && old.b == 0) {
                *claimed = true;
                return h;
            }
            if (old.a == a && old.b == b) return h;
        }
        if ((probes & 31) == 31 && *(volatile uint32_t*)ctl) return ~0ull;
        h = (h + 1) & mask;
    }
    atomicExch(ctl, 1u);
    return ~0ull;
}

// Claimed slots, counted once per warp (ctl[1]); past the load limit (3/4 of
// the table) the table is abandoned (ctl[0] = 1), so an undersized table costs
// O(limit) claims instead of being probed to saturation.  Every claimed slot is
// appended to clist (claim order), so the compaction visits the claimed slots
// only, not the whole table.  Called by the active lanes together.
__device__ __forceinline__ void claim_count(bool claimed, uint64_t g, uint32_t* ctl, uint32_t limit,
                                            uint32_t* __restrict__ clist) {
    const uint32_t m = __activemask();
    const uint32_t b = __ballot_sync(m, claimed);
    if (!b) return;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)(threadIdx.x & 31) == leader) {
        const uint32_t c = __popc(b);
        base = atomicAdd(&ctl[1], c);
        if (base + c > limit) atomicExch(ctl, 1u);
    }
    base = __shfl_sync(m, base, leader);
    if (claimed) clist[base + __popc(b & lanemask_lt())] = (uint32_t)g;
}

// Items: t in [0, n_items) -> item list[t] (or t).  Each CTA first aggregates a
// chunk of items in a shared-memory table keyed by (k1, k2) -- so a hot variant
// (Zipf head) costs one global atomic per CTA, not one per case -- then
// publishes every distinct key of the chunk to the global table.
constexpr int INS_THREADS = 256, INS_IPT = 4, INS_CHUNK = INS_THREADS * INS_IPT, INS_SLOTS = 2048;
constexpr size_t INS_SMEM = (size_t)INS_SLOTS * (8 + 8 + 4 + 4 + 8 + 2);

template <class OFF>
__global__ __launch_bounds__(INS_THREADS) void k_insert(
    const uint32_t* __restrict__ list, uint64_t n_items, const uint64_t* __restrict__ k1,
    const uint64_t* __restrict__ k2, const OFF* __restrict__ off, const uint64_t* __restrict__ weight,
    const uint32_t* __restrict__ order, Slot* table, uint64_t mask, uint32_t limit, uint64_t salt,
    uint32_t* __restrict__ item_slot, uint8_t* __restrict__ pending, uint32_t* ctl,
    const uint64_t* __restrict__ d_n, uint32_t* __restrict__ clist) {
    extern __shared__ __align__(16) unsigned char ins_sm[];
    unsigned long long* s_k1 = (unsigned long long*)ins_sm;
    unsigned long long* s_k2 = s_k1 + INS_SLOTS;
    unsigned long long* s_g = s_k2 + INS_SLOTS;
    uint32_t* s_w = (uint32_t*)(s_g + INS_SLOTS);
    uint32_t* s_rep = s_w + INS_SLOTS;
    uint16_t* s_list = (uint16_t*)(s_rep + INS_SLOTS);
    __shared__ uint32_t s_scan[INS_THREADS / 32 + 1];
    __shared__ uint32_t s_stop;
    (void)off;
    if (d_n) n_items = min(n_items, *d_n);   // round 0 sized by an upper bound: the device count rules
    for (uint64_t chunk = blockIdx.x; chunk * INS_CHUNK < n_items; chunk += gridDim.x) {
        if (threadIdx.x == 0) s_stop = *(volatile uint32_t*)ctl;   // table abandoned: stop early
        for (int i = threadIdx.x; i < INS_SLOTS; i += INS_THREADS) {
            s_k1[i] = 0;
            s_w[i] = 0;
            s_rep[i] = 0xffffffffu;
        }
        __syncthreads();
        if (s_stop) break;
        uint32_t it[INS_IPT], loc[INS_IPT], ord[INS_IPT], w[INS_IPT];
        uint64_t ka[INS_IPT], kb[INS_IPT];
        bool claimed[INS_IPT], live[INS_IPT];
#pragma unroll
        for (int u = 0; u < INS_IPT; ++u) {
            const uint64_t t = chunk * INS_CHUNK + u * INS_THREADS + threadIdx.x;
            live[u] = t < n_items;
            claimed[u] = false;
            if (!live[u]) continue;
            it[u] = list ? list[t] : (uint32_t)t;
            uint64_t a = k1[it[u]], b = k2[it[u]];
            if (salt) {
                a = vmix(a ^ salt) | 1ull;
                b = vmix(b + salt);
            }
            ka[u] = a;
            kb[u] = b;
            w[u] = weight ? (uint32_t)weight[it[u]] : 1u;
            ord[u] = order ? order[it[u]] : it[u];
        }
        // phase A: claim / find the local slot by k1 (k1 is odd, never 0)
#pragma unroll
        for (int u = 0; u < INS_IPT; ++u) {
            if (!live[u]) continue;
            uint32_t h = (uint32_t)(ka[u] ^ (ka[u] >> 31)) & (INS_SLOTS - 1);
            while (true) {
                unsigned long long cur = s_k1[h];
                if (cur == ka[u]) break;
                if (cur == 0) {
                    unsigned long long old = atomicCAS(&s_k1[h], 0ull, (unsigned long long)ka[u]);
                    if (old == 0) { claimed[u] = true; break; }
                    if (old == ka[u]) break;
                }
                h = (h + 1) & (INS_SLOTS - 1);
            }
            loc[u] = h;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < INS_IPT; ++u)
            if (live[u] && claimed[u]) s_k2[loc[u]] = kb[u];
        __syncthreads();
        // phase B: aggregate; a k1 match with a different k2 goes straight to global
        bool direct[INS_IPT];
#pragma unroll
        for (int u = 0; u < INS_IPT; ++u) {
            direct[u] = live[u] && s_k2[loc[u]] != kb[u];
            if (live[u] && !direct[u]) {
                atomicAdd(&s_w[loc[u]], w[u]);
                atomicMin(&s_rep[loc[u]], ord[u]);
            }
        }
        __syncthreads();
        // phase C: compact the occupied local slots (so every thread probes ~2
        // keys, not 8 mostly-empty slots in sequence), then publish each
        // distinct local key once
        uint32_t nocc;
        {
            constexpr int PER = INS_SLOTS / INS_THREADS;
            uint32_t occ = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int sl = threadIdx.x + j * INS_THREADS;
                occ |= (s_k1[sl] != 0 && s_w[sl] != 0) ? (1u << j) : 0u;
            }
            uint32_t pos = block_excl_scan<INS_THREADS>(__popc(occ), s_scan, &nocc);
#pragma unroll
            for (int j = 0; j < PER; ++j)
                if (occ & (1u << j)) s_list[pos++] = (uint16_t)(threadIdx.x + j * INS_THREADS);
            __syncthreads();
        }
        for (uint32_t q = threadIdx.x; q < nocc; q += INS_THREADS) {
            const int sl = s_list[q];
            bool claimed = false;
            uint64_t g = table_slot(table, mask, s_k1[sl], s_k2[sl], ctl, &claimed);
            claim_count(claimed, g, ctl, limit, clist);
            s_g[sl] = g;
            if (g == ~0ull) continue;
            atomicAdd(&table[g].weight, (unsigned long long)s_w[sl]);
            atomicMin(&table[g].rep, s_rep[sl]);
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < INS_IPT; ++u) {
            if (!live[u]) continue;
            uint64_t g;
            if (direct[u]) {
                bool claimed = false;
                g = table_slot(table, mask, ka[u], kb[u], ctl, &claimed);
                claim_count(claimed, g, ctl, limit, clist);
                if (g != ~0ull) {
                    atomicAdd(&table[g].weight, (unsigned long long)w[u]);
                    atomicMin(&table[g].rep, ord[u]);
                }
            } else {
                g = s_g[loc[u]];
            }
            if (g == ~0ull) continue;
            item_slot[it[u]] = (uint32_t)g;
            pending[it[u]] = 0;
        }
        __syncthreads();
    }
}

// 8 bytes starting at an arbitrary byte offset, from two aligned 8-byte loads
// (the activity arrays carry >= 16 bytes of tail padding).
__device__ __forceinline__ uint64_t load8_at(const uint8_t* b, uint64_t off) {
    const uint64_t* w = (const uint64_t*)(b + (off & ~7ull));
    const uint32_t sh = (uint32_t)(off & 7) * 8;
    const uint64_t w0 = w[0];
    return sh ? (w0 >> sh) | (w[1] << (64 - sh)) : w0;
}

// exact sequence equality of acts[f, f+len) and acts[rf, rf+len): 8 bytes per
// step for byte-wide activities, branch-free (no early exit)
template <class ACT>
__device__ __forceinline__ bool seq_equal(const ACT* acts, uint64_t f, uint64_t rf, uint64_t len) {
    if constexpr (sizeof(ACT) == 1) {
        const uint8_t* b = (const uint8_t*)acts;
        uint64_t diff = 0;
        for (uint64_t i = 0; i < len; i += 8) {
            const uint64_t m = (len - i >= 8) ? ~0ull : ((1ull << (8 * (len - i))) - 1);
            diff |= (load8_at(b, f + i) ^ load8_at(b, rf + i)) & m;
        }
        return diff == 0;
    } else {
        uint32_t diff = 0;
        for (uint64_t i = 0; i < len; ++i) diff |= (uint32_t)acts[f + i] ^ (uint32_t)acts[rf + i];
        return diff == 0;
    }
}

// Each item compares its sequence with its slot representative's; the rep is
// the item whose order key equals slot.rep: item_of_order maps order -> item
// (identity when order == nullptr).
template <class OFF, class ACT>
__global__ void k_verify(const uint32_t* __restrict__ list, uint64_t n_items,
                         const OFF* __restrict__ off, const ACT* __restrict__ acts,
                         const uint64_t* __restrict__ weight, const uint32_t* __restrict__ order,
                         const uint32_t* __restrict__ item_of_rep_slot, Slot* table,
                         const uint32_t* __restrict__ item_slot, uint8_t* __restrict__ pending,
                         uint32_t* __restrict__ next_list, uint32_t* __restrict__ next_count,
                         const uint32_t* __restrict__ overflow, const uint64_t* __restrict__ d_n) {
    if (*overflow) return;   // this attempt's table is abandoned (item_slot incomplete)
    if (d_n) n_items = min(n_items, *d_n);
    // VU items per trip, their dependent loads (slot -> rep -> offsets ->
    // sequences) interleaved: the kernel is L2-latency bound
    constexpr int VU = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_items; t += VU * stride) {
        uint32_t it[VU], sl[VU], ord[VU], rep[VU], rep_it[VU];
        bool ok[VU];
#pragma unroll
        for (int u = 0; u < VU; ++u) {
            const uint64_t tu = t + u * stride;
            ok[u] = tu < n_items;
            it[u] = ok[u] ? (list ? list[tu] : (uint32_t)tu) : (list ? list[t] : (uint32_t)t);
        }
#pragma unroll
        for (int u = 0; u < VU; ++u) {
            sl[u] = item_slot[it[u]];
            ord[u] = order ? order[it[u]] : it[u];
        }
#pragma unroll
        for (int u = 0; u < VU; ++u) rep[u] = table[sl[u]].rep;
        // with the identity order the representative item IS the slot's rep
#pragma unroll
        for (int u = 0; u < VU; ++u) rep_it[u] = order ? item_of_rep_slot[sl[u]] : rep[u];
        OFF f[VU], l[VU], rf[VU], rl[VU];
#pragma unroll
        for (int u = 0; u < VU; ++u) {
            f[u] = off[it[u]];
            l[u] = off[it[u] + 1];
            rf[u] = off[rep_it[u]];
            rl[u] = off[rep_it[u] + 1];
        }
#pragma unroll
        for (int u = 0; u < VU; ++u) {
            if (!ok[u] || rep[u] == ord[u]) continue;        // past the end / the representative itself
            bool same = (l[u] - f[u]) == (rl[u] - rf[u]);
            if (same) same = seq_equal(acts, (uint64_t)f[u], (uint64_t)rf[u], (uint64_t)(l[u] - f[u]));
            if (!same) {
                atomicAdd(&table[sl[u]].weight, (unsigned long long)(0ull - (weight ? weight[it[u]] : 1ull)));
                pending[it[u]] = 1;
                next_list[atomicAdd(next_count, 1u)] = it[u];
            }
        }
    }
}

// slot -> representative item (the item whose order == slot.rep)
__global__ void k_rep_item(const uint32_t* __restrict__ list, uint64_t n_items,
                           const uint32_t* __restrict__ order, const Slot* __restrict__ table,
                           const uint32_t* __restrict__ item_slot, uint32_t* __restrict__ item_of_rep_slot,
                           const uint32_t* __restrict__ overflow, const uint64_t* __restrict__ d_n) {
    if (*overflow) return;
    if (d_n) n_items = min(n_items, *d_n);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_items;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t it = list ? list[t] : (uint32_t)t;
        const uint32_t sl = item_slot[it];
        if (table[sl].rep == (order ? order[it] : it)) item_of_rep_slot[sl] = it;
    }
}

// claimed slots (clist) with weight > 0 -> groups (append order is irrelevant:
// the final sort is a total order)
// also sums the new groups' sequence lengths (one atomic per block) so the
// host learns the total variant length with the round's counters
template <class OFF>
__global__ __launch_bounds__(256) void k_compact(const Slot* __restrict__ table, uint64_t cap,
                                                 const uint32_t* __restrict__ clist,
                                                 const uint32_t* __restrict__ n_claims,
                                                 const uint32_t* __restrict__ item_of_rep_slot,
                                                 uint32_t* __restrict__ slot_group, uint64_t* __restrict__ g_weight,
                                                 uint32_t* __restrict__ g_rep_item, uint32_t* __restrict__ g_order,
                                                 uint32_t* __restrict__ n_groups, const uint32_t* __restrict__ overflow,
                                                 const OFF* __restrict__ off, unsigned long long* total_len) {
    __shared__ unsigned long long s_tot;
    if (*overflow) return;
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    unsigned long long tl = 0;
    const uint64_t nc = min((uint64_t)*n_claims, cap);
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nc;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t sl = clist[q];
        const Slot& s = table[sl];
        if ((s.k1 | s.k2) == 0 || s.weight == 0) continue;
        uint32_t g = atomicAdd(n_groups, 1u);
        const uint32_t rep_item = item_of_rep_slot ? item_of_rep_slot[sl] : s.rep;
        g_weight[g] = s.weight;
        g_rep_item[g] = rep_item;
        g_order[g] = s.rep;
        slot_group[sl] = g;
        tl += (unsigned long long)(off[rep_item + 1] - off[rep_item]);
    }
    if (tl) atomicAdd(&s_tot, tl);
    __syncthreads();
    if (threadIdx.x == 0 && s_tot) atomicAdd(total_len, s_tot);
}

__global__ void k_item_group(const uint32_t* __restrict__ list, uint64_t n_items,
                             const uint32_t* __restrict__ item_slot, const uint8_t* __restrict__ pending,
                             const uint32_t* __restrict__ slot_group, uint32_t* __restrict__ item_group,
                             const uint32_t* __restrict__ overflow, const uint64_t* __restrict__ d_n) {
    if (*overflow) return;
    if (d_n) n_items = min(n_items, *d_n);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_items;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t it = list ? list[t] : (uint32_t)t;
        if (!pending[it]) item_group[it] = slot_group[item_slot[it]];
    }
}

// sort key of a group: (Wmax - weight) above the order key, Wmax = 2^wbits - 1
// (wbits = bit width of the item count when weights are 1, else 32 with
// clipping), so one LSD sort orders by weight desc, then order asc
__global__ void k_sort_keys(const uint64_t* __restrict__ g_weight, const uint32_t* __restrict__ g_order,
                            uint64_t G, int wbits, int order_bits, uint64_t* __restrict__ key,
                            uint32_t* __restrict__ val) {
    const uint64_t wmax = (1ull << wbits) - 1;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < G;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = min(g_weight[g], wmax);
        key[g] = ((wmax - w) << order_bits) | g_order[g];
        val[g] = (uint32_t)g;
    }
}

// Small group counts: every key's output position = #(keys smaller) + #(equal
// keys at lower index), all pairs compared (keys staged through shared memory
// in chunks) -- one launch instead of ~6 latency-bound radix passes.
constexpr uint64_t RANK_SORT_MAX = 4096;
__global__ __launch_bounds__(256) void k_rank_sort(const uint64_t* __restrict__ key, uint32_t n,
                                                   uint32_t* __restrict__ sorted) {
    __shared__ uint64_t s_k[2048];
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t ki = i < n ? key[i] : 0;
    uint32_t r = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 2048) {
        const uint32_t cn = min(2048u, n - c0);
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < cn; t += blockDim.x) s_k[t] = key[c0 + t];
        __syncthreads();
        if (i < n)
            for (uint32_t t = 0; t < cn; ++t) {
                const uint64_t kj = s_k[t];
                r += (kj < ki) | ((kj == ki) & (c0 + t < i));
            }
    }
    if (i < n) sorted[r] = i;
}

struct Groups {
    uint64_t G = 0;
    uint64_t Ga = 0;                // group ids (>= G: the one-pass grouping's unused reserved ids)
    uint64_t total_len = 0;         // sum of the groups' sequence lengths
    uint64_t* weight = nullptr;     // [G]
    uint32_t* rep_item = nullptr;   // [G]
    uint32_t* order = nullptr;      // [G] (rep's order key)
    uint32_t* item_group = nullptr; // [n_items]
    uint32_t* sorted = nullptr;     // [G] group ids in output order
    uint32_t* inv = nullptr;        // [G] group -> output position
    void free(cudaStream_t s) {
        dfree(weight, s);
        dfree(rep_item, s);
        dfree(order, s);
        dfree(item_group, s);
        dfree(sorted, s);
        dfree(inv, s);
    }
};

__global__ void k_inv(const uint32_t* __restrict__ sorted, uint64_t G, uint32_t* __restrict__ inv) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < G;
         p += (uint64_t)gridDim.x * blockDim.x)
        inv[sorted[p]] = (uint32_t)p;
}

static int gsz(uint64_t n) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 8));
}

static uint64_t pow2_at_least(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Group n_items items by exact sequence.  order: unique u32 per item (nullptr
// = item index).  order_bits: bits needed by the order key (for the sort).
template <class OFF, class ACT>
// d_n (optional): the device item count when n_items is only an upper bound
// (round 0 clamps to it; the true count comes back with round 0's counters in
// *n_true), which spares a host round trip before the grouping starts.
static pm4g_status group_items(uint64_t n_items, const uint64_t* k1, const uint64_t* k2,
                               const OFF* off, const ACT* acts, const uint64_t* weight,
                               const uint32_t* order, int order_bits, cudaStream_t s, Groups* out,
                               const uint64_t* d_n = nullptr, uint64_t* n_true = nullptr) {
    if (n_true) *n_true = n_items;
    Groups g;
    auto bail = [&](pm4g_status st) {
        g.free(s);
        return st;
    };
    pm4g_status st;
    const uint64_t N = std::max<uint64_t>(n_items, 1);
    if ((st = dalloc_t(&g.item_group, N, s))) return bail(st);
    if ((st = dalloc_t(&g.weight, N, s))) return bail(st);
    if ((st = dalloc_t(&g.rep_item, N, s))) return bail(st);
    if ((st = dalloc_t(&g.order, N, s))) return bail(st);
    if (n_items == 0) {
        *out = g;
        return PM4G_OK;
    }
    Scratch work(s);
    // item_slot u32 | pending u8 | list_a u32 | list_b u32 | counters
    const size_t wbytes = N * 4 + N + 16 + N * 4 * 2 + 64;
    if ((st = work.alloc(wbytes))) return bail(st);
    uint32_t* item_slot = work.as<uint32_t>();
    uint8_t* pending = (uint8_t*)(item_slot + N);
    uint32_t* list_a = (uint32_t*)(((uintptr_t)(pending + N) + 15) & ~(uintptr_t)15);
    uint32_t* list_b = list_a + N;
    // [0] next_count, [1] overflow, [2] claimed slots, [3] n_groups
    uint32_t* counters = list_b + N;
    unsigned long long* d_total = (unsigned long long*)(((uintptr_t)(counters + 4) + 7) & ~(uintptr_t)7);
    PM4G_CK(cudaMemsetAsync(counters, 0, 16, s));
    PM4G_CK(cudaMemsetAsync(d_total, 0, 8, s));

    const uint32_t* list = nullptr;   // round 0: all items
    uint64_t n_active = n_items;
    uint64_t G = 0;
    const bool weak = debug_weak_hash();
    for (int round = 0; n_active > 0; ++round) {
        // A table of `full` slots holds every item at load <= 1/2 and never
        // overflows; the first try is smaller (distinct sequences are usually
        // far fewer than items) and grows 4x whenever its load limit trips.
        const uint64_t full = pow2_at_least(std::max<uint64_t>(1024, 2 * n_active));
        uint64_t cap = std::min<uint64_t>(full, std::max<uint64_t>(1ull << 21, pow2_at_least(n_active / 16)));
        if (const uint64_t dc = debug_variant_cap()) cap = std::min<uint64_t>(full, pow2_at_least(std::max<uint64_t>(dc, 64)));
        for (int attempt = 0;; ++attempt) {
            Scratch tab(s), aux(s);
            if ((st = tab.alloc(cap * sizeof(Slot)))) return bail(st);
            if ((st = aux.alloc(cap * 12))) return bail(st);
            Slot* table = tab.as<Slot>();
            uint32_t* item_of_rep_slot = aux.as<uint32_t>();
            uint32_t* slot_group = item_of_rep_slot + cap;
            uint32_t* clist = slot_group + cap;   // claimed slots, claim order
            PM4G_LAUNCH("k_variant_init", cap * 32.0, s, (k_init_table<<<gsz(cap), 256, 0, s>>>(table, cap)));
            PM4G_CK(cudaMemsetAsync(counters, 0, 12, s));
            const uint32_t limit = cap == full ? 0xffffffffu : (uint32_t)(cap / 4 * 3);
            uint64_t salt = (round == 0 || weak) ? 0ull : 0x9E3779B97F4A7C15ull * (uint64_t)round;
            uint32_t* next_list = (list == list_a) ? list_b : list_a;
            const int gs = gsz(n_active);
            {
                PM4G_MAX_SMEM(k_insert<OFF>);
                uint64_t chunks = (n_active + INS_CHUNK - 1) / INS_CHUNK;
                int gi = (int)std::max<uint64_t>(1, std::min<uint64_t>(chunks, (uint64_t)num_sms() * 3));
                PM4G_LAUNCH("k_variant_insert", n_active * 24.0, s,
                            (k_insert<OFF><<<gi, INS_THREADS, INS_SMEM, s>>>(
                                list, n_active, k1, k2, off, weight, order, table, cap - 1, limit, salt,
                                item_slot, pending, counters + 1, list ? nullptr : d_n, clist)));
            }
            uint32_t* ior = order ? item_of_rep_slot : nullptr;   // identity order: rep item = slot.rep
            if (order)
                PM4G_LAUNCH("k_variant_rep", n_active * 8.0, s,
                            (k_rep_item<<<gs, 256, 0, s>>>(list, n_active, order, table, item_slot, item_of_rep_slot,
                                                            counters + 1, list ? nullptr : d_n)));
            PM4G_LAUNCH("k_variant_verify", n_active * 16.0, s,
                        (k_verify<OFF, ACT><<<gs, 256, 0, s>>>(list, n_active, off, acts, weight, order,
                                                               ior, table, item_slot,
                                                               pending, next_list, counters, counters + 1,
                                                               list ? nullptr : d_n)));
            PM4G_LAUNCH("k_variant_compact", n_active * 8.0, s,
                        (k_compact<OFF><<<gsz(n_active), 256, 0, s>>>(table, cap, clist, counters + 2, ior, slot_group,
                                                                 g.weight, g.rep_item, g.order,
                                                                 counters + 3, counters + 1, off, d_total)));
            PM4G_LAUNCH("k_variant_item_group", n_active * 12.0, s,
                        (k_item_group<<<gs, 256, 0, s>>>(list, n_active, item_slot, pending, slot_group,
                                                         g.item_group, counters + 1, list ? nullptr : d_n)));
            // one host round trip per round: next_count, overflow, claims, n_groups
            // (counters and the length total in one copy, into pinned staging)
            uint32_t h[4] = {0, 0, 0, 0};
            unsigned long long htot = 0;
            uint64_t hn = n_items;
            static thread_local unsigned char* h_stage = nullptr;
            if (!h_stage) PM4G_CK(cudaHostAlloc((void**)&h_stage, 64, cudaHostAllocDefault));
            const size_t o_tot = (size_t)((const char*)d_total - (const char*)counters);   // <= 20
            PM4G_TRY(copy_words_to_host(h_stage, counters, o_tot + 8, s));
            if (d_n && !list) PM4G_TRY(copy_words_to_host(h_stage + 32, d_n, 8, s));
            PM4G_TRY(stream_sync(s));
            memcpy(h, h_stage, 16);
            memcpy(&htot, h_stage + o_tot, 8);
            if (d_n && !list) memcpy(&hn, h_stage + 32, 8);
            if (d_n && !list) {
                n_items = std::min(n_items, hn);
                if (n_true) *n_true = n_items;
            }
            if (h[1]) {  // load limit hit: verify/compact/item_group skipped on the device; regrow
                if (cap >= full || attempt > 16) return bail(fail(PM4G_ENOMEM, "variant table overflow"));
                cap = std::min<uint64_t>(full, cap * 4);
                continue;
            }
            G = h[3];
            g.total_len = htot;
            n_active = h[0];
            list = next_list;
            if (round > 64 * 1024) return bail(fail(PM4G_ECUDA, "variant grouping did not converge"));
            break;
        }
    }
    g.G = G;
    // sort groups: count desc, order asc
    const int wbits = weight ? 32 : std::max(1, bit_width_u64(n_items));
    Scratch sk(s);   // keys [G] u64 | group ids [G] u32 (the radix payload)
    if ((st = sk.alloc(G * 12 + 16))) return bail(st);
    uint32_t* sk_val = (uint32_t*)(sk.as<uint64_t>() + G);
    if ((st = dalloc_t(&g.sorted, std::max<uint64_t>(G, 1), s))) return bail(st);
    if ((st = dalloc_t(&g.inv, std::max<uint64_t>(G, 1), s))) return bail(st);
    PM4G_LAUNCH("k_variant_sortkeys", G * 16.0, s,
                (k_sort_keys<<<gsz(G), 256, 0, s>>>(g.weight, g.order, G, wbits, order_bits, sk.as<uint64_t>(),
                                                     sk_val)));
    if (G <= RANK_SORT_MAX) {
        if (G)
            PM4G_LAUNCH("k_rank_sort", G * 8.0 + G * 4.0, s,
                        (k_rank_sort<<<(unsigned)((G + 255) / 256), 256, 0, s>>>(sk.as<uint64_t>(), (uint32_t)G,
                                                                               g.sorted)));
    } else {
        PM4G_TRY(radix_sort_u64_to(sk.as<uint64_t>(), sk_val, g.sorted, (int64_t)G, wbits + order_bits, s));
    }
    PM4G_LAUNCH("k_variant_inv", G * 8.0, s, (k_inv<<<gsz(G), 256, 0, s>>>(g.sorted, G, g.inv)));
    *out = g;
    return PM4G_OK;
}


// ------------------------------------------------------------------ exclusive scan
constexpr int SCAN_THREADS = 256, SCAN_IPT = 8, SCAN_TILE = SCAN_THREADS * SCAN_IPT;

template <class OUT>
__global__ __launch_bounds__(SCAN_THREADS) void k_excl_scan(const uint32_t* __restrict__ in,
                                                            OUT* __restrict__ out, int64_t n,
                                                            st_t* status, uint32_t* counter) {
    __shared__ uint32_t s_tile, s_scan[SCAN_THREADS / 32 + 1], s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t b = (int64_t)tile * SCAN_TILE + threadIdx.x * SCAN_IPT;
    uint32_t v[SCAN_IPT], sum = 0;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; ++j) {
        v[j] = (b + j < n) ? in[b + j] : 0u;
        sum += v[j];
    }
    uint32_t total;
    uint32_t ex = block_excl_scan<SCAN_THREADS>(sum, s_scan, &total);
    if (threadIdx.x < 32) {
        uint32_t pf = lookback_warp_k<8>(status, tile, total);
        if (threadIdx.x == 0) s_prefix = pf;
    }
    __syncthreads();
    OUT r = (OUT)s_prefix + ex;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; ++j) {
        if (b + j < n) out[b + j] = r;
        r += v[j];
    }
    if (threadIdx.x == 0 && (int64_t)(tile + 1) * SCAN_TILE >= n) out[n] = (OUT)s_prefix + total;
}

// out[0..n] = exclusive prefix sums of in[0..n), out[n] = total (< 2^31)
template <class OUT>
static pm4g_status excl_scan_u32(const uint32_t* in, OUT* out, int64_t n, cudaStream_t s) {
    if (n == 0) {
        PM4G_CK(cudaMemsetAsync(out, 0, sizeof(OUT), s));
        return PM4G_OK;
    }
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    Scratch st(s);
    PM4G_TRY(st.alloc((tiles + 1) * sizeof(st_t)));
    PM4G_CK(cudaMemsetAsync(st.p, 0, (tiles + 1) * sizeof(st_t), s));
    PM4G_LAUNCH("k_excl_scan", n * 12.0, s,
                (k_excl_scan<OUT><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, n, st.as<st_t>() + 1,
                                                                          st.as<uint32_t>())));
    return PM4G_OK;
}

pm4g_status excl_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t n, cudaStream_t s) {
    return excl_scan_u32<uint64_t>(in, out, n, s);
}

// ------------------------------------------------------------------ emission
// rep_code: per item -> case code of the item (local: case code of the case;
// merge: the entry's representative code).
template <class OFF>
__global__ void k_emit(const Groups g, const OFF* __restrict__ off, const uint32_t* __restrict__ rep_code,
                       const uint64_t* __restrict__ k1, const uint64_t* __restrict__ k2,
                       uint64_t* __restrict__ count, uint32_t* __restrict__ len,
                       uint32_t* __restrict__ rep_case, uint64_t* __restrict__ ok1,
                       uint64_t* __restrict__ ok2) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < g.G;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t gid = g.sorted[p];
        const uint32_t it = g.rep_item[gid];
        count[p] = g.weight[gid];
        len[p] = (uint32_t)(off[it + 1] - off[it]);
        rep_case[p] = rep_code[it];
        ok1[p] = k1[it];
        ok2[p] = k2[it];
    }
}

// one warp per variant: copy the representative's sequence
constexpr int SEQ_LANES = 8;
template <class OFF, class ACT>
__global__ void k_seq_gather(const Groups g, const OFF* __restrict__ off, const ACT* __restrict__ acts,
                             const uint64_t* __restrict__ seq_off, uint32_t* __restrict__ seq_act) {
    // SEQ_LANES lanes per variant (sequences are short: more of them in flight)
    const uint64_t teams = (uint64_t)gridDim.x * blockDim.x / SEQ_LANES;
    const uint32_t ln = threadIdx.x & (SEQ_LANES - 1);
    for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / SEQ_LANES; p < g.G; p += teams) {
        const uint32_t it = g.rep_item[g.sorted[p]];
        const OFF f = off[it];
        const uint64_t o = seq_off[p], L = seq_off[p + 1] - o;
        for (uint64_t i = ln; i < L; i += SEQ_LANES) seq_act[o + i] = (uint32_t)acts[f + i];
    }
}

__global__ void k_case_variant(const uint32_t* __restrict__ item_group, const uint32_t* __restrict__ inv,
                               uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < n;
         c += (uint64_t)gridDim.x * blockDim.x)
        out[c] = inv[item_group[c]];
}

void free_variants(pm4g_variant_table* v) {
    if (!v) return;
    cudaStream_t s = v->stream;
    dfree(v->count, s);
    dfree(v->len, s);
    dfree(v->rep_case, s);
    dfree(v->seq_off, s);
    dfree(v->seq_act, s);
    dfree(v->k1, s);
    dfree(v->k2, s);
    dfree(v->case_variant, s);
    delete v;
}

// ------------------------------------------------------------------ the case grouping, one pass
// The usual call (items = the cases of one log, weight 1, order = case rank,
// full-strength hash) groups, counts, finds representatives and verifies in
// ONE persistent kernel, k_vgroup:
//   * the global open-addressing table maps a key (k1, k2) to a dense group id
//     (claim order) and the group's canonical case (its claimer): one 128-bit
//     CAS claims a slot, the claimer then publishes (gid, case) in one 64-bit
//     store that finders wait for;
//   * every CTA keeps a shared-memory cache of the keys it has met (key, gid,
//     canonical offset / length, local count, local min case) across its chunks,
//     so a Zipf-hot variant costs shared-memory work only; the cache is flushed
//     into the dense per-group arrays once at the end;
//   * every case is verified against its group's canonical sequence on the
//     spot (sequence equality is an equivalence, so any member serves as the
//     reference); a mismatch (a hash collision) is counted, and the host then
//     reruns the general round-based engine (group_items) from scratch.
// Result: item_group[c] = dense gid, per-group count / min case / total length,
// i.e. the Groups of group_items without a compaction or item pass.
// a warp's task: 32 * IPT consecutive cases (IPT = PM4G_VG_IPT; IPT = 1 for small logs,
// so their few tasks spread over more warps and CTAs instead of one CTA's latency chain)
#ifndef PM4G_VG_THREADS
#define PM4G_VG_THREADS 256
#endif
constexpr int VG_THREADS = PM4G_VG_THREADS;
// per-CTA key cache entries, minimum CTAs per SM and cases per lane per task
// (sweep, 100M / 1B-8 shard: 2 cases per lane, 1024 entries, 4 CTAs per SM
// 0.36 / 0.36 ms; 4 per lane 0.50 / 0.55; 1 per lane 0.43 / 0.40; 8 per lane
// 0.62 / 0.97; 2048 entries with 3 CTAs 0.60 / 0.45)
#ifndef PM4G_VG_CACHE
#define PM4G_VG_CACHE 1024
#endif
#ifndef PM4G_VG_MINB
#define PM4G_VG_MINB 4
#endif
#ifndef PM4G_VG_IPT
#define PM4G_VG_IPT 2   // cases per lane per task (large logs)
#endif
constexpr int VG_CACHE = PM4G_VG_CACHE, VG_FILL = VG_CACHE / 2, VG_PROBES = 8;
constexpr size_t VG_SMEM = (size_t)VG_CACHE * (8 + 8 + 4 + 4 + 4 + 4 + 4);
constexpr unsigned long long VG_NOMETA = ~0ull;

// global slot: key, then (gid << 32 | canonical offset, canonical length)
// published by the claimer in one 16-byte atomic
struct alignas(32) VSlot {
    unsigned long long k1, k2;
    alignas(16) unsigned long long meta;
    unsigned long long len;
};

__global__ void k_vinit(VSlot* table, uint64_t cap, uint32_t* g_w, uint32_t* g_rep, uint64_t gcap) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap || i < gcap;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < cap) {
            VSlot z;
            z.k1 = 0;
            z.k2 = 0;
            z.meta = VG_NOMETA;
            z.len = 0;
            table[i] = z;
        }
        if (i < gcap) {
            g_w[i] = 0;
            g_rep[i] = 0xffffffffu;
        }
    }
}

// exact equality of two activity sequences of length len (u8: aligned 8-byte
// words, the first five of each issued together -- 33+ rows take the loop)
template <class ACT>
__device__ __forceinline__ bool seq_same(const ACT* acts, uint32_t f, uint32_t rf, uint32_t len) {
    if (f == rf) return true;
    if constexpr (sizeof(ACT) == 1) {
        if (len <= 32) {
            const uint64_t* wa = (const uint64_t*)((const uint8_t*)acts + (f & ~7u));
            const uint64_t* wb = (const uint64_t*)((const uint8_t*)acts + (rf & ~7u));
            const uint32_t sa = (f & 7) * 8, sb = (rf & 7) * 8;
            uint64_t a[5], b[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const bool need = 8u * i < len + 8u;
                a[i] = need ? wa[i] : 0;
                b[i] = need ? wb[i] : 0;
            }
            uint64_t diff = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (8u * i >= len) break;
                const uint64_t x = sa ? (a[i] >> sa) | (a[i + 1] << (64 - sa)) : a[i];
                const uint64_t y = sb ? (b[i] >> sb) | (b[i + 1] << (64 - sb)) : b[i];
                const uint64_t m = (len - 8u * i >= 8) ? ~0ull : ((1ull << (8 * (len - 8u * i))) - 1);
                diff |= (x ^ y) & m;
            }
            return diff == 0;
        }
    }
    return seq_equal(acts, (uint64_t)f, (uint64_t)rf, (uint64_t)len);
}

// ctl: [0] overflow, [1] gids reserved (the warps' blocks), [2] collisions, [3] groups claimed
// weight / order (nullptr: 1 / the item index): the merge of shard tables groups
// their entries (weight = count, order = representative case code).  Weighted
// counts stay u32: a weight or a sum past 2^32 - 1 counts as a collision (the
// general engine then groups with u64 weights).
__device__ __forceinline__ void vg_add_w(uint32_t* p, uint32_t w, bool checked, uint32_t* ctl) {
    if (!checked) {
        atomicAdd(p, w);
    } else if (atomicAdd(p, w) > 0xffffffffu - w) {
        atomicAdd(&ctl[2], 1u);
    }
}

template <class ACT, int VG_IPT, int VG_GBLOCK>
__global__ __launch_bounds__(VG_THREADS, PM4G_VG_MINB) void k_vgroup(
    uint64_t n_items, const uint64_t* __restrict__ d_n, const uint64_t* __restrict__ k1,
    const uint64_t* __restrict__ k2, const uint32_t* __restrict__ off, const ACT* __restrict__ acts,
    const uint64_t* __restrict__ weight, const uint32_t* __restrict__ order,
    VSlot* table, uint64_t mask, uint32_t gcap, uint32_t* __restrict__ g_w, uint32_t* __restrict__ g_rep,
    uint32_t* __restrict__ item_gid, uint32_t* ctl, unsigned long long* total_len, uint32_t* task_counter) {
    extern __shared__ __align__(16) unsigned char vg_sm[];
    unsigned long long* c_k1 = (unsigned long long*)vg_sm;   // claim word (0: free)
    unsigned long long* c_k2 = c_k1 + VG_CACHE;              // written last: the entry is ready
    uint32_t* c_gid = (uint32_t*)(c_k2 + VG_CACHE);
    uint32_t* c_off = c_gid + VG_CACHE;   // canonical sequence: offset and length
    uint32_t* c_len = c_off + VG_CACHE;
    uint32_t* c_cnt = c_len + VG_CACHE;   // local count / min case of the entry
    uint32_t* c_rep = c_cnt + VG_CACHE;
    __shared__ uint32_t s_fill, s_claims;
    __shared__ unsigned long long s_len;
    for (int i = threadIdx.x; i < VG_CACHE; i += VG_THREADS) {
        c_k1[i] = 0;
        c_k2[i] = 0;
        c_cnt[i] = 0;
        c_rep[i] = 0xffffffffu;
    }
    if (threadIdx.x == 0) {
        s_fill = 0;
        s_claims = 0;
        s_len = 0;
    }
    __syncthreads();
    if (d_n) n_items = min(n_items, *d_n);
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    auto chash = [](uint64_t a) { return (uint32_t)(a ^ (a >> 29)) & (VG_CACHE - 1); };
    constexpr int VG_TASK = 32 * VG_IPT;
    // VG_GBLOCK: gids reserved per warp at a time (one by one for logs whose table
    // may take the single-CTA emission: no empty gids)
    uint32_t claims = 0, gnext = 0, gend = 0;   // gend - gnext: the warp's unused reserved gids
    unsigned long long lensum = 0;
    for (;;) {
        uint64_t task = 0;
        if (lane == 0) task = atomicAdd((unsigned long long*)task_counter, 1ull);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task * VG_TASK >= n_items) break;
        uint32_t f[VG_IPT], l[VG_IPT], gid[VG_IPT], cof[VG_IPT], cln[VG_IPT], wt[VG_IPT], od[VG_IPT];
        uint64_t ka[VG_IPT], kb[VG_IPT];
        int hit[VG_IPT];   // cache entry, -1: miss, -2: none (past the end / abandoned / collision)
#pragma unroll
        for (int u = 0; u < VG_IPT; ++u) {
            const uint64_t t = task * VG_TASK + u * 32 + lane;
            hit[u] = -2;
            if (t >= n_items) continue;
            hit[u] = -1;
            ka[u] = k1[t];
            kb[u] = k2[t];
            f[u] = off[t];
            l[u] = off[t + 1];
            wt[u] = 1u;
            if (weight) {
                const uint64_t w = weight[t];
                wt[u] = (uint32_t)w;
                if ((w >> 32) || !w) atomicAdd(&ctl[2], 1u);
            }
            od[u] = order ? order[t] : (uint32_t)t;
        }
        // A: the CTA's cache (an entry is used once its k2 is written)
#pragma unroll
        for (int u = 0; u < VG_IPT; ++u) {
            if (hit[u] != -1) continue;
            uint32_t h = chash(ka[u]);
            for (int p = 0; p < VG_PROBES; ++p) {
                const unsigned long long c = ld_volatile(&c_k1[h]);
                if (c == 0) break;
                if (c == ka[u] && ld_volatile(&c_k2[h]) == kb[u]) {
                    __threadfence_block();
                    hit[u] = (int)h;
                    gid[u] = c_gid[h];
                    cof[u] = c_off[h];
                    cln[u] = c_len[h];
                    break;
                }
                h = (h + 1) & (VG_CACHE - 1);
            }
        }
        // B: misses find or claim their global slot (key and meta read together).
        // A claimer takes its gid from the warp's block of reserved gids and
        // publishes (gid, canonical offset, length) in one 16-byte atomic;
        // finders wait for that.
#pragma unroll
        for (int u = 0; u < VG_IPT; ++u) {
            const bool miss = hit[u] == -1;
            VSlot* sp = nullptr;
            bool mine = false;
            K128 m{VG_NOMETA, 0};
            if (miss) {
                uint64_t h = (ka[u] ^ (ka[u] >> 29) ^ (kb[u] * 0x9E3779B97F4A7C15ull)) & mask;
                for (uint64_t probes = 0;; ++probes) {
                    sp = &table[h];
                    K128 cur = ld_k128(sp);
                    m = ld_k128(&sp->meta);
                    if (cur.a == 0 && cur.b == 0) {
                        K128 exp{0, 0}, des{ka[u], kb[u]};
                        cur = atomicCAS((K128*)sp, exp, des);
                        mine = cur.a == 0 && cur.b == 0;
                    }
                    if (mine || (cur.a == ka[u] && cur.b == kb[u])) break;
                    if (probes >= mask || ((probes & 31) == 31 && ld_volatile(&ctl[0]))) {
                        atomicExch(&ctl[0], 1u);
                        sp = nullptr;
                        m = K128{VG_NOMETA, 0};   // (m held the last probed slot's: not this key's)
                        break;
                    }
                    h = (h + 1) & mask;
                }
            }
            const uint32_t cm = __ballot_sync(0xffffffffu, mine);
            if (cm) {
                const uint32_t nc = __popc(cm);
                if (gnext + nc > gend) {   // refill the warp's gid block
                    const uint32_t take = max(nc, (uint32_t)VG_GBLOCK);
                    uint32_t b = 0;
                    if (lane == 0) b = atomicAdd(&ctl[1], take);
                    gnext = __shfl_sync(0xffffffffu, b, 0);
                    gend = gnext + take;
                }
                if (mine) {
                    const uint32_t g = gnext + __popc(cm & lt);
                    if (g >= gcap) atomicExch(&ctl[0], 1u);
                    K128 exp{VG_NOMETA, 0}, des{((unsigned long long)g << 32) | f[u], (unsigned long long)(l[u] - f[u])};
                    atomicCAS((K128*)&sp->meta, exp, des);
                    gid[u] = g;
                    cof[u] = f[u];
                    cln[u] = l[u] - f[u];
                    ++claims;
                    lensum += l[u] - f[u];
                    if (g >= gcap) hit[u] = -2;
                }
                gnext += nc;
            }
            if (miss && !mine) {
                if (sp) {
                    while (m.a == VG_NOMETA && !ld_volatile(&ctl[0])) {
                        __nanosleep(16);
                        m = ld_k128(&sp->meta);
                    }
                }
                if (m.a == VG_NOMETA || (uint32_t)(m.a >> 32) >= gcap) {   // table abandoned
                    hit[u] = -2;
                } else {
                    gid[u] = (uint32_t)(m.a >> 32);
                    cof[u] = (uint32_t)m.a;
                    cln[u] = (uint32_t)m.b;
                }
            }
        }
        // C: verify against the canonical sequence, count, and cache the misses
#pragma unroll
        for (int u = 0; u < VG_IPT; ++u) {
            if (hit[u] == -2) continue;
            const uint32_t t = (uint32_t)(task * VG_TASK + u * 32 + lane);
            const uint32_t len = l[u] - f[u];
            if (len != cln[u] || !seq_same(acts, f[u], cof[u], len)) {   // hash collision: rerun exactly
                atomicAdd(&ctl[2], 1u);
                continue;
            }
            item_gid[t] = gid[u];
            if (hit[u] >= 0) {
                vg_add_w(&c_cnt[hit[u]], wt[u], weight != nullptr, ctl);
                atomicMin(&c_rep[hit[u]], od[u]);
                continue;
            }
            bool cached = false;
            if (ld_volatile(&s_fill) < VG_FILL) {
                uint32_t h = chash(ka[u]);
                for (int p = 0; p < VG_PROBES; ++p) {
                    if (ld_volatile(&c_k1[h]) == 0 && atomicCAS(&c_k1[h], 0ull, (unsigned long long)ka[u]) == 0ull) {
                        atomicAdd(&s_fill, 1u);
                        c_gid[h] = gid[u];
                        c_off[h] = cof[u];
                        c_len[h] = cln[u];
                        vg_add_w(&c_cnt[h], wt[u], weight != nullptr, ctl);
                        atomicMin(&c_rep[h], od[u]);
                        __threadfence_block();
                        st_volatile(&c_k2[h], (unsigned long long)kb[u]);
                        cached = true;
                        break;
                    }
                    h = (h + 1) & (VG_CACHE - 1);
                }
            }
            if (!cached) {
                vg_add_w(&g_w[gid[u]], wt[u], weight != nullptr, ctl);
                atomicMin(&g_rep[gid[u]], od[u]);
            }
        }
    }
    if (claims) atomicAdd(&s_claims, claims);
    if (lensum) atomicAdd(&s_len, lensum);
    __syncthreads();
    // flush the cache's counts and minimum cases into the dense group arrays
    for (int i = threadIdx.x; i < VG_CACHE; i += VG_THREADS) {
        if (c_cnt[i]) {
            vg_add_w(&g_w[c_gid[i]], c_cnt[i], weight != nullptr, ctl);
            atomicMin(&g_rep[c_gid[i]], c_rep[i]);
        }
    }
    if (threadIdx.x == 0) {
        if (s_claims) atomicAdd(&ctl[3], s_claims);
        if (s_len) atomicAdd(total_len, s_len);
    }
}

// (the radix fallback) the groups' u64 weights and order keys as the u32
// arrays k_vfinal reads
__global__ void k_vrekey(const uint64_t* __restrict__ weight, const uint32_t* __restrict__ rep, uint64_t G,
                         uint32_t* __restrict__ w32, uint32_t* __restrict__ r32) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < G; g += (uint64_t)gridDim.x * blockDim.x) {
        w32[g] = (uint32_t)weight[g];
        r32[g] = rep[g];
    }
}

// (weighted merge) the representative item of each group: the one holding the
// group's minimum order (orders are unique per item)
__global__ void k_vrepitem(const uint32_t* __restrict__ order, const uint32_t* __restrict__ item_gid,
                           const uint32_t* __restrict__ g_rep, uint64_t n_items, uint32_t* __restrict__ rep_item) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_items; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t g = item_gid[t];
        if (order[t] == g_rep[g]) rep_item[g] = (uint32_t)t;
    }
}

// dense groups -> Groups arrays (u64 weight, rep item = min case = order) and
// the sort key ((Wmax - weight) << order_bits) | rep of each group
__global__ void k_vfinal(const uint32_t* __restrict__ g_w, const uint32_t* __restrict__ g_rep, uint64_t G,
                         int wbits, int order_bits, uint64_t* __restrict__ weight, uint32_t* __restrict__ rep_item,
                         uint32_t* __restrict__ order, uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
    const uint64_t wmax = (1ull << wbits) - 1;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < G; g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = g_w[g];
        const uint32_t r = g_rep[g];
        weight[g] = w;
        if (rep_item) rep_item[g] = r;   // nullptr: already set
        order[g] = r;
        if (!key) continue;   // small tables: ordered by k_small_variants
        // an empty (reserved, unused) gid sorts after every group
        key[g] = w ? ((wmax - min(w, wmax)) << order_bits) | r : low_mask(wbits + order_bits);
        val[g] = (uint32_t)g;
    }
}

// ------------------------------------------------------------------ small variant tables, one launch
// Up to SV_MAX groups (e.g. the RoadTraffic shape's 231 variants, PAPER.md
// Table 1; one SM's instruction throughput makes the spread-out path below
// faster beyond ~2k groups): ONE CTA orders the groups by (count desc, rep asc) with a
// shared-memory LSD radix sort of a compacted key ((maxw - w) << rbits | rep),
// then emits count / len / rep_case / keys, scans the lengths and copies the
// representatives' sequences -- instead of ~11 launches (sort keys, histogram,
// scan, radix passes, inverse, emit, scan, gather), each a few microseconds of
// latency at these sizes.
constexpr int SV_THREADS = 1024, SV_WARPS = SV_THREADS / 32, SV_MAX = 2048, SV_IPT = SV_MAX / SV_THREADS;
constexpr size_t SV_SMEM = (size_t)SV_MAX * 8 + 2 * (size_t)SV_MAX * 2 + (size_t)SV_WARPS * 256 * 4;

template <class ACT>
__global__ __launch_bounds__(SV_THREADS) void k_small_variants(
    const uint64_t* __restrict__ weight, const uint32_t* __restrict__ order, const uint32_t* __restrict__ rep,
    uint32_t Ga, uint32_t G, const uint32_t* __restrict__ off, const ACT* __restrict__ acts, const uint32_t* __restrict__ rep_code,
    const uint64_t* __restrict__ k1, const uint64_t* __restrict__ k2, uint64_t* __restrict__ count,
    uint32_t* __restrict__ len, uint32_t* __restrict__ rep_case, uint64_t* __restrict__ seq_off,
    uint32_t* __restrict__ seq_act, uint64_t* __restrict__ ok1, uint64_t* __restrict__ ok2,
    uint32_t* __restrict__ inv) {
    extern __shared__ __align__(16) unsigned char sv_sm[];
    uint64_t* s_key = (uint64_t*)sv_sm;                        // [SV_MAX] in gid order
    uint16_t* s_idx = (uint16_t*)(s_key + SV_MAX);             // [2][SV_MAX] gid at each position
    uint32_t(*s_whist)[256] = (uint32_t(*)[256])(s_idx + 2 * SV_MAX);   // [SV_WARPS][256]
    __shared__ uint32_t s_scan[SV_WARPS + 1];
    __shared__ unsigned long long s_maxw;
    __shared__ uint32_t s_maxr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_maxw = 0;
        s_maxr = 0;
    }
    __syncthreads();
    unsigned long long mw = 0;
    uint32_t mr = 0;
    for (uint32_t g = tid; g < Ga; g += SV_THREADS)
        if (weight[g]) {
            mw = max(mw, (unsigned long long)weight[g]);
            mr = max(mr, order[g]);
        }
    for (int o = 16; o; o >>= 1) {
        mw = max(mw, __shfl_xor_sync(0xffffffffu, mw, o));
        mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    }
    if (lane == 0) {
        atomicMax(&s_maxw, mw);
        atomicMax(&s_maxr, mr);
    }
    __syncthreads();
    const int rbits = max(1, bit_width_u64(s_maxr)), bits = rbits + max(1, bit_width_u64(s_maxw));
    for (uint32_t g = tid; g < Ga; g += SV_THREADS) {
        const uint64_t w = weight[g];
        // an empty (reserved, unused) gid sorts after every group
        s_key[g] = w ? ((s_maxw - w) << rbits) | order[g] : low_mask(bits);
        s_idx[g] = (uint16_t)g;
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    int cur = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        for (int i = tid; i < SV_WARPS * 256; i += SV_THREADS) (&s_whist[0][0])[i] = 0;
        __syncthreads();
        const uint16_t* src = s_idx + cur * SV_MAX;
        uint16_t* dst = s_idx + (cur ^ 1) * SV_MAX;
        uint32_t dp[SV_IPT];
        uint16_t gv[SV_IPT];
#pragma unroll
        for (int j = 0; j < SV_IPT; ++j) {   // striped: (warp, j, lane) is position order (stable)
            const uint32_t pos = warp * (32 * SV_IPT) + j * 32 + lane;
            uint32_t d = 255;
            gv[j] = 0;
            if (pos < Ga) {
                gv[j] = src[pos];
                d = (uint32_t)(s_key[gv[j]] >> shift) & 255u;
            }
            uint32_t peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
                peers &= ((d >> b) & 1u) ? bal : ~bal;
            }
            const int leader = __ffs(peers) - 1;
            uint32_t bse = 0;
            if (lane == leader) {
                bse = s_whist[warp][d];
                s_whist[warp][d] = bse + __popc(peers);
            }
            bse = __shfl_sync(0xffffffffu, bse, leader);
            dp[j] = (d << 16) | (bse + __popc(peers & lt));
            __syncwarp();
        }
        __syncthreads();
        // digit-major, warp-minor exclusive offsets (digit d = thread d of the first 256)
        uint32_t tot = 0;
        if (tid < 256)
            for (int w = 0; w < SV_WARPS; ++w) {
                const uint32_t c = s_whist[w][tid];
                s_whist[w][tid] = tot;
                tot += c;
            }
        const uint32_t start = block_excl_scan<SV_THREADS>(tid < 256 ? tot : 0u, s_scan, nullptr);
        if (tid < 256)
            for (int w = 0; w < SV_WARPS; ++w) s_whist[w][tid] += start;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < SV_IPT; ++j) {
            const uint32_t pos = warp * (32 * SV_IPT) + j * 32 + lane;
            if (pos < Ga) dst[(dp[j] & 0xffffu) + s_whist[warp][dp[j] >> 16]] = gv[j];
        }
        __syncthreads();
        cur ^= 1;
    }
    // emit position p (< G: the real groups come first) and scan the lengths.  The
    // keys' shared memory now holds s_it (the representative item, then its first
    // row) and s_len (lengths, then their exclusive prefix).
    const uint16_t* ord = s_idx + cur * SV_MAX;
    uint32_t* s_it = (uint32_t*)s_key;
    uint32_t* s_len = s_it + SV_MAX;
    __syncthreads();
#pragma unroll 4
    for (uint32_t p = tid; p < Ga; p += SV_THREADS) {
        const uint32_t g = ord[p];
        inv[g] = p;
        s_it[p] = rep[g];
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t p = tid; p < SV_MAX; p += SV_THREADS) {
        uint32_t L = 0;
        if (p < G) {
            const uint32_t it = s_it[p], f = off[it];
            L = off[it + 1] - f;
            count[p] = weight[ord[p]];
            len[p] = L;
            rep_case[p] = rep_code[it];
            ok1[p] = k1[it];
            ok2[p] = k2[it];
            s_it[p] = f;
        }
        s_len[p] = L;
    }
    __syncthreads();
    // exclusive scan of s_len[0..SV_MAX): SV_IPT consecutive entries per thread
    uint32_t loc[SV_IPT], sum = 0;
#pragma unroll
    for (int j = 0; j < SV_IPT; ++j) {
        loc[j] = s_len[tid * SV_IPT + j];
        sum += loc[j];
    }
    uint32_t total = 0;
    uint32_t ex = block_excl_scan<SV_THREADS>(sum, s_scan, &total);
#pragma unroll
    for (int j = 0; j < SV_IPT; ++j) {
        const uint32_t p = tid * SV_IPT + j;
        if (p < G) seq_off[p] = ex;
        s_len[p] = ex;   // in place: each thread rewrites only its own entries
        ex += loc[j];
    }
    if (tid == 0) seq_off[G] = total;
    __syncthreads();
    // the representatives' sequences, flattened: element i belongs to the last
    // variant p with s_len[p] <= i (binary search over the G prefix sums)
#pragma unroll 4
    for (uint32_t i = tid; i < total; i += SV_THREADS) {
        uint32_t lo = 0, hi = G;
        while (hi - lo > 1) {
            const uint32_t m = (lo + hi) >> 1;
            if (s_len[m] <= i) lo = m; else hi = m;
        }
        seq_act[i] = (uint32_t)acts[s_it[lo] + (i - s_len[lo])];
    }
}

// ------------------------------------------------------------------ medium variant tables, one launch
// Up to VO_MAX groups: ONE cooperative kernel (grid-wide barriers instead of
// kernel boundaries) orders the groups by (count desc, rep asc) with an LSD
// radix sort in the reduce-then-scan form -- every CTA owns a contiguous chunk
// of <= 4096 groups; per pass it histograms its chunk, reads every chunk's
// histogram to place its digits (no look-back chain), and scatters stably with
// the ballot ranking -- then emits count / len / rep_case / keys, the sequence
// offsets (chunk totals + in-chunk scan) and the representatives' sequences,
// and finally every case's variant index.  Replaces ~14 launches (sort keys,
// histogram, scan, 5-6 radix passes, inverse, emit, scan, gather, case index)
// whose latency dominated at these sizes.
#ifndef PM4G_VO_IPT
#define PM4G_VO_IPT 8
#endif
constexpr int VO_THREADS = 512, VO_WARPS = VO_THREADS / 32, VO_IPT = PM4G_VO_IPT, VO_CHUNK = VO_THREADS * VO_IPT;
constexpr uint64_t VO_MAX_GROUPS = 296ull * VO_CHUNK;   // chunks of <= 4096 over co-resident CTAs (order_medium checks the real occupancy)
constexpr pm4g_status VO_NOT_LAUNCHED = (pm4g_status)100;   // internal: the cooperative grid was refused
#ifndef PM4G_VO_TARGET
#define PM4G_VO_TARGET 256   // groups per chunk aimed at (more CTAs, but each reads every chunk's histogram)
#endif

struct VoArgs {
    const uint64_t* weight;
    const uint32_t* order;     // the groups' order keys (min order of their items)
    const uint32_t* rep;       // the groups' representative items
    uint32_t Ga, G, chunk;
    const uint32_t* off;
    const uint32_t* rep_code;
    const uint64_t* k1;
    const uint64_t* k2;
    const uint32_t* item_group;
    uint64_t n_items;
    uint64_t* count;
    uint32_t* len;
    uint32_t* rep_case;
    uint64_t* seq_off;
    uint32_t* seq_act;
    uint64_t* ok1;
    uint64_t* ok2;
    uint32_t* inv;
    uint32_t* case_variant;    // nullptr: not requested
    uint64_t* key[2];          // [Ga] each
    uint32_t* val[2];          // [Ga] each
    uint32_t* hist;            // [gridDim.x][256]
    uint32_t* tot;             // [max(gridDim.x, 256)]: digit totals, then chunk length totals
    unsigned long long* mx;    // [2]: max weight, max rep (zeroed)
    unsigned long long* trace; // debug (PM4G_VO_TRACE): CTA 0's %globaltimer at each phase
};
__device__ __forceinline__ unsigned long long vo_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <class ACT>
__global__ __launch_bounds__(VO_THREADS) void k_vorder(VoArgs a, const ACT* __restrict__ acts) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t s_whist[VO_WARPS][256];
    __shared__ uint32_t s_run[256], s_hist[256];
    __shared__ uint32_t s_scan[VO_WARPS + 1];
    extern __shared__ __align__(16) uint32_t vo_dyn[];   // [VO_CHUNK] first rows | [VO_CHUNK] prefixes
    uint32_t* s_f = vo_dyn;
    uint32_t* s_ex = vo_dyn + VO_CHUNK;
    __shared__ unsigned long long s_pre;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t c = blockIdx.x, nc = gridDim.x;
    const uint32_t lo = min(a.Ga, c * a.chunk), hi = min(a.Ga, lo + a.chunk), cn = hi - lo;
    const uint32_t lt = lanemask_lt();
    int ntr = 0;
    auto mark = [&]() { if (a.trace && c == 0 && tid == 0) a.trace[ntr++] = vo_now(); };
    mark();
    // 1. key bits from the largest weight and representative
    {
        unsigned long long mw = 0, mr = 0;
        for (uint32_t g = lo + tid; g < hi; g += VO_THREADS)
            if (a.weight[g]) {
                mw = max(mw, (unsigned long long)a.weight[g]);
                mr = max(mr, (unsigned long long)a.order[g]);
            }
        for (int o = 16; o; o >>= 1) {
            mw = max(mw, __shfl_xor_sync(0xffffffffu, mw, o));
            mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        }
        if (lane == 0) {
            if (mw) atomicMax(&a.mx[0], mw);
            if (mr) atomicMax(&a.mx[1], mr);
        }
    }
    grid.sync();
    mark();
    const unsigned long long maxw = ld_volatile(&a.mx[0]), maxr = ld_volatile(&a.mx[1]);
    const int rbits = max(1, bit_width_u64(maxr)), bits = rbits + max(1, bit_width_u64(maxw));
    for (uint32_t g = lo + tid; g < hi; g += VO_THREADS) {
        const uint64_t w = a.weight[g];
        // an empty (reserved, unused) gid sorts after every group
        a.key[0][g] = w ? ((maxw - w) << rbits) | a.order[g] : low_mask(bits);
        a.val[0][g] = g;
    }
    grid.sync();
    mark();
    // 2. LSD passes, 8 bits each
    int cur = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        const uint64_t* ik = a.key[cur];
        const uint32_t* iv = a.val[cur];
        uint64_t* okey = a.key[cur ^ 1];
        uint32_t* oval = a.val[cur ^ 1];
        uint64_t kk[VO_IPT];
        uint32_t vv[VO_IPT], dp[VO_IPT];
        for (int i = tid; i < VO_WARPS * 256; i += VO_THREADS) (&s_whist[0][0])[i] = 0;
        __syncthreads();
        // the chunk's items, striped (warp, j, lane) = position order; stable ranks per warp
#pragma unroll
        for (int j = 0; j < VO_IPT; ++j) {
            const uint32_t li = warp * (32 * VO_IPT) + j * 32 + lane;
            uint32_t d = 255;
            kk[j] = ~0ull;
            vv[j] = 0;
            if (li < cn) {
                kk[j] = ik[lo + li];
                vv[j] = iv[lo + li];
                d = (uint32_t)(kk[j] >> shift) & 255u;
            }
            uint32_t peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
                peers &= ((d >> b) & 1u) ? bal : ~bal;
            }
            const int leader = __ffs(peers) - 1;
            uint32_t bse = 0;
            if (lane == leader) {
                bse = s_whist[warp][d];
                s_whist[warp][d] = bse + __popc(peers);
            }
            bse = __shfl_sync(0xffffffffu, bse, leader);
            dp[j] = (d << 16) | (bse + __popc(peers & lt));
            __syncwarp();
        }
        __syncthreads();
        // the chunk's digit counts (padding ranks last under digit 255, not counted)
        if (tid < 256) {
            uint32_t t = 0;
            for (int w = 0; w < VO_WARPS; ++w) {
                const uint32_t x = s_whist[w][tid];
                s_whist[w][tid] = t;   // warp-exclusive prefix inside the chunk
                t += x;
            }
            if (tid == 255) t -= VO_CHUNK - cn;
            a.hist[(size_t)c * 256 + tid] = t;
        }
        uint32_t tot = 0, pre = 0;
        grid.sync();
        mark();
        // digit base: every chunk's counts of smaller digits, plus earlier chunks' of
        // this digit.  Each CTA reads the whole [nc][256] matrix (rows coalesced;
        // thread t sums digit t & 255 over half t >> 8 of the chunks), so no
        // separate scan phase and barrier is needed.
        {
            const uint32_t d = tid & 255, half = tid >> 8;
            const uint32_t q0 = half ? (nc + 1) / 2 : 0u, q1 = half ? nc : (nc + 1) / 2;
            uint32_t t = 0, pr = 0;
#pragma unroll 8
            for (uint32_t q = q0; q < q1; ++q) {
                const uint32_t h = a.hist[(size_t)q * 256 + d];
                t += h;
                pr += q < c ? h : 0u;
            }
            if (half) {
                s_hist[d] = t;
                s_run[d] = pr;
            }
            __syncthreads();
            if (!half) {
                t += s_hist[d];
                pr += s_run[d];
            }
            __syncthreads();
            tot = half ? 0u : t;
            pre = half ? 0u : pr;
        }
        const uint32_t base = block_excl_scan<VO_THREADS>(tot, s_scan, nullptr);
        if (tid < 256) s_run[tid] = base + pre;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < VO_IPT; ++j) {
            const uint32_t li = warp * (32 * VO_IPT) + j * 32 + lane;
            if (li >= cn) continue;
            const uint32_t d = dp[j] >> 16;
            const uint32_t pos = s_run[d] + s_whist[warp][d] + (dp[j] & 0xffffu);
            okey[pos] = kk[j];
            oval[pos] = vv[j];
        }
        grid.sync();
        mark();
        cur ^= 1;
    }
    // 3. emission of this chunk's output positions [lo, hi)
    const uint32_t* ord = a.val[cur];
    uint32_t myL[VO_IPT], sum = 0;
#pragma unroll
    for (int j = 0; j < VO_IPT; ++j) {   // thread tid owns positions lo + tid * VO_IPT + j (consecutive)
        const uint32_t li = tid * VO_IPT + j, p = lo + li;
        myL[j] = 0;
        if (li >= cn) continue;
        const uint32_t g = ord[p];
        a.inv[g] = p;
        if (p < a.G) {
            const uint32_t it = a.rep[g], f = a.off[it];
            myL[j] = a.off[it + 1] - f;
            a.count[p] = a.weight[g];
            a.len[p] = myL[j];
            a.rep_case[p] = a.rep_code[it];
            a.ok1[p] = a.k1[it];
            a.ok2[p] = a.k2[it];
            s_f[li] = f;
        }
        sum += myL[j];
    }
    uint32_t ctot = 0;
    uint32_t ex = block_excl_scan<VO_THREADS>(sum, s_scan, &ctot);
#pragma unroll
    for (int j = 0; j < VO_IPT; ++j) {
        s_ex[tid * VO_IPT + j] = ex;
        ex += myL[j];
    }
    if (tid == 0) a.tot[c] = ctot;
    grid.sync();
    mark();
    if (tid == 0) {
        unsigned long long pr = 0;
        for (uint32_t q = 0; q < c; ++q) pr += a.tot[q];
        s_pre = pr;
    }
    __syncthreads();
    const unsigned long long pre = s_pre;
    const uint32_t creal = a.G > lo ? min(cn, a.G - lo) : 0u;   // real groups in this chunk
    for (uint32_t li = tid; li < creal; li += VO_THREADS) a.seq_off[lo + li] = pre + s_ex[li];
    if (creal && lo + creal == a.G && tid == 0) a.seq_off[a.G] = pre + ctot;
    if (a.G == 0 && c == 0 && tid == 0) a.seq_off[0] = 0;
    // the chunk's sequences, flattened: thread t writes output elements
    // [t E, (t + 1) E) of the chunk -- one binary search for its first element's
    // variant, then a walk across the variant boundaries (work balanced whatever
    // the lengths; a search per element cost 2x at 100M)
    {
        const uint32_t E = (ctot + VO_THREADS - 1) / VO_THREADS;
        const uint32_t i0 = min(ctot, tid * E), i1 = min(ctot, i0 + E);
        if (i0 < i1) {
            uint32_t l = 0, h = creal;
            while (h - l > 1) {
                const uint32_t m = (l + h) >> 1;
                if (s_ex[m] <= i0) l = m; else h = m;
            }
            uint32_t nxt = l + 1 < creal ? s_ex[l + 1] : ctot;
            uint32_t src = s_f[l] + (i0 - s_ex[l]);
            uint32_t* dst = a.seq_act + pre;
            for (uint32_t i = i0; i < i1; ++i) {
                while (i == nxt) {   // next variant (every length >= 1)
                    ++l;
                    src = s_f[l];
                    nxt = l + 1 < creal ? s_ex[l + 1] : ctot;
                }
                dst[i] = (uint32_t)acts[src++];
            }
        }
    }
    // 4. every case's variant index (inv complete after the barrier)
    if (a.case_variant) {
        grid.sync();
        for (uint64_t q = (uint64_t)c * VO_THREADS + tid; q < a.n_items; q += (uint64_t)nc * VO_THREADS)
            a.case_variant[q] = a.inv[a.item_group[q]];
    }
    __syncthreads();
    mark();
    if (a.trace && c == 0 && tid == 0) a.trace[63] = ntr;
}

// The one-pass grouping of a log's cases.  *fallback = true when the general
// engine must run instead (a hash collision); otherwise *out holds the groups
// in output order (sorted, inv) exactly as group_items leaves them.
template <class ACT>
static pm4g_status group_cases_fast(uint64_t n_items, const uint64_t* k1, const uint64_t* k2, const uint32_t* off,
                                    const ACT* acts, const uint64_t* weight, const uint32_t* order, int order_bits,
                                    cudaStream_t s, Groups* out,
                                    const uint64_t* d_n, uint64_t* n_true, bool* fallback) {
    *fallback = false;
    if (n_true) *n_true = n_items;
    Groups g;
    auto bail = [&](pm4g_status st) {
        g.free(s);
        return st;
    };
    pm4g_status st;
    const uint64_t N = std::max<uint64_t>(n_items, 1);
    if ((st = dalloc_t(&g.item_group, N, s))) return bail(st);
    if (n_items == 0) {
        *out = g;
        return PM4G_OK;
    }
    const uint64_t full = pow2_at_least(std::max<uint64_t>(1024, 2 * n_items));
    // a log's cases hold few distinct sequences; the merge's items (the shards'
    // variants) are mostly distinct: a table that never trips its load limit
    uint64_t cap = std::min<uint64_t>(full, weight ? pow2_at_least(n_items)
                                                   : std::max<uint64_t>(1ull << 19, pow2_at_least(n_items / 8)));
    if (const uint64_t dc = debug_variant_cap()) cap = std::min<uint64_t>(full, pow2_at_least(std::max<uint64_t>(dc, 64)));
    uint64_t G = 0, Ga = 0, htot = 0, gcap = 0;
    Scratch gw(s);
    const bool small = n_items < (uint64_t)num_sms() * 8 * 128;   // fewer 128-case tasks than warps
    const bool fine = small;   // gids one by one (no empty ones: the table may take k_small_variants)
    const int ipt = small ? 1 : PM4G_VG_IPT;
    auto kern = small ? k_vgroup<ACT, 1, 1> : k_vgroup<ACT, PM4G_VG_IPT, 8>;
    PM4G_MAX_SMEM((k_vgroup<ACT, 1, 1>));
    PM4G_MAX_SMEM((k_vgroup<ACT, PM4G_VG_IPT, 8>));
    static int per_sm = -1;
    if (per_sm < 0)
        PM4G_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vgroup<ACT, PM4G_VG_IPT, 8>, VG_THREADS, VG_SMEM));
    const uint64_t tasks = (n_items + 32 * ipt - 1) / (32 * ipt);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((tasks + VG_THREADS / 32 - 1) / (VG_THREADS / 32),
                                                                    (uint64_t)std::max(per_sm, 1) * num_sms()));
    const uint64_t slack = (uint64_t)grid * (VG_THREADS / 32) * 2 * (fine ? 1 : 8);   // unused reserved gids
    for (int attempt = 0;; ++attempt) {
        // groups never exceed the items; the table's claims stop near 3/4 load
        // (reserved gids past gcap abandon the table)
        gcap = std::min<uint64_t>(n_items, cap == full ? cap : cap / 4 * 3) + slack;
        Scratch tab(s);
        if ((st = tab.alloc(cap * sizeof(VSlot)))) return bail(st);
        if ((st = gw.alloc(gcap * 8 + 64))) return bail(st);
        uint32_t* g_w = gw.as<uint32_t>();
        uint32_t* g_rep = g_w + gcap;
        uint32_t* ctl = g_rep + gcap;   // [0] overflow [1] reserved gids [2] collisions [3] groups
        unsigned long long* d_tot = (unsigned long long*)(ctl + 4);
        uint32_t* d_task = ctl + 6;     // u64 task counter
        PM4G_CK(cudaMemsetAsync(ctl, 0, 32, s));
        PM4G_LAUNCH("k_variant_init", cap * 32.0 + gcap * 8.0, s,
                    (k_vinit<<<gsz(std::max(cap, gcap)), 256, 0, s>>>(tab.as<VSlot>(), cap, g_w, g_rep, gcap)));
        PM4G_LAUNCH("k_variant_group", n_items * 36.0, s,
                    (kern<<<grid, VG_THREADS, VG_SMEM, s>>>(n_items, d_n, k1, k2, off, acts, weight, order, tab.as<VSlot>(),
                                                                     cap - 1, (uint32_t)gcap, g_w, g_rep,
                                                                     g.item_group, ctl, d_tot, d_task)));
        // one host round trip: overflow, gids, collisions, groups, total length (+ the case count)
        static thread_local unsigned char* h_stage = nullptr;
        if (!h_stage) PM4G_CK(cudaHostAlloc((void**)&h_stage, 64, cudaHostAllocDefault));
        PM4G_TRY(copy_words_to_host(h_stage, ctl, 24, s));
        if (d_n) PM4G_TRY(copy_words_to_host(h_stage + 32, d_n, 8, s));
        PM4G_TRY(stream_sync(s));
        uint32_t h[4];
        memcpy(h, h_stage, 16);
        memcpy(&htot, h_stage + 16, 8);
        if (d_n) {
            uint64_t hn;
            memcpy(&hn, h_stage + 32, 8);
            n_items = std::min(n_items, hn);
            if (n_true) *n_true = n_items;
        }
        if (h[2]) {   // a collision: the general engine handles it exactly
            *fallback = true;
            return bail(PM4G_OK);
        }
        if (h[0]) {
            if (cap >= full || attempt > 16) return bail(fail(PM4G_ENOMEM, "variant table overflow"));
            cap = std::min<uint64_t>(full, cap * 4);
            continue;
        }
        Ga = h[1];   // reserved gids: the groups plus the warps' unused ones (empty, sorted last)
        G = h[3];
        if (G > Ga) return bail(fail(PM4G_ECUDA, "variant grouping: gid count mismatch"));
        break;
    }
    g.G = G;
    g.Ga = Ga;
    g.total_len = htot;
    const uint64_t Ga1 = std::max<uint64_t>(Ga, 1);
    if ((st = dalloc_t(&g.weight, Ga1, s))) return bail(st);
    if ((st = dalloc_t(&g.rep_item, Ga1, s))) return bail(st);
    if ((st = dalloc_t(&g.order, Ga1, s))) return bail(st);
    if ((st = dalloc_t(&g.inv, Ga1, s))) return bail(st);
    const int wbits = weight ? 32 : std::max(1, bit_width_u64(n_items));   // u32 counts
    const uint32_t* g_w = gw.as<uint32_t>();
    // the weighted merge: the item holding each group's minimum order represents it
    auto rep_items = [&]() -> pm4g_status {
        if (order && Ga)
            PM4G_LAUNCH("k_variant_rep", n_items * 12.0, s,
                        (k_vrepitem<<<gsz(n_items), 256, 0, s>>>(order, g.item_group, g_w + gcap, n_items, g.rep_item)));
        return PM4G_OK;
    };
    static const uint64_t vo_max = getenv("PM4G_VO_MAX") ? strtoull(getenv("PM4G_VO_MAX"), nullptr, 10) : VO_MAX_GROUPS;
    if (Ga <= std::min(vo_max, VO_MAX_GROUPS)) {   // ordered and emitted in one launch (k_small_variants / k_vorder)
        if (Ga)
            PM4G_LAUNCH("k_variant_sortkeys", Ga * 20.0, s,
                        (k_vfinal<<<gsz(Ga), 256, 0, s>>>(g_w, g_w + gcap, Ga, wbits, order_bits, g.weight,
                                                          g.rep_item, g.order, nullptr, nullptr)));
        if ((st = rep_items())) return bail(st);
        *out = g;
        return PM4G_OK;
    }
    if ((st = dalloc_t(&g.sorted, Ga1, s))) return bail(st);
    Scratch sk(s);   // keys [Ga] u64 | group ids [Ga] u32 (the radix payload)
    if ((st = sk.alloc(Ga * 12 + 16))) return bail(st);
    uint32_t* sk_val = (uint32_t*)(sk.as<uint64_t>() + Ga);
    if (Ga) {
        PM4G_LAUNCH("k_variant_sortkeys", Ga * 28.0, s,
                    (k_vfinal<<<gsz(Ga), 256, 0, s>>>(g_w, g_w + gcap, Ga, wbits, order_bits, g.weight, g.rep_item,
                                                      g.order, sk.as<uint64_t>(), sk_val)));
        if ((st = rep_items())) return bail(st);
        if (Ga <= RANK_SORT_MAX)
            PM4G_LAUNCH("k_rank_sort", Ga * 12.0, s,
                        (k_rank_sort<<<(unsigned)((Ga + 255) / 256), 256, 0, s>>>(sk.as<uint64_t>(), (uint32_t)Ga, g.sorted)));
        else if ((st = radix_sort_u64_to(sk.as<uint64_t>(), sk_val, g.sorted, (int64_t)Ga, wbits + order_bits, s)))
            return bail(st);
        PM4G_LAUNCH("k_variant_inv", Ga * 8.0, s, (k_inv<<<gsz(Ga), 256, 0, s>>>(g.sorted, Ga, g.inv)));
    }
    *out = g;
    return PM4G_OK;
}

// The one-pass table's ordering with the library radix sort (the general path;
// used when the cooperative kernel cannot be launched): g.sorted / g.inv.
static pm4g_status order_groups_radix(Groups& g, int order_bits, uint64_t n_items, bool weighted, cudaStream_t s) {
    const uint64_t Ga = g.Ga, Ga1 = std::max<uint64_t>(Ga, 1);
    const int wbits = weighted ? 32 : std::max(1, bit_width_u64(n_items));
    PM4G_TRY(dalloc_t(&g.sorted, Ga1, s));
    Scratch sk(s), gw(s);   // keys [Ga] | vals [Ga]; the u32 weights / reps k_vfinal reads
    PM4G_TRY(sk.alloc(Ga * 12 + 16));
    PM4G_TRY(gw.alloc(Ga * 8 + 16));
    uint64_t* key = sk.as<uint64_t>();
    uint32_t* val = (uint32_t*)(key + Ga);
    uint32_t* w32 = gw.as<uint32_t>();
    uint32_t* r32 = w32 + Ga;
    if (!Ga) return PM4G_OK;
    PM4G_LAUNCH("k_variant_sortkeys", Ga * 28.0, s,
                (k_vrekey<<<gsz(Ga), 256, 0, s>>>(g.weight, g.order, Ga, w32, r32)));
    PM4G_LAUNCH("k_variant_sortkeys", Ga * 28.0, s,
                (k_vfinal<<<gsz(Ga), 256, 0, s>>>(w32, r32, Ga, wbits, order_bits, g.weight, nullptr, g.order,
                                                  key, val)));
    PM4G_TRY(radix_sort_u64_to(key, val, g.sorted, (int64_t)Ga, wbits + order_bits, s));
    PM4G_LAUNCH("k_variant_inv", Ga * 8.0, s, (k_inv<<<gsz(Ga), 256, 0, s>>>(g.sorted, Ga, g.inv)));
    return PM4G_OK;
}

// k_vorder: the medium one-pass table ordered, emitted and indexed in one cooperative launch
template <class ACT>
static pm4g_status order_medium(Groups& g, pm4g_variant_table* v, const uint32_t* off, const ACT* acts,
                                const uint32_t* rep_code, const uint64_t* k1, const uint64_t* k2, uint64_t n_items,
                                bool with_case_variant, cudaStream_t s) {
    constexpr size_t dyn = 2 * VO_CHUNK * 4;
    PM4G_MAX_SMEM(k_vorder<ACT>);
    static int per_sm = -1;
    if (per_sm < 0)
        PM4G_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vorder<ACT>, VO_THREADS, dyn));
    const uint64_t Ga = g.Ga;
    const uint64_t maxc = (uint64_t)std::max(per_sm, 1) * num_sms();
    // one chunk per SM at most, unless the table needs more (every CTA reads every
    // chunk's histogram per pass: 296 chunks of a 300k table cost 15 us more than 148)
    uint64_t nc = std::min<uint64_t>((uint64_t)num_sms(), std::max<uint64_t>((Ga + PM4G_VO_TARGET - 1) / PM4G_VO_TARGET, 1));
    nc = std::max<uint64_t>(nc, (Ga + VO_CHUNK - 1) / VO_CHUNK);
    nc = std::min<uint64_t>(nc, 2 * VO_THREADS);
    if (nc > maxc || nc * VO_CHUNK < Ga) {   // more groups than co-resident chunks hold: radix passes
        if (getenv("PM4G_VO_TRACE")) fprintf(stderr, "k_vorder: Ga=%llu past capacity\n", (unsigned long long)Ga);
        return VO_NOT_LAUNCHED;
    }
    Scratch sc(s);
    const size_t kb = ((Ga * 8 + 15) & ~(size_t)15), vb = ((Ga * 4 + 15) & ~(size_t)15);
    PM4G_TRY(sc.alloc(2 * kb + 2 * vb + nc * 256 * 4 + std::max<uint64_t>(nc, 256) * 4 + 64));
    char* b = (char*)sc.p;
    VoArgs a{};
    a.weight = g.weight;
    a.order = g.order;
    a.rep = g.rep_item;
    a.Ga = (uint32_t)Ga;
    a.G = (uint32_t)g.G;
    a.chunk = (uint32_t)((Ga + nc - 1) / nc);
    a.off = off;
    a.rep_code = rep_code;
    a.k1 = k1;
    a.k2 = k2;
    a.item_group = g.item_group;
    a.n_items = n_items;
    a.count = v->count;
    a.len = v->len;
    a.rep_case = v->rep_case;
    a.seq_off = v->seq_off;
    a.seq_act = v->seq_act;
    a.ok1 = v->k1;
    a.ok2 = v->k2;
    a.inv = g.inv;
    a.key[0] = (uint64_t*)b;
    a.key[1] = (uint64_t*)(b + kb);
    a.val[0] = (uint32_t*)(b + 2 * kb);
    a.val[1] = (uint32_t*)(b + 2 * kb + vb);
    a.hist = (uint32_t*)(b + 2 * kb + 2 * vb);
    a.tot = a.hist + nc * 256;
    a.mx = (unsigned long long*)(((uintptr_t)(a.tot + std::max<uint64_t>(nc, 256)) + 15) & ~(uintptr_t)15);
    // the per-case index in the same launch for small logs; a wide grid gathers it faster otherwise
    const bool cv_inside = with_case_variant && n_items <= (1ull << 20);
    if (with_case_variant) PM4G_TRY(dalloc_t(&v->case_variant, std::max<uint64_t>(n_items, 1), s));
    if (cv_inside) a.case_variant = v->case_variant;
    PM4G_CK(cudaMemsetAsync(a.mx, 0, 16, s));
    static const bool trace = getenv("PM4G_VO_TRACE") != nullptr;
    static unsigned long long* d_trace = nullptr;
    if (trace && !d_trace) PM4G_CK(cudaMalloc(&d_trace, 64 * 8));
    a.trace = trace ? d_trace : nullptr;
    void* args[] = {(void*)&a, (void*)&acts};
    // a cooperative grid can be refused (e.g. too large while other work holds the
    // device, or under a tool): the caller then orders the table with the radix passes
    const bool no_coop = getenv("PM4G_DEBUG_NO_COOP") != nullptr;   // test hook: force the fallback
    if (no_coop) return VO_NOT_LAUNCHED;
    prof_begin("k_variant_order", Ga * 60.0 + g.total_len * 5.0 + (cv_inside ? n_items * 8.0 : 0.0), s);
    const cudaError_t le = cudaLaunchCooperativeKernel((const void*)k_vorder<ACT>, dim3((unsigned)nc),
                                                       dim3(VO_THREADS), args, dyn, s);
    prof_end(s);
    if (le != cudaSuccess) {
        cudaGetLastError();
        if (trace)
            fprintf(stderr, "k_vorder not launched (%s): G=%llu Ga=%llu nc=%llu per_sm=%d\n", cudaGetErrorString(le),
                    (unsigned long long)g.G, (unsigned long long)Ga, (unsigned long long)nc, per_sm);
        return VO_NOT_LAUNCHED;
    }
    count_launch();
    if (trace) {
        unsigned long long h[64];
        pm4g_status gs;
        const bool seg = gseg_suspend(s, &gs);
        PM4G_TRY(gs);
        PM4G_CK(cudaMemcpyAsync(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost, s));
        PM4G_CK(cudaStreamSynchronize(s));
        if (seg) PM4G_TRY(gseg_resume());
        fprintf(stderr, "k_vorder G=%llu Ga=%llu nc=%llu chunk=%u phases(us):", (unsigned long long)g.G, (unsigned long long)Ga, (unsigned long long)nc, a.chunk);
        for (unsigned i = 1; i < h[63] && i < 63; ++i) fprintf(stderr, " %.1f", (h[i] - h[i - 1]) / 1e3);
        fprintf(stderr, "\n");
    }
    if (with_case_variant && !cv_inside && n_items)
        PM4G_LAUNCH("k_case_variant", n_items * 8.0, s,
                    (k_case_variant<<<gsz(n_items), 256, 0, s>>>(g.item_group, g.inv, n_items, v->case_variant)));
    return PM4G_OK;
}

// the per-case variant index (output position of each item's group), then the
// groups' scratch is released and the table handed out
static pm4g_status case_variant_index(const Groups& g, pm4g_variant_table* v, uint64_t n_items, cudaStream_t s) {
    PM4G_TRY(dalloc_t(&v->case_variant, std::max<uint64_t>(n_items, 1), s));
    if (n_items)
        PM4G_LAUNCH("k_case_variant", n_items * 8.0, s,
                    (k_case_variant<<<gsz(n_items), 256, 0, s>>>(g.item_group, g.inv, n_items, v->case_variant)));
    return PM4G_OK;
}

static pm4g_status finish_variants(Groups& g, pm4g_variant_table* v, uint64_t n_items, bool with_case_variant,
                                   cudaStream_t s, pm4g_variant_table** out) {
    const pm4g_status st = with_case_variant ? case_variant_index(g, v, n_items, s) : PM4G_OK;
    g.free(s);
    if (st) {
        free_variants(v);
        return st;
    }
    *out = v;
    return PM4G_OK;
}

template <class OFF, class ACT>
static pm4g_status build_variants(uint64_t n_items, const uint64_t* k1, const uint64_t* k2,
                                  const OFF* off, const ACT* acts, const uint64_t* weight,
                                  const uint32_t* order, int order_bits, const uint32_t* rep_code,
                                  bool with_case_variant, cudaStream_t s, pm4g_variant_table** out,
                                  const uint64_t* d_n = nullptr, uint64_t* n_true = nullptr) {
    Groups g;
    uint64_t nt = n_items;
    bool general = true;
    const uint64_t* dn = d_n;
    if constexpr (sizeof(OFF) == 4) {   // a log's cases: the one-pass grouping unless it meets a collision
        // (weak debug keys collide: they exercise the fallback)
        if (!weight == !order) {
            PM4G_TRY((group_cases_fast<ACT>(n_items, k1, k2, (const uint32_t*)off, acts, weight, order, order_bits, s,
                                            &g, d_n, &nt, &general)));
            if (general) {   // the case count is known now
                n_items = nt;
                dn = nullptr;
            }
        }
    }
    if (general)
        PM4G_TRY((group_items<OFF, ACT>(n_items, k1, k2, off, acts, weight, order, order_bits, s, &g,
                                        dn, &nt)));
    n_items = nt;
    if (n_true) *n_true = nt;
    pm4g_variant_table* v = new pm4g_variant_table();
    v->stream = s;
    v->V = g.G;
    v->n_cases = with_case_variant ? n_items : 0;
    auto bail = [&](pm4g_status st) {
        g.free(s);
        free_variants(v);
        return st;
    };
    pm4g_status st;
    const uint64_t V1 = std::max<uint64_t>(g.G, 1);
    if ((st = dalloc_t(&v->count, V1, s))) return bail(st);
    if ((st = dalloc_t(&v->len, V1, s))) return bail(st);
    if ((st = dalloc_t(&v->rep_case, V1, s))) return bail(st);
    if ((st = dalloc_t(&v->seq_off, V1 + 1, s))) return bail(st);
    if ((st = dalloc_t(&v->k1, V1, s))) return bail(st);
    if ((st = dalloc_t(&v->k2, V1, s))) return bail(st);
    const uint64_t total = g.total_len;   // summed with the grouping, read with its counters
    v->total_len = total;
    if ((st = dalloc_t(&v->seq_act, std::max<uint64_t>(total, 1), s))) return bail(st);
    if constexpr (sizeof(OFF) == 4) {
        if (!g.sorted && g.Ga > (uint64_t)SV_MAX) {   // a medium one-pass table: one cooperative launch
            const pm4g_status vs = order_medium<ACT>(g, v, (const uint32_t*)off, acts, rep_code, k1, k2, n_items,
                                                     with_case_variant, s);
            if (vs == PM4G_OK) {
                g.free(s);
                *out = v;
                return PM4G_OK;
            }
            if (vs != VO_NOT_LAUNCHED) return bail(vs);
            // not launched: order with the radix passes, then the general emission below
            if (v->case_variant) {
                dfree(v->case_variant, s);
                v->case_variant = nullptr;
            }
            const pm4g_status os = order_groups_radix(g, order_bits, n_items, weight != nullptr, s);
            if (os) return bail(os);
        }
        if (!g.sorted) {   // a small one-pass table: ordered and emitted by one CTA
            PM4G_MAX_SMEM(k_small_variants<ACT>);
            PM4G_LAUNCH("k_variant_small", g.Ga * 24.0 + g.G * 40.0 + total * 5.0, s,
                        (k_small_variants<ACT><<<1, SV_THREADS, SV_SMEM, s>>>(
                            g.weight, g.order, g.rep_item, (uint32_t)g.Ga, (uint32_t)g.G, (const uint32_t*)off, acts, rep_code,
                            k1, k2, v->count, v->len, v->rep_case, v->seq_off, v->seq_act, v->k1, v->k2, g.inv)));
            return finish_variants(g, v, n_items, with_case_variant, s, out);
        }
    }
    if (g.G) {
        PM4G_LAUNCH("k_variant_emit", g.G * 40.0, s,
                    (k_emit<OFF><<<gsz(g.G), 256, 0, s>>>(g, off, rep_code, k1, k2, v->count, v->len,
                                                          v->rep_case, v->k1, v->k2)));
    }
    if ((st = excl_scan_u32_to_u64(v->len, v->seq_off, (int64_t)g.G, s))) return bail(st);
    if (g.G) {
        int gs = (int)std::max<uint64_t>(1, std::min<uint64_t>((g.G * SEQ_LANES + 255) / 256, (uint64_t)num_sms() * 64));
        PM4G_LAUNCH("k_variant_seq", (double)total * 8.0, s,
                    (k_seq_gather<OFF, ACT><<<gs, 256, 0, s>>>(g, off, acts, v->seq_off, v->seq_act)));
    }
    return finish_variants(g, v, n_items, with_case_variant, s, out);
}

pm4g_status variants_from_keys(const pm4g_log* L, const uint64_t* k1, const uint64_t* k2,
                               cudaStream_t s, pm4g_variant_table** out) {
    // without a known case count, start from the host bound (the aggregate
    // filled the keys of the true cases); round 0 reads the count itself
    const bool known = L->n_cases >= 0;
    const uint64_t C = known ? (uint64_t)L->n_cases
                             : std::min<uint64_t>((uint64_t)L->n, (uint64_t)(L->case_max - L->case_min) + 1);
    const uint64_t* dn = known ? nullptr : L->d_n_cases;
    int order_bits = bit_width_u64(C);
    uint64_t nt = C;
    pm4g_status st;
    switch (L->act_bytes) {
        case 1: st = build_variants<uint32_t, uint8_t>(C, k1, k2, L->off, (const uint8_t*)L->s_act, nullptr, nullptr, order_bits, L->s_case_code, true, s, out, dn, &nt); break;
        case 2: st = build_variants<uint32_t, uint16_t>(C, k1, k2, L->off, (const uint16_t*)L->s_act, nullptr, nullptr, order_bits, L->s_case_code, true, s, out, dn, &nt); break;
        default: st = build_variants<uint32_t, uint32_t>(C, k1, k2, L->off, (const uint32_t*)L->s_act, nullptr, nullptr, order_bits, L->s_case_code, true, s, out, dn, &nt); break;
    }
    if (st == PM4G_OK && !known) const_cast<pm4g_log*>(L)->n_cases = (int64_t)nt;
    return st;
}

// Merge R per-shard tables (disjoint case ranges): items = entries.  With
// local_part >= 0, the merged table also carries the case -> variant index of
// that part's cases: its local index composed with the merged position of the
// part's entries (the merge groups entries, so entry i of part r lands at
// item_out[offset_r + i]).
__global__ void k_compose_case_variant(const uint32_t* __restrict__ local_cv, uint64_t C,
                                       const uint32_t* __restrict__ item_out, uint64_t offset,
                                       uint32_t* __restrict__ out) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < C; c += (uint64_t)gridDim.x * blockDim.x)
        out[c] = item_out[offset + local_cv[c]];
}

// The merge's items, flat: entry i (of every part, part-major) has keys k1/k2,
// weight w (its count), order ord (its representative case) and sequence
// sa[so[i], so[i + 1]).  lp (optional) is the part whose per-case index the
// merged table carries; its entries start at item lp_first.
pm4g_status merge_flat(const MergeItems& in, const pm4g_variant_table* lp, uint64_t lp_first, cudaStream_t s,
                       pm4g_variant_table** out) {
    // the entries' sequences are addressed with u32 offsets
    if (in.V > 0xfffffffeull || in.T > (uint64_t)MAX_SHARD_EVENTS)
        return fail(PM4G_EINVAL, "merged variant tables exceed 2^31 - 2 activities");
    const bool compose = lp && lp->case_variant && lp->n_cases;
    pm4g_variant_table* v = nullptr;
    PM4G_TRY((build_variants<uint32_t, uint32_t>(in.V, in.k1, in.k2, in.so, in.sa, in.w, in.ord, 32, in.ord, compose,
                                                 s, &v)));
    if (compose) {   // v->case_variant holds item -> output for the V merged entries
        uint32_t* cv = nullptr;
        pm4g_status st = dalloc_t(&cv, std::max<uint64_t>(lp->n_cases, 1), s);
        if (st) {
            free_variants(v);
            return st;
        }
        PM4G_LAUNCH("k_compose_case_variant", lp->n_cases * 12.0, s,
                    (k_compose_case_variant<<<gsz(lp->n_cases), 256, 0, s>>>(lp->case_variant, lp->n_cases,
                                                                             v->case_variant, lp_first, cv)));
        dfree(v->case_variant, s);
        v->case_variant = cv;
        v->n_cases = lp->n_cases;
    }
    *out = v;
    return PM4G_OK;
}

// one part's entries into the flat items (its sequences start at tbase)
__global__ void k_flat_part(const pm4g_variant_table p, uint64_t tbase, MergeItems m, uint64_t vbase) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.V; i += (uint64_t)gridDim.x * blockDim.x) {
        m.k1[vbase + i] = p.k1[i];
        m.k2[vbase + i] = p.k2[i];
        m.w[vbase + i] = p.count[i];
        m.ord[vbase + i] = p.rep_case[i];
        m.so[vbase + i] = (uint32_t)(tbase + p.seq_off[i]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && vbase + p.V == m.V) m.so[m.V] = (uint32_t)m.T;
}

pm4g_status merge_items_alloc(uint64_t V, uint64_t T, Scratch& buf, MergeItems* m) {
    // k1 k2 w (u64, V) | so (u32, V + 1) | ord (u32, V) | sa (u32, T)
    PM4G_TRY(buf.alloc(V * 24 + 16 + (V + 1) * 4 + V * 4 + 16 + (T + 1) * 4));
    m->V = V;
    m->T = T;
    m->k1 = buf.as<uint64_t>();
    m->k2 = m->k1 + V;
    m->w = m->k2 + V;
    m->so = (uint32_t*)(m->w + V);
    m->ord = m->so + V + 1;
    m->sa = (uint32_t*)(((uintptr_t)(m->ord + V) + 15) & ~(uintptr_t)15);
    return PM4G_OK;
}

// Merge R per-shard tables (disjoint case ranges): items = entries.  With
// local_part >= 0, the merged table also carries the case -> variant index of
// that part's cases: its local index composed with the merged position of the
// part's entries (the merge groups entries, so entry i of part r lands at
// item_out[offset_r + i]).
pm4g_status merge_variant_tables(const pm4g_variant_table* const* parts, int n_parts, cudaStream_t s,
                                 pm4g_variant_table** out, int local_part) {
    uint64_t V = 0, T = 0;
    for (int r = 0; r < n_parts; ++r) {
        V += parts[r]->V;
        T += parts[r]->total_len;
    }
    if (V > 0xfffffffeull || T > (uint64_t)MAX_SHARD_EVENTS)
        return fail(PM4G_EINVAL, "merged variant tables exceed 2^31 - 2 activities");
    Scratch buf(s);
    MergeItems m;
    PM4G_TRY(merge_items_alloc(V, T, buf, &m));
    uint64_t vo = 0, to = 0, lp_first = 0;
    for (int r = 0; r < n_parts; ++r) {
        const pm4g_variant_table* p = parts[r];
        if (r == local_part) lp_first = vo;
        if (!p->V) continue;
        PM4G_LAUNCH("k_merge_flat", p->V * 64.0, s, (k_flat_part<<<gsz(p->V), 256, 0, s>>>(*p, to, m, vo)));
        PM4G_CK(cudaMemcpyAsync(m.sa + to, p->seq_act, p->total_len * 4, cudaMemcpyDeviceToDevice, s));
        vo += p->V;
        to += p->total_len;
    }
    if (!V) PM4G_CK(cudaMemsetAsync(m.so, 0, 4, s));   // (else the last part's k_flat_part writes so[V] = T)
    return merge_flat(m, local_part >= 0 ? parts[local_part] : nullptr, lp_first, s, out);
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_variants_size(const pm4g_variant_table* v, uint64_t* n_variants, uint64_t* total_len) {
    if (!v) return fail(PM4G_EINVAL, "null variants");
    if (n_variants) *n_variants = v->V;
    if (total_len) *total_len = v->total_len;
    return PM4G_OK;
}

pm4g_status pm4g_variants_get(const pm4g_variant_table* v, uint64_t* count, uint32_t* len,
                              uint32_t* rep_case, uint64_t* seq_off, uint32_t* seq_act,
                              pm4g_stream_t stream) {
    if (!v) return fail(PM4G_EINVAL, "null variants");
    cudaStream_t s = (cudaStream_t)stream;
    auto cp = [&](void* dst, const void* src, size_t b) -> pm4g_status {
        if (dst && b) PM4G_CK(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, s));
        return PM4G_OK;
    };
    PM4G_TRY(cp(count, v->count, v->V * 8));
    PM4G_TRY(cp(len, v->len, v->V * 4));
    PM4G_TRY(cp(rep_case, v->rep_case, v->V * 4));
    PM4G_TRY(cp(seq_off, v->seq_off, (v->V + 1) * 8));
    PM4G_TRY(cp(seq_act, v->seq_act, v->total_len * 4));
    return PM4G_OK;
}

pm4g_status pm4g_variants_case_index(const pm4g_variant_table* v, uint32_t* case_variant,
                                     pm4g_stream_t stream) {
    if (!v) return fail(PM4G_EINVAL, "null variants");
    if (v->n_cases && !case_variant) return fail(PM4G_EINVAL, "null output");
    if (!v->case_variant) return fail(PM4G_EINVAL, "merged tables carry no per-case index");
    if (v->n_cases)
        PM4G_CK(cudaMemcpyAsync(case_variant, v->case_variant, v->n_cases * 4,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return PM4G_OK;
}

pm4g_status pm4g_variants_destroy(pm4g_variant_table* v) {
    free_variants(v);
    return PM4G_OK;
}

pm4g_status pm4g_variants_merge(const pm4g_variant_table* const* parts, int32_t n_parts, int32_t local_part,
                                pm4g_stream_t stream, pm4g_variant_table** out) {
    PM4G_NVTX("pm4g_variants_merge");
    if (!parts || n_parts <= 0 || !out || local_part >= n_parts) return fail(PM4G_EINVAL, "bad arguments");
    for (int i = 0; i < n_parts; ++i)
        if (!parts[i]) return fail(PM4G_EINVAL, "null part");
    *out = nullptr;
    return merge_variant_tables(parts, n_parts, (cudaStream_t)stream, out, local_part < 0 ? -1 : local_part);
}

}  // extern "C"
