// NEXT-4: global repartition of an ingested (unsorted) log by case range
// (P:75-88 ingest of a columnar table; S:128-136,
// S:146, S:228-241 sharding by contiguous case ranges, R19).
//
// partition_rows: the stable split of a log's rows by destination rank,
// dest(row) = r with bounds[r] <= case < bounds[r + 1].  One radix pass keyed by
// the destination (stable, so each destination keeps the rows' original order)
// gives the permutation; every column is then gathered into one send buffer
// grouped by destination.  The exchange itself (pm4g_repartition) is in
// comm.cu: grouped ncclSend / ncclRecv over NVLink; pm4g_partition_by_case +
// pm4g_log_concat perform the same data movement on one device (tests, and
// single-process multi-shard use).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

__global__ void k_dest_keys(const uint32_t* __restrict__ cs, int64_t n, const uint32_t* __restrict__ bounds, int R,
                            uint64_t* __restrict__ key, uint32_t* __restrict__ val, unsigned long long* __restrict__ cnt) {
    __shared__ unsigned long long s_cnt[1024];
    for (int i = threadIdx.x; i < R; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cs[i];
        int a = 0, b = R;   // last r with bounds[r] <= c
        while (b - a > 1) {
            const int m = (a + b) >> 1;
            if (bounds[m] <= c) a = m; else b = m;
        }
        key[i] = (uint64_t)a;
        val[i] = (uint32_t)i;
        atomicAdd(&s_cnt[a], 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < R; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&cnt[i], s_cnt[i]);
}

template <class T>
__global__ void k_gather_rows(const T* __restrict__ in, const uint32_t* __restrict__ perm, int64_t n, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}

static pm4g_status gather_col(const void* in, int elem, const uint32_t* perm, int64_t n, void* out, cudaStream_t s) {
    if (n == 0) return PM4G_OK;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
    switch (elem) {
        case 1: PM4G_LAUNCH("k_gather_rows", n * 6.0, s, (k_gather_rows<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)in, perm, n, (uint8_t*)out))); break;
        case 2: PM4G_LAUNCH("k_gather_rows", n * 8.0, s, (k_gather_rows<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)in, perm, n, (uint16_t*)out))); break;
        case 4: PM4G_LAUNCH("k_gather_rows", n * 12.0, s, (k_gather_rows<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)in, perm, n, (uint32_t*)out))); break;
        default: PM4G_LAUNCH("k_gather_rows", n * 20.0, s, (k_gather_rows<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)in, perm, n, (uint64_t*)out))); break;
    }
    return PM4G_OK;
}

// the columns of an ingested log, in a fixed order: case, act, ts, then each
// extra column's data and (if nullable) its validity bytes
void log_columns(const pm4g_log* L, std::vector<const void*>* cols, std::vector<int>* elems) {
    cols->clear();
    elems->clear();
    cols->push_back(L->case_);
    elems->push_back(4);
    cols->push_back(L->act);
    elems->push_back(L->act_bytes);
    cols->push_back(L->ts);
    elems->push_back(8);
    for (const auto& x : L->extra) {
        cols->push_back(x.data);
        elems->push_back(x.elem);
        if (x.valid) {
            cols->push_back(x.valid);
            elems->push_back(1);
        }
    }
}

pm4g_status partition_rows(const pm4g_log* in, const uint32_t* bounds, int R, cudaStream_t s, PartitionedRows* out) {
    PM4G_TRY(materialize(const_cast<pm4g_log*>(in), s));   // a lazily filtered log: its kept rows
    PM4G_TRY(check_log(in));
    if (in->sorted) return fail(PM4G_EINVAL, "repartition needs an ingested (unsorted) log");
    if (R < 1 || R > 1024) return fail(PM4G_EINVAL, "1 <= R <= 1024 destinations");
    for (int r = 0; r < R; ++r)
        if (bounds[r] > bounds[r + 1]) return fail(PM4G_EINVAL, "bounds must be ascending");
    if ((uint64_t)bounds[R] > in->n_case_codes) return fail(PM4G_EINVAL, "bounds[R] > n_case_codes");
    if (in->n > 0 && (in->case_min < bounds[0] || (uint64_t)in->case_max >= (uint64_t)bounds[R]))
        return fail(PM4G_EINVAL, "a case code lies outside [bounds[0], bounds[R])");
    const int64_t n = in->n;
    std::vector<const void*> cols;
    std::vector<int> elems;
    log_columns(in, &cols, &elems);
    out->elems = elems;
    out->counts.assign(R, 0);
    // [bounds R+1 u32] [counts R u64] | keys u64[n] | perm u32[n] | columns (16-byte aligned each)
    Scratch meta(s), kv(s);
    PM4G_TRY(meta.alloc((R + 1) * 4 + 16 + R * 8));
    uint32_t* d_bounds = meta.as<uint32_t>();
    unsigned long long* d_cnt = (unsigned long long*)(((uintptr_t)(d_bounds + R + 1) + 15) & ~(uintptr_t)15);
    PM4G_CK(cudaMemcpyAsync(d_bounds, bounds, (R + 1) * 4, cudaMemcpyHostToDevice, s));
    PM4G_CK(cudaMemsetAsync(d_cnt, 0, R * 8, s));
    const int64_t N = std::max<int64_t>(n, 1);
    size_t col_off = 0;
    std::vector<size_t> offs;
    for (int e : elems) {
        offs.push_back(col_off);
        col_off += ((size_t)N * e + 15) & ~(size_t)15;
    }
    PM4G_TRY(out->buf.alloc(col_off + 16));
    PM4G_TRY(kv.alloc((size_t)N * 12 + 16));
    uint64_t* key = kv.as<uint64_t>();
    uint32_t* perm = (uint32_t*)(key + N);
    if (n > 0) {
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 4));
        PM4G_LAUNCH("k_dest_keys", n * 16.0, s, (k_dest_keys<<<g, 256, 0, s>>>(in->case_, n, d_bounds, R, key, perm, d_cnt)));
        if (R > 1) PM4G_TRY(radix_sort_u64(key, perm, n, bit_width_u64((uint64_t)(R - 1)), s));   // stable
    }
    std::vector<unsigned long long> hc(R, 0);
    PM4G_CK(cudaMemcpyAsync(hc.data(), d_cnt, R * 8, cudaMemcpyDeviceToHost, s));
    out->cols.clear();
    for (size_t c = 0; c < cols.size(); ++c) {
        void* dst = (char*)out->buf.p + offs[c];
        out->cols.push_back(dst);
        if (n > 0 && R > 1) PM4G_TRY(gather_col(cols[c], elems[c], perm, n, dst, s));
        else if (n > 0) PM4G_CK(cudaMemcpyAsync(dst, cols[c], (size_t)n * elems[c], cudaMemcpyDeviceToDevice, s));
    }
    PM4G_CK(cudaStreamSynchronize(s));
    for (int r = 0; r < R; ++r) out->counts[r] = hc[r];
    return PM4G_OK;
}

// a new ingested log owning columns filled by `fill` (dst pointers in
// log_columns order), with the case range [case_lo, case_hi), validated
pm4g_status make_ingested_log(const pm4g_log* like, int64_t n, uint32_t case_lo, uint32_t case_hi,
                              const std::function<pm4g_status(const std::vector<void*>&)>& fill, cudaStream_t s,
                              pm4g_log** out) {
    pm4g_log* L = new pm4g_log();
    L->n = n;
    L->A = like->A;
    L->act_bytes = like->act_bytes;
    L->n_case_codes = like->n_case_codes;
    L->case_lo = case_lo;
    L->case_hi = case_hi;
    L->stream = s;
    L->owns_cols = true;
    LogGuard guard(L);
    auto bail = [&](pm4g_status st) { return st; };   // the guard destroys L
    pm4g_status st;
    const int64_t N = std::max<int64_t>(n, 1);
    if ((st = dalloc((void**)&L->case_, N * 4, s))) return bail(st);
    if ((st = dalloc(&L->act, N * L->act_bytes, s))) return bail(st);
    if ((st = dalloc((void**)&L->ts, N * 8, s))) return bail(st);
    std::vector<void*> dst = {L->case_, L->act, L->ts};
    for (const auto& x : like->extra) {
        ExtraCol y = x;
        y.owned = true;
        y.data = nullptr;
        y.valid = nullptr;
        if ((st = dalloc(&y.data, N * x.elem, s))) return bail(st);
        if (x.valid && (st = dalloc((void**)&y.valid, N, s))) return bail(st);
        L->extra.push_back(y);
        dst.push_back(y.data);
        if (y.valid) dst.push_back(y.valid);
    }
    if ((st = fill(dst))) return bail(st);
    if ((st = dalloc((void**)&L->d_n_cases, 8, s))) return bail(st);
    if ((st = validate_and_meta(L, s))) return bail(st);
    *out = guard.release();
    return PM4G_OK;
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_partition_by_case(const pm4g_log* in, const uint32_t* bounds, int32_t n_parts,
                                   pm4g_stream_t stream, pm4g_log** parts) {
    PM4G_NVTX("pm4g_partition_by_case");
    if (!in || !bounds || !parts || n_parts < 1) return fail(PM4G_EINVAL, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    for (int r = 0; r < n_parts; ++r) parts[r] = nullptr;
    PartitionedRows pr(s);
    PM4G_TRY(partition_rows(in, bounds, n_parts, s, &pr));
    uint64_t start = 0;
    for (int r = 0; r < n_parts; ++r) {
        const uint64_t cnt = pr.counts[r];
        auto fill = [&](const std::vector<void*>& dst) -> pm4g_status {
            for (size_t c = 0; c < dst.size(); ++c)
                if (cnt) PM4G_CK(cudaMemcpyAsync(dst[c], (char*)pr.cols[c] + start * pr.elems[c], cnt * pr.elems[c],
                                                 cudaMemcpyDeviceToDevice, s));
            return PM4G_OK;
        };
        pm4g_status st = make_ingested_log(in, (int64_t)cnt, bounds[r], bounds[r + 1], fill, s, &parts[r]);
        if (st) {
            for (int q = 0; q < n_parts; ++q) {
                pm4g_log_destroy(parts[q]);
                parts[q] = nullptr;
            }
            return st;
        }
        start += cnt;
    }
    return PM4G_OK;
}

pm4g_status pm4g_log_concat(const pm4g_log* const* logs, int32_t n_logs, uint32_t case_lo, uint32_t case_hi,
                            pm4g_stream_t stream, pm4g_log** out) {
    PM4G_NVTX("pm4g_log_concat");
    if (!logs || n_logs < 1 || !out) return fail(PM4G_EINVAL, "bad arguments");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = 0;
    for (int i = 0; i < n_logs; ++i) {
        const pm4g_log* L = logs[i];
        PM4G_TRY(check_log(L));
        if (L->sorted) return fail(PM4G_EINVAL, "concat needs ingested (unsorted) logs");
        PM4G_TRY(materialize(const_cast<pm4g_log*>(L), s));
        if (L->A != logs[0]->A || L->act_bytes != logs[0]->act_bytes || L->extra.size() != logs[0]->extra.size())
            return fail(PM4G_EINVAL, "logs differ in activity dictionary or columns");
        for (size_t e = 0; e < L->extra.size(); ++e)
            if (L->extra[e].kind != logs[0]->extra[e].kind || (!L->extra[e].valid) != (!logs[0]->extra[e].valid))
                return fail(PM4G_EINVAL, "logs differ in extra columns");
        n += L->n;
    }
    if (n > MAX_SHARD_EVENTS) return fail(PM4G_EINVAL, "n_events exceeds 2^31-2 per shard");
    auto fill = [&](const std::vector<void*>& dst) -> pm4g_status {
        uint64_t at = 0;
        std::vector<const void*> cols;
        std::vector<int> elems;
        for (int i = 0; i < n_logs; ++i) {
            log_columns(logs[i], &cols, &elems);
            for (size_t c = 0; c < dst.size(); ++c)
                if (logs[i]->n)
                    PM4G_CK(cudaMemcpyAsync((char*)dst[c] + at * elems[c], cols[c], (size_t)logs[i]->n * elems[c],
                                            cudaMemcpyDeviceToDevice, s));
            at += logs[i]->n;
        }
        return PM4G_OK;
    };
    return make_ingested_log(logs[0], n, case_lo, case_hi, fill, s, out);
}

}  // extern "C"
