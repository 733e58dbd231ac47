// A11: cross-GPU merge over NCCL (NVLink 5 / NVSwitch on an 8xB200 node).
//
// The log is sharded by contiguous case-code ranges (R19), so every
// per-case quantity is local; only the A x A / A tables and the variant tables
// need an exchange (associative, commutative merge with identity).
//   C1  one ncclAllReduce(sum, uint64) of the packed [cnt | sum | start | end]
//       table: integer sums are exact in any order (two's complement wraps
//       identically), so the result is independent of the rank count.
//   C2  ncclAllGather of (V_r, T_r), then grouped ncclSend / ncclRecv of every
//       rank's variant entries and representative sequences straight into the
//       flat merge input (rank order), merged on every rank with the same
//       exact hash-and-verify grouping used locally.
// NCCL is loaded with dlopen on first use so that libpm4g itself has no hard
// link-time dependency on it; torch.distributed only carries the unique id.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pm4g_internal.cuh"

namespace pm4g {

typedef struct { char internal[128]; } NcclUid;
typedef void* NcclComm;
typedef int NcclResult;  // ncclSuccess = 0
enum { NCCL_UINT64 = 5, NCCL_UINT8 = 1 };  // ncclDataType_t: ncclUint8 = 1, ncclUint64 = 5
enum { NCCL_SUM = 0 };
// NCCL is dlopen'ed (no link-time dependency); where its header is present the
// ABI constants used here are checked against it at compile time.
#if __has_include(<nccl.h>)
}  // namespace pm4g
#include <nccl.h>
namespace pm4g {
static_assert(NCCL_UINT64 == (int)ncclUint64 && NCCL_UINT8 == (int)ncclUint8, "ncclDataType_t values");
static_assert(NCCL_SUM == (int)ncclSum && COMM_SUM == (int)ncclSum && COMM_MIN == (int)ncclMin &&
                  COMM_MAX == (int)ncclMax, "ncclRedOp_t values");
static_assert(sizeof(NcclUid) == sizeof(ncclUniqueId), "ncclUniqueId size");
#endif

struct NcclApi {
    void* h = nullptr;
    NcclResult (*getUniqueId)(NcclUid*) = nullptr;
    NcclResult (*commInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
    NcclResult (*commDestroy)(NcclComm) = nullptr;
    NcclResult (*allReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    NcclResult (*allGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
    NcclResult (*send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    NcclResult (*recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    NcclResult (*groupStart)() = nullptr;
    NcclResult (*groupEnd)() = nullptr;
    const char* (*getErrorString)(NcclResult) = nullptr;
};

static NcclApi g_nccl;

static pm4g_status load_nccl() {
    if (g_nccl.h) return PM4G_OK;
    // PM4G_NCCL_LIB: an explicit library path (tests load a loopback NCCL that
    // runs several ranks as threads of one process on one device)
    const char* forced = getenv("PM4G_NCCL_LIB");
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    if (forced && *forced) {
        h = dlopen(forced, RTLD_NOW | RTLD_LOCAL);
    } else {
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    }
    if (!h) return fail(PM4G_ENCCL, std::string("cannot load NCCL: ") + dlerror());
    g_nccl.h = h;
    g_nccl.getUniqueId = (NcclResult(*)(NcclUid*))dlsym(h, "ncclGetUniqueId");
    g_nccl.commInitRank = (NcclResult(*)(NcclComm*, int, NcclUid, int))dlsym(h, "ncclCommInitRank");
    g_nccl.commDestroy = (NcclResult(*)(NcclComm))dlsym(h, "ncclCommDestroy");
    g_nccl.allReduce = (NcclResult(*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllReduce");
    g_nccl.allGather = (NcclResult(*)(const void*, void*, size_t, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllGather");
    g_nccl.getErrorString = (const char* (*)(NcclResult))dlsym(h, "ncclGetErrorString");
    g_nccl.send = (NcclResult(*)(const void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclSend");
    g_nccl.recv = (NcclResult(*)(void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclRecv");
    g_nccl.groupStart = (NcclResult(*)())dlsym(h, "ncclGroupStart");
    g_nccl.groupEnd = (NcclResult(*)())dlsym(h, "ncclGroupEnd");
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.commDestroy || !g_nccl.allReduce ||
        !g_nccl.allGather || !g_nccl.send || !g_nccl.recv || !g_nccl.groupStart || !g_nccl.groupEnd) {
        g_nccl = NcclApi();
        return fail(PM4G_ENCCL, "NCCL symbols missing");
    }
    return PM4G_OK;
}

static pm4g_status nccl_fail(NcclResult r, const char* what) {
    std::string m = std::string("NCCL error in ") + what + ": " +
                    (g_nccl.getErrorString ? g_nccl.getErrorString(r) : std::to_string(r));
    return fail(PM4G_ENCCL, m);
}

}  // namespace pm4g

struct pm4g_comm {
    pm4g::NcclComm comm = nullptr;
    int nranks = 1, rank = 0;
};

namespace pm4g {

pm4g_status comm_allreduce_u64(pm4g_comm* c, uint64_t* buf, size_t count, cudaStream_t s) {
    return comm_allreduce_u64_op(c, buf, count, COMM_SUM, s);
}

pm4g_status comm_allreduce_u64_op(pm4g_comm* c, uint64_t* buf, size_t count, int op, cudaStream_t s) {
    if (c->nranks == 1) return PM4G_OK;
    NcclResult r = g_nccl.allReduce(buf, buf, count, NCCL_UINT64, op, c->comm, s);
    if (r) return nccl_fail(r, "ncclAllReduce");
    return PM4G_OK;
}

__global__ void k_pack_entries(const pm4g_variant_table v, uint64_t* out) {
    // per entry: k1, k2, count, (rep_case | sequence offset << 32)
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < v.V;
         i += (uint64_t)gridDim.x * blockDim.x) {
        out[4 * i + 0] = v.k1[i];
        out[4 * i + 1] = v.k2[i];
        out[4 * i + 2] = v.count[i];
        out[4 * i + 3] = (uint64_t)v.rep_case[i] | (v.seq_off[i] << 32);
    }
}

// every rank's packed entries (rank-major, contiguous) -> the merge's flat
// items; the sequences stay where they were received.  sz: [R][2] (V_r, T_r).
__global__ void k_unpack_entries(const uint64_t* __restrict__ in, const uint64_t* __restrict__ sz, int R,
                                 MergeItems m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m.V;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t vb = 0, tb = 0;
        for (int r = 0; r < R; ++r) {   // the entry's rank (R is small)
            if (i < vb + sz[2 * r]) break;
            vb += sz[2 * r];
            tb += sz[2 * r + 1];
        }
        m.k1[i] = in[4 * i + 0];
        m.k2[i] = in[4 * i + 1];
        m.w[i] = in[4 * i + 2];
        m.ord[i] = (uint32_t)in[4 * i + 3];
        m.so[i] = (uint32_t)(tb + (in[4 * i + 3] >> 32));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) m.so[m.V] = (uint32_t)m.T;
}

pm4g_status comm_variants_allgather_merge(pm4g_comm* c, pm4g_variant_table* local, cudaStream_t s,
                                          pm4g_variant_table** out) {
    const int R = c->nranks, me = c->rank;
    if (R == 1) {
        const pm4g_variant_table* parts[1] = {local};
        return merge_variant_tables(parts, 1, s, out, 0);
    }
    // sizes
    Scratch sz(s);
    PM4G_TRY(sz.alloc((size_t)R * 16 + 16));
    uint64_t* d_sz = sz.as<uint64_t>();
    uint64_t mine[2] = {local->V, local->total_len};
    PM4G_CK(cudaMemcpyAsync(d_sz + 2 * R, mine, 16, cudaMemcpyHostToDevice, s));
    NcclResult r = g_nccl.allGather(d_sz + 2 * R, d_sz, 2, NCCL_UINT64, c->comm, s);
    if (r) return nccl_fail(r, "ncclAllGather(sizes)");
    std::vector<uint64_t> sizes(2 * R);
    PM4G_CK(cudaMemcpyAsync(sizes.data(), d_sz, 16 * R, cudaMemcpyDeviceToHost, s));
    PM4G_CK(cudaStreamSynchronize(s));
    std::vector<uint64_t> vb(R + 1, 0), tb(R + 1, 0);
    for (int i = 0; i < R; ++i) {
        vb[i + 1] = vb[i] + sizes[2 * i];
        tb[i + 1] = tb[i] + sizes[2 * i + 1];
    }
    const uint64_t V = vb[R], T = tb[R];
    if (V > 0xfffffffeull || T > (uint64_t)MAX_SHARD_EVENTS)
        return fail(PM4G_EINVAL, "merged variant tables exceed 2^31 - 2 activities");
    // an all-gather with per-rank sizes (grouped sends / receives): every rank's
    // entries and sequences land contiguously, in rank order, where the merge
    // reads them -- this rank's own are written in place
    Scratch ent(s), acts(s), items(s);
    PM4G_TRY(ent.alloc(V * 32 + 16));
    PM4G_TRY(acts.alloc(T * 4 + 16));
    uint64_t* re = ent.as<uint64_t>();
    uint32_t* ra = acts.as<uint32_t>();
    if (local->V) {
        int g = (int)std::max<uint64_t>(1, std::min<uint64_t>((local->V + 255) / 256, 1024));
        PM4G_LAUNCH("k_pack_entries", local->V * 64.0, s, k_pack_entries<<<g, 256, 0, s>>>(*local, re + 4 * vb[me]));
        PM4G_CK(cudaMemcpyAsync(ra + tb[me], local->seq_act, local->total_len * 4, cudaMemcpyDeviceToDevice, s));
    }
    if ((r = g_nccl.groupStart())) return nccl_fail(r, "ncclGroupStart");
    for (int p = 0; p < R && !r; ++p) {
        if (p == me) continue;
        if (local->V) r = g_nccl.send(re + 4 * vb[me], local->V * 32, NCCL_UINT8, p, c->comm, s);
        if (!r && local->total_len) r = g_nccl.send(ra + tb[me], local->total_len * 4, NCCL_UINT8, p, c->comm, s);
        if (!r && sizes[2 * p]) r = g_nccl.recv(re + 4 * vb[p], sizes[2 * p] * 32, NCCL_UINT8, p, c->comm, s);
        if (!r && sizes[2 * p + 1]) r = g_nccl.recv(ra + tb[p], sizes[2 * p + 1] * 4, NCCL_UINT8, p, c->comm, s);
    }
    const NcclResult re_end = g_nccl.groupEnd();
    if (r) return nccl_fail(r, "ncclSend/ncclRecv(variants)");
    if (re_end) return nccl_fail(re_end, "ncclGroupEnd");
    MergeItems m;
    PM4G_TRY(merge_items_alloc(V, 0, items, &m));
    m.T = T;
    m.sa = ra;
    const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>((V + 255) / 256, (uint64_t)num_sms() * 8));
    PM4G_LAUNCH("k_unpack_entries", V * 64.0, s, (k_unpack_entries<<<g, 256, 0, s>>>(re, d_sz, R, m)));
    return merge_flat(m, local, vb[me], s, out);
}

__global__ void k_sum_parts(const uint64_t* parts, int R, uint64_t len, uint64_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a = 0;
        for (int r = 0; r < R; ++r) a += parts[(uint64_t)r * len + i];
        out[i] = a;
    }
}

}  // namespace pm4g

using namespace pm4g;

extern "C" {

pm4g_status pm4g_comm_unique_id(void* id_out, size_t* id_bytes) {
    if (!id_out) return fail(PM4G_EINVAL, "null id");
    PM4G_TRY(load_nccl());
    NcclUid uid;
    NcclResult r = g_nccl.getUniqueId(&uid);
    if (r) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, &uid, sizeof(uid));
    if (id_bytes) *id_bytes = sizeof(uid);
    return PM4G_OK;
}

pm4g_status pm4g_comm_create(const void* id, int32_t nranks, int32_t rank, pm4g_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(PM4G_EINVAL, "bad arguments");
    *out = nullptr;
    pm4g_comm* c = new pm4g_comm();
    c->nranks = nranks;
    c->rank = rank;
    if (nranks > 1) {
        pm4g_status st = load_nccl();
        if (st) {
            delete c;
            return st;
        }
        NcclUid uid;
        std::memcpy(&uid, id, sizeof(uid));
        NcclResult r = g_nccl.commInitRank(&c->comm, nranks, uid, rank);
        if (r) {
            delete c;
            return nccl_fail(r, "ncclCommInitRank");
        }
    }
    *out = c;
    return PM4G_OK;
}

pm4g_status pm4g_comm_destroy(pm4g_comm* c) {
    if (!c) return PM4G_OK;
    if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
    delete c;
    return PM4G_OK;
}

pm4g_status pm4g_repartition(const pm4g_log* in, const uint32_t* bounds, pm4g_comm* c, pm4g_stream_t stream,
                             pm4g_log** out) {
    PM4G_NVTX("pm4g_repartition");
    if (!in || !bounds || !c || !out) return fail(PM4G_EINVAL, "bad arguments");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    const int R = c->nranks, me = c->rank;
    PartitionedRows pr(s);
    PM4G_TRY(partition_rows(in, bounds, R, s, &pr));
    // counts matrix M[src][dst] through one allgather
    std::vector<uint64_t> M((size_t)R * R, 0);
    if (R == 1) {
        M[0] = pr.counts[0];
    } else {
        Scratch cb(s);
        PM4G_TRY(cb.alloc((size_t)R * (R + 1) * 8));
        uint64_t* d_all = cb.as<uint64_t>();
        uint64_t* d_mine = d_all + (size_t)R * R;
        PM4G_CK(cudaMemcpyAsync(d_mine, pr.counts.data(), R * 8, cudaMemcpyHostToDevice, s));
        NcclResult r = g_nccl.allGather(d_mine, d_all, R, NCCL_UINT64, c->comm, s);
        if (r) return nccl_fail(r, "ncclAllGather(counts)");
        PM4G_CK(cudaMemcpyAsync(M.data(), d_all, (size_t)R * R * 8, cudaMemcpyDeviceToHost, s));
        PM4G_CK(cudaStreamSynchronize(s));
    }
    std::vector<uint64_t> soff(R, 0), roff(R, 0);
    uint64_t n_recv = 0;
    for (int p = 0; p < R; ++p) {
        soff[p] = p ? soff[p - 1] + M[(size_t)me * R + p - 1] : 0;
        roff[p] = n_recv;
        n_recv += M[(size_t)p * R + me];
    }
    if (n_recv > (uint64_t)MAX_SHARD_EVENTS) return fail(PM4G_EINVAL, "a destination shard exceeds 2^31-2 events");
    auto fill = [&](const std::vector<void*>& dst) -> pm4g_status {
        if (R == 1) {
            for (size_t k = 0; k < dst.size(); ++k)
                if (n_recv) PM4G_CK(cudaMemcpyAsync(dst[k], pr.cols[k], n_recv * pr.elems[k], cudaMemcpyDeviceToDevice, s));
            return PM4G_OK;
        }
        // one NCCL group: every column to / from every peer (self included)
        NcclResult r = g_nccl.groupStart();
        for (size_t k = 0; k < dst.size() && !r; ++k) {
            const int e = pr.elems[k];
            for (int p = 0; p < R && !r; ++p) {
                const uint64_t ns = M[(size_t)me * R + p], nr = M[(size_t)p * R + me];
                if (ns) r = g_nccl.send((char*)pr.cols[k] + soff[p] * e, ns * e, NCCL_UINT8, p, c->comm, s);
                if (!r && nr) r = g_nccl.recv((char*)dst[k] + roff[p] * e, nr * e, NCCL_UINT8, p, c->comm, s);
            }
        }
        NcclResult r2 = g_nccl.groupEnd();
        if (r) return nccl_fail(r, "ncclSend/ncclRecv");
        if (r2) return nccl_fail(r2, "ncclGroupEnd");
        return PM4G_OK;
    };
    return make_ingested_log(in, (int64_t)n_recv, bounds[me], bounds[me + 1], fill, s, out);
}

pm4g_status pm4g_sum_u64(const uint64_t* parts, int32_t n_parts, uint64_t len, uint64_t* out,
                         pm4g_stream_t stream) {
    if (!parts || !out || n_parts <= 0) return fail(PM4G_EINVAL, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (!len) return PM4G_OK;
    int g = (int)std::max<uint64_t>(1, std::min<uint64_t>((len + 255) / 256, (uint64_t)num_sms() * 4));
    PM4G_LAUNCH("k_sum_parts", (double)len * 8 * (n_parts + 1), s,
                k_sum_parts<<<g, 256, 0, s>>>(parts, n_parts, len, out));
    return PM4G_OK;
}

}  // extern "C"
