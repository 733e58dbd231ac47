// Loopback NCCL -- TEST INFRASTRUCTURE ONLY (tests/test_gpu_fake_nccl.py).
//
// Implements the subset of the NCCL API that libpm4g's comm.cu calls, for R
// ranks that are threads of ONE process on ONE device (real NCCL refuses two
// ranks on one GPU).  Every collective is a rendezvous of the R ranks: the
// last rank to arrive synchronises every rank's stream (stream-ordered inputs
// are then final), moves / reduces the data through host memory, and releases
// the others.  Point-to-point calls between ncclGroupStart/End are queued and
// executed at the group's rendezvous, matched per (sender, receiver) in call
// order.  Semantics follow NCCL's: allreduce sum / max / min on uint64 / uint8,
// allgather rank-major, send / recv byte counts.  Blocking, not asynchronous --
// sufficient for correctness tests of the callers' logic.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace {

struct Op {
    int kind = 0;             // 1 allreduce, 2 allgather
    const void* send = nullptr;
    void* recv = nullptr;
    size_t count = 0;
    int dtype = 0, redop = 0;
    cudaStream_t stream = nullptr;
};

struct P2P {
    bool is_send;
    int peer;
    const void* sbuf;
    void* rbuf;
    size_t bytes;
    cudaStream_t stream;
};

struct Group {
    int R = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<Op> ops;                  // per rank, current collective
    std::vector<std::vector<P2P>> p2p;    // per rank, current group
};

struct Comm {
    Group* g;
    int rank;
};

std::mutex g_registry_mu;
std::map<uint64_t, Group*> g_groups;
thread_local std::vector<P2P>* t_pending = nullptr;   // inside ncclGroupStart/End
thread_local Comm* t_group_comm = nullptr;

size_t elem(int dtype) { return dtype == 5 || dtype == 4 ? 8 : (dtype == 2 || dtype == 3 ? 4 : 1); }

// rendezvous: `work` runs on the last arriving rank with the group locked
template <class F>
void rendezvous(Group* g, F&& work) {
    std::unique_lock<std::mutex> lk(g->mu);
    const uint64_t gen = g->generation;
    if (++g->arrived == g->R) {
        work();
        g->arrived = 0;
        ++g->generation;
        g->cv.notify_all();
    } else {
        g->cv.wait(lk, [&] { return g->generation != gen; });
    }
}

}  // namespace

extern "C" {

typedef struct { char internal[128]; } ncclUniqueId;

int ncclGetUniqueId(ncclUniqueId* id) {
    static uint64_t next = 1;
    std::lock_guard<std::mutex> lk(g_registry_mu);
    std::memset(id, 0, sizeof(*id));
    const uint64_t v = next++;
    std::memcpy(id->internal, &v, 8);
    return 0;
}

int ncclCommInitRank(void** comm, int nranks, ncclUniqueId id, int rank) {
    uint64_t key;
    std::memcpy(&key, id.internal, 8);
    std::lock_guard<std::mutex> lk(g_registry_mu);
    Group*& g = g_groups[key];
    if (!g) {
        g = new Group();
        g->R = nranks;
        g->ops.resize(nranks);
        g->p2p.resize(nranks);
    }
    if (g->R != nranks || rank < 0 || rank >= nranks) return 4;   // invalid usage
    *comm = new Comm{g, rank};
    return 0;
}

int ncclCommDestroy(void* comm) {
    delete (Comm*)comm;
    return 0;
}

const char* ncclGetErrorString(int r) { return r ? "fake nccl error" : "no error"; }

int ncclAllReduce(const void* send, void* recv, size_t count, int dtype, int redop, void* comm, cudaStream_t s) {
    Comm* c = (Comm*)comm;
    Group* g = c->g;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->ops[c->rank] = Op{1, send, recv, count, dtype, redop, s};
    }
    int err = 0;
    rendezvous(g, [&] {
        const size_t bytes = count * elem(dtype);
        std::vector<std::vector<uint8_t>> in(g->R, std::vector<uint8_t>(bytes));
        for (int r = 0; r < g->R; ++r) {
            cudaStreamSynchronize(g->ops[r].stream);
            if (bytes && cudaMemcpy(in[r].data(), g->ops[r].send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) err = 1;
        }
        std::vector<uint8_t> out(in[0]);
        for (size_t i = 0; i < count; ++i)
            for (int r = 1; r < g->R; ++r) {
                if (dtype == 5) {   // uint64
                    uint64_t a, b;
                    std::memcpy(&a, &out[i * 8], 8);
                    std::memcpy(&b, &in[r][i * 8], 8);
                    const uint64_t v = redop == 0 ? a + b : redop == 2 ? (a > b ? a : b) : (a < b ? a : b);
                    std::memcpy(&out[i * 8], &v, 8);
                } else {            // uint8
                    const uint8_t a = out[i], b = in[r][i];
                    out[i] = redop == 0 ? (uint8_t)(a + b) : redop == 2 ? (a > b ? a : b) : (a < b ? a : b);
                }
            }
        for (int r = 0; r < g->R; ++r)
            if (bytes && cudaMemcpy(g->ops[r].recv, out.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) err = 1;
    });
    return err;
}

int ncclAllGather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s) {
    Comm* c = (Comm*)comm;
    Group* g = c->g;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->ops[c->rank] = Op{2, send, recv, count, dtype, 0, s};
    }
    int err = 0;
    rendezvous(g, [&] {
        const size_t bytes = count * elem(dtype);
        std::vector<uint8_t> all(bytes * g->R);
        for (int r = 0; r < g->R; ++r) {
            cudaStreamSynchronize(g->ops[r].stream);
            if (bytes && cudaMemcpy(all.data() + r * bytes, g->ops[r].send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
                err = 1;
        }
        for (int r = 0; r < g->R; ++r)
            if (bytes && cudaMemcpy(g->ops[r].recv, all.data(), all.size(), cudaMemcpyHostToDevice) != cudaSuccess) err = 1;
    });
    return err;
}

int ncclGroupStart() {
    if (!t_pending) t_pending = new std::vector<P2P>();
    t_pending->clear();
    t_group_comm = nullptr;
    return 0;
}

int ncclSend(const void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t s) {
    if (!t_pending) return 4;
    t_group_comm = (Comm*)comm;
    t_pending->push_back(P2P{true, peer, buf, nullptr, count * elem(dtype), s});
    return 0;
}

int ncclRecv(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t s) {
    if (!t_pending) return 4;
    t_group_comm = (Comm*)comm;
    t_pending->push_back(P2P{false, peer, nullptr, buf, count * elem(dtype), s});
    return 0;
}

int ncclGroupEnd() {
    if (!t_pending) return 4;
    Comm* c = t_group_comm;
    if (!c) {   // empty group
        t_pending->clear();
        return 0;
    }
    Group* g = c->g;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->p2p[c->rank] = *t_pending;
    }
    t_pending->clear();
    int err = 0;
    rendezvous(g, [&] {
        for (int r = 0; r < g->R; ++r)
            for (auto& op : g->p2p[r]) cudaStreamSynchronize(op.stream);
        // match the k-th send r -> p with the k-th recv at p from r
        for (int r = 0; r < g->R; ++r) {
            std::map<int, int> sent;   // peer -> count of sends matched so far
            for (auto& op : g->p2p[r]) {
                if (!op.is_send) continue;
                const int p = op.peer, k = sent[p]++;
                int seen = 0;
                bool matched = false;
                for (auto& rv : g->p2p[p]) {
                    if (rv.is_send || rv.peer != r) continue;
                    if (seen++ != k) continue;
                    if (rv.bytes != op.bytes) err = 1;
                    else if (op.bytes && cudaMemcpy(rv.rbuf, op.sbuf, op.bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
                        err = 1;
                    matched = true;
                    break;
                }
                if (!matched) err = 1;
            }
        }
        for (int r = 0; r < g->R; ++r) g->p2p[r].clear();
    });
    return err;
}

}  // extern "C"
