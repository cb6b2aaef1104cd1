// comm.cu — the in-library data plane of a multi-GPU round (collectives
// C0-C3 of SURVEY §2.5).
//
// One process per GPU; the ctx of rank r of P owns a communicator.  The exchange steps of a
// round are
//   a6 transpose (usfft_transpose): samples [G][B/P] on each rank -> P slabs [G/P][B_p], one
//      all-to-all as grouped ncclSend / ncclRecv (the NCCL headers have no all-to-all-v);
//   C2 all-reduce MAX of the fp64 kappa_max (inside usfft_detect_select, the threshold basis Z5);
//   C3 all-reduce SUM of the int32 votes (inside usfft_detect_union, Alg. 1 Step 2e P:318).
// All three are data movement or order-free (MAX, integer SUM): results are bit-identical for
// every P.  NCCL is loaded at run time (dlopen of libnccl.so.2: the copy torch already loaded,
// else the system one), so the library loads on machines without it.
//
// Loopback (T4): P virtual ranks in one process on one GPU, each driven by its own host thread
// with its own ctx and stream.  A collective is a rendezvous of the P threads in a process-wide
// hub keyed by the 128-byte id: every rank posts its buffers, then pulls what it receives with
// device-to-device copies on its own stream after the senders' "ready" events, and every rank's
// stream waits for all the copies before it may touch its buffers again.  The same index math
// as NCCL runs, so one GPU tests the sharding of the product path.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"

using namespace usfft;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);       // torch's copy, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char *n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
                 api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

#define USFFT_NCCL(c, expr)                                                                   \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            (c)->sticky = true;                                                               \
            return usfft::fail((c), USFFT_ENCCL, "%s: %s", #expr, nccl().GetErrorString(r_)); \
        }                                                                                     \
    } while (0)

// ---- loopback hub -------------------------------------------------------------------------------
struct Hub {
    int P;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    // posted by each rank for the current collective
    std::vector<const void *> send;
    std::vector<const int64_t *> sdispl, scount;   // all-to-all: per destination (doubles)
    std::vector<cudaEvent_t> ready, done;
    // all-reduce scratch: P slots
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    explicit Hub(int p) : P(p), send(p), sdispl(p), scount(p), ready(p), done(p) {
        for (int r = 0; r < p; ++r) {
            cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
        }
    }
    ~Hub() {
        for (int r = 0; r < P; ++r) {
            cudaEventDestroy(ready[r]);
            cudaEventDestroy(done[r]);
        }
        if (scratch) cudaFree(scratch);
    }
    // all P threads meet; `last` runs in the last arriving thread, under the lock
    template <class F>
    void barrier(F &&last) {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == P) {
            last();
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
    void barrier() {
        barrier([] {});
    }
};

std::mutex &hub_mutex() {
    static std::mutex m;
    return m;
}
std::map<std::string, std::weak_ptr<Hub>> &hub_table() {
    static std::map<std::string, std::weak_ptr<Hub>> t;
    return t;
}

template <class T, int OP>      // OP 0: max, 1: sum
__global__ void k_reduce_slots(const T *__restrict__ slots, int P, int64_t count, T *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        T v = slots[i];
        for (int p = 1; p < P; ++p) {                    // rank order (max / integer sum: order-free)
            const T w = slots[(int64_t)p * count + i];
            v = OP == 0 ? (w > v ? w : v) : v + w;
        }
        out[i] = v;
    }
}

}  // namespace

struct usfft_comm {
    int rank = 0, nranks = 1;
    bool loopback = false;
    ncclComm_t nccl = nullptr;
    std::shared_ptr<Hub> hub;
};

namespace usfft {

int comm_size(const usfft_ctx *c) { return c->comm ? c->comm->nranks : 1; }

void comm_destroy(usfft_ctx *c) {
    if (!c->comm) return;
    if (c->comm->nccl) nccl().CommDestroy(c->comm->nccl);
    delete c->comm;
    c->comm = nullptr;
}

usfft_status comm_create(usfft_ctx *c, int rank, int nranks, const void *id, int loopback) {
    if (nranks <= 1) return USFFT_OK;
    if (!id) return fail(c, USFFT_EINVAL, "nranks > 1 needs a 128-byte id");
    auto *cm = new usfft_comm();
    cm->rank = rank;
    cm->nranks = nranks;
    cm->loopback = loopback != 0;
    c->comm = cm;
    if (cm->loopback) {
        std::lock_guard<std::mutex> lk(hub_mutex());
        const std::string key(static_cast<const char *>(id), NCCL_UNIQUE_ID_BYTES);
        auto &slot = hub_table()[key];
        cm->hub = slot.lock();
        if (!cm->hub) {
            cm->hub = std::make_shared<Hub>(nranks);
            slot = cm->hub;
        }
        if (cm->hub->P != nranks) return fail(c, USFFT_EINVAL, "loopback id reused with another nranks");
        return USFFT_OK;
    }
    if (!nccl().ok) return fail(c, USFFT_ENCCL, "NCCL unavailable: %s", nccl().why.c_str());
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    USFFT_NCCL(c, nccl().CommInitRank(&cm->nccl, nranks, uid, rank));
    return USFFT_OK;
}

// All-to-all of doubles: to rank q the scount[q] values at send + sdispl[q]; from rank p the
// rcount[p] values into recv + rdispl[p].  Stream-ordered on the ctx stream.
usfft_status comm_alltoallv(usfft_ctx *c, const double *send, const int64_t *scount, const int64_t *sdispl,
                            double *recv, const int64_t *rcount, const int64_t *rdispl) {
    usfft_comm *cm = c->comm;
    const int P = cm->nranks, r = cm->rank;
    if (!cm->loopback) {
        if (rcount[r]) USFFT_CUDA(c, cudaMemcpyAsync(recv + rdispl[r], send + sdispl[r], 8 * rcount[r],
                                                      cudaMemcpyDeviceToDevice, c->stream));
        USFFT_NCCL(c, nccl().GroupStart());
        for (int q = 0; q < P; ++q) {
            if (q == r) continue;
            if (scount[q]) USFFT_NCCL(c, nccl().Send(send + sdispl[q], scount[q], ncclFloat64, q, cm->nccl, c->stream));
            if (rcount[q]) USFFT_NCCL(c, nccl().Recv(recv + rdispl[q], rcount[q], ncclFloat64, q, cm->nccl, c->stream));
        }
        USFFT_NCCL(c, nccl().GroupEnd());
        return USFFT_OK;
    }
    Hub &h = *cm->hub;
    h.send[r] = send;
    h.sdispl[r] = sdispl;
    h.scount[r] = scount;
    USFFT_CUDA(c, cudaEventRecord(h.ready[r], c->stream));
    h.barrier();                                         // every rank posted
    for (int p = 0; p < P; ++p) {
        if (rcount[p] != h.scount[p][r])
            return fail(c, USFFT_EINVAL, "loopback all-to-all: rank %d sends %lld, rank %d expects %lld", p,
                        (long long)h.scount[p][r], r, (long long)rcount[p]);
        if (!rcount[p]) continue;
        USFFT_CUDA(c, cudaStreamWaitEvent(c->stream, h.ready[p], 0));
        USFFT_CUDA(c, cudaMemcpyAsync(recv + rdispl[p], static_cast<const double *>(h.send[p]) + h.sdispl[p][r],
                                      8 * rcount[p], cudaMemcpyDeviceToDevice, c->stream));
    }
    USFFT_CUDA(c, cudaEventRecord(h.done[r], c->stream));
    h.barrier();                                         // every rank enqueued its pulls
    for (int p = 0; p < P; ++p)                          // nobody reuses a send buffer before they ran
        if (p != r) USFFT_CUDA(c, cudaStreamWaitEvent(c->stream, h.done[p], 0));
    h.barrier();                                         // the posted arrays may be released now
    return USFFT_OK;
}

template <class T, int OP>
usfft_status comm_allreduce(usfft_ctx *c, T *buf, int64_t count) {
    usfft_comm *cm = c->comm;
    const int P = cm->nranks, r = cm->rank;
    if (!cm->loopback) {
        USFFT_NCCL(c, nccl().AllReduce(buf, buf, (size_t)count, sizeof(T) == 8 ? ncclFloat64 : ncclInt32,
                                       OP == 0 ? ncclMax : ncclSum, cm->nccl, c->stream));
        return USFFT_OK;
    }
    Hub &h = *cm->hub;
    const size_t need = sizeof(T) * (size_t)count * P;
    cudaError_t alloc_err = cudaSuccess;
    h.barrier([&] {                                      // grow the shared slots (last arriver)
        if (need > h.scratch_bytes) {
            if (h.scratch) cudaFree(h.scratch);
            h.scratch = nullptr;
            alloc_err = cudaMalloc(&h.scratch, need);
            h.scratch_bytes = alloc_err == cudaSuccess ? need : 0;
        }
    });
    if (!h.scratch || h.scratch_bytes < need) return fail(c, USFFT_ENOMEM, "loopback all-reduce scratch");
    T *slots = static_cast<T *>(h.scratch);
    USFFT_CUDA(c, cudaMemcpyAsync(slots + (int64_t)r * count, buf, sizeof(T) * count, cudaMemcpyDeviceToDevice,
                                  c->stream));
    USFFT_CUDA(c, cudaEventRecord(h.ready[r], c->stream));
    h.barrier();
    for (int p = 0; p < P; ++p)
        if (p != r) USFFT_CUDA(c, cudaStreamWaitEvent(c->stream, h.ready[p], 0));
    k_reduce_slots<T, OP><<<grid1d(count, 256), 256, 0, c->stream>>>(slots, P, count, buf);
    USFFT_CHECK_LAUNCH(c);
    USFFT_CUDA(c, cudaEventRecord(h.done[r], c->stream));
    h.barrier();
    for (int p = 0; p < P; ++p)                          // the slots are reused by the next call
        if (p != r) USFFT_CUDA(c, cudaStreamWaitEvent(c->stream, h.done[p], 0));
    h.barrier();
    return USFFT_OK;
}

usfft_status comm_max_f64(usfft_ctx *c, double *buf, int64_t count) { return comm_allreduce<double, 0>(c, buf, count); }
usfft_status comm_sum_i32(usfft_ctx *c, int32_t *buf, int64_t count) { return comm_allreduce<int32_t, 1>(c, buf, count); }

}  // namespace usfft

// ---- C-ABI ---------------------------------------------------------------------------------------
extern "C" usfft_status usfft_comm_unique_id(void *out) {
    if (!out) return USFFT_EINVAL;
    if (!nccl().ok) return USFFT_ENCCL;
    ncclUniqueId uid;
    if (nccl().GetUniqueId(&uid) != ncclSuccess) return USFFT_ENCCL;
    std::memcpy(out, &uid, sizeof uid);
    return USFFT_OK;
}

extern "C" usfft_status usfft_comm_info(const usfft_ctx *c, int32_t *rank, int32_t *nranks, int32_t *loopback) {
    if (!c) return USFFT_EINVAL;
    if (rank) *rank = c->comm ? c->comm->rank : 0;
    if (nranks) *nranks = c->comm ? c->comm->nranks : 1;
    if (loopback) *loopback = c->comm && c->comm->loopback ? 1 : 0;
    return USFFT_OK;
}

// a6: [G][nb_r] sample columns of this rank -> slabs [G_loc][B] (slab p = samples of rank p at
// offset G_loc * b0_p), G and B partitioned in contiguous balanced ranges (first G % P ranks one
// more node, same for samples).  One rank: a device copy.
extern "C" usfft_status usfft_transpose(usfft_ctx *c, int64_t G, int64_t B, const double *u_local, int64_t ldu,
                                        double *slabs) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, G >= 0 && B >= 0, "negative sizes");
    const int P = c->comm ? c->comm->nranks : 1, r = c->comm ? c->comm->rank : 0;
    auto part = [](int64_t n, int P_, int q, int64_t *lo, int64_t *hi) {
        const int64_t base = n / P_, rem = n % P_;
        *lo = q * base + (q < rem ? q : rem);
        *hi = *lo + base + (q < rem ? 1 : 0);
    };
    int64_t b0, b1, g0, g1;
    part(B, P, r, &b0, &b1);
    part(G, P, r, &g0, &g1);
    const int64_t nb = b1 - b0, Gl = g1 - g0;
    USFFT_REQUIRE(c, ldu == nb, "u_local must be [G][nb] contiguous (ldu == nb = %lld)", (long long)nb);
    USFFT_REQUIRE(c, (G * nb == 0 || u_local) && (Gl * B == 0 || slabs), "NULL buffer");
    if (P == 1) {
        if (G * B && slabs != u_local)
            USFFT_CUDA(c, cudaMemcpyAsync(slabs, u_local, 8 * G * B, cudaMemcpyDeviceToDevice, c->stream));
        return USFFT_OK;
    }
    std::vector<int64_t> sc(P), sd(P), rc(P), rd(P);
    for (int q = 0; q < P; ++q) {
        int64_t qg0, qg1, qb0, qb1;
        part(G, P, q, &qg0, &qg1);
        part(B, P, q, &qb0, &qb1);
        sc[q] = (qg1 - qg0) * nb;                        // rows qg0 .. qg1 of the local block
        sd[q] = qg0 * nb;
        rc[q] = Gl * (qb1 - qb0);                        // slab q
        rd[q] = Gl * qb0;
    }
    return comm_alltoallv(c, u_local, sc.data(), sd.data(), slabs, rc.data(), rd.data());
}
