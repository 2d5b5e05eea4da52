// comm.cu — NCCL inside libptg: communicators and the per-evaluation
// exchange of sharded plans (north_star: "scan positions shard
// across the 8 GPUs of one box ... summed with NCCL allreduce over NVLink").
//
// NCCL is bound at run time (dlopen of libnccl.so.2, the same library
// torch.distributed loads), so libptg stays loadable -- and its single-GPU
// entry points usable -- where NCCL is absent.  One communicator per process
// (one rank per GPU), created from an ncclUniqueId the caller distributes
// (ptg_comm_unique_id on rank 0, any out-of-band broadcast, ptg_comm_init).
//
// Two layouts (plan.cuh Shard):
//   REPLICATED  every rank holds the whole object and a contiguous block of
//               the scan; after its frames, the gradient and the value are
//               summed by two ncclAllReduce calls in one NCCL group --
//               north_star's baseline layout;
//   BANDS       rank r holds only object rows [R_r, R_r + rows) (its own
//               rows plus the halo its windows reach into rank r+1's rows);
//               after its frames, the halo gradient rows go to rank r+1
//               (ncclSend / ncclRecv in one group) and are added there, and
//               the misfit (with the owned rows' <v,z>) is one scalar
//               allreduce.  Traffic per evaluation: halo x n x 8 B per
//               boundary instead of the whole gradient.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "plan.cuh"

namespace ptg {

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) {
            err = std::string("NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [](const char* s) {
            void* p = dlsym(n.h, s);
            if (!p) err = std::string("NCCL symbol missing: ") + s;
            return p;
        };
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(sym("ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(sym("ncclCommInitRank"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
        n.allReduce = reinterpret_cast<decltype(n.allReduce)>(sym("ncclAllReduce"));
        n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
        n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
        n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) raise(PTG_ERR_CUDA, err);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(PTG_ERR_CUDA, std::string(what) + ": " + nccl().errorString(r));
}

// grad[0 : rows*n) += recv (the previous rank's halo rows)
template <typename C>
__global__ void k_add_rows(C* __restrict__ g, const C* __restrict__ add, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        g[i] = cadd(g[i], add[i]);
}

}  // namespace

struct Comm {
    ncclComm_t c = nullptr;
    int world = 1, rank = 0, device = 0;
};

void comm_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
}

Comm* comm_init(const unsigned char id[128], int world, int rank, int device) {
    if (world < 1 || rank < 0 || rank >= world) raise(PTG_ERR_CONFIG, "comm: bad rank / world size");
    check_device_public(device);
    auto c = std::make_unique<Comm>();
    c->world = world;
    c->rank = rank;
    c->device = device;
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    nccl_check(nccl().commInitRank(&c->c, world, uid, rank), "ncclCommInitRank");
    return c.release();
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->c) nccl().commDestroy(c->c);
    delete c;
}

int comm_world(const Comm* c) { return c ? c->world : 1; }
int comm_rank(const Comm* c) { return c ? c->rank : 0; }

// after the local frames: the global value (value_dev) and gradient on this rank
void comm_exchange(Plan& p, void* grad, double* value_dev) {
    Comm* c = p.comm;
    if (!c) return;
    const Nccl& N = nccl();
    const size_t ce = p.celem();
    const ncclDataType_t real_t = p.prec == PTG_C64 ? ncclFloat32 : ncclFloat64;
    if (p.shard.layout == PTG_SHARD_REPLICATED) {
        // the whole gradient + the value in one call is not possible across
        // dtypes in c64; two calls grouped (one launch from NCCL's view)
        nccl_check(N.groupStart(), "ncclGroupStart");
        nccl_check(N.allReduce(grad, grad, 2 * p.nn(), real_t, ncclSum, c->c, p.stream), "ncclAllReduce(grad)");
        nccl_check(N.allReduce(value_dev, value_dev, 1, ncclFloat64, ncclSum, c->c, p.stream), "ncclAllReduce(value)");
        nccl_check(N.groupEnd(), "ncclGroupEnd");
        return;
    }
    // BANDS: halo rows to the next rank, the previous rank's halo added here
    const int n = p.n, r = c->rank, W = c->world;
    const size_t send_rows = (size_t)(p.rows - p.shard.own_rows), recv_rows = (size_t)p.shard.halo_prev;
    if (recv_rows) p.halo_buf.ensure(recv_rows * n * ce);
    nccl_check(N.groupStart(), "ncclGroupStart");
    if (r + 1 < W && send_rows)
        nccl_check(N.send(static_cast<const char*>(grad) + (size_t)p.shard.own_rows * n * ce, 2 * send_rows * n, real_t,
                          r + 1, c->c, p.stream),
                   "ncclSend(halo)");
    if (r > 0 && recv_rows)
        nccl_check(N.recv(p.halo_buf.p, 2 * recv_rows * n, real_t, r - 1, c->c, p.stream), "ncclRecv(halo)");
    nccl_check(N.allReduce(value_dev, value_dev, 1, ncclFloat64, ncclSum, c->c, p.stream), "ncclAllReduce(value)");
    nccl_check(N.groupEnd(), "ncclGroupEnd");
    if (r > 0 && recv_rows) {
        const size_t len = recv_rows * n;
        const int blocks = (int)std::min<size_t>((len + 255) / 256, 148 * 8);
        if (p.prec == PTG_C64)
            k_add_rows<float2><<<blocks, 256, 0, p.stream>>>(static_cast<float2*>(grad), p.halo_buf.as<const float2>(), len);
        else
            k_add_rows<double2><<<blocks, 256, 0, p.stream>>>(static_cast<double2*>(grad), p.halo_buf.as<const double2>(),
                                                              len);
        PTG_CHECK_LAUNCH();
        ++p.launches;
    }
}

// BANDS: the iterate's halo rows [own_rows, rows) <- rank r+1's first rows
void comm_sync_halo(Plan& p, void* z) {
    Comm* c = p.comm;
    if (!c || p.shard.layout != PTG_SHARD_BANDS) return;
    const Nccl& N = nccl();
    const size_t ce = p.celem();
    const ncclDataType_t real_t = p.prec == PTG_C64 ? ncclFloat32 : ncclFloat64;
    const int n = p.n, r = c->rank, W = c->world;
    const size_t need = (size_t)(p.rows - p.shard.own_rows), give = (size_t)p.shard.halo_prev;
    nccl_check(N.groupStart(), "ncclGroupStart");
    if (r + 1 < W && need)
        nccl_check(N.recv(static_cast<char*>(z) + (size_t)p.shard.own_rows * n * ce, 2 * need * n, real_t, r + 1, c->c,
                          p.stream),
                   "ncclRecv(z halo)");
    if (r > 0 && give) nccl_check(N.send(z, 2 * give * n, real_t, r - 1, c->c, p.stream), "ncclSend(z halo)");
    nccl_check(N.groupEnd(), "ncclGroupEnd");
}

}  // namespace ptg
