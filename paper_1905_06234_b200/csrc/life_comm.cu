// life_comm.cu -- the library's own NCCL communicator for voxel-sharded runs
// (the reference itself is threads only, engine.py:86-106).
//
// libnccl.so.2 is resolved at run time with dlopen: inside a PyTorch process
// that returns the copy torch already loaded (one NCCL per process), a plain
// C caller gets the system library.  Only the few entry points used here are
// declared; their ABI (ncclUniqueId = 128 bytes, enum values) is NCCL's
// stable public one.  The all-reduce is enqueued on the caller's stream and
// is capturable, so the solver keeps its CUDA graphs for nranks > 1.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "life_common.cuh"

namespace {
typedef int ncclResult;  // ncclSuccess = 0
typedef struct ncclComm *ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
enum { kNcclInt64 = 4, kNcclFloat32 = 7, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2 };

struct Nccl {
    void *h = nullptr;
    ncclResult (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult (*allReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult) = nullptr;
    std::string err;
};

const Nccl &nccl()
{
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) {
            n.err = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(n.h, "ncclCommInitRank"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.allReduce = reinterpret_cast<decltype(n.allReduce)>(dlsym(n.h, "ncclAllReduce"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(n.h, "ncclGetErrorString"));
        if (!n.getUniqueId || !n.commInitRank || !n.commDestroy || !n.allReduce || !n.errorString)
            n.err = "libnccl.so.2 lacks an entry point";
    });
    return n;
}

int nccl_fail(const Nccl &n, const char *what, ncclResult r)
{
    return life::fail(LIFE_ERR_NCCL, std::string(what) + ": " + (n.errorString ? n.errorString(r) : "?"));
}

// life_allreduce_fn over NCCL: in place, on the caller's stream
int nccl_allreduce(void *buf, int64_t count, int dtype, int op, void *stream, void *ctx)
{
    const Nccl &n = nccl();
    const int dt = dtype == LIFE_DT_I64 ? kNcclInt64 : dtype == LIFE_DT_F32 ? kNcclFloat32 : kNcclFloat64;
    const int ro = op == LIFE_OP_MAX ? kNcclMax : kNcclSum;
    const ncclResult r = n.allReduce(buf, buf, (size_t)count, dt, ro, static_cast<ncclComm_t>(ctx),
                                     static_cast<cudaStream_t>(stream));
    return r == 0 ? 0 : 1;
}
}  // namespace

extern "C" {

int life_nccl_unique_id(void *unique_id_out)
{
    if (!unique_id_out) return life::fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    const Nccl &n = nccl();
    if (!n.err.empty()) return life::fail(LIFE_ERR_NCCL, n.err);
    ncclUniqueId id;
    const ncclResult r = n.getUniqueId(&id);
    if (r != 0) return nccl_fail(n, "ncclGetUniqueId", r);
    std::memcpy(unique_id_out, id.internal, sizeof(id.internal));
    return life::ok();
}

int life_comm_init_nccl(const void *unique_id, int rank, int nranks, life_comm *comm)
{
    if (!unique_id || !comm) return life::fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return life::fail(LIFE_ERR_INVALID_ARGUMENT, "bad rank / nranks");
    const Nccl &n = nccl();
    if (!n.err.empty()) return life::fail(LIFE_ERR_NCCL, n.err);
    ncclUniqueId id;
    std::memcpy(id.internal, unique_id, sizeof(id.internal));
    ncclComm_t c = nullptr;
    const ncclResult r = n.commInitRank(&c, nranks, id, rank);
    if (r != 0) return nccl_fail(n, "ncclCommInitRank", r);
    comm->allreduce = nccl_allreduce;
    comm->ctx = c;
    comm->rank = rank;
    comm->nranks = nranks;
    comm->capturable = 1;
    comm->reserved = 0;
    return life::ok();
}

int life_comm_destroy_nccl(life_comm *comm)
{
    if (!comm || !comm->ctx) return life::ok();
    const Nccl &n = nccl();
    if (n.commDestroy) n.commDestroy(static_cast<ncclComm_t>(comm->ctx));
    comm->ctx = nullptr;
    comm->allreduce = nullptr;
    return life::ok();
}

}  // extern "C"
