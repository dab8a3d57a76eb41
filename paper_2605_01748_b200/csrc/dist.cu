// Multi-GPU plumbing: one process per GPU, NCCL over NVLink / NVSwitch.
//
// libnccl is dlopen'ed (the torch-bundled libnccl.so.2 when torch is loaded,
// else the system one), so the library has no link-time NCCL dependency and a
// single-GPU run never touches it.  The unique id is exchanged by the caller
// (torch.distributed / any host channel); the communicator reduces the per-edge
// partial vectors and residual scalars of the fast solver (fused.cu).
#include <dlfcn.h>
#include <nccl.h>

#include "fused.cuh"
#include "pf_internal.cuh"

namespace pf {
namespace {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
        api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    });
    require(api.h && api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy,
            "NCCL (libnccl.so.2) could not be loaded", PF_ERR_COMM);
    return api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) {
        const char *m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw Error(PF_ERR_COMM, std::string(what) + ": " + m);
    }
}

}  // namespace
}  // namespace pf

struct pf_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    pf::CommOps ops{};
};

namespace pf {

static void comm_allreduce(void *ctx, double *buf, int64_t n, cudaStream_t s) {
    pf_comm *c = (pf_comm *)ctx;
    nccl_check(nccl().AllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, c->comm, s), "ncclAllReduce");
}

const CommOps *comm_ops(pf_comm *c) { return c ? &c->ops : nullptr; }
int comm_nranks(const pf_comm *c) { return c ? c->nranks : 1; }

}  // namespace pf

using namespace pf;

extern "C" {

int pf_comm_unique_id(void *id128) {
    return guard([&] {
        require(id128 != nullptr, "null id buffer");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        memcpy(id128, &id, sizeof(id));
    });
}

int pf_comm_create(int nranks, int rank, const void *id128, int device, pf_comm **out) {
    return guard([&] {
        require(out && id128, "null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
        ensure_device(device);
        DeviceGuard g(device);
        std::unique_ptr<pf_comm> c(new pf_comm());
        ncclUniqueId id;
        memcpy(&id, id128, sizeof(id));
        nccl_check(nccl().CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        c->ops.ctx = c.get();
        c->ops.allreduce_sum = comm_allreduce;
        *out = c.release();
    });
}

int pf_comm_destroy(pf_comm *c) {
    return guard([&] {
        if (!c) return;
        if (c->comm) nccl().CommDestroy(c->comm);
        delete c;
    });
}

}  // extern "C"
