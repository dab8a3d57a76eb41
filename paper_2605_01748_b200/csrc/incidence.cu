// GPU-resident incidence store: model.py:206-271 build_instance (index part).
//
// From the pre-drop flat path set (commodity CSR over paths, path CSR over
// edge ids) the device builds, bit-identically to the reference:
//   kept_rows, demand, com_path_ptr, path_com, hops, pair_ptr, pair_edge,
//   pair_path, edge_path_count, edge_pair_ptr, edge_pairs.
// Dropping (demand <= 0 or no path, model.py:226-229) is a stream compaction
// (CUB scans); edge_pairs, the reference's stable argsort of pair_edge
// (model.py:254), is a stable LSD radix sort of (pair_edge, pair id) -- the
// same permutation.  All arrays are int32 on device; export widens to int64.
#include <cub/cub.cuh>

#include <climits>

#include "pf_internal.cuh"

namespace pf {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
const std::string &get_error() { return g_err; }

void ensure_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Error(PF_ERR_CUDA, std::string("no CUDA device available: ") +
                                     (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    require(device >= 0 && device < n, "device index out of range");
}

namespace {

__global__ void k_flags_commodity(int64_t C0, const int64_t *cpp0, const double *demand0, int32_t *cflag) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C0) return;
    cflag[c] = (demand0[c] > 0.0 && cpp0[c + 1] > cpp0[c]) ? 1 : 0;
}

// path -> owning commodity, pair -> owning path (original spaces)
__global__ void k_owner_paths(int64_t C0, const int64_t *cpp0, int32_t *path_owner) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C0) return;
    for (int64_t p = cpp0[c]; p < cpp0[c + 1]; ++p) path_owner[p] = (int32_t)c;
}
__global__ void k_owner_pairs(int64_t P0, const int64_t *pep0, int32_t *pair_owner) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P0) return;
    for (int64_t t = pep0[p]; t < pep0[p + 1]; ++t) pair_owner[t] = (int32_t)p;
}
__global__ void k_gather_flag(int64_t n, const int32_t *owner, const int32_t *owner_flag, int32_t *flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = owner_flag[owner[i]];
}

__global__ void k_emit_commodities(int64_t C0, const int32_t *cflag, const int32_t *cpos, const int64_t *cpp0,
                                   const int32_t *ppos, const double *demand0, int64_t *kept_rows, double *demand,
                                   int32_t *com_path_ptr) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= C0 || !cflag[c]) return;
    int32_t nc = cpos[c];
    kept_rows[nc] = c;
    demand[nc] = demand0[c];
    com_path_ptr[nc] = ppos[cpp0[c]];
}

__global__ void k_emit_paths(int64_t P0, const int32_t *pflag, const int32_t *ppos, const int32_t *path_owner,
                             const int32_t *cpos, const int64_t *pep0, const int32_t *tpos, int32_t *path_com,
                             int32_t *hops, int32_t *pair_ptr) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P0 || !pflag[p]) return;
    int32_t np_ = ppos[p];
    path_com[np_] = cpos[path_owner[p]];
    hops[np_] = (int32_t)(pep0[p + 1] - pep0[p]);
    pair_ptr[np_] = tpos[pep0[p]];
}

__global__ void k_emit_pairs(int64_t NP0, const int32_t *tflag, const int32_t *tpos, const int32_t *pair_owner,
                             const int32_t *ppos, const int64_t *pe0, int64_t E, int32_t *pair_edge,
                             int32_t *pair_path, int32_t *iota, Flags *flags) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= NP0) return;
    int64_t e = pe0[t];
    if (e < 0 || e >= E) atomicMin(&flags->bad_edge, (int32_t)(t < INT_MAX ? t : INT_MAX - 1));
    if (!tflag[t]) return;
    int32_t nt = tpos[t];
    pair_edge[nt] = (int32_t)(e < 0 || e >= E ? 0 : e);
    pair_path[nt] = ppos[pair_owner[t]];
    iota[nt] = nt;
}

__global__ void k_set_tail(int32_t *ptr, int64_t at, int32_t v) { ptr[at] = v; }

__global__ void k_edge_count(int32_t NP, const int32_t *pair_edge, int32_t *cnt) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < NP) atomicAdd(&cnt[pair_edge[t]], 1);
}

__global__ void k_widen(int64_t n, const int32_t *a, int64_t *b) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

template <class T>
void exclusive_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t tmp = 0;
    PF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s));
    DevBuf<char> t(tmp ? tmp : 1);
    PF_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, (int)n, s));
    PF_CUDA(cudaStreamSynchronize(s));
}

int32_t last_plus(const int32_t *flag, const int32_t *pos, int64_t n, cudaStream_t s) {
    if (n == 0) return 0;
    int32_t a = 0, b = 0;
    d2h(&a, flag + n - 1, 1, s);
    d2h(&b, pos + n - 1, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    return a + b;
}

}  // namespace

static pf_instance *build(int device, int64_t C0, int64_t E, const int64_t *h_cpp0, const int64_t *h_pep0,
                          const int64_t *h_pe0, const double *h_demand0, const double *h_capacity) {
    ensure_device(device);
    DeviceGuard g(device);
    require(C0 >= 0 && E >= 0, "negative sizes");
    require(C0 < INT_MAX && E < INT_MAX, "too many commodities / edges for int32 indices");
    int64_t P0 = h_cpp0[C0];
    require(P0 >= 0 && P0 < INT_MAX, "path count out of range");
    int64_t NP0 = h_pep0[P0];
    require(NP0 >= 0 && NP0 < INT_MAX, "pair count out of range for int32 indices");
    for (int64_t c = 0; c < C0; ++c) require(h_cpp0[c + 1] >= h_cpp0[c], "com_path_ptr not monotone");

    std::unique_ptr<pf_instance> inst(new pf_instance());
    PF_CUDA(cudaStreamCreateWithFlags(&inst->stream, cudaStreamNonBlocking));
    cudaStream_t s = inst->stream;
    auto idx = std::make_shared<Index>();
    idx->device = device;
    idx->C0 = C0;
    idx->E = E;

    DevBuf<int64_t> cpp0(C0 + 1), pep0(P0 + 1), pe0(NP0 ? NP0 : 1);
    DevBuf<double> dem0(C0 ? C0 : 1);
    h2d(cpp0.p, h_cpp0, C0 + 1, s);
    h2d(pep0.p, h_pep0, P0 + 1, s);
    h2d(pe0.p, h_pe0, NP0, s);
    h2d(dem0.p, h_demand0, C0, s);
    inst->capacity.alloc(E ? E : 1);
    h2d(inst->capacity.p, h_capacity, E, s);

    const int B = 256;
    DevBuf<int32_t> cflag(C0 + 1), cpos(C0 + 1), path_owner(P0 + 1), pflag(P0 + 1), ppos(P0 + 1);
    DevBuf<int32_t> pair_owner(NP0 + 1), tflag(NP0 + 1), tpos(NP0 + 1);
    DevBuf<Flags> flags(1);
    Flags f0{INT_MAX, INT_MAX, INT_MAX, 0};
    h2d(flags.p, &f0, 1, s);
    if (C0) {
        k_flags_commodity<<<ceil_div(C0, B), B, 0, s>>>(C0, cpp0.p, dem0.p, cflag.p);
        k_owner_paths<<<ceil_div(C0, B), B, 0, s>>>(C0, cpp0.p, path_owner.p);
        PF_CHECK_LAUNCH();
    }
    if (P0) {
        k_owner_pairs<<<ceil_div(P0, B), B, 0, s>>>(P0, pep0.p, pair_owner.p);
        k_gather_flag<<<ceil_div(P0, B), B, 0, s>>>(P0, path_owner.p, cflag.p, pflag.p);
        PF_CHECK_LAUNCH();
    }
    if (NP0) {
        k_gather_flag<<<ceil_div(NP0, B), B, 0, s>>>(NP0, pair_owner.p, pflag.p, tflag.p);
        PF_CHECK_LAUNCH();
    }
    exclusive_scan(cflag.p, cpos.p, C0, s);
    exclusive_scan(pflag.p, ppos.p, P0, s);
    exclusive_scan(tflag.p, tpos.p, NP0, s);
    const int32_t C = last_plus(cflag.p, cpos.p, C0, s);
    const int32_t P = last_plus(pflag.p, ppos.p, P0, s);
    const int32_t NP = last_plus(tflag.p, tpos.p, NP0, s);
    // ppos/tpos are indexed at cpp0[c] / pep0[p] which may equal P0 / NP0 only for
    // empty ranges of dropped entries; give the tail a defined value.
    if (P0) k_set_tail<<<1, 1, 0, s>>>(ppos.p, P0, P);
    if (NP0) k_set_tail<<<1, 1, 0, s>>>(tpos.p, NP0, NP);
    idx->C = C;
    idx->P = P;
    idx->NP = NP;

    idx->kept_rows.alloc(C ? C : 1);
    inst->demand.alloc(C ? C : 1);
    idx->com_path_ptr.alloc(C + 1);
    idx->path_com.alloc(P ? P : 1);
    idx->hops.alloc(P ? P : 1);
    idx->pair_ptr.alloc(P + 1);
    idx->pair_edge.alloc(NP ? NP : 1);
    idx->pair_path.alloc(NP ? NP : 1);
    idx->edge_path_count.alloc(E ? E : 1);
    idx->edge_pair_ptr.alloc(E + 1);
    idx->edge_pairs.alloc(NP ? NP : 1);
    DevBuf<int32_t> iota(NP ? NP : 1);

    if (C0)
        k_emit_commodities<<<ceil_div(C0, B), B, 0, s>>>(C0, cflag.p, cpos.p, cpp0.p, ppos.p, dem0.p,
                                                          idx->kept_rows.p, inst->demand.p, idx->com_path_ptr.p);
    k_set_tail<<<1, 1, 0, s>>>(idx->com_path_ptr.p, C, P);
    if (P0)
        k_emit_paths<<<ceil_div(P0, B), B, 0, s>>>(P0, pflag.p, ppos.p, path_owner.p, cpos.p, pep0.p, tpos.p,
                                                    idx->path_com.p, idx->hops.p, idx->pair_ptr.p);
    k_set_tail<<<1, 1, 0, s>>>(idx->pair_ptr.p, P, NP);
    if (NP0)
        k_emit_pairs<<<ceil_div(NP0, B), B, 0, s>>>(NP0, tflag.p, tpos.p, pair_owner.p, ppos.p, pe0.p, E,
                                                     idx->pair_edge.p, idx->pair_path.p, iota.p, flags.p);
    PF_CHECK_LAUNCH();
    Flags fh;
    d2h(&fh, flags.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    require(fh.bad_edge == INT_MAX, "path edge id out of range at flat position " + std::to_string(fh.bad_edge));

    // edge_path_count = bincount(pair_edge); edge_pair_ptr = cumsum (model.py:249-252)
    PF_CUDA(cudaMemsetAsync(idx->edge_path_count.p, 0, sizeof(int32_t) * (E ? E : 1), s));
    if (NP) k_edge_count<<<ceil_div(NP, B), B, 0, s>>>(NP, idx->pair_edge.p, idx->edge_path_count.p);
    PF_CHECK_LAUNCH();
    {
        DevBuf<int32_t> cnt1(E + 1);
        PF_CUDA(cudaMemsetAsync(cnt1.p, 0, sizeof(int32_t) * (E + 1), s));
        if (E) PF_CUDA(cudaMemcpyAsync(cnt1.p, idx->edge_path_count.p, sizeof(int32_t) * E, cudaMemcpyDeviceToDevice, s));
        exclusive_scan(cnt1.p, idx->edge_pair_ptr.p, E + 1, s);
    }
    // edge_pairs = stable argsort(pair_edge) (model.py:254): stable radix sort by edge id.
    if (NP) {
        int end_bit = 1;
        while ((int64_t(1) << end_bit) < E) ++end_bit;
        DevBuf<int32_t> keys_out(NP);
        size_t tmp = 0;
        PF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, idx->pair_edge.p, keys_out.p, iota.p,
                                                idx->edge_pairs.p, NP, 0, end_bit, s));
        DevBuf<char> t(tmp ? tmp : 1);
        PF_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, idx->pair_edge.p, keys_out.p, iota.p,
                                                idx->edge_pairs.p, NP, 0, end_bit, s));
    }
    PF_CUDA(cudaStreamSynchronize(s));
    inst->idx = idx;
    return inst.release();
}

}  // namespace pf

using namespace pf;

namespace pf {
void instance_release(const pf_instance *inst) {
    if (!inst || inst->refs.fetch_sub(1) != 1) return;
    pf_instance *p = const_cast<pf_instance *>(inst);
    DeviceGuard g(p->device());
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
}
}  // namespace pf

extern "C" {

int pf_last_error(char *buf, size_t cap) {
    if (buf && cap) {
        const std::string &e = get_error();
        size_t n = e.size() < cap - 1 ? e.size() : cap - 1;
        memcpy(buf, e.data(), n);
        buf[n] = 0;
    }
    return PF_OK;
}

int pf_device_info(int device, int *sm_count, int64_t *l2_bytes, int64_t *hbm_bytes, char *name, size_t name_cap) {
    return guard([&] {
        ensure_device(device);
        cudaDeviceProp p;
        PF_CUDA(cudaGetDeviceProperties(&p, device));
        if (sm_count) *sm_count = p.multiProcessorCount;
        if (l2_bytes) *l2_bytes = p.l2CacheSize;
        if (hbm_bytes) *hbm_bytes = (int64_t)p.totalGlobalMem;
        if (name && name_cap) snprintf(name, name_cap, "%s", p.name);
    });
}

int pf_instance_create(int device, int64_t C0, int64_t E, const int64_t *cpp0, const int64_t *pep0,
                       const int64_t *pe0, const double *demand0, const double *capacity, pf_instance **out) {
    return guard([&] {
        require(out != nullptr, "null output handle");
        *out = build(device, C0, E, cpp0, pep0, pe0, demand0, capacity);
    });
}

int pf_instance_with_conditions(const pf_instance *base, const double *capacity, const double *demand,
                                pf_instance **out) {
    return guard([&] {
        require(base && out, "null handle");
        DeviceGuard g(base->device());
        std::unique_ptr<pf_instance> inst(new pf_instance());
        PF_CUDA(cudaStreamCreateWithFlags(&inst->stream, cudaStreamNonBlocking));
        inst->idx = base->idx;  // same index spaces (model.py:274-294)
        const Index &I = *base->idx;
        inst->demand.alloc(I.C ? I.C : 1);
        inst->capacity.alloc(I.E ? I.E : 1);
        if (demand)
            h2d(inst->demand.p, demand, I.C, inst->stream);
        else if (I.C)
            PF_CUDA(cudaMemcpyAsync(inst->demand.p, base->demand.p, sizeof(double) * I.C, cudaMemcpyDeviceToDevice,
                                    inst->stream));
        if (capacity)
            h2d(inst->capacity.p, capacity, I.E, inst->stream);
        else if (I.E)
            PF_CUDA(cudaMemcpyAsync(inst->capacity.p, base->capacity.p, sizeof(double) * I.E,
                                    cudaMemcpyDeviceToDevice, inst->stream));
        PF_CUDA(cudaStreamSynchronize(inst->stream));
        *out = inst.release();
    });
}

int pf_instance_destroy(pf_instance *inst) {
    return guard([&] { pf::instance_release(inst); });
}

int pf_instance_sizes(const pf_instance *inst, int64_t *C, int64_t *P, int64_t *E, int64_t *NP) {
    return guard([&] {
        require(inst != nullptr, "null instance");
        if (C) *C = inst->idx->C;
        if (P) *P = inst->idx->P;
        if (E) *E = inst->idx->E;
        if (NP) *NP = inst->idx->NP;
    });
}

int pf_instance_export_index(const pf_instance *inst, int field, int64_t *out) {
    return guard([&] {
        require(inst && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        if (field == PF_KEPT_ROWS) {
            d2h(out, I.kept_rows.p, I.C, s);
            PF_CUDA(cudaStreamSynchronize(s));
            return;
        }
        const int32_t *src = nullptr;
        int64_t n = 0;
        switch (field) {
            case PF_COM_PATH_PTR: src = I.com_path_ptr.p; n = I.C + 1; break;
            case PF_PATH_COM: src = I.path_com.p; n = I.P; break;
            case PF_HOPS: src = I.hops.p; n = I.P; break;
            case PF_PAIR_PTR: src = I.pair_ptr.p; n = I.P + 1; break;
            case PF_PAIR_EDGE: src = I.pair_edge.p; n = I.NP; break;
            case PF_PAIR_PATH: src = I.pair_path.p; n = I.NP; break;
            case PF_EDGE_PATH_COUNT: src = I.edge_path_count.p; n = I.E; break;
            case PF_EDGE_PAIR_PTR: src = I.edge_pair_ptr.p; n = I.E + 1; break;
            case PF_EDGE_PAIRS: src = I.edge_pairs.p; n = I.NP; break;
            default: throw Error(PF_ERR_INPUT, "unknown index field");
        }
        if (n == 0) return;
        DevBuf<int64_t> w(n);
        k_widen<<<ceil_div(n, 256), 256, 0, s>>>(n, src, w.p);
        PF_CHECK_LAUNCH();
        d2h(out, w.p, n, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_instance_export_values(const pf_instance *inst, int field, double *out) {
    return guard([&] {
        require(inst && out, "null argument");
        DeviceGuard g(inst->device());
        if (field == PF_DEMAND)
            d2h(out, inst->demand.p, inst->idx->C, inst->stream);
        else if (field == PF_CAPACITY)
            d2h(out, inst->capacity.p, inst->idx->E, inst->stream);
        else
            throw Error(PF_ERR_INPUT, "unknown value field");
        PF_CUDA(cudaStreamSynchronize(inst->stream));
    });
}

}  // extern "C"
