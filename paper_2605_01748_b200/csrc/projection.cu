// GPU feasibility projection: projection.py:22-107 (score_paths, project).
//
//   phase 1  clamp negatives                                  (projection.py:59)
//   phase 2  per-commodity demand trims, one thread per commodity, paths in
//            stable descending-score order, _trim_slice with 16 re-sum passes
//                                                              (:63-74, :35-48)
//   phase 3  per violated edge in stable descending-overload order, trim the
//            edge's paths in stable descending-score order with re-sums
//                                                              (:76-106)
// Phase 3 is sequential across edges in the reference (a trim on one edge
// unloads others), so it runs in ONE CTA that walks the violated edges in
// order; inside an edge the re-sum is a CTA-parallel 32-chunk reduction
// combined in chunk order (exactly _sum_gather_range) and the trim walk is a
// warp that prefetches 32 candidates at a time.  The per-edge path orders
// (scores are fixed during phase 3) are one segmented stable radix sort.
// All arithmetic keeps the reference's order, so the projection is bitwise
// identical to the reference whenever its inputs are (alpha <= 1 scores).
#include <cub/cub.cuh>

#include <climits>

#include "pf_internal.cuh"

namespace pf {
namespace {

constexpr int BLK = 32;

__device__ __forceinline__ double sum_range_d(const double *v, int64_t lo, int64_t hi) {
    double total = 0.0;
    int64_t i = lo;
    while (i < hi) {
        int64_t j = i + BLK;
        if (j > hi) j = hi;
        double part = 0.0;
        for (int64_t t = i; t < j; ++t) part += v[t];
        total += part;
        i = j;
    }
    return total;
}

// Order key so that an ascending sort == numpy argsort(-key, kind="stable"):
// descending key, NaN last, -0.0 == +0.0.
__device__ __forceinline__ uint64_t desc_key(double k) {
    double nk = -k + 0.0;
    if (isnan(nk)) return ~0ull;
    uint64_t b = (uint64_t)__double_as_longlong(nk);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_clamp(int32_t P, const double *r, double *x, int32_t *bad) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    double v = r[p];
    if (!isfinite(v)) atomicMin(bad, p);
    x[p] = npmax0(v);
}

__global__ void k_violated_edges(int32_t E, const double *loads, const double *cap, double tol, uint8_t *viol) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) viol[e] = (loads[e] - cap[e]) > tol ? 1 : 0;
}

// projection.py:26-32
__global__ void k_scores(InstView I, const double *x_sums, const uint8_t *viol, int64_t alpha, double *scores) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= I.P) return;
    int32_t lo = I.pair_ptr[p], hi = I.pair_ptr[p + 1];
    double total = 0.0;
    for (int32_t i = lo; i < hi;) {
        int32_t j = i + BLK < hi ? i + BLK : hi;
        double part = 0.0;
        for (int32_t t = i; t < j; ++t) part += viol[I.pair_edge[t]] ? 1.0 : 0.0;
        total += part;
        i = j;
    }
    double s = npmax0(x_sums[I.path_com[p]]);
    scores[p] = pow(s, (double)alpha) * total;
}

// projection.py:63-74 + _trim_slice :35-48; one thread per commodity.
__global__ void k_demand_trim(InstView I, const double *scores, double *x, int32_t *order) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= I.C) return;
    int32_t lo = I.com_path_ptr[c], hi = I.com_path_ptr[c + 1];
    double demand = I.demand[c];
    double excess = sum_range_d(x, lo, hi) - demand;
    if (excess <= 0.0) return;
    // stable insertion sort of [lo,hi) by descending score, NaN last
    int32_t *ord = order + lo;
    int32_t n = hi - lo;
    for (int32_t i = 0; i < n; ++i) {
        int32_t p = lo + i;
        uint64_t kp = desc_key(scores[p]);
        int32_t j = i;
        while (j > 0 && desc_key(scores[ord[j - 1]]) > kp) {
            ord[j] = ord[j - 1];
            --j;
        }
        ord[j] = p;
    }
    for (int pass = 0; pass < 16; ++pass) {
        for (int32_t i = 0; i < n; ++i) {
            if (excess <= 0.0) break;
            int32_t p = ord[i];
            double d = x[p] < excess ? x[p] : excess;
            x[p] -= d;
            excess -= d;
        }
        excess = sum_range_d(x, lo, hi) - demand;
        if (excess <= 0.0) break;
    }
}

__global__ void k_over(int32_t E, const double *loads, const double *cap, double *over, uint64_t *keys,
                       int32_t *ids, int32_t *nviol) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    double o = loads[e] - cap[e];
    over[e] = o;
    keys[e] = o > 0.0 ? desc_key(o) : ~0ull;  // non-violated sort after every violated edge
    ids[e] = e;
    if (o > 0.0) atomicAdd(nviol, 1);
}

// keys for the per-edge stable path orders, in edge-major (edge_pairs) order
__global__ void k_edge_path_keys(InstView I, const double *scores, uint64_t *keys, int32_t *vals) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= I.NP) return;
    int32_t p = I.pair_path[I.edge_pairs[t]];
    keys[t] = desc_key(scores[p]);
    vals[t] = p;
}

// CTA-wide _sum_gather_range of x over the edge's pairs (projection.py:87-88).
__device__ double cta_edge_resum(const InstView &I, const double *x, int32_t lo, int32_t hi, double *parts) {
    __shared__ double s_total;
    int32_t n = hi - lo;
    int32_t nch = (n + BLK - 1) / BLK;
    for (int32_t ch = threadIdx.x; ch < nch; ch += blockDim.x) {
        int32_t cs = lo + ch * BLK, ce = cs + BLK < hi ? cs + BLK : hi;
        double part = 0.0;
        for (int32_t t = cs; t < ce; ++t) part += x[I.pair_path[I.edge_pairs[t]]];
        parts[ch] = part;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int32_t ch = 0; ch < nch; ++ch) total += parts[ch];
        s_total = total;
    }
    __syncthreads();
    double r = s_total;
    __syncthreads();
    return r;
}

// projection.py:83-106, one CTA walks the violated edges in order.
__global__ void __launch_bounds__(1024) k_edge_trim(InstView I, const int32_t *edge_order, const int32_t *nviol_p,
                                                     const int32_t *path_order, double *x, double *parts) {
    int32_t nviol = *nviol_p;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int32_t vi = 0; vi < nviol; ++vi) {
        int32_t e = edge_order[vi];
        int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
        double cap = I.capacity[e];
        double excess = cta_edge_resum(I, x, lo, hi, parts) - cap;
        if (excess <= 0.0) continue;
        for (int pass = 0; pass < 16; ++pass) {
            if (warp == 0) {
                double ex = excess;
                for (int32_t base = lo; base < hi && ex > 0.0; base += 32) {
                    int32_t t = base + lane;
                    int32_t p = t < hi ? path_order[t] : -1;
                    double xv = p >= 0 ? x[p] : 0.0;
                    int n = hi - base < 32 ? hi - base : 32;
                    for (int j = 0; j < n; ++j) {
                        if (ex <= 0.0) break;
                        double xj = __shfl_sync(0xffffffffu, xv, j);
                        double d = xj < ex ? xj : ex;
                        if (d > 0.0) {
                            if (lane == j) x[p] = xj - d;
                            ex -= d;
                        }
                    }
                }
            }
            __syncthreads();
            excess = cta_edge_resum(I, x, lo, hi, parts) - cap;
            if (excess <= 0.0) break;
        }
    }
}

}  // namespace

constexpr int TB = 256;

void score_paths_device(const pf_instance *inst, const double *x, int64_t alpha, double *scores, cudaStream_t s) {
    InstView I = inst->view();
    DevBuf<double> sums(I.C + 1), loads(I.E + 1);
    DevBuf<uint8_t> viol(I.E + 1);
    exact_commodity_sums(I, x, sums.p, s);
    exact_edge_loads_of_rates(I, x, loads.p, s);
    if (I.E) k_violated_edges<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, loads.p, I.capacity, 1e-9, viol.p);
    if (I.P) k_scores<<<ceil_div(I.P, TB), TB, 0, s>>>(I, sums.p, viol.p, alpha, scores);
    PF_CHECK_LAUNCH();
    PF_CUDA(cudaStreamSynchronize(s));
}

void project_device(const pf_instance *inst, const double *rates, int64_t alpha, double *x, cudaStream_t s) {
    InstView I = inst->view();
    DevBuf<int32_t> bad(1);
    int32_t init = INT_MAX;
    h2d(bad.p, &init, 1, s);
    if (I.P) k_clamp<<<ceil_div(I.P, TB), TB, 0, s>>>(I.P, rates, x, bad.p);
    PF_CHECK_LAUNCH();
    int32_t hb;
    d2h(&hb, bad.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    require(hb == INT_MAX, "projection input contains non-finite rates");
    if (I.P == 0) return;

    DevBuf<double> scores(I.P);
    DevBuf<int32_t> order(I.P);
    score_paths_device(inst, x, alpha, scores.p, s);
    if (I.C) k_demand_trim<<<ceil_div(I.C, 128), 128, 0, s>>>(I, scores.p, x, order.p);
    PF_CHECK_LAUNCH();

    // phase 3
    DevBuf<double> loads(I.E + 1), over(I.E + 1);
    DevBuf<uint64_t> ekeys(I.E + 1), ekeys_out(I.E + 1);
    DevBuf<int32_t> eids(I.E + 1), eorder(I.E + 1), nviol(1);
    PF_CUDA(cudaMemsetAsync(nviol.p, 0, sizeof(int32_t), s));
    exact_edge_loads_of_rates(I, x, loads.p, s);
    if (I.E) k_over<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, loads.p, I.capacity, over.p, ekeys.p, eids.p, nviol.p);
    PF_CHECK_LAUNCH();
    int32_t hn = 0;
    d2h(&hn, nviol.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    if (hn == 0) return;
    {
        size_t tmp = 0;
        PF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ekeys.p, ekeys_out.p, eids.p, eorder.p, I.E, 0, 64, s));
        DevBuf<char> t(tmp ? tmp : 1);
        PF_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, ekeys.p, ekeys_out.p, eids.p, eorder.p, I.E, 0, 64, s));
    }
    score_paths_device(inst, x, alpha, scores.p, s);  // projection.py:81 (post-phase-2 rates)
    DevBuf<uint64_t> pkeys(I.NP), pkeys_out(I.NP);
    DevBuf<int32_t> pvals(I.NP), porder(I.NP);
    k_edge_path_keys<<<ceil_div(I.NP, TB), TB, 0, s>>>(I, scores.p, pkeys.p, pvals.p);
    PF_CHECK_LAUNCH();
    {
        size_t tmp = 0;
        PF_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, pkeys.p, pkeys_out.p, pvals.p, porder.p,
                                                         I.NP, I.E, I.edge_pair_ptr, I.edge_pair_ptr + 1, 0, 64, s));
        DevBuf<char> t(tmp ? tmp : 1);
        PF_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(t.p, tmp, pkeys.p, pkeys_out.p, pvals.p, porder.p, I.NP,
                                                         I.E, I.edge_pair_ptr, I.edge_pair_ptr + 1, 0, 64, s));
    }
    int32_t max_ne = 0;
    {
        std::vector<int32_t> eptr(I.E + 1);
        d2h(eptr.data(), I.edge_pair_ptr, I.E + 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        for (int32_t e = 0; e < I.E; ++e) max_ne = std::max(max_ne, eptr[e + 1] - eptr[e]);
    }
    DevBuf<double> parts((max_ne + BLK - 1) / BLK + 1);
    k_edge_trim<<<1, 1024, 0, s>>>(I, eorder.p, nviol.p, porder.p, x, parts.p);
    PF_CHECK_LAUNCH();
    PF_CUDA(cudaStreamSynchronize(s));
}

}  // namespace pf
