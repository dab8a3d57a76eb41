// Drift carry of a stale allocation (oracles.py:262-287 dao_carry_rates) on the
// device, in the reference's operation order (bitwise equal to it):
//   1. commodity sums S (blk sums, model.py:297-302); every commodity with
//      S > D + tol has its rates multiplied by D / S;
//   2. up to 4 E + 4 passes: edge loads L (blk sums through the incidence,
//      model.py:305-311), over = L - cap, e = argmax(over) (first index; NaN
//      wins, as numpy's argmax); stop when over[e] <= tol; else every path
//      crossing e (each once: np.unique) is multiplied by cap[e] / (over[e] + cap[e]).
// A pass is three launches with no host round trip: the exact edge loads (an
// edge-major copy of the rates, then the reference's blocked sums), a one-CTA
// argmax that also decides the factor and a stop flag, and the path scaling.
// The host checks the stop flag once per batch of passes.

#include <algorithm>
#include <cfloat>

#include "pf_internal.cuh"

namespace pf {
namespace {

constexpr int TB = 256;

// oracles.py:271-274: sums above the new demand scale down proportionally
__global__ void k_dao_commodities(InstView I, const double *sums, double tol, double *x) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= I.C) return;
    const double D = I.demand[c];
    if (!(sums[c] > D + tol)) return;
    const double f = D / sums[c];
    for (int p = I.com_path_ptr[c]; p < I.com_path_ptr[c + 1]; ++p) x[p] *= f;
}

struct DaoPass {
    int32_t e;       // edge scaled by this pass, or -1
    int32_t stop;    // sticky: the loop has ended
    int32_t passes;  // passes that scaled an edge
    int32_t pad;
    double factor;
};

// oracles.py:278-283: over = L - cap, e = argmax(over), stop or the factor.
// One CTA; ties keep the first index, a NaN is the maximum (numpy's argmax).
__global__ void __launch_bounds__(1024) k_dao_argmax(int32_t E, const double *loads, const double *cap, double tol,
                                                     DaoPass *st) {
    __shared__ double sv[32];
    __shared__ int32_t si[32];
    if (st->stop) return;
    double best = -DBL_MAX;
    int32_t bi = -1;
    bool bnan = false;
    for (int32_t e = threadIdx.x; e < E; e += blockDim.x) {
        const double v = loads[e] - cap[e];
        if (bnan) continue;
        if (isnan(v)) {
            best = v;
            bi = e;
            bnan = true;
        } else if (bi < 0 || v > best) {
            best = v;
            bi = e;
        }
    }
    // combine (value, index): NaN first, then larger value, then smaller index
    auto better = [](double v1, int32_t i1, double v2, int32_t i2) {
        if (i2 < 0) return true;
        if (i1 < 0) return false;
        const bool n1 = isnan(v1), n2 = isnan(v2);
        if (n1 != n2) return n1;
        if (n1) return i1 < i2;
        if (v1 != v2) return v1 > v2;
        return i1 < i2;
    };
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_down_sync(0xffffffffu, best, o);
        const int32_t i2 = __shfl_down_sync(0xffffffffu, bi, o);
        if (!better(best, bi, v2, i2)) {
            best = v2;
            bi = i2;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        sv[w] = best;
        si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = sv[0];
        int32_t i = si[0];
        for (int k = 1; k < nw; ++k)
            if (!better(b, i, sv[k], si[k])) {
                b = sv[k];
                i = si[k];
            }
        if (i < 0 || b <= tol) {  // NaN is not <= tol: it goes on, like the reference
            st->stop = 1;
            st->e = -1;
        } else {
            const double load = b + cap[i];  // oracles.py:281 (over + cap, not the sum)
            st->factor = cap[i] / load;
            st->e = i;
            st->passes += 1;
        }
    }
}

// oracles.py:284-286: the paths crossing e, each scaled once (np.unique):
// the last pass that scaled a path is stamped on it
__global__ void k_dao_scale(InstView I, const DaoPass *st, int32_t pass, int32_t *stamp, double *x) {
    const int32_t e = st->e;
    if (st->stop || e < 0) return;
    const int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
    const double f = st->factor;
    for (int32_t t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) {
        const int32_t p = I.pair_path[I.edge_pairs[t]];
        if (atomicExch(&stamp[p], pass) != pass) x[p] *= f;
    }
}

}  // namespace

int64_t dao_carry_device(const pf_instance *inst, double *x, double tol, cudaStream_t s) {
    const InstView I = inst->view();
    {
        DevBuf<double> sums(I.C + 1);
        exact_commodity_sums(I, x, sums.p, s);
        if (I.C) k_dao_commodities<<<ceil_div(I.C, TB), TB, 0, s>>>(I, sums.p, tol, x);
        PF_CHECK_LAUNCH();
        PF_CUDA(cudaStreamSynchronize(s));  // before `sums` is freed
    }
    if (I.E == 0) return 0;
    DevBuf<double> loads(I.E + 1), scratch(I.NP + 1);
    DevBuf<int32_t> stamp(I.P + 1);
    DevBuf<DaoPass> st(1);
    PF_CUDA(cudaMemsetAsync(stamp.p, 0xff, sizeof(int32_t) * (I.P + 1), s));  // -1: never scaled
    PF_CUDA(cudaMemsetAsync(st.p, 0, sizeof(DaoPass), s));
    const int64_t max_pass = 4 * (int64_t)I.E + 4;  // oracles.py:277
    constexpr int blocks = 148;  // grid-stride over the edge's pairs
    constexpr int BATCH = 16;  // passes between two host checks of the stop flag
    DaoPass h{};
    for (int64_t pass = 0; pass < max_pass;) {
        const int64_t end = std::min(max_pass, pass + BATCH);
        for (; pass < end; ++pass) {
            exact_edge_loads_of_rates_em_pairs(I, x, scratch.p, loads.p, s);
            k_dao_argmax<<<1, 1024, 0, s>>>(I.E, loads.p, I.capacity, tol, st.p);
            k_dao_scale<<<blocks, TB, 0, s>>>(I, st.p, (int32_t)pass, stamp.p, x);
            PF_CHECK_LAUNCH();
        }
        d2h(&h, st.p, 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        if (h.stop) break;
    }
    if (!h.stop) {
        d2h(&h, st.p, 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
    }
    return h.passes;
}

}  // namespace pf
