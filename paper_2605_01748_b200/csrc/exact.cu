// Exact-order kernels: the reference's iterate math with its fp64 operation
// order preserved (compiled -fmad=false), one kernel per reference step.
//
// Each kernel cites the numba kernel / numpy expression it reproduces
// (pathfair/kernels.py, pathfair/_reduce.py, pathfair/model.py).  These back
// (a) the kernel-level C-ABI (pf_update_duals ...), (b) PF_MODE_EXACT solves,
// which are bit-identical to the reference for alpha in {0, 1}, and (c) the
// model-level reductions used by validation, projection and tracing.
//
// Parallel structure: one owner per output element, sequential where the
// reference is sequential.  Where the reference sums in 32-element chunks
// (_reduce.py:18-49) each chunk partial is computed by one lane in parallel
// and the partials are then combined in chunk order, which is the same
// rounding sequence.  Long sequential chains (the per-edge total of
// _k_suggest) are walked by one warp with the gathers issued 32-wide.
#include <climits>

#include <math_constants.h>

#include "pf_internal.cuh"

namespace pf {
namespace {

constexpr int BLK = 32;    // _reduce.py:14
constexpr int PART = 4096; // _reduce.py:15

// _reduce.py:18-33 _sum_range over values[lo:hi] (sequential; used for short segments)
__device__ __forceinline__ double sum_range(const double *v, int64_t lo, int64_t hi) {
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

// _reduce.py:52-57 segment_sums (thread per segment)
__global__ void k_segment_sums(const double *__restrict__ v, const int32_t *__restrict__ ptr, int32_t nseg,
                               double *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nseg) out[i] = sum_range(v, ptr[i], ptr[i + 1]);
}

// _reduce.py:60-65 gather_segment_sums, one warp per edge.  MODE 0: values are
// per-pair (vals[edge_pairs[t]]); MODE 1: values are per-path rates gathered
// through pair_path (model.py:305-311 edge_loads).
template <int MODE>
__global__ void k_edge_gather_blk(InstView I, const double *__restrict__ vals, double *__restrict__ out) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= I.E) return;
    int64_t lo = I.edge_pair_ptr[warp], hi = I.edge_pair_ptr[warp + 1];
    double total = 0.0;
    for (int64_t base = lo; base < hi; base += BLK * 32) {
        int64_t cs = base + (int64_t)lane * BLK;
        double part = 0.0;
        if (cs < hi) {
            int64_t ce = cs + BLK < hi ? cs + BLK : hi;
            for (int64_t t = cs; t < ce; ++t) {
                int32_t pr = I.edge_pairs[t];
                double v = MODE == 0 ? vals[pr] : vals[I.pair_path[pr]];
                part += v;
            }
        }
        int64_t rem = hi - base;
        int nch = rem >= BLK * 32 ? 32 : (int)((rem + BLK - 1) / BLK);
        for (int j = 0; j < nch; ++j) total += __shfl_sync(0xffffffffu, part, j);
    }
    if (lane == 0) out[warp] = total;
}

// kernels.py:209-215 (+ _k_dual_consensus :69-73)
__global__ void k_dual_dd(int32_t C, const double *dd, const double *sums, const double *D, double *out) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C) out[c] = npmax0(dd[c] + (sums[c] - D[c]));
}
__global__ void k_dual_dc(int32_t E, const double *dc, const double *loads, const double *cap, double *out) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) out[e] = npmax0(dc[e] + (loads[e] - cap[e]));
}
__global__ void k_dual_dcon(int32_t NP, const double *dcon, const double *x, const int32_t *pair_path,
                            const double *y, double *out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < NP) out[t] = max0(dcon[t] + x[pair_path[t]] - y[t]);
}
__global__ void k_dual_dn(int32_t P, const double *dn, const double *x, double *out) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) out[p] = npmax0(dn[p] - x[p]);
}

// kernels.py:228-231
__global__ void k_slack_sd(int32_t C, const double *dd, double beta, const double *D, const double *sums,
                           double *out) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C) out[c] = npmax0(dd[c] / beta + (D[c] - sums[c]));
}
__global__ void k_slack_sc(int32_t E, const double *dc, double beta, const double *cap, const double *loads,
                           double *out) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) out[e] = npmax0(dc[e] / beta + (cap[e] - loads[e]));
}

// edge-major copy of a per-pair array: vals[t] = pv[edge_pairs[t]]
__global__ void k_gather_edge_major(InstView I, const double *__restrict__ pv, double *__restrict__ vals) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < I.NP) vals[t] = pv[I.edge_pairs[t]];
}

// edge-major copy of the per-path rates through the incidence: vals[t] = x[pair_path[edge_pairs[t]]]
__global__ void k_gather_rates_em_pairs(InstView I, const double *__restrict__ x, double *__restrict__ vals) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < I.NP) vals[t] = x[I.pair_path[I.edge_pairs[t]]];
}

// edge-major copy of the per-path rates: vals[t] = x[pair_path[edge_pairs[t]]]
__global__ void k_gather_rates_edge_major(int64_t NP, const int32_t *__restrict__ epath,
                                          const double *__restrict__ x, double *__restrict__ vals) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < NP) vals[t] = x[epath[t]];
}

// _reduce.py:60-65 over an edge-major contiguous array: one warp per edge,
// lane j sums the j-th 32-element chunk of each 1024-block (a full chunk's 32
// loads are independent of the sum and issue together), chunk partials added in
// chunk order -- the same association as k_edge_gather_blk.
__global__ void k_edge_blk_contig(InstView I, const double *__restrict__ vals, double *__restrict__ out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= I.E) return;
    const int64_t lo = I.edge_pair_ptr[warp], hi = I.edge_pair_ptr[warp + 1];
    double total = 0.0;
    for (int64_t base = lo; base < hi; base += BLK * 32) {
        const int64_t cs = base + (int64_t)lane * BLK;
        double part = 0.0;
        if (cs + BLK <= hi) {
            double b[BLK];
#pragma unroll
            for (int u = 0; u < BLK; ++u) b[u] = vals[cs + u];
#pragma unroll
            for (int u = 0; u < BLK; ++u) part += b[u];
        } else if (cs < hi) {
            for (int64_t t = cs; t < hi; ++t) part += vals[t];
        }
        const int64_t rem = hi - base;
        const int nch = rem >= BLK * 32 ? 32 : (int)((rem + BLK - 1) / BLK);
        for (int j = 0; j < nch; ++j) total += __shfl_sync(0xffffffffu, part, j);
    }
    if (lane == 0) out[warp] = total;
}

// kernels.py:90-91 values of _k_suggest's per-edge sums, x[pair_path] + dcon',
// laid out in edge-major order (one thread per edge-major position: the same
// single addition the sequential walk does)
__global__ void k_suggest_vals(InstView I, const double *__restrict__ x, const double *__restrict__ dcon,
                               double *__restrict__ vals) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= I.NP) return;
    const int32_t pr = I.edge_pairs[t];
    vals[t] = x[I.pair_path[pr]] + dcon[pr];
}

// kernels.py:88-100 from the edge-major values: lane 0 of the edge's warp walks
// the sequential total (ascending pair order, exactly the reference's chain)
// over the contiguous values with 8 loads in flight; then the warp writes y.
__global__ void k_suggest_seq(InstView I, const double *__restrict__ vals, const double *__restrict__ dc,
                              double *__restrict__ y) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= I.E) return;
    const int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
    if (hi == lo) return;
    // the warp loads 32-value chunks two ahead (coalesced); every lane adds the
    // current chunk's values in order via shuffles (identical totals on all lanes)
    double total = 0.0;
    double v0 = lo + lane < hi ? vals[lo + lane] : 0.0;
    double v1 = lo + 32 + lane < hi ? vals[lo + 32 + lane] : 0.0;
    for (int32_t base = lo; base < hi; base += 32) {
        const int32_t t2 = base + 64 + lane;
        const double v2 = t2 < hi ? vals[t2] : 0.0;
        const int n = hi - base < 32 ? hi - base : 32;
        if (n == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) total += __shfl_sync(0xffffffffu, v0, j);
        } else {
            for (int j = 0; j < n; ++j) total += __shfl_sync(0xffffffffu, v0, j);
        }
        v0 = v1;
        v1 = v2;
    }
    double adjust = (total + dc[e] - I.capacity[e]) / ((double)I.edge_path_count[e] + 1.0);
    if (adjust < 0.0) adjust = 0.0;
    for (int32_t t = lo + lane; t < hi; t += 32) y[I.edge_pairs[t]] = max0(vals[t] - adjust);
}

// kernels.py:76-100 _k_suggest: warp per edge; the per-edge total is one
// sequential chain (total += x + dcon) walked 32 gathered values at a time.
__global__ void k_suggest(InstView I, const double *__restrict__ x, const double *__restrict__ dcon,
                          const double *__restrict__ dc, double *__restrict__ y) {
    int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (e >= I.E) return;
    int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
    if (hi == lo) return;
    double total = 0.0;
    for (int32_t base = lo; base < hi; base += 32) {
        int32_t t = base + lane;
        double v = 0.0;
        if (t < hi) {
            int32_t pr = I.edge_pairs[t];
            v = x[I.pair_path[pr]] + dcon[pr];
        }
        int n = hi - base < 32 ? hi - base : 32;
        for (int j = 0; j < n; ++j) total += __shfl_sync(0xffffffffu, v, j);
    }
    double adjust = (total + dc[e] - I.capacity[e]) / ((double)I.edge_path_count[e] + 1.0);
    if (adjust < 0.0) adjust = 0.0;
    for (int32_t t = lo + lane; t < hi; t += 32) {
        int32_t pr = I.edge_pairs[t];
        double v = x[I.pair_path[pr]] + dcon[pr] - adjust;
        y[pr] = max0(v);
    }
}

// kernels.py:103-119 _k_path_coeffs
__global__ void k_path_coeffs(InstView I, const double *__restrict__ y, const double *__restrict__ dcon,
                              const double *__restrict__ x_prev, const double *__restrict__ dn,
                              double *__restrict__ pk, double *__restrict__ pw) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= I.P) return;
    double acc = 0.0;
    for (int32_t t = I.pair_ptr[p]; t < I.pair_ptr[p + 1]; ++t) acc += y[t] - dcon[t];
    double h = (double)I.hops[p];
    if (x_prev[p] < dn[p]) {
        pk[p] = acc + dn[p];
        pw[p] = 1.0 / (h + 1.0);
    } else {
        pk[p] = acc;
        pw[p] = 1.0 / h;
    }
}

// kernels.py:122-131 _k_com_coeffs
__global__ void k_com_coeffs(InstView I, const double *__restrict__ pk, const double *__restrict__ pw,
                             double *__restrict__ wsum, double *__restrict__ q) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= I.C) return;
    double ws = 0.0, qw = 0.0;
    for (int32_t p = I.com_path_ptr[c]; p < I.com_path_ptr[c + 1]; ++p) {
        ws += pw[p];
        qw += pw[p] * pk[p];
    }
    wsum[c] = ws;
    q[c] = qw;
}

// kernels.py:267-282 + _k_roots :176-189
__global__ void k_roots(InstView I, const double *__restrict__ wsum, const double *__restrict__ q,
                        const double *__restrict__ dd, double beta, int64_t alpha, double *__restrict__ out,
                        Flags *flags) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= I.C) return;
    double w = wsum[c], qc = q[c];
    if (!(isfinite(w) && isfinite(qc))) {
        atomicMin(&flags->bad_coef, c);
        out[c] = NAN;
        return;
    }
    double d_eff = I.demand[c] - dd[c];  // kernels.py:275
    double s = commodity_root(w, qc, d_eff, beta, alpha);
    out[c] = s;
    if (!isfinite(s)) atomicMin(&flags->bad_root, c);
}

// kernels.py:285-296 update_rates (+ _k_rates :192-195)
__global__ void k_rates(InstView I, const double *__restrict__ pk, const double *__restrict__ pw,
                        const double *__restrict__ sums, const double *__restrict__ dd, double beta, int64_t alpha,
                        double *__restrict__ x) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= I.P) return;
    int32_t c = I.path_com[p];
    double ct = commodity_term(sums[c], I.demand[c], dd[c], beta, alpha);
    x[p] = pw[p] * (pk[p] + ct);
}

// _reduce.py:79-99 _sqdiff_partials: one CTA per 4096 block, one lane per 32-chunk.
__global__ void k_sqdiff_blocks(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                                double *__restrict__ out) {
    __shared__ double parts[PART / BLK];
    int64_t lo = (int64_t)blockIdx.x * PART;
    int64_t hi = lo + PART < n ? lo + PART : n;
    int j = threadIdx.x;  // chunk index, blockDim == 128
    int64_t cs = lo + (int64_t)j * BLK;
    double part = 0.0;
    if (cs < hi) {
        int64_t ce = cs + BLK < hi ? cs + BLK : hi;
        for (int64_t t = cs; t < ce; ++t) {
            double d = a[t] - b[t];
            part += d * d;
        }
    }
    parts[j] = part;
    __syncthreads();
    if (j == 0) {
        int nch = (int)((hi - lo + BLK - 1) / BLK);
        double total = 0.0;
        for (int i = 0; i < nch; ++i) total += parts[i];
        out[blockIdx.x] = total;
    }
}

// _reduce.py:18-33 over the block totals (single thread; nb <= n / 4096).
__global__ void k_sum_range_1(const double *__restrict__ v, int64_t n, double *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = sum_range(v, 0, n);
}

__global__ void k_scale(double *a, int64_t n, double f) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = a[i] * f;
}

__global__ void k_reset_flags(Flags *f) {
    f->bad_coef = INT_MAX;
    f->bad_root = INT_MAX;
    f->bad_edge = INT_MAX;
    f->pad = 0;
}

// ---------------- trace / validation helpers

// numpy pairwise_sum (PW_BLOCKSIZE 128) -- np.sum/np.mean order.
// np_pairwise's leaf branches (n <= 128): no recursion, no stack
__device__ __forceinline__ double np_pairwise_leaf(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
}

__device__ double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// np_pairwise's split of a node of m > 128 elements: the left child's size.
__device__ __forceinline__ int32_t np_split(int32_t m) {
    int32_t n2 = m / 2;
    return n2 - n2 % 8;
}

constexpr int NPW_DEPTH = 5;  // the top of the tree expanded by thread 0 (<= 32 subtrees)

// np_pairwise(a, n) by one CTA, bitwise the same.
//  1. thread 0 expands the top NPW_DEPTH levels of numpy's split tree, in order:
//     <= 32 frontier nodes (subtrees, or leaves above that depth);
//  2. lane j of warp 0 counts its subtree's leaves (<= 128 elements, >= 64
//     unless n <= 128), a warp scan places them, lane j enumerates them;
//  3. the block sums the leaves in parallel (np_pairwise's leaf branch);
//  4. lane j adds its subtree up numpy's tree (post-order), thread 0 adds the
//     frontier values up the top levels.
// leaf_lo and leaf_sum hold n / 32 + 8 entries; n < 2^31.  Every thread gets
// the result.
__device__ double cta_np_pairwise(const double *a, int64_t n64, int64_t *leaf_lo, double *leaf_sum) {
    __shared__ int32_t f_lo[2][32], f_n[2][32];
    __shared__ int32_t f_cnt, f_off[33];
    __shared__ double f_val[32], s_res;
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t n = (int32_t)n64;
    if (tid == 0) {
        int cnt = 0, cur = 0;
        if (n > 0) {
            f_lo[0][0] = 0;
            f_n[0][0] = n;
            cnt = 1;
            for (int d = 0; d < NPW_DEPTH; ++d) {  // in-order expansion, level by level
                int k = 0;
                for (int i = 0; i < cnt; ++i) {
                    const int32_t lo = f_lo[cur][i], m = f_n[cur][i];
                    if (m > 128) {
                        const int32_t n2 = np_split(m);
                        f_lo[cur ^ 1][k] = lo;
                        f_n[cur ^ 1][k++] = n2;
                        f_lo[cur ^ 1][k] = lo + n2;
                        f_n[cur ^ 1][k++] = m - n2;
                    } else {
                        f_lo[cur ^ 1][k] = lo;
                        f_n[cur ^ 1][k++] = m;
                    }
                }
                cur ^= 1;
                cnt = k;
            }
        }
        if (cur) {
            for (int i = 0; i < cnt; ++i) {
                f_lo[0][i] = f_lo[1][i];
                f_n[0][i] = f_n[1][i];
            }
        }
        f_cnt = cnt;
    }
    __syncthreads();
    const int F = f_cnt;
    if (tid < 32) {  // leaves per frontier node, placed by a warp scan, enumerated in order
        int32_t stk[64];
        int32_t c = 0;
        if (lane < F) {
            int sp = 0;
            stk[sp++] = f_n[0][lane];
            while (sp) {
                const int32_t mm = stk[--sp];
                if (mm <= 128) {
                    ++c;
                } else {
                    const int32_t n2 = np_split(mm);
                    stk[sp++] = mm - n2;
                    stk[sp++] = n2;
                }
            }
        }
        int32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        f_off[lane] = incl - c;
        if (lane == 31) f_off[32] = incl;
        if (lane < F) {
            int64_t L = incl - c;
            int sp = 0;
            stk[sp++] = f_lo[0][lane];
            stk[sp++] = f_n[0][lane];
            while (sp) {
                sp -= 2;
                const int32_t lo = stk[sp], mm = stk[sp + 1];
                if (mm <= 128) {
                    leaf_lo[L++] = lo;
                } else {
                    const int32_t n2 = np_split(mm);
                    stk[sp] = lo + n2;
                    stk[sp + 1] = mm - n2;
                    stk[sp + 2] = lo;
                    stk[sp + 3] = n2;
                    sp += 4;
                }
            }
        }
        const int32_t total = __shfl_sync(0xffffffffu, incl, 31);  // (f_off[32] is not yet visible to lane 0)
        if (lane == 0) leaf_lo[total] = n;
    }
    __syncthreads();
    const int64_t L = f_off[32];
    for (int64_t l = tid; l < L; l += blockDim.x)
        leaf_sum[l] = np_pairwise_leaf(a + leaf_lo[l], leaf_lo[l + 1] - leaf_lo[l]);
    __syncthreads();
    if (tid < 32 && lane < F) {  // each frontier subtree added up numpy's tree
        int32_t stk[64];
        double val[32];
        int sp = 0, vp = 0;
        int64_t i = f_off[lane];
        stk[sp++] = f_n[0][lane];
        while (sp) {
            const int32_t mm = stk[--sp];
            if (mm < 0) {
                const double b = val[--vp], c2 = val[--vp];
                val[vp++] = c2 + b;
            } else if (mm <= 128) {
                val[vp++] = leaf_sum[i++];
            } else {
                const int32_t n2 = np_split(mm);
                stk[sp++] = ~mm;
                stk[sp++] = mm - n2;
                stk[sp++] = n2;
            }
        }
        f_val[lane] = val[0];
    }
    __syncthreads();
    if (tid == 0) {  // the top levels: a node at depth NPW_DEPTH or a leaf is a frontier value
        double res = 0.0;
        if (F > 0) {
            int32_t stk[2 * NPW_DEPTH + 4];
            int32_t dep[2 * NPW_DEPTH + 4];
            double val[NPW_DEPTH + 2];
            int sp = 0, vp = 0, fi = 0;
            stk[sp] = n;
            dep[sp++] = 0;
            while (sp) {
                --sp;
                const int32_t mm = stk[sp];
                const int d = dep[sp];
                if (mm < 0) {
                    const double b = val[--vp], c2 = val[--vp];
                    val[vp++] = c2 + b;
                } else if (mm <= 128 || d == NPW_DEPTH) {
                    val[vp++] = f_val[fi++];
                } else {
                    const int32_t n2 = np_split(mm);
                    stk[sp] = ~mm;
                    dep[sp++] = d;
                    stk[sp] = mm - n2;
                    dep[sp++] = d + 1;
                    stk[sp] = n2;
                    dep[sp++] = d + 1;
                }
            }
            res = val[0];
        }
        s_res = res;
    }
    __syncthreads();
    return s_res;
}

__global__ void __launch_bounds__(1024) k_np_sum(const double *a, int64_t n, double *out, int64_t *leaf_lo,
                                                 double *leaf_sum) {
    const double r = cta_np_pairwise(a, n, leaf_lo, leaf_sum);
    if (threadIdx.x == 0) *out = r;
}

// oracles.py:244-254 per-commodity term min(S_c / max(OPT_c, theta), 1) (the
// host metric's expressions: NaN becomes 1 as in min(v, 1) written v < 1 ? v : 1)
__global__ void k_opt_ratio(int32_t C, const double *sums, const double *ref, double theta, double *r) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const double den = ref[c] > theta ? ref[c] : theta;
    const double v = sums[c] / den;
    r[c] = v < 1.0 ? v : 1.0;
}

// kernels.py:47-66 utility of max(S, 1e-12) (controller.py:175)
__global__ void k_utility(int32_t C, const double *sums, int64_t alpha, double *u) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double s = sums[c] > 1e-12 ? sums[c] : 1e-12;
    if (alpha == 0)
        u[c] = s - 1.0;
    else if (alpha == 1)
        u[c] = log(s);
    else
        u[c] = (pow(s, 1.0 - (double)alpha) - 1.0) / (1.0 - (double)alpha);
}

// k_utility with alpha read from the device controller (traced runs)
__global__ void k_utility_dev(int32_t C, const double *sums, const int64_t *alpha_p, double *u) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const int64_t alpha = *alpha_p;
    double s = sums[c] > 1e-12 ? sums[c] : 1e-12;
    if (alpha == 0)
        u[c] = s - 1.0;
    else if (alpha == 1)
        u[c] = log(s);
    else
        u[c] = (pow(s, 1.0 - (double)alpha) - 1.0) / (1.0 - (double)alpha);
}

// the host's pct_violated / n_violated arithmetic (violation_stats) on the device
__global__ void k_row_pct(const int32_t *cnt, int64_t total, double *row_pct, double *row_nv) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t nv = (int64_t)cnt[0] + cnt[1] + cnt[2];
    *row_pct = total ? 100.0 * (double)nv / (double)total : 0.0;
    *row_nv = (double)nv;
}

// model.py:346-362: overload / excess, violation flags and relative violations.
__global__ void k_violations(InstView I, const double *x, const double *loads, const double *sums, double tol,
                             double *overload, double *excess, double *rel_e, double *rel_c, int32_t *cnt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < I.E) {
        double ov = npmax0(loads[i] - I.capacity[i]);
        if (overload) overload[i] = ov;
        bool bad = ov > tol;
        rel_e[i] = bad ? ov / (I.capacity[i] > 1e-12 ? I.capacity[i] : 1e-12) : NAN;
        if (bad) atomicAdd(&cnt[0], 1);
    }
    if (i < I.C) {
        double ex = npmax0(sums[i] - I.demand[i]);
        if (excess) excess[i] = ex;
        bool bad = ex > tol;
        rel_c[i] = bad ? ex / (I.demand[i] > 1e-12 ? I.demand[i] : 1e-12) : NAN;
        if (bad) atomicAdd(&cnt[1], 1);
    }
    if (i < I.P && x[i] < -tol) {
        atomicAdd(&cnt[2], 1);
    }
}

// max of -x over x < -tol, grid-wide (order-free: max is exact).  *out must
// hold +0.0 before the launch; the maxima are >= 0, so their bit patterns
// order like the values.
__global__ void k_worst_negative(int32_t P, const double *x, double tol, double *out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
        if (x[i] < -tol && -x[i] > m) m = -x[i];
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax((unsigned long long *)out, (unsigned long long)__double_as_longlong(m));
}

// Stable compaction of the non-NaN relative violations (edges first, then
// commodities: np.concatenate order, model.py:358-362) followed by np.mean,
// one CTA: block-scan compaction, then the pairwise tree with parallel leaves.
__global__ void __launch_bounds__(1024) k_compact_mean(const double *rel_e, int32_t E, const double *rel_c,
                                                       int32_t C, double *tmp, double *out, int64_t *leaf_lo,
                                                       double *leaf_sum) {
    constexpr int PER = 8;  // contiguous elements per thread per block step
    __shared__ int32_t wcnt[32];
    __shared__ int64_t s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int64_t N = (int64_t)E + C;
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < N; c0 += (int64_t)PER * blockDim.x) {
        const int64_t i0 = c0 + (int64_t)PER * tid;
        double v[PER];
        int32_t cnt = 0;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int64_t i = i0 + u;
            v[u] = i < E ? rel_e[i] : (i < N ? rel_c[i - E] : CUDART_NAN);
            cnt += !isnan(v[u]);
        }
        int32_t incl = cnt;  // warp inclusive scan of the per-thread counts
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wcnt[warp] = incl;
        __syncthreads();
        int32_t before = 0, total = 0;
        for (int w = 0; w < nw; ++w) {
            before += w < warp ? wcnt[w] : 0;
            total += wcnt[w];
        }
        int64_t pos = s_base + before + (incl - cnt);
#pragma unroll
        for (int u = 0; u < PER; ++u)
            if (!isnan(v[u])) tmp[pos++] = v[u];
        __syncthreads();
        if (tid == 0) s_base += total;
    }
    __syncthreads();
    const int64_t n = s_base;
    const double r = cta_np_pairwise(tmp, n, leaf_lo, leaf_sum);
    if (tid == 0) *out = n ? r / (double)n : 0.0;
}

}  // namespace

// ---------------------------------------------------------------- host wrappers

constexpr int TB = 256;

void exact_commodity_sums(const InstView &I, const double *x, double *out, cudaStream_t s) {
    if (I.C) k_segment_sums<<<ceil_div(I.C, TB), TB, 0, s>>>(x, I.com_path_ptr, I.C, out);
    PF_CHECK_LAUNCH();
}

void exact_edge_loads_from_pairs(const InstView &I, const double *pv, double *out, cudaStream_t s) {
    if (I.E) k_edge_gather_blk<0><<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, pv, out);
    PF_CHECK_LAUNCH();
}

void exact_edge_loads_of_rates(const InstView &I, const double *rates, double *out, cudaStream_t s) {
    if (I.E) k_edge_gather_blk<1><<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, rates, out);
    PF_CHECK_LAUNCH();
}

void exact_edge_loads_of_rates_em(const InstView &I, const double *rates, const int32_t *epath, double *scratch,
                                  double *out, cudaStream_t s) {
    if (!I.E) return;
    if (I.NP) k_gather_rates_edge_major<<<ceil_div(I.NP, 256), 256, 0, s>>>(I.NP, epath, rates, scratch);
    k_edge_blk_contig<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, scratch, out);
    PF_CHECK_LAUNCH();
}

void exact_edge_loads_of_rates_em_pairs(const InstView &I, const double *rates, double *scratch, double *out,
                                        cudaStream_t s) {
    if (!I.E) return;
    if (!I.NP) {
        exact_edge_loads_of_rates(I, rates, out, s);
        return;
    }
    k_gather_rates_em_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, rates, scratch);
    k_edge_blk_contig<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, scratch, out);
    PF_CHECK_LAUNCH();
}

void exact_update_duals(const InstView &I, const StatePtrs &st, double *sums, double *loads, double *dd, double *dc,
                        double *dcon, double *dn, cudaStream_t s, double *scratch) {
    exact_commodity_sums(I, st.x, sums, s);
    if (scratch && I.NP && I.E) {  // edge-major copy, then blocked sums over contiguous memory
        k_gather_edge_major<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, st.y, scratch);
        k_edge_blk_contig<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, scratch, loads);
    } else {
        exact_edge_loads_from_pairs(I, st.y, loads, s);
    }
    if (I.C) k_dual_dd<<<ceil_div(I.C, TB), TB, 0, s>>>(I.C, st.dd, sums, I.demand, dd);
    if (I.E) k_dual_dc<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, st.dc, loads, I.capacity, dc);
    if (I.NP) k_dual_dcon<<<ceil_div(I.NP, TB), TB, 0, s>>>(I.NP, st.dcon, st.x, I.pair_path, st.y, dcon);
    if (I.P) k_dual_dn<<<ceil_div(I.P, TB), TB, 0, s>>>(I.P, st.dn, st.x, dn);
    PF_CHECK_LAUNCH();
}

void exact_update_slacks(const InstView &I, const StatePtrs &st, double beta, double *sums, double *loads,
                         double *sd, double *sc, cudaStream_t s) {
    exact_commodity_sums(I, st.x, sums, s);
    exact_edge_loads_from_pairs(I, st.y, loads, s);
    if (I.C) k_slack_sd<<<ceil_div(I.C, TB), TB, 0, s>>>(I.C, st.dd, beta, I.demand, sums, sd);
    if (I.E) k_slack_sc<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, st.dc, beta, I.capacity, loads, sc);
    PF_CHECK_LAUNCH();
}

void exact_suggest(const InstView &I, const StatePtrs &st, double *y_out, cudaStream_t s, double *scratch) {
    if (!I.E) return;
    if (scratch && I.NP) {  // parallel value pass, then the sequential totals over a contiguous array
        k_suggest_vals<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, st.x, st.dcon, scratch);
        k_suggest_seq<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, scratch, st.dc, y_out);
    } else {
        k_suggest<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, st.x, st.dcon, st.dc, y_out);
    }
    PF_CHECK_LAUNCH();
}

void exact_coefficients(const InstView &I, const StatePtrs &st, double *pk, double *pw, double *wsum, double *q,
                        cudaStream_t s) {
    if (I.P) k_path_coeffs<<<ceil_div(I.P, TB), TB, 0, s>>>(I, st.y, st.dcon, st.x, st.dn, pk, pw);
    if (I.C) k_com_coeffs<<<ceil_div(I.C, TB), TB, 0, s>>>(I, pk, pw, wsum, q);
    PF_CHECK_LAUNCH();
}

void exact_roots(const InstView &I, const double *wsum, const double *q, const double *dd, double beta,
                 int64_t alpha, double *sums, Flags *flags, cudaStream_t s) {
    if (I.C) k_roots<<<ceil_div(I.C, 128), 128, 0, s>>>(I, wsum, q, dd, beta, alpha, sums, flags);
    PF_CHECK_LAUNCH();
}

void exact_rates(const InstView &I, const double *pk, const double *pw, const double *sums, const double *dd,
                 double beta, int64_t alpha, double *x_out, cudaStream_t s) {
    if (I.P) k_rates<<<ceil_div(I.P, TB), TB, 0, s>>>(I, pk, pw, sums, dd, beta, alpha, x_out);
    PF_CHECK_LAUNCH();
}

size_t sqdiff_tmp_len(int64_t n) { return (size_t)((n + PART - 1) / PART) + 1; }

void exact_sqdiff_sum(const double *a, const double *b, int64_t n, double *block_tmp, double *out, cudaStream_t s) {
    if (n == 0) {
        PF_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
        return;
    }
    int64_t nb = (n + PART - 1) / PART;
    k_sqdiff_blocks<<<(unsigned)nb, PART / BLK, 0, s>>>(a, b, n, block_tmp);
    k_sum_range_1<<<1, 32, 0, s>>>(block_tmp, nb, out);
    PF_CHECK_LAUNCH();
}

void scale_inplace(double *a, int64_t n, double f, cudaStream_t s) {
    if (n) k_scale<<<ceil_div(n, TB), TB, 0, s>>>(a, n, f);
    PF_CHECK_LAUNCH();
}

void reset_flags(Flags *f, cudaStream_t s) {
    k_reset_flags<<<1, 1, 0, s>>>(f);
    PF_CHECK_LAUNCH();
}

static void ensure_trace_scratch(const InstView &I, TraceScratch &ts) {
    if (ts.loads.n < (size_t)I.E + 1) ts.loads.alloc(I.E + 1);
    if (ts.sums.n < (size_t)I.C + 1) ts.sums.alloc(I.C + 1);
    if (ts.rel.n < (size_t)(I.E + I.C) + 1) ts.rel.alloc(I.E + I.C + 1);
    if (ts.tmp.n < (size_t)(I.E + I.C) + 1) ts.tmp.alloc(I.E + I.C + 1);
    const size_t nleaf = (size_t)(I.E + I.C) / 32 + 8;
    if (ts.leaf_sum.n < nleaf) ts.leaf_sum.alloc(nleaf);
    if (ts.leaf_lo.n < nleaf) ts.leaf_lo.alloc(nleaf);
    if (ts.cnt.n < 4) ts.cnt.alloc(4);
    if (ts.out.n < 8) ts.out.alloc(8);
    if (ts.em.n < (size_t)I.NP + 1) ts.em.alloc(I.NP + 1);
}

// controller.py:173-194 _trace_row: objective + pct_violated + mean_relative_violation.
void trace_stats(const InstView &I, const double *x, const double *root_sums, int64_t alpha, TraceScratch &ts,
                 double tol, double *host_out4, cudaStream_t s) {
    ensure_trace_scratch(I, ts);
    if (I.C) {
        k_utility<<<ceil_div(I.C, TB), TB, 0, s>>>(I.C, root_sums, alpha, ts.tmp.p);
        k_np_sum<<<1, 1024, 0, s>>>(ts.tmp.p, I.C, ts.out.p + 0, ts.leaf_lo.p, ts.leaf_sum.p);
    } else {
        PF_CUDA(cudaMemsetAsync(ts.out.p, 0, sizeof(double), s));
    }
    pf_violation rep;
    violation_stats(I, x, tol, nullptr, nullptr, ts, &rep, s);
    double obj;
    d2h(&obj, ts.out.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    host_out4[0] = obj;
    host_out4[1] = rep.pct_violated;
    host_out4[2] = rep.mean_relative_violation;
    host_out4[3] = (double)rep.n_violated;
}

// optimality_from_sums' numerator on the device: the numpy pairwise sum of the
// per-commodity terms into *d_sum (the mean divides by C on the host)
void optimality_sum_dev(const InstView &I, const double *sums, const double *ref, double theta, TraceScratch &ts,
                        double *d_sum, cudaStream_t s) {
    ensure_trace_scratch(I, ts);
    if (!I.C) {
        PF_CUDA(cudaMemsetAsync(d_sum, 0, sizeof(double), s));
        return;
    }
    k_opt_ratio<<<ceil_div(I.C, TB), TB, 0, s>>>(I.C, sums, ref, theta, ts.tmp.p);
    k_np_sum<<<1, 1024, 0, s>>>(ts.tmp.p, I.C, d_sum, ts.leaf_lo.p, ts.leaf_sum.p);
    PF_CHECK_LAUNCH();
}

// trace_stats without a host round trip (traced fast runs): row[0] objective,
// row[1] pct_violated, row[2] mean_relative_violation, row[3] n_violated, all
// on the device; alpha from the device controller
void trace_stats_dev(const InstView &I, const double *x, const double *root_sums, const int64_t *d_alpha,
                     TraceScratch &ts, double tol, double *row, cudaStream_t s) {
    ensure_trace_scratch(I, ts);
    if (I.C) {
        k_utility_dev<<<ceil_div(I.C, TB), TB, 0, s>>>(I.C, root_sums, d_alpha, ts.tmp.p);
        k_np_sum<<<1, 1024, 0, s>>>(ts.tmp.p, I.C, row + 0, ts.leaf_lo.p, ts.leaf_sum.p);
    } else {
        PF_CUDA(cudaMemsetAsync(row, 0, sizeof(double), s));
    }
    if (I.NP && I.E) {
        k_gather_rates_em_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, x, ts.em.p);
        k_edge_blk_contig<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, ts.em.p, ts.loads.p);
    } else {
        exact_edge_loads_of_rates(I, x, ts.loads.p, s);
    }
    exact_commodity_sums(I, x, ts.sums.p, s);
    PF_CUDA(cudaMemsetAsync(ts.cnt.p, 0, sizeof(int32_t) * 4, s));
    int32_t n = I.E > I.C ? I.E : I.C;
    n = n > I.P ? n : I.P;
    if (n)
        k_violations<<<ceil_div(n, TB), TB, 0, s>>>(I, x, ts.loads.p, ts.sums.p, tol, nullptr, nullptr, ts.rel.p,
                                                     ts.rel.p + I.E, ts.cnt.p);
    k_compact_mean<<<1, 1024, 0, s>>>(ts.rel.p, I.E, ts.rel.p + I.E, I.C, ts.tmp.p, row + 2, ts.leaf_lo.p,
                                      ts.leaf_sum.p);
    k_row_pct<<<1, 32, 0, s>>>(ts.cnt.p, (int64_t)I.E + I.C + I.P, row + 1, row + 3);
    PF_CHECK_LAUNCH();
}

// model.py:335-369 validate_allocation
void violation_stats(const InstView &I, const double *x, double tol, double *d_overload, double *d_excess,
                     TraceScratch &ts, pf_violation *rep, cudaStream_t s) {
    ensure_trace_scratch(I, ts);
    // exact-order edge loads through an edge-major copy (same association as
    // exact_edge_loads_of_rates, one parallel gather instead of per-lane chains)
    if (I.NP && I.E) {
        k_gather_rates_em_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, x, ts.em.p);
        k_edge_blk_contig<<<ceil_div((int64_t)I.E * 32, 128), 128, 0, s>>>(I, ts.em.p, ts.loads.p);
        PF_CHECK_LAUNCH();
    } else {
        exact_edge_loads_of_rates(I, x, ts.loads.p, s);
    }
    exact_commodity_sums(I, x, ts.sums.p, s);
    PF_CUDA(cudaMemsetAsync(ts.cnt.p, 0, sizeof(int32_t) * 4, s));
    int32_t n = I.E > I.C ? I.E : I.C;
    n = n > I.P ? n : I.P;
    if (n)
        k_violations<<<ceil_div(n, TB), TB, 0, s>>>(I, x, ts.loads.p, ts.sums.p, tol, d_overload, d_excess, ts.rel.p,
                                                     ts.rel.p + I.E, ts.cnt.p);
    k_compact_mean<<<1, 1024, 0, s>>>(ts.rel.p, I.E, ts.rel.p + I.E, I.C, ts.tmp.p, ts.out.p + 1, ts.leaf_lo.p,
                                      ts.leaf_sum.p);
    PF_CUDA(cudaMemsetAsync(ts.out.p + 2, 0, sizeof(double), s));
    if (I.P) k_worst_negative<<<std::min<int64_t>(ceil_div(I.P, 256), 592), 256, 0, s>>>(I.P, x, tol, ts.out.p + 2);
    PF_CHECK_LAUNCH();
    int32_t cnt[4];
    double mr[2];
    d2h(cnt, ts.cnt.p, 4, s);
    d2h(mr, ts.out.p + 1, 2, s);
    PF_CUDA(cudaStreamSynchronize(s));
    int64_t nv = (int64_t)cnt[0] + cnt[1] + cnt[2];
    int64_t total = (int64_t)I.E + I.C + I.P;
    rep->n_violated = nv;
    rep->negative_count = cnt[2];
    rep->worst_negative = mr[1];
    rep->pct_violated = total ? 100.0 * (double)nv / (double)total : 0.0;
    rep->mean_relative_violation = mr[0];
}

}  // namespace pf
