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
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>

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
    // np.power(s, 0.0) == 1 and np.power(s, 1.0) == s exactly; CUDA's pow is
    // only within an ulp of the latter
    const double sa = alpha == 0 ? 1.0 : alpha == 1 ? s : pow(s, (double)alpha);
    scores[p] = sa * total;
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

// CTA-wide _sum_gather_range of x over the edge's pairs (projection.py:87-88):
// the values are gathered in parallel into shared memory one block at a time,
// each 32-element chunk is summed sequentially and the chunk partials are added
// in chunk order by one thread -- the reference's exact association.
constexpr int RB = 7936;  // gather block (a multiple of the 32-element chunk; RB + RB / 32 pad slots fit the 8,192-double buffer)

__device__ double cta_edge_resum(const int32_t *epath, const double *x, int32_t lo, int32_t hi, double *buf) {
    __shared__ double s_parts[RB / BLK];
    __shared__ double s_total;
    if (threadIdx.x == 0) s_total = 0.0;
    for (int32_t b0 = lo; b0 < hi; b0 += RB) {
        const int32_t n = hi - b0 < RB ? hi - b0 : RB;
        // 8 independent gathers in flight per thread
        for (int32_t j0 = threadIdx.x; j0 < n; j0 += 8 * blockDim.x) {
            int32_t pi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int32_t j = j0 + u * blockDim.x;
                pi[u] = j < n ? epath[b0 + j] : -1;
            }
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = pi[u] >= 0 ? x[pi[u]] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int32_t j = j0 + u * blockDim.x;
                if (j < n) buf[j + (j >> 5)] = v[u];  // one pad slot per chunk: chunk c at 33 c
            }
        }
        __syncthreads();
        const int32_t nch = (n + BLK - 1) / BLK;
        for (int32_t ch = threadIdx.x; ch < nch; ch += blockDim.x) {
            const int32_t cs = ch * BLK, ce = cs + BLK < n ? cs + BLK : n;
            const double *cb = buf + ch * (BLK + 1);  // the padding keeps a warp's chunks on distinct banks
            double part = 0.0;
            if (ce - cs == BLK) {  // the loads in flight, the adds in the same order
                double b[BLK];
#pragma unroll
                for (int u = 0; u < BLK; ++u) b[u] = cb[u];
#pragma unroll
                for (int u = 0; u < BLK; ++u) part += b[u];
            } else {
                for (int32_t t = 0; t < ce - cs; ++t) part += cb[t];
            }
            s_parts[ch] = part;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double total = s_total;
            int32_t ch = 0;
            for (; ch + 8 <= nch; ch += 8) {  // 8 partials loaded ahead, added in order
                double b[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) b[u] = s_parts[ch + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) total += b[u];
            }
            for (; ch < nch; ++ch) total += s_parts[ch];
            s_total = total;
        }
        __syncthreads();
    }
    const double r = s_total;
    __syncthreads();
    return r;
}

// store a trimmed rate and mark the edges of its path for an exact re-sum
__device__ __forceinline__ void write_back(const InstView &I, double *x, uint8_t *dirty, int32_t p, double v) {
    if (x[p] != v) {
        x[p] = v;
        for (int32_t t = I.pair_ptr[p]; t < I.pair_ptr[p + 1]; ++t) dirty[I.pair_edge[t]] = 1;
    }
}

constexpr int TCH = 4096;  // chunk of ordered candidates (dynamic shared memory: 2 x 48 KB)

__global__ void __launch_bounds__(1024) k_edge_trim(InstView I, const int32_t *edge_order, const int32_t *nviol_p,
                                                     const int32_t *path_order, const int32_t *epath, double *x,
                                                     const double *over, uint8_t *dirty, int stats) {
    long long st_pass = 0, st_chain = 0, st_resum = 0, st_edges = 0;
    extern __shared__ __align__(16) char dsm[];
    double(*sx)[TCH] = (double(*)[TCH])dsm;                        // [2][TCH], also the re-sum buffer
    int32_t(*sp)[TCH] = (int32_t(*)[TCH])(dsm + 2 * TCH * sizeof(double));  // [2][TCH]
    __shared__ double s_ex;
    __shared__ int32_t s_done;
    const int32_t nviol = *nviol_p;
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int32_t vi = 0; vi < nviol; ++vi) {
        const int32_t e = edge_order[vi];
        const int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
        const double cap = I.capacity[e];
        // an edge none of whose paths was trimmed since phase 3 began still has
        // its exact starting load (same association as the re-sum)
        double excess;
        if (dirty[e]) {
            excess = cta_edge_resum(epath, x, lo, hi, &sx[0][0]) - cap;
            st_resum += hi - lo;
        } else {
            excess = over[e];
        }
        if (excess <= 0.0) continue;
        ++st_edges;
        const int32_t nch = (hi - lo + TCH - 1) / TCH;
        for (int pass = 0; pass < 16; ++pass) {
            if (tid == 0) {
                s_ex = excess;
                s_done = 0;
            }
            // chunk 0
            for (int32_t j = tid; j < TCH && lo + j < hi; j += nthr) {
                const int32_t p = path_order[lo + j];
                sp[0][j] = p;
                sx[0][j] = x[p];
            }
            __syncthreads();
            int32_t t = 0;
            for (; t < nch; ++t) {
                const int b = t & 1;
                const int32_t base = lo + t * TCH;
                const int32_t n = hi - base < TCH ? hi - base : TCH;
                if (tid == 0) {  // the exact sequential chain (projection.py:95-102)
                    // Once excess <= 0 every later step is a no-op (d <= 0), so
                    // the chain runs unrolled without a per-element exit.
                    double ex = s_ex;
                    double *v = sx[b];
                    int32_t j = 0;
                    for (; j < n && ex > 0.0; j += 8) {
                        double xv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) xv[u] = j + u < n ? v[j + u] : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            // d = min(x, ex); if d > 0: x -= d, ex -= d  (projection.py:97-101):
                            // x < ex:  d = x,  x - x = +0,  ex - x
                            // x >= ex: d = ex, x - ex,      ex - ex = +0
                            const double xu = xv[u];
                            const bool c = xu < ex;
                            const double t = ex - xu;
                            const double nx = c ? (xu > 0.0 ? 0.0 : xu) : (ex > 0.0 ? xu - ex : xu);
                            ex = c ? (xu > 0.0 ? t : ex) : (ex > 0.0 ? 0.0 : ex);
                            if (j + u < n) v[j + u] = nx;
                        }
                    }
                    s_ex = ex;
                    st_chain += j;
                    if (!(ex > 0.0)) s_done = 1;
                } else if (tid >= 32) {
                    const int nb = b ^ 1;
                    const int ltid = tid - 32, lthr = nthr - 32;
                    if (t >= 1) {  // write back chunk t-1
                        const int32_t pbase = base - TCH;
                        for (int32_t j = ltid; j < TCH && pbase + j < hi; j += lthr)
                            write_back(I, x, dirty, sp[nb][j], sx[nb][j]);
                    }
                    if (t + 1 < nch) {  // gather chunk t+1
                        const int32_t nbase = base + TCH;
                        for (int32_t j = ltid; j < TCH && nbase + j < hi; j += lthr) {
                            const int32_t p = path_order[nbase + j];
                            sp[nb][j] = p;
                            sx[nb][j] = x[p];
                        }
                    }
                }
                __syncthreads();
                if (s_done) break;
            }
            {  // write back the last chained chunk
                const int32_t tt = t < nch ? t : nch - 1;
                const int b = tt & 1;
                const int32_t base = lo + tt * TCH;
                for (int32_t j = tid; j < TCH && base + j < hi; j += nthr) write_back(I, x, dirty, sp[b][j], sx[b][j]);
            }
            __syncthreads();
            excess = cta_edge_resum(epath, x, lo, hi, &sx[0][0]) - cap;
            st_resum += hi - lo;
            ++st_pass;
            if (excess <= 0.0) break;
        }
    }
    if (stats && threadIdx.x == 0)
        printf("[k_edge_trim] violated %d trimmed %lld passes %lld chained %lld resummed %lld\n", nviol, st_edges,
               st_pass, st_chain, st_resum);
}

}  // namespace

constexpr int TB = 256;

// segments for the per-edge stable path orders: only violated edges get a
// non-empty segment (the others are never walked by k_edge_trim)
__global__ void k_violated_segments(int32_t E, const double *over, const int32_t *eptr, int32_t *sb, int32_t *se) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    bool v = over[e] > 0.0;
    sb[e] = v ? eptr[e] : 0;
    se[e] = v ? eptr[e + 1] : 0;
}

__global__ void k_edge_path_keys_violated(InstView I, const double *scores, const double *over, uint64_t *keys,
                                          int32_t *vals) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= I.NP) return;
    int32_t pr = I.edge_pairs[t];
    if (!(over[I.pair_edge[pr]] > 0.0)) return;
    int32_t p = I.pair_path[pr];
    keys[t] = desc_key(scores[p]);
    vals[t] = p;
}

// alpha = 0: a path's score is its count of violated edges (S^0 = 1), an
// integer <= hmax, so the descending stable order is the ascending stable order
// of hmax - count: a few-bit radix key (one sort pass instead of eight)
__global__ void k_edge_path_keys_violated_count(InstView I, const double *scores, const double *over, int32_t hmax,
                                                uint64_t *keys, int32_t *vals) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= I.NP) return;
    int32_t pr = I.edge_pairs[t];
    if (!(over[I.pair_edge[pr]] > 0.0)) return;
    int32_t p = I.pair_path[pr];
    keys[t] = (uint64_t)(hmax - (int32_t)scores[p]);
    vals[t] = p;
}

__global__ void k_edge_paths(InstView I, int32_t *epath) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < I.NP) epath[t] = I.pair_path[I.edge_pairs[t]];
}


// Fast-mode phase 3 (tolerance-matched, deterministic): the same walk over the
// violated edges in order, but each pass trims an edge's paths with a CTA-wide
// prefix sum of the score-ordered rates instead of the reference's sequential
// `excess -= d` chain: the paths before the first prefix >= excess are zeroed,
// that path keeps prefix - excess.  The re-sum (a fixed-order tree here) and
// the up-to-16 passes are the reference's, so any rounding excess left by the
// reassociated sums is trimmed by the next pass and the result is feasible.
__device__ double cta_sum_tree(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        double r = l < nw ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
        if (l == 0) red[32] = r;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

__device__ double cta_edge_resum_fast(const int32_t *epath, const double *x, int32_t lo, int32_t hi, double *red) {
    double v = 0.0;
    const int32_t nt = blockDim.x;
    int32_t t = lo + threadIdx.x;
    for (; t + 7 * nt < hi; t += 8 * nt) {  // 8 independent gathers in flight
        int32_t pi[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pi[u] = epath[t + u * nt];
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = x[pi[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u) v += xv[u];
    }
    for (; t < hi; t += nt) v += x[epath[t]];
    return cta_sum_tree(v, red);
}

constexpr int FCH = 4096;  // chunk of ordered candidates: 4 per thread

__global__ void __launch_bounds__(1024) k_edge_trim_fast(InstView I, const int32_t *edge_order,
                                                          const int32_t *nviol_p, const int32_t *path_order,
                                                          const int32_t *epath, double *x, const double *over,
                                                          uint8_t *dirty) {
    extern __shared__ __align__(16) char dsm[];
    double *sx = (double *)dsm;                                      // [FCH]
    int32_t *sp = (int32_t *)(dsm + FCH * sizeof(double));          // [FCH]
    __shared__ double red[33], wsum[32];
    __shared__ int32_t s_jstar;
    const int32_t nviol = *nviol_p;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int32_t vi = 0; vi < nviol; ++vi) {
        const int32_t e = edge_order[vi];
        const int32_t lo = I.edge_pair_ptr[e], hi = I.edge_pair_ptr[e + 1];
        const double cap = I.capacity[e];
        double excess = dirty[e] ? cta_edge_resum_fast(epath, x, lo, hi, red) - cap : over[e];
        if (excess <= 0.0) continue;
        for (int pass = 0; pass < 16; ++pass) {
            double carry = 0.0;  // prefix of the chunks already zeroed
            for (int32_t base = lo; base < hi; base += FCH) {
                const int32_t n = hi - base < FCH ? hi - base : FCH;
                double v[4], incl[4];
                double tsum = 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t j = 4 * tid + u;
                    double xv = 0.0;
                    if (j < n) {
                        const int32_t p = path_order[base + j];
                        sp[j] = p;
                        xv = x[p];
                    }
                    v[u] = xv;
                    tsum += xv;
                    incl[u] = tsum;
                }
                // block exclusive scan of the thread sums
                double ws = tsum;
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(0xffffffffu, ws, o);
                    if (lane >= o) ws += t;
                }
                if (lane == 31) wsum[warp] = ws;
                if (tid == 0) s_jstar = INT_MAX;
                __syncthreads();
                if (warp == 0) {
                    double a = lane < nw ? wsum[lane] : 0.0;
                    for (int o = 1; o < 32; o <<= 1) {
                        const double t = __shfl_up_sync(0xffffffffu, a, o);
                        if (lane >= o) a += t;
                    }
                    if (lane < nw) wsum[lane] = a;  // inclusive warp prefixes
                }
                __syncthreads();
                const double before = carry + (warp ? wsum[warp - 1] : 0.0) + (ws - tsum);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (4 * tid + u < n && before + incl[u] >= excess) atomicMin(&s_jstar, 4 * tid + u);
                __syncthreads();
                const int32_t js = s_jstar;
                const double total = wsum[nw - 1];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int32_t j = 4 * tid + u;
                    if (j >= n) continue;
                    double nx = v[u];
                    if (j < js)
                        nx = 0.0;
                    else if (j == js)
                        nx = max0(before + incl[u] - excess);  // prefix - excess (>= 0)
                    sx[j] = nx;
                }
                __syncthreads();
                for (int32_t j = tid; j < n; j += blockDim.x) write_back(I, x, dirty, sp[j], sx[j]);
                __syncthreads();
                if (js != INT_MAX) break;
                carry += total;
            }
            excess = cta_edge_resum_fast(epath, x, lo, hi, red) - cap;
            if (excess <= 0.0) break;
        }
    }
}

// Fast-mode phase 3 on a thread-block cluster (same trim rule as
// k_edge_trim_fast, fewer round trips): the violated edge's score-ordered
// paths are split into contiguous slices, one per CTA, gathered ONCE into
// shared memory; every pass is a local block scan plus two DSMEM exchanges
// (slice totals, then each slice's first crossing index), the trim and the
// re-check of the load stay on chip, and the changed rates are written back
// once per edge.  The load, the carries and the cut index are computed from
// values every CTA holds identically, so all decisions are uniform across the
// cluster and the result is deterministic.
namespace cg = cooperative_groups;
constexpr int CL_NT = 1024;
constexpr int CL_CAP = 18432;  // slice capacity per CTA (12 B per entry: 216 KB)
constexpr int CL_SMEM = CL_CAP * (sizeof(double) + sizeof(int32_t));

__global__ void __launch_bounds__(CL_NT, 1) k_edge_trim_cluster(InstView I, const int32_t *edge_order,
                                                               const int32_t *nviol_p, const int32_t *path_order,
                                                               double *x, int stats) {
    extern __shared__ __align__(16) char dsm[];
    double *sx = (double *)dsm;                                  // [CL_CAP]
    int32_t *sp = (int32_t *)(dsm + CL_CAP * sizeof(double));   // [CL_CAP]
    __shared__ double s_part[2][8];                              // slice totals, by rank (written remotely)
    __shared__ int32_t s_found[2][8];                            // slice-local cut index or INT_MAX
    __shared__ double wsum[32];
    __shared__ int32_t s_js;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = CL_NT >> 5;
    const int32_t nviol = *nviol_p;
    long long st_trimmed = 0, st_passes = 0;
    int ph = 0;
    cl.sync();  // every CTA of the cluster is running before any DSMEM access
    // every edge is gathered anyway, so its load is always the fresh sum of the
    // gathered rates (the reference re-sums each edge at its turn,
    // projection.py:84-88); no dirty-edge bookkeeping
    for (int32_t vi = 0; vi < nviol; ++vi) {
        const int32_t e = edge_order[vi];
        const int32_t lo = I.edge_pair_ptr[e], n = I.edge_pair_ptr[e + 1] - lo;
        const double cap = I.capacity[e];
        const int32_t chunk = (n + ncl - 1) / ncl;
        const int32_t a = min(n, rank * chunk), len = min(n, a + chunk) - a;
        if (vi + 1 < nviol) {  // the next edge's slice of the path order into L2 (independent of x)
            const int32_t e2 = edge_order[vi + 1];
            const int32_t lo2 = I.edge_pair_ptr[e2], n2 = I.edge_pair_ptr[e2 + 1] - lo2;
            const int32_t c2 = (n2 + ncl - 1) / ncl, a2 = min(n2, rank * c2), l2 = min(n2, a2 + c2) - a2;
            for (int32_t j = tid * 32; j < l2; j += CL_NT * 32)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(path_order + lo2 + a2 + j));
        }
        for (int32_t j0 = tid; j0 < len && !(stats & 2 && vi); j0 += 8 * CL_NT) {  // gather: 8 independent loads in flight
            int32_t pi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int32_t j = j0 + u * CL_NT;
                pi[u] = j < len ? __ldcg(path_order + lo + a + j) : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int32_t j = j0 + u * CL_NT;
                if (j < len) {
                    sp[j] = pi[u];
                    sx[j] = __ldcg(x + pi[u]);
                }
            }
        }
        const int32_t m = (len + CL_NT - 1) / CL_NT;  // each thread owns a contiguous run
        const int32_t r0 = min(len, tid * m), r1 = min(len, r0 + m);
        int32_t maxchg = -1;  // highest slice index changed on this edge (uniform in the CTA)
        __syncthreads();
        for (int pass = 0;; ++pass) {
            double ts = 0.0;
            for (int32_t j = r0; j < r1; ++j) ts += sx[j];
            double ws = ts;
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += t;
            }
            if (lane == 31) wsum[warp] = ws;
            if (tid == 0) s_js = INT_MAX;
            __syncthreads();
            if (warp == 0) {
                double v = lane < nw ? wsum[lane] : 0.0;
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += t;
                }
                if (lane < nw) wsum[lane] = v;
            }
            __syncthreads();
            if (tid < ncl) *cl.map_shared_rank(&s_part[ph][rank], tid) = wsum[nw - 1];
            cl.sync();
            double load = 0.0, carry = 0.0;
            for (int q = 0; q < ncl; ++q) {
                if (q == rank) carry = load;
                load += s_part[ph][q];
            }
            const double excess = load - cap;
            if (!(excess > 0.0) || pass == 16) break;  // uniform
            st_passes += 1;
            // first index of the slice whose prefix reaches the excess
            double pre = carry + (warp ? wsum[warp - 1] : 0.0) + (ws - ts);
            for (int32_t j = r0; j < r1; ++j) {
                pre += sx[j];
                if (pre >= excess) {
                    atomicMin(&s_js, j);
                    break;
                }
            }
            __syncthreads();
            const int32_t js = s_js;
            if (tid < ncl) *cl.map_shared_rank(&s_found[ph][rank], tid) = js;
            cl.sync();
            bool earlier = false;
            for (int q = 0; q < rank; ++q) earlier |= s_found[ph][q] != INT_MAX;
            if (!earlier) {
                // zero up to the cut; the cut keeps prefix - excess (recomputed by its owner)
                const int32_t cut = js == INT_MAX ? len : js;
                if (cut < len && cut >= r0 && cut < r1) {
                    double p2 = carry + (warp ? wsum[warp - 1] : 0.0) + (ws - ts);
                    for (int32_t j = r0; j <= cut; ++j) p2 += sx[j];
                    sx[cut] = max0(p2 - excess);
                }
                __syncthreads();
                for (int32_t j = tid; j < cut; j += CL_NT) sx[j] = 0.0;
                maxchg = max(maxchg, cut < len ? cut : len - 1);
            }
            ph ^= 1;
            __syncthreads();
        }
        ph ^= 1;
        for (int32_t j = tid; j <= maxchg; j += CL_NT) x[sp[j]] = sx[j];
        st_trimmed += maxchg >= 0;
        cl.sync();  // the written rates are visible to the whole cluster before the next gather
    }
    if ((stats & 1) && tid == 0)
        printf("[k_edge_trim_cluster] rank %d/%d violated %d slices trimmed %lld passes %lld\n", rank, ncl, nviol,
               st_trimmed, st_passes);
}

// The cluster trim with the gathers pipelined across edges: the score-ordered
// path slice (static during phase 3) is loaded two edges ahead, and the rates of
// the next edge are gathered speculatively while the current edge is trimmed.
// The speculative rates are used only when the current edge changed nothing
// (a cluster-uniform fact: its load did not exceed its capacity on the first
// pass); otherwise they are gathered again after the current edge's
// write-back.  Every decision and every sum is the one k_edge_trim_cluster
// makes: the result is bitwise the same.  Shared memory per CTA: three path
// slices and two rate slices of `cap` entries (cap <= PIPE_PF * CL_NT).
constexpr int PIPE_PF = 8;  // slice entries per thread held in registers while prefetching
constexpr int PIPE_ENTRY = 3 * sizeof(int32_t) + 2 * sizeof(double);
constexpr size_t PIPE_SMEM_MAX = 224 * 1024;

__device__ __forceinline__ void slice_of(const InstView &I, const int32_t *edge_order, int32_t v, int rank, int ncl,
                                         int32_t &lo, int32_t &len) {
    const int32_t e = edge_order[v];
    const int32_t l0 = I.edge_pair_ptr[e], n = I.edge_pair_ptr[e + 1] - l0;
    const int32_t chunk = (n + ncl - 1) / ncl;
    const int32_t a = min(n, rank * chunk);
    lo = l0 + a;
    len = min(n, a + chunk) - a;
}

__global__ void __launch_bounds__(CL_NT, 1) k_edge_trim_cluster_pipe(InstView I, const int32_t *edge_order,
                                                                    const int32_t *nviol_p, const int32_t *path_order,
                                                                    double *x, int32_t cap, int stats) {
    extern __shared__ __align__(16) char dsm[];
    double *sxb = (double *)dsm;                          // [2][cap]
    int32_t *spb = (int32_t *)(dsm + 2 * (size_t)cap * sizeof(double));  // [3][cap]
    __shared__ double s_part[2][8];
    __shared__ int32_t s_found[2][8];
    __shared__ double wsum[32];
    __shared__ int32_t s_js;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = CL_NT >> 5;
    const int32_t nviol = *nviol_p;
    long long st_trimmed = 0, st_passes = 0, st_regather = 0;
    int ph = 0;
    cl.sync();
    // prologue: the path slices of edges 0 and 1, the rates of edge 0
    for (int v = 0; v < 2 && v < nviol; ++v) {
        int32_t lo, len;
        slice_of(I, edge_order, v, rank, ncl, lo, len);
        for (int32_t j = tid; j < len; j += CL_NT) spb[v * cap + j] = __ldcg(path_order + lo + j);
    }
    __syncthreads();
    bool fresh = false;  // the rate slice of the current edge holds current rates
    for (int32_t vi = 0; vi < nviol; ++vi) {
        const int32_t e = edge_order[vi];
        int32_t lo, len;
        slice_of(I, edge_order, vi, rank, ncl, lo, len);
        const double cap_e = I.capacity[e];
        double *sx = sxb + (vi & 1) * cap;
        int32_t *sp = spb + (vi % 3) * cap;
        if (!fresh) {  // (edge 0, or the previous edge trimmed): gather the rates now
            for (int32_t j0 = tid; j0 < len; j0 += 8 * CL_NT) {
                double xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int32_t j = j0 + u * CL_NT;
                    xv[u] = j < len ? __ldcg(x + sp[j]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int32_t j = j0 + u * CL_NT;
                    if (j < len) sx[j] = xv[u];
                }
            }
            st_regather += vi > 0;
            __syncthreads();
        }
        // prefetch into registers: the next edge's rates (speculative) and the
        // path slice two edges ahead
        int32_t len1 = 0, len2 = 0, lo2 = 0;
        if (vi + 1 < nviol) {
            int32_t lo1;
            slice_of(I, edge_order, vi + 1, rank, ncl, lo1, len1);
        }
        if (vi + 2 < nviol) slice_of(I, edge_order, vi + 2, rank, ncl, lo2, len2);
        const int32_t *sp1 = spb + ((vi + 1) % 3) * cap;
        double nx[PIPE_PF];
        int32_t np2[PIPE_PF];
#pragma unroll
        for (int u = 0; u < PIPE_PF; ++u) {
            const int32_t j = tid + u * CL_NT;
            nx[u] = j < len1 ? __ldcg(x + sp1[j]) : 0.0;
            np2[u] = j < len2 ? __ldcg(path_order + lo2 + j) : 0;
        }
        const int32_t m = (len + CL_NT - 1) / CL_NT;  // each thread owns a contiguous run
        const int32_t r0 = min(len, tid * m), r1 = min(len, r0 + m);
        int32_t maxchg = -1;
        int npass = 0;
        for (int pass = 0;; ++pass) {
            double ts = 0.0;
            for (int32_t j = r0; j < r1; ++j) ts += sx[j];
            double ws = ts;
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += t;
            }
            if (lane == 31) wsum[warp] = ws;
            if (tid == 0) s_js = INT_MAX;
            __syncthreads();
            if (warp == 0) {
                double v = lane < nw ? wsum[lane] : 0.0;
                for (int o = 1; o < 32; o <<= 1) {
                    const double t = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += t;
                }
                if (lane < nw) wsum[lane] = v;
            }
            __syncthreads();
            if (tid < ncl) *cl.map_shared_rank(&s_part[ph][rank], tid) = wsum[nw - 1];
            cl.sync();
            double load = 0.0, carry = 0.0;
            for (int q = 0; q < ncl; ++q) {
                if (q == rank) carry = load;
                load += s_part[ph][q];
            }
            const double excess = load - cap_e;
            if (!(excess > 0.0) || pass == 16) break;  // uniform across the cluster
            ++npass;
            st_passes += 1;
            double pre = carry + (warp ? wsum[warp - 1] : 0.0) + (ws - ts);
            for (int32_t j = r0; j < r1; ++j) {
                pre += sx[j];
                if (pre >= excess) {
                    atomicMin(&s_js, j);
                    break;
                }
            }
            __syncthreads();
            const int32_t js = s_js;
            if (tid < ncl) *cl.map_shared_rank(&s_found[ph][rank], tid) = js;
            cl.sync();
            bool earlier = false;
            for (int q = 0; q < rank; ++q) earlier |= s_found[ph][q] != INT_MAX;
            if (!earlier) {
                const int32_t cut = js == INT_MAX ? len : js;
                if (cut < len && cut >= r0 && cut < r1) {
                    double p2 = carry + (warp ? wsum[warp - 1] : 0.0) + (ws - ts);
                    for (int32_t j = r0; j <= cut; ++j) p2 += sx[j];
                    sx[cut] = max0(p2 - excess);
                }
                __syncthreads();
                for (int32_t j = tid; j < cut; j += CL_NT) sx[j] = 0.0;
                maxchg = max(maxchg, cut < len ? cut : len - 1);
            }
            ph ^= 1;
            __syncthreads();
        }
        ph ^= 1;
        for (int32_t j = tid; j <= maxchg; j += CL_NT) x[sp[j]] = sx[j];
        st_trimmed += maxchg >= 0;
        // the prefetched slices into shared memory (buffers of finished edges)
        double *sx1 = sxb + ((vi + 1) & 1) * cap;
        int32_t *sp2 = spb + ((vi + 2) % 3) * cap;
#pragma unroll
        for (int u = 0; u < PIPE_PF; ++u) {
            const int32_t j = tid + u * CL_NT;
            if (j < len1) sx1[j] = nx[u];
            if (j < len2) sp2[j] = np2[u];
        }
        fresh = npass == 0;  // this edge changed nothing: the speculative rates are current
        cl.sync();  // write-back and prefetched slices visible before the next edge
    }
    if ((stats & 1) && tid == 0)
        printf("[k_edge_trim_cluster_pipe] rank %d/%d violated %d slices trimmed %lld passes %lld regathers %lld\n",
               rank, ncl, nviol, st_trimmed, st_passes, st_regather);
}

constexpr int TRIM_SMEM = 2 * TCH * (sizeof(double) + sizeof(int32_t));
constexpr int TRIM_FAST_SMEM = FCH * (sizeof(double) + sizeof(int32_t));

// Persistent scratch for the projection of one instance's index spaces (allocated
// once; no cudaMalloc / host synchronisation inside a projection).
struct ProjWS {
    DevBuf<double> scores, sums, loads, over, parts;
    DevBuf<uint8_t> viol, dirty;
    DevBuf<int32_t> order, bad, nviol, eids, eorder, pvals, porder, sb, se, epath;
    DevBuf<uint64_t> ekeys, ekeys_out, pkeys, pkeys_out;
    DevBuf<char> cub;
    size_t cub_bytes = 0;
    int32_t max_ne = 0;
    int32_t max_hops = 0;  // most edges of one path (the alpha = 0 score bound)
};

static ProjWS &workspace(const pf_instance *inst, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(inst->ws_mu);
    if (inst->proj_ws) return *static_cast<ProjWS *>(inst->proj_ws.get());
    InstView I = inst->view();
    static const bool timing = getenv("PF_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (timing)
            fprintf(stderr, "[proj_workspace] %s at %.2f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    auto ws = std::make_shared<ProjWS>();
    ws->scores.alloc(I.P + 1);
    ws->sums.alloc(I.C + 1);
    ws->loads.alloc(I.E + 1);
    ws->over.alloc(I.E + 1);
    ws->viol.alloc(I.E + 1);
    ws->dirty.alloc(I.E + 1);
    ws->order.alloc(I.P + 1);
    ws->bad.alloc(1);
    ws->nviol.alloc(1);
    ws->eids.alloc(I.E + 1);
    ws->eorder.alloc(I.E + 1);
    ws->ekeys.alloc(I.E + 1);
    ws->ekeys_out.alloc(I.E + 1);
    ws->pkeys.alloc(I.NP + 1);
    ws->pkeys_out.alloc(I.NP + 1);
    ws->pvals.alloc(I.NP + 1);
    ws->porder.alloc(I.NP + 1);
    ws->sb.alloc(I.E + 1);
    ws->se.alloc(I.E + 1);
    lap("allocs");
    ws->epath.alloc(I.NP + 1);  // path of each edge-major pair: pair_path[edge_pairs[t]]
    if (I.NP) k_edge_paths<<<ceil_div(I.NP, 256), 256, 0, s>>>(I, ws->epath.p);
    PF_CHECK_LAUNCH();
    std::vector<int32_t> eptr(I.E + 1);
    d2h(eptr.data(), I.edge_pair_ptr, I.E + 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    lap("edge paths + sync");
    for (int32_t e = 0; e < I.E; ++e) ws->max_ne = std::max(ws->max_ne, eptr[e + 1] - eptr[e]);
    {
        std::vector<int32_t> pptr(I.P + 1);
        d2h(pptr.data(), I.pair_ptr, I.P + 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        for (int64_t p = 0; p < I.P; ++p) ws->max_hops = std::max(ws->max_hops, pptr[p + 1] - pptr[p]);
    }
    ws->parts.alloc((ws->max_ne + BLK - 1) / BLK + 1);
    size_t a = 0, b = 0;
    PF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, a, ws->ekeys.p, ws->ekeys_out.p, ws->eids.p, ws->eorder.p,
                                            I.E, 0, 64, s));
    PF_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, b, ws->pkeys.p, ws->pkeys_out.p, ws->pvals.p,
                                                     ws->porder.p, I.NP, I.E, ws->sb.p, ws->se.p, 0, 64, s));
    ws->cub_bytes = std::max<size_t>(std::max(a, b), 16);
    lap("cub sizing");
    ws->cub.alloc(ws->cub_bytes);
    PF_CUDA(cudaFuncSetAttribute(k_edge_trim, cudaFuncAttributeMaxDynamicSharedMemorySize, TRIM_SMEM));
    PF_CUDA(cudaFuncSetAttribute(k_edge_trim_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, TRIM_FAST_SMEM));
    PF_CUDA(cudaFuncSetAttribute(k_edge_trim_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));
    PF_CUDA(cudaFuncSetAttribute(k_edge_trim_cluster_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 PIPE_SMEM_MAX));
    lap("attributes");
    inst->proj_ws = ws;
    return *ws;
}

// Fast-mode edge loads: one CTA per edge, 8 gathers in flight per thread, fixed
// tree (deterministic; a reassociation of model.py:305-311).
__global__ void __launch_bounds__(256) k_edge_loads_fast(InstView I, const int32_t *__restrict__ epath,
                                                         const double *__restrict__ x, double *__restrict__ out) {
    __shared__ double red[33];
    const int32_t e = blockIdx.x;
    out[e] = cta_edge_resum_fast(epath, x, I.edge_pair_ptr[e], I.edge_pair_ptr[e + 1], red);
}

static void edge_loads_ws(const InstView &I, ProjWS &ws, const double *x, bool fast, cudaStream_t s) {
    if (fast) {
        if (I.E) k_edge_loads_fast<<<I.E, 256, 0, s>>>(I, ws.epath.p, x, ws.loads.p);
        PF_CHECK_LAUNCH();
    } else {  // pkeys_out is dead outside the phase-3 sort: edge-major scratch
        exact_edge_loads_of_rates_em(I, x, ws.epath.p, (double *)ws.pkeys_out.p, ws.loads.p, s);
    }
}

static void score_paths_ws(const pf_instance *inst, ProjWS &ws, const double *x, int64_t alpha, double *scores,
                           cudaStream_t s, bool fast = false, bool loads_ready = false) {
    InstView I = inst->view();
    exact_commodity_sums(I, x, ws.sums.p, s);
    if (!loads_ready) edge_loads_ws(I, ws, x, fast, s);
    if (I.E) k_violated_edges<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, ws.loads.p, I.capacity, 1e-9, ws.viol.p);
    if (I.P) k_scores<<<ceil_div(I.P, TB), TB, 0, s>>>(I, ws.sums.p, ws.viol.p, alpha, scores);
    PF_CHECK_LAUNCH();
}

void score_paths_device(const pf_instance *inst, const double *x, int64_t alpha, double *scores, cudaStream_t s) {
    ProjWS &ws = workspace(inst, s);
    score_paths_ws(inst, ws, x, alpha, scores, s);
    PF_CUDA(cudaStreamSynchronize(s));
}

void project_device(const pf_instance *inst, const double *rates, int64_t alpha, double *x, cudaStream_t s,
                    bool fast) {
    InstView I = inst->view();
    if (I.P == 0) return;
    ProjWS &ws = workspace(inst, s);
    int32_t init[2] = {INT_MAX, 0};
    h2d(ws.bad.p, &init[0], 1, s);
    h2d(ws.nviol.p, &init[1], 1, s);
    k_clamp<<<ceil_div(I.P, TB), TB, 0, s>>>(I.P, rates, x, ws.bad.p);
    PF_CHECK_LAUNCH();
    // phase 2 (projection.py:63-74)
    score_paths_ws(inst, ws, x, alpha, ws.scores.p, s, fast);
    if (I.C) k_demand_trim<<<ceil_div(I.C, 128), 128, 0, s>>>(I, ws.scores.p, x, ws.order.p);
    PF_CHECK_LAUNCH();
    // phase 3 (projection.py:76-106): violated edges in stable descending overload
    edge_loads_ws(I, ws, x, fast, s);
    if (I.E)
        k_over<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, ws.loads.p, I.capacity, ws.over.p, ws.ekeys.p, ws.eids.p,
                                                 ws.nviol.p);
    PF_CHECK_LAUNCH();
    if (I.E) {
        size_t bytes = ws.cub_bytes;
        PF_CUDA(cub::DeviceRadixSort::SortPairs(ws.cub.p, bytes, ws.ekeys.p, ws.ekeys_out.p, ws.eids.p, ws.eorder.p,
                                                I.E, 0, 64, s));
    }
    // projection.py:81 (post-phase-2 rates): the loads of these rates were just computed
    score_paths_ws(inst, ws, x, alpha, ws.scores.p, s, fast, true);
    if (I.E) k_violated_segments<<<ceil_div(I.E, TB), TB, 0, s>>>(I.E, ws.over.p, I.edge_pair_ptr, ws.sb.p, ws.se.p);
    int end_bit = 64;
    if (alpha == 0) {
        end_bit = 1;
        while ((1ll << end_bit) <= ws.max_hops) ++end_bit;
        if (I.NP)
            k_edge_path_keys_violated_count<<<ceil_div(I.NP, TB), TB, 0, s>>>(I, ws.scores.p, ws.over.p, ws.max_hops,
                                                                            ws.pkeys.p, ws.pvals.p);
    } else if (I.NP) {
        k_edge_path_keys_violated<<<ceil_div(I.NP, TB), TB, 0, s>>>(I, ws.scores.p, ws.over.p, ws.pkeys.p,
                                                                  ws.pvals.p);
    }
    PF_CHECK_LAUNCH();
    if (I.NP) {
        size_t bytes = ws.cub_bytes;
        PF_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(ws.cub.p, bytes, ws.pkeys.p, ws.pkeys_out.p, ws.pvals.p,
                                                         ws.porder.p, I.NP, I.E, ws.sb.p, ws.se.p, 0, end_bit, s));
    }
    static const int stats = (getenv("PF_PROJ_STATS") ? 1 : 0) | (getenv("PF_PROJ_ABLATE") ? 2 : 0);  // 2: timing ablation
    PF_CUDA(cudaMemsetAsync(ws.dirty.p, 0, I.E + 1, s));
    // PF_PROJ_CLUSTER: CTAs per cluster for the fast trim (0 = single-CTA kernel)
    static const int cl_env = getenv("PF_PROJ_CLUSTER") ? atoi(getenv("PF_PROJ_CLUSTER")) : -1;
    int ncl = 0;
    if (fast && ws.max_ne <= 8 * CL_CAP) {
        const int need = (ws.max_ne + CL_CAP - 1) / CL_CAP, want = (ws.max_ne + 6143) / 6144;
        ncl = 1;
        while (ncl < 8 && (ncl < need || ncl < want)) ncl *= 2;
        if (cl_env == 0) {
            ncl = 0;
        } else if (cl_env > 0) {  // the requested size, at least what the largest edge needs
            ncl = 1;
            while (ncl < 8 && (ncl < cl_env || ncl < need)) ncl *= 2;
        }
    }
    // the pipelined cluster trim when the slices of the largest edge fit its
    // shared memory (config 2: 8 CTAs x 6,656 entries); PF_PROJ_PIPE=0 disables it
    static const bool pipe_env = !getenv("PF_PROJ_PIPE") || atoi(getenv("PF_PROJ_PIPE")) != 0;
    const int32_t pcap = ncl > 0 ? ((ws.max_ne + ncl - 1) / ncl + 31) / 32 * 32 : 0;
    if (fast && ncl > 0 && pipe_env && pcap <= PIPE_PF * CL_NT && (size_t)pcap * PIPE_ENTRY <= PIPE_SMEM_MAX) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(ncl);
        lc.blockDim = dim3(CL_NT);
        lc.dynamicSmemBytes = (size_t)pcap * PIPE_ENTRY;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ncl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        PF_CUDA(cudaLaunchKernelEx(&lc, k_edge_trim_cluster_pipe, I, (const int32_t *)ws.eorder.p,
                                   (const int32_t *)ws.nviol.p, (const int32_t *)ws.porder.p, x, pcap, stats));
    } else if (fast && ncl > 0) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(ncl);
        lc.blockDim = dim3(CL_NT);
        lc.dynamicSmemBytes = CL_SMEM;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ncl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        PF_CUDA(cudaLaunchKernelEx(&lc, k_edge_trim_cluster, I, (const int32_t *)ws.eorder.p,
                                   (const int32_t *)ws.nviol.p, (const int32_t *)ws.porder.p, x, stats));
    } else if (fast)
        k_edge_trim_fast<<<1, 1024, TRIM_FAST_SMEM, s>>>(I, ws.eorder.p, ws.nviol.p, ws.porder.p, ws.epath.p, x,
                                                         ws.over.p, ws.dirty.p);
    else
    k_edge_trim<<<1, 1024, TRIM_SMEM, s>>>(I, ws.eorder.p, ws.nviol.p, ws.porder.p, ws.epath.p, x, ws.over.p, ws.dirty.p,
                                   stats);
    PF_CHECK_LAUNCH();
    int32_t hb;
    d2h(&hb, ws.bad.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    require(hb == INT_MAX, "projection input contains non-finite rates");
}

}  // namespace pf
