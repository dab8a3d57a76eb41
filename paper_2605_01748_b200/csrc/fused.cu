// Fast mode: the whole GATE iteration (controller.py:225-273 with kernels.py's
// five steps) as ONE persistent, grid-synchronised kernel per run of iterations.
//
// Layout (built once per instance, TileLayout):
//   Commodities are cut into TILES of <= TP consecutive pairs (commodity-major,
//   the reference's own pair order).  Inside a tile the pairs are stored in
//   SLOTS sorted by edge id (stable), so every edge's pairs inside a tile form one
//   contiguous run.  Per slot: `slot_eid` (u16 edge id); per tile-local pair (in
//   path-major order, stored at the tile's slot base): `pos` (u16 slot of that
//   pair).  Tiles start at a 64-slot boundary so every per-slot array is 16-byte
//   aligned per tile.  The only per-pair STATE is dual_consensus (fp64, slot order):
//   y is never stored -- y_k = max0((x_{k-1} + dcon_k) - adj_k) is recomputed from
//   per-path x_{k-1}, per-slot dcon_k and per-edge adj_k (bitwise the value
//   _k_suggest produced), removing 16 B/pair/iteration of HBM traffic.
//
// One iteration = 3 grid barriers:
//   ctrl   residual partials -> s, r -> EMA / beta / alpha / stop (every CTA
//          evaluates the same scalar logic redundantly; no host round trip)
//   A      per tile: S_c + dual_demand (thread per commodity), dual_nonneg (thread
//          per path), then per slot: y_{k-1} recompute, dual_consensus update, T value
//          (x + dcon'); the tile's edge runs are reduced by a block-wide segmented
//          scan into a CTA-private smem accumulator (no atomics)
//   R      CTA partials -> per-edge totals in a fixed order; dual_capacity and the
//          suggestion adjustment per edge (kernels.py:94-96, :212)
//   B      per tile: y_k, path coefficients K/w (path order, kernels.py:110-119),
//          commodity coefficients + sum roots (thread per commodity), new rates;
//          y_k edge runs reduced for the next iteration's capacity dual.
// Tile inputs are staged into shared memory with cp.async (LDGSTS), double
// buffered: the copies of tile k+1 are in flight while tile k is computed.
// Reductions are deterministic (fixed tile->CTA map and operator trees); the
// per-edge sums differ in association from the reference's sequential sums, so
// fast mode is tolerance-matched (exact mode is the bitwise path).
//
// The dual rescale on a beta change (controller.py:255-266) is applied lazily:
// the factor is folded into the next read of each dual array.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "fused.cuh"

namespace cg = cooperative_groups;

namespace pf {

constexpr int NT = 256;        // threads per CTA (several CTAs per SM)
constexpr int TP = 1024;       // max pairs (slots) per tile
constexpr int ITEMS = TP / NT; // slots per thread in the segmented scan
constexpr int TPATH = 256;     // max paths per tile
constexpr int TCOM = 128;      // max commodities per tile
constexpr int SLOT_ALIGN = 64; // tile slot start alignment
constexpr int RGRP = 32;       // edges per reduction group (one lane per edge)
static_assert(ITEMS * NT == TP, "tile = ITEMS slots per thread");

struct TileDesc {
    int32_t c0, c1, p0, p1, t0, np, sb, pad;
};

struct TileLayout {
    int32_t ntiles = 0;
    int64_t nslots = 0;
    DevBuf<TileDesc> desc;      // per tile
    DevBuf<uint16_t> slot_eid;  // [nslots] edge id per slot (sorted within a tile)
    DevBuf<uint16_t> pos;       // [nslots] slot of the tile's l-th pair (path-major), at sb + l
    DevBuf<uint16_t> pair_slot; // [NP] tile-local slot of pair t (export only)
    DevBuf<int32_t> pair_tile;  // [NP] tile of pair t (export only)
    std::vector<TileDesc> h_desc;
    int32_t max_pairs = 0, max_paths = 0;
};

struct Ctrl {
    double beta, beta_used, ema_s, ema_r, f, s, r;
    int64_t alpha, alpha_used, iteration, evaluated, cooldown, target;
    int32_t just_incremented, stopped, status, first, cur, pad;
    int64_t bad;
};

struct Params {
    InstView I;
    int32_t ntiles, G, nred_items, nslices;
    const TileDesc *desc;
    const uint16_t *slot_eid, *pos;
    double *dcon, *x0, *x1, *dn, *dd, *dc, *adj;
    double *partT, *partL;  // [G][E]
    double *sub;            // [2][nslices][E]
    double *res;            // [G][8]
    double *res_dc;         // [ngroups]
    int32_t *grp_count;     // [ngroups]
    double *root_sums;      // [C] or null
    Ctrl *ctrl;
    int32_t *err;           // [2]: bad_coef, bad_root (INT_MAX = none)
    // config
    double gamma, residual_ratio, beta_scale, beta_min, beta_max;
    int64_t alpha_target, max_iterations;
    int32_t adapt;
};

// ------------------------------------------------------------------ shared memory

// One staging buffer: every global input of one tile (filled by cp.async).
struct Stage {
    TileDesc d;
    double dcon[TP];
    double x[TPATH], xp[TPATH], dn[TPATH];
    double D[TCOM], dd[TCOM];
    uint16_t eid[TP], pos[TP];
    int32_t poff[TPATH + 4];  // raw pair_ptr[p0 .. p1]
    int32_t cpp[TCOM + 4];    // raw com_path_ptr[c0 .. c1]
};

struct Work {
    double v[TP];
    double pK[TPATH], pw[TPATH];
    uint16_t pidx[TP];
    double wval[NT / 32];
    int32_t wflag[NT / 32];
    double red[NT / 32];
};

struct Smem {
    Stage *st[2];
    Work *w;
    double *acc;
};

__device__ __forceinline__ Smem carve(char *base, int E) {
    Smem s;
    char *p = base;
    s.st[0] = (Stage *)p;
    p += sizeof(Stage);
    s.st[1] = (Stage *)p;
    p += sizeof(Stage);
    s.w = (Work *)p;
    p += sizeof(Work);
    s.acc = (double *)p;
    return s;
}

static size_t smem_bytes(int E) { return 2 * sizeof(Stage) + sizeof(Work) + sizeof(double) * (size_t)E; }

// ------------------------------------------------------------------ cp.async

__device__ __forceinline__ void cp16(void *smem, const void *g) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp8(void *smem, const void *g) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp4(void *smem, const void *g) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

enum { MODE_A = 0, MODE_B = 1, MODE_L0 = 2 };

// Issue the copies of one tile's inputs into a staging buffer.
template <int MODE>
__device__ __forceinline__ void stage_tile(const Params &P, const TileDesc &d, Stage &st, const double *xk,
                                           const double *xp) {
    const int tid = threadIdx.x;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    if (MODE != MODE_L0)
        for (int i = tid; i < (np + 1) / 2; i += NT) cp16(&st.dcon[2 * i], &P.dcon[d.sb + 2 * i]);
    for (int i = tid; i < (np + 7) / 8; i += NT) {
        cp16(&st.eid[8 * i], &P.slot_eid[d.sb + 8 * i]);
        cp16(&st.pos[8 * i], &P.pos[d.sb + 8 * i]);
    }
    for (int i = tid; i < npath; i += NT) {
        cp8(&st.x[i], &xk[d.p0 + i]);
        if (MODE == MODE_A) cp8(&st.xp[i], &xp[d.p0 + i]);
        if (MODE != MODE_L0) cp8(&st.dn[i], &P.dn[d.p0 + i]);
    }
    for (int i = tid; i <= npath; i += NT) cp4(&st.poff[i], &P.I.pair_ptr[d.p0 + i]);
    if (MODE != MODE_L0) {
        for (int i = tid; i <= nc; i += NT) cp4(&st.cpp[i], &P.I.com_path_ptr[d.c0 + i]);
        for (int i = tid; i < nc; i += NT) {
            cp8(&st.D[i], &P.I.demand[d.c0 + i]);
            cp8(&st.dd[i], &P.dd[d.c0 + i]);
        }
    }
}

// Block reduction of one double in a fixed tree order (deterministic).
__device__ double block_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NT / 32 ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

// Segmented-sum operator on (head flag, value): associative.
__device__ __forceinline__ void seg_op(int f1, double x1, int &f2, double &x2) {
    if (!f2) x2 = x1 + x2;
    f2 |= f1;
}

// Block-wide segmented inclusive scan over the tile's slots (ITEMS consecutive
// slots per thread) keyed by edge id; the value at the last slot of each edge
// run is the run total and is added to acc[eid] by the thread owning that slot
// (each edge has exactly one run per tile: no write conflicts).  The operator
// tree is fixed, so the result is deterministic.
__device__ void seg_reduce_runs(const double *vals, const uint16_t *eid, int np, double *acc, Work &W) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = ITEMS * tid;
    int key[ITEMS + 1];
    double v[ITEMS];
    int h[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        int sl = base + i;
        key[i] = sl < np ? (int)eid[sl] : -1 - i;
        v[i] = sl < np ? vals[sl] : 0.0;
    }
    key[ITEMS] = base + ITEMS < np ? (int)eid[base + ITEMS] : -100;
    const int kprev = (base > 0 && base - 1 < np) ? (int)eid[base - 1] : -200;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) h[i] = (i == 0 ? key[0] != kprev : key[i] != key[i - 1]);
    // thread aggregate
    int f = h[0];
    double x = v[0];
#pragma unroll
    for (int i = 1; i < ITEMS; ++i) {
        int fi = h[i];
        double xi = v[i];
        seg_op(f, x, fi, xi);
        f = fi;
        x = xi;
    }
    // warp inclusive scan of the thread aggregates
    for (int o = 1; o < 32; o <<= 1) {
        int fo = __shfl_up_sync(0xffffffffu, f, o);
        double xo = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) seg_op(fo, xo, f, x);
    }
    if (lane == 31) {
        W.wflag[warp] = f;
        W.wval[warp] = x;
    }
    int fe = __shfl_up_sync(0xffffffffu, f, 1);
    double xe = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) {
        fe = 0;
        xe = 0.0;
    }
    __syncthreads();
    if (warp == 0) {
        int wf = lane < NT / 32 ? W.wflag[lane] : 0;
        double wx = lane < NT / 32 ? W.wval[lane] : 0.0;
        for (int o = 1; o < NT / 32; o <<= 1) {
            int fo = __shfl_up_sync(0xffffffffu, wf, o);
            double xo = __shfl_up_sync(0xffffffffu, wx, o);
            if (lane >= o) seg_op(fo, xo, wf, wx);
        }
        int pf_ = __shfl_up_sync(0xffffffffu, wf, 1);
        double px = __shfl_up_sync(0xffffffffu, wx, 1);
        if (lane < NT / 32) {
            W.wflag[lane] = lane ? pf_ : 0;
            W.wval[lane] = lane ? px : 0.0;
        }
    }
    __syncthreads();
    int fp = fe;
    double xr = xe;
    seg_op(W.wflag[warp], W.wval[warp], fp, xr);  // exclusive prefix of this thread
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        int fi = h[i];
        double xi = v[i];
        seg_op(fp, xr, fi, xi);
        fp = fi;
        xr = xi;
        if (base + i < np && key[i + 1] != key[i]) acc[key[i]] += xi;
    }
    __syncthreads();
}

// ------------------------------------------------------------------ controller

// controller.py:237-273 on the residuals of the iteration just completed.
__device__ __noinline__ void controller_step(const Params &P, Ctrl &c, double s, double r, int32_t ec, int32_t er) {
    c.evaluated = c.iteration;
    c.s = s;
    c.r = r;
    if (ec != INT_MAX) {
        c.status = PF_ERR_KERNEL_COEF;
        c.bad = ec;
        return;
    }
    if (er != INT_MAX) {
        c.status = PF_ERR_KERNEL_ROOT;
        c.bad = er;
        return;
    }
    if (!(isfinite(s) && isfinite(r))) {
        c.status = PF_ERR_SOLVER;
        return;
    }
    bool converged = r <= P.gamma && s <= P.gamma;
    int decision = 0;
    if (converged) {
        if (P.alpha_target >= 0 && c.alpha >= P.alpha_target)
            decision = 1;
        else if (c.just_incremented)
            decision = 1;
        else
            decision = 2;
    }
    c.f = 1.0;
    if (P.adapt) {
        if (c.ema_s < 0.0) {
            c.ema_s = s;
            c.ema_r = r;
        } else {
            c.ema_s += 0.1 * (s - c.ema_s);
            c.ema_r += 0.1 * (r - c.ema_r);
        }
        if (c.cooldown > 0) {
            c.cooldown -= 1;
        } else {
            double b = c.beta;
            if (c.ema_r > P.residual_ratio * c.ema_s)
                b = b * P.beta_scale;
            else if (c.ema_s > P.residual_ratio * c.ema_r)
                b = b / P.beta_scale;
            double lo = b > P.beta_min ? b : P.beta_min;
            double nb = lo < P.beta_max ? lo : P.beta_max;
            if (nb != c.beta) {
                c.f = c.beta / nb;
                c.beta = nb;
                c.cooldown = 10;
            }
        }
    }
    c.just_incremented = 0;
    if (decision == 1) {
        c.stopped = 1;
    } else if (decision == 2) {
        c.alpha += 1;
        c.just_incremented = 1;
    }
}

// Runs in every CTA on its shared-memory copy of the controller state.
__device__ void controller_eval(const Params &P, Ctrl &c) {
    if (threadIdx.x < 32) {
        double acc[5] = {0, 0, 0, 0, 0};
        for (int g = threadIdx.x; g < P.G; g += 32)
            for (int j = 0; j < 5; ++j) acc[j] += __ldcg(&P.res[g * 8 + j]);
        int ngroups = (P.I.E + RGRP - 1) / RGRP;
        double dcs = 0.0;
        for (int g = threadIdx.x; g < ngroups; g += 32) dcs += __ldcg(&P.res_dc[g]);
        acc[2] += dcs;
        for (int j = 0; j < 5; ++j)
            for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_down_sync(0xffffffffu, acc[j], o);
        if (threadIdx.x == 0) controller_step(P, c, sqrt(acc[0]), sqrt(((acc[1] + acc[2]) + acc[3]) + acc[4]),
                                              __ldcg(&P.err[0]), __ldcg(&P.err[1]));
    }
    __syncthreads();
}

// ------------------------------------------------------------------ edge phase

// Work item (group, slice): lanes = 32 edges of the group, sum CTA partials of
// the slice in CTA order; the last item of a group combines slices in order and
// applies kernels.py:212 (dual_capacity) and :94-96 (adjustment).
__device__ __noinline__ void edge_phase(const Params &P, const Ctrl &c, int g) {
    const InstView &I = P.I;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int ngroups = (I.E + RGRP - 1) / RGRP;
    int nitems = ngroups * P.nslices;
    int per = (P.G + P.nslices - 1) / P.nslices;
    for (int item = g * (NT / 32) + warp; item < nitems; item += P.G * (NT / 32)) {
        int grp = item / P.nslices, sl = item % P.nslices;
        int e = grp * RGRP + lane;
        int g0 = sl * per, g1 = g0 + per < P.G ? g0 + per : P.G;
        double sT = 0.0, sL = 0.0;
        if (e < I.E) {
            for (int gg = g0; gg < g1; ++gg) {
                sT += __ldcg(&P.partT[(size_t)gg * I.E + e]);
                sL += __ldcg(&P.partL[(size_t)gg * I.E + e]);
            }
            P.sub[(size_t)sl * I.E + e] = sT;
            P.sub[(size_t)(P.nslices + sl) * I.E + e] = sL;
        }
        __threadfence();
        __syncwarp();
        int ticket = 0;
        if (lane == 0) ticket = atomicAdd(&P.grp_count[grp], 1);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket == P.nslices - 1) {
            __threadfence();
            double T = 0.0, L = 0.0, rdc = 0.0;
            if (e < I.E) {
                for (int k = 0; k < P.nslices; ++k) {
                    T += __ldcg(&P.sub[(size_t)k * I.E + e]);
                    L += __ldcg(&P.sub[(size_t)(P.nslices + k) * I.E + e]);
                }
                double cap = I.capacity[e];
                double dold = __ldcg(&P.dc[e]) * c.f;
                double dnew = npmax0(dold + (L - cap));
                double adj = (T + dnew - cap) / ((double)I.edge_path_count[e] + 1.0);
                if (adj < 0.0) adj = 0.0;
                P.dc[e] = dnew;
                P.adj[e] = adj;
                double d = dnew - dold;
                rdc = d * d;
            }
            for (int o = 16; o > 0; o >>= 1) rdc += __shfl_down_sync(0xffffffffu, rdc, o);
            if (lane == 0) {
                P.res_dc[grp] = rdc;
                P.grp_count[grp] = 0;
            }
        }
    }
}

// ------------------------------------------------------------------ sweeps

// Per-tile compute of sweep A (kernels.py:206-216 duals of iteration k+1, and the
// per-edge T = sum(x + dcon') of _k_suggest :88-91).
__device__ __forceinline__ void tile_A(const Params &P, const TileDesc &d, const Stage &st, Smem &S, double f,
                                       int first, double &r_dd, double &r_dn, double &r_dcon) {
    Work &W = *S.w;
    const int tid = threadIdx.x;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    if (tid < TPATH) {
        // per path: dual_nonneg (kernels.py:215) and the slot -> path scatter
        for (int i = tid; i < npath; i += TPATH) {
            double dold = st.dn[i] * f;
            double dnew = npmax0(dold - st.x[i]);
            P.dn[d.p0 + i] = dnew;
            double df = dnew - dold;
            r_dn += df * df;
            int lo = st.poff[i] - d.t0, hi = st.poff[i + 1] - d.t0;
            for (int l = lo; l < hi; ++l) W.pidx[st.pos[l]] = (uint16_t)i;
        }
    } else {
        // per commodity: S_c in model.py:297-302 order, dual_demand (kernels.py:211)
        for (int j = tid - TPATH; j < nc; j += NT - TPATH) {
            int lo = st.cpp[j] - d.p0, hi = st.cpp[j + 1] - d.p0;
            double total = 0.0;
            for (int i = lo; i < hi;) {
                int k2 = i + 32 < hi ? i + 32 : hi;
                double part = 0.0;
                for (int t = i; t < k2; ++t) part += st.x[t];
                total += part;
                i = k2;
            }
            double dold = st.dd[j] * f;
            double dnew = npmax0(dold + (total - st.D[j]));
            P.dd[d.c0 + j] = dnew;
            double df = dnew - dold;
            r_dd += df * df;
        }
    }
    __syncthreads();
    // per slot: y_{k-1} (recomputed), dual_consensus (kernels.py:72), T value (:91)
    for (int sl = tid; sl < np; sl += NT) {
        int i = W.pidx[sl];
        double dk = st.dcon[sl];
        double y = first ? st.xp[i] : max0(st.xp[i] + dk - P.adj[st.eid[sl]]);
        double dks = dk * f;
        double dnew = max0(dks + st.x[i] - y);
        P.dcon[d.sb + sl] = dnew;
        double df = dnew - dks;
        r_dcon += df * df;
        W.v[sl] = st.x[i] + dnew;
    }
    __syncthreads();
    seg_reduce_runs(W.v, st.eid, np, S.acc, W);
}

// Per-tile compute of sweep B (kernels.py:235-296 for iteration k+1).
__device__ __forceinline__ void tile_B(const Params &P, const TileDesc &d, const Stage &st, Smem &S, double beta,
                                       int64_t alpha, double *xn, double &r_x) {
    Work &W = *S.w;
    const int tid = threadIdx.x;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    // per path: y_k and K_p in path order (kernels.py:98-100, :110-119)
    for (int i = tid; i < npath; i += NT) {
        double x = st.x[i];
        double acc = 0.0;
        int lo = st.poff[i] - d.t0, hi = st.poff[i + 1] - d.t0;
        for (int l = lo; l < hi; ++l) {
            int sl = st.pos[l];
            double dk = st.dcon[sl];
            double y = max0(x + dk - P.adj[st.eid[sl]]);
            W.v[sl] = y;
            acc += y - dk;
        }
        double dn = st.dn[i];
        double h = (double)(hi - lo);
        if (x < dn) {
            W.pK[i] = acc + dn;
            W.pw[i] = 1.0 / (h + 1.0);
        } else {
            W.pK[i] = acc;
            W.pw[i] = 1.0 / h;
        }
    }
    __syncthreads();
    // per commodity: W, Q, root, rates (kernels.py:122-131, 176-195, 285-296)
    for (int j = tid; j < nc; j += NT) {
        int lo = st.cpp[j] - d.p0, hi = st.cpp[j + 1] - d.p0;
        int cc = d.c0 + j;
        double ws = 0.0, qw = 0.0;
        for (int i = lo; i < hi; ++i) {
            ws += W.pw[i];
            qw += W.pw[i] * W.pK[i];
        }
        if (!(isfinite(ws) && isfinite(qw))) {
            atomicMin(&P.err[0], cc);
            continue;
        }
        double D = st.D[j], dd = st.dd[j];
        double Sc = commodity_root(ws, qw, D - dd, beta, alpha);
        if (!isfinite(Sc)) atomicMin(&P.err[1], cc);
        if (P.root_sums) P.root_sums[cc] = Sc;
        double ct = commodity_term(Sc, D, dd, beta, alpha);
        for (int i = lo; i < hi; ++i) {
            double xv = W.pw[i] * (W.pK[i] + ct);
            xn[d.p0 + i] = xv;
            double df = xv - st.x[i];
            r_x += df * df;
        }
    }
    seg_reduce_runs(W.v, st.eid, np, S.acc, W);
}

// Initial capacity-dual load L(y_0), y_0 = x_0[pair_path] (controller.py:118).
__device__ __forceinline__ void tile_L0(const TileDesc &d, const Stage &st, Smem &S) {
    Work &W = *S.w;
    const int npath = d.p1 - d.p0;
    for (int i = threadIdx.x; i < npath; i += NT) {
        int lo = st.poff[i] - d.t0, hi = st.poff[i + 1] - d.t0;
        for (int l = lo; l < hi; ++l) W.v[st.pos[l]] = st.x[i];
    }
    __syncthreads();
    seg_reduce_runs(W.v, st.eid, d.np, S.acc, W);
}

// One sweep over this CTA's tiles with double-buffered cp.async staging.
// Sweep B walks the tiles in reverse so it first re-reads what sweep A wrote last.
template <int MODE>
__device__ __noinline__ void sweep(const Params &P, const Ctrl &c, Smem &S, int g, double *part, double *res3) {
    const int E = P.I.E;
    const double *xk = c.cur ? P.x1 : P.x0;
    double *xo = c.cur ? P.x0 : P.x1;  // x_{k-1} (A: read) / x_{k+1} (B: write)
    for (int e = threadIdx.x; e < E; e += NT) S.acc[e] = 0.0;
    const int my = g < P.ntiles ? (P.ntiles - 1 - g) / P.G + 1 : 0;
    auto tile_of = [&](int k) { return MODE == MODE_B ? g + (my - 1 - k) * P.G : g + k * P.G; };
    double ra = 0.0, rb = 0.0, rc = 0.0;
    if (my > 0) {
        TileDesc d = P.desc[tile_of(0)];
        stage_tile<MODE>(P, d, *S.st[0], xk, xo);
        if (threadIdx.x == 0) S.st[0]->d = d;
        cp_commit();
    }
    for (int k = 0; k < my; ++k) {
        if (k + 1 < my) {
            TileDesc d = P.desc[tile_of(k + 1)];
            stage_tile<MODE>(P, d, *S.st[(k + 1) & 1], xk, xo);
            if (threadIdx.x == 0) S.st[(k + 1) & 1]->d = d;
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const Stage &st = *S.st[k & 1];
        if (MODE == MODE_A)
            tile_A(P, st.d, st, S, c.f, c.first, ra, rb, rc);
        else if (MODE == MODE_B)
            tile_B(P, st.d, st, S, c.beta, c.alpha, xo, ra);
        else
            tile_L0(st.d, st, S);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += NT) part[(size_t)g * E + e] = S.acc[e];
    if (MODE == MODE_A) {
        double t = block_sum(ra, S.w->red);
        if (threadIdx.x == 0) res3[1] = t;
        t = block_sum(rc, S.w->red);
        if (threadIdx.x == 0) res3[3] = t;
        t = block_sum(rb, S.w->red);
        if (threadIdx.x == 0) res3[4] = t;
    } else if (MODE == MODE_B) {
        double t = block_sum(ra, S.w->red);
        if (threadIdx.x == 0) res3[0] = t;
    }
}

// ------------------------------------------------------------------ kernels

__global__ void __launch_bounds__(NT, 3) k_fused(const __grid_constant__ Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ Ctrl c;
    Smem S = carve(smem_raw, P.I.E);
    cg::grid_group grid = cg::this_grid();
    const int g = blockIdx.x;
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    for (;;) {
        if (c.iteration > c.evaluated) controller_eval(P, c);
        if (c.stopped || c.status || c.iteration >= c.target || c.iteration >= P.max_iterations) break;
        sweep<MODE_A>(P, c, S, g, P.partT, P.res + g * 8);
        grid.sync();
        edge_phase(P, c, g);
        grid.sync();
        sweep<MODE_B>(P, c, S, g, P.partL, P.res + g * 8);
        __syncthreads();
        if (threadIdx.x == 0) {
            c.alpha_used = c.alpha;
            c.beta_used = c.beta;
            c.f = 1.0;
            c.first = 0;
            c.cur ^= 1;
            c.iteration += 1;
        }
        grid.sync();
    }
    if (g == 0 && threadIdx.x == 0) *P.ctrl = c;
}

__global__ void __launch_bounds__(NT, 3) k_init_L0(const __grid_constant__ Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ Ctrl c;
    Smem S = carve(smem_raw, P.I.E);
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    sweep<MODE_L0>(P, c, S, blockIdx.x, P.partL, nullptr);
}

// Export helpers: reference pair order <- slot order.
__global__ void k_export_pairs(Params P, const int32_t *pair_tile, const uint16_t *pair_slot, double *y_out,
                               double *dcon_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.I.NP) return;
    Ctrl c = *P.ctrl;
    TileDesc d = P.desc[pair_tile[t]];
    int sl = d.sb + pair_slot[t];
    int p = P.I.pair_path[t];
    const double *xp = c.cur ? P.x0 : P.x1;  // x_{k-1}
    const double *xk = c.cur ? P.x1 : P.x0;
    double dk = P.dcon[sl];
    if (y_out) {
        if (c.iteration == 0)
            y_out[t] = xk[p];
        else
            y_out[t] = max0(xp[p] + dk - P.adj[P.slot_eid[sl]]);
    }
    if (dcon_out) dcon_out[t] = dk * c.f;
}

__global__ void k_scaled_copy(const double *a, int64_t n, const Ctrl *ctrl, double *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] * ctrl->f;
}

// ------------------------------------------------------------------ host side

static std::shared_ptr<TileLayout> build_tiles(const pf_instance *inst, cudaStream_t s) {
    const Index &I = *inst->idx;
    std::vector<int32_t> cpp(I.C + 1), pptr(I.P + 1), pedge(I.NP);
    d2h(cpp.data(), I.com_path_ptr.p, I.C + 1, s);
    d2h(pptr.data(), I.pair_ptr.p, I.P + 1, s);
    d2h(pedge.data(), I.pair_edge.p, I.NP, s);
    PF_CUDA(cudaStreamSynchronize(s));
    require(I.E <= 65535, "fast mode supports up to 65535 edges (u16 edge ids)");
    auto L = std::make_shared<TileLayout>();
    std::vector<TileDesc> tiles;
    int64_t slot = 0;
    int32_t c = 0;
    while (c < I.C) {
        int32_t c0 = c;
        int32_t p0 = cpp[c0];
        int32_t t0 = pptr[p0];
        while (c < I.C) {
            int32_t np_ = pptr[cpp[c + 1]] - t0;
            int32_t npath = cpp[c + 1] - p0;
            if (c > c0 && (np_ > TP || npath > TPATH || c + 1 - c0 > TCOM)) break;
            require(np_ <= TP && npath <= TPATH,
                    "commodity " + std::to_string(c) + " has more pairs/paths than a fast-mode tile holds");
            ++c;
        }
        TileDesc d;
        d.c0 = c0;
        d.c1 = c;
        d.p0 = p0;
        d.p1 = cpp[c];
        d.t0 = t0;
        d.np = pptr[cpp[c]] - t0;
        d.sb = (int32_t)slot;
        d.pad = 0;
        tiles.push_back(d);
        L->max_pairs = std::max(L->max_pairs, d.np);
        L->max_paths = std::max(L->max_paths, d.p1 - d.p0);
        slot += (d.np + SLOT_ALIGN - 1) / SLOT_ALIGN * SLOT_ALIGN;
        require(slot < INT_MAX, "too many slots");
    }
    L->ntiles = (int32_t)tiles.size();
    L->nslots = slot;
    std::vector<uint16_t> pair_slot(I.NP), slot_eid(slot ? slot : 1, (uint16_t)0), pos(slot ? slot : 1, (uint16_t)0);
    std::vector<int32_t> pair_tile(I.NP);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t ti = 0; ti < (int64_t)tiles.size(); ++ti) {
        const TileDesc &T = tiles[ti];
        std::vector<int32_t> ord(T.np);
        for (int32_t l = 0; l < T.np; ++l) ord[l] = l;
        std::stable_sort(ord.begin(), ord.end(),
                         [&](int32_t a, int32_t b) { return pedge[T.t0 + a] < pedge[T.t0 + b]; });
        for (int32_t sl = 0; sl < T.np; ++sl) {
            int32_t l = ord[sl];
            pair_slot[T.t0 + l] = (uint16_t)sl;
            pair_tile[T.t0 + l] = (int32_t)ti;
            slot_eid[T.sb + sl] = (uint16_t)pedge[T.t0 + l];
            pos[T.sb + l] = (uint16_t)sl;
        }
    }
    L->desc.alloc(tiles.size() ? tiles.size() : 1);
    L->slot_eid.alloc(slot ? slot : 1);
    L->pos.alloc(slot ? slot : 1);
    L->pair_slot.alloc(I.NP ? I.NP : 1);
    L->pair_tile.alloc(I.NP ? I.NP : 1);
    h2d(L->desc.p, tiles.data(), tiles.size(), s);
    h2d(L->slot_eid.p, slot_eid.data(), slot, s);
    h2d(L->pos.p, pos.data(), slot, s);
    h2d(L->pair_slot.p, pair_slot.data(), I.NP, s);
    h2d(L->pair_tile.p, pair_tile.data(), I.NP, s);
    PF_CUDA(cudaStreamSynchronize(s));
    L->h_desc = std::move(tiles);
    return L;
}

struct FastSolver {
    const pf_instance *inst;
    pf_config cfg;
    std::shared_ptr<TileLayout> L;
    int G = 0, nslices = 1;
    size_t smem = 0;
    DevBuf<double> dcon, x0, x1, dn, dd, dc, adj, partT, partL, sub, res, res_dc, root_sums;
    DevBuf<int32_t> grp_count, err;
    DevBuf<Ctrl> ctrl;
    Params P{};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int64_t launches = 0;
    const CommOps *comm = nullptr;
};

FastSolver *fast_create(const pf_instance *inst, const pf_config &cfg, cudaStream_t s) {
    const Index &I = *inst->idx;
    std::unique_ptr<FastSolver> F(new FastSolver());
    F->inst = inst;
    F->cfg = cfg;
    {
        std::lock_guard<std::mutex> lk(inst->idx->tiles_mu);
        if (!inst->idx->tiles) inst->idx->tiles = build_tiles(inst, s);
        F->L = inst->idx->tiles;
    }
    F->smem = smem_bytes((int)I.E);
    int dev = inst->device();
    cudaDeviceProp prop;
    PF_CUDA(cudaGetDeviceProperties(&prop, dev));
    require(F->smem <= (size_t)prop.sharedMemPerBlockOptin,
            "fast mode: edge tables do not fit in shared memory (too many edges)");
    PF_CUDA(cudaFuncSetAttribute(k_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_init_L0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    int per_sm = 0;
    PF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused, NT, F->smem));
    require(per_sm >= 1, "fast kernel does not fit on an SM");
    int G = prop.multiProcessorCount * per_sm;
    G = std::max(1, std::min(G, F->L->ntiles));
    F->G = G;
    int ngroups = (int)((I.E + RGRP - 1) / RGRP);
    int warps = G * (NT / 32);
    F->nslices = std::max(1, std::min(G, warps / std::max(ngroups, 1)));
    F->nslices = std::min(F->nslices, 32);
    int64_t E = I.E ? I.E : 1;
    F->dcon.alloc(F->L->nslots ? F->L->nslots : 1);
    F->x0.alloc(I.P ? I.P : 1);
    F->x1.alloc(I.P ? I.P : 1);
    F->dn.alloc(I.P ? I.P : 1);
    F->dd.alloc(I.C ? I.C : 1);
    F->dc.alloc(E);
    F->adj.alloc(E);
    F->partT.alloc((size_t)G * E);
    F->partL.alloc((size_t)G * E);
    F->sub.alloc((size_t)2 * F->nslices * E);
    F->res.alloc((size_t)G * 8);
    F->res_dc.alloc(ngroups ? ngroups : 1);
    F->grp_count.alloc(ngroups ? ngroups : 1);
    F->err.alloc(2);
    F->ctrl.alloc(1);
    if (cfg.trace) F->root_sums.alloc(I.C ? I.C : 1);
    PF_CUDA(cudaMemsetAsync(F->grp_count.p, 0, sizeof(int32_t) * (ngroups ? ngroups : 1), s));
    PF_CUDA(cudaEventCreate(&F->e0));
    PF_CUDA(cudaEventCreate(&F->e1));
    Params &P = F->P;
    P.I = inst->view();
    P.ntiles = F->L->ntiles;
    P.G = G;
    P.nslices = F->nslices;
    P.desc = F->L->desc.p;
    P.slot_eid = F->L->slot_eid.p;
    P.pos = F->L->pos.p;
    P.dcon = F->dcon.p;
    P.x0 = F->x0.p;
    P.x1 = F->x1.p;
    P.dn = F->dn.p;
    P.dd = F->dd.p;
    P.dc = F->dc.p;
    P.adj = F->adj.p;
    P.partT = F->partT.p;
    P.partL = F->partL.p;
    P.sub = F->sub.p;
    P.res = F->res.p;
    P.res_dc = F->res_dc.p;
    P.grp_count = F->grp_count.p;
    P.root_sums = cfg.trace ? F->root_sums.p : nullptr;
    P.ctrl = F->ctrl.p;
    P.err = F->err.p;
    P.gamma = cfg.gamma;
    P.residual_ratio = cfg.residual_ratio;
    P.beta_scale = cfg.beta_scale;
    P.beta_min = cfg.beta_min;
    P.beta_max = cfg.beta_max;
    P.alpha_target = cfg.alpha_target;
    P.max_iterations = cfg.max_iterations;
    P.adapt = cfg.adapt;
    PF_CUDA(cudaStreamSynchronize(s));
    return F.release();
}

void fast_destroy(FastSolver *F) {
    if (!F) return;
    if (F->e0) cudaEventDestroy(F->e0);
    if (F->e1) cudaEventDestroy(F->e1);
    delete F;
}

void fast_set_comm(FastSolver *F, const CommOps *ops) { F->comm = ops; }

void fast_init(FastSolver *F, const double *d_x0, int64_t alpha0, double beta0, cudaStream_t s) {
    const Index &I = *F->inst->idx;
    PF_CUDA(cudaMemcpyAsync(F->x0.p, d_x0, sizeof(double) * I.P, cudaMemcpyDeviceToDevice, s));
    PF_CUDA(cudaMemcpyAsync(F->x1.p, d_x0, sizeof(double) * I.P, cudaMemcpyDeviceToDevice, s));
    PF_CUDA(cudaMemsetAsync(F->dcon.p, 0, F->dcon.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->dn.p, 0, F->dn.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->dd.p, 0, F->dd.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->dc.p, 0, F->dc.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->adj.p, 0, F->adj.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->partL.p, 0, F->partL.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->res.p, 0, F->res.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->res_dc.p, 0, F->res_dc.bytes(), s));
    int32_t e2[2] = {INT_MAX, INT_MAX};
    h2d(F->err.p, e2, 2, s);
    Ctrl c;
    std::memset(&c, 0, sizeof(c));
    c.beta = c.beta_used = beta0;
    c.ema_s = c.ema_r = -1.0;
    c.f = 1.0;
    c.alpha = c.alpha_used = alpha0;
    c.iteration = 0;
    c.evaluated = 0;
    c.first = 1;
    c.cur = 0;
    c.s = c.r = NAN;
    c.bad = -1;
    h2d(F->ctrl.p, &c, 1, s);
    if (I.P) {
        k_init_L0<<<F->G, NT, F->smem, s>>>(F->P);
        PF_CHECK_LAUNCH();
        ++F->launches;
    }
    PF_CUDA(cudaStreamSynchronize(s));
}

int64_t fast_run(FastSolver *F, int64_t max_steps, cudaStream_t s, float *ms) {
    Ctrl c;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    int64_t start = c.iteration;
    if (F->inst->idx->P == 0 || max_steps <= 0) {
        if (ms) *ms = 0.f;
        return 0;
    }
    int64_t target = start + max_steps;
    // write the new target into the device controller
    PF_CUDA(cudaMemcpyAsync((char *)F->ctrl.p + offsetof(Ctrl, target), &target, sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
    Params P = F->P;
    void *args[] = {&P};
    PF_CUDA(cudaEventRecord(F->e0, s));
    PF_CUDA(cudaLaunchCooperativeKernel((const void *)k_fused, dim3(F->G), dim3(NT), args, F->smem, s));
    PF_CHECK_LAUNCH();
    PF_CUDA(cudaEventRecord(F->e1, s));
    ++F->launches;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    float t = 0.f;
    PF_CUDA(cudaEventElapsedTime(&t, F->e0, F->e1));
    if (ms) *ms = t;
    return c.iteration - start;
}

FastStatus fast_status(FastSolver *F, cudaStream_t s) {
    Ctrl c;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    FastStatus fs;
    fs.iteration = c.iteration;
    fs.alpha = c.alpha;
    fs.alpha_used = c.alpha_used;
    fs.beta = c.beta;
    fs.beta_used = c.beta_used;
    fs.s = c.s;
    fs.r = c.r;
    fs.stopped = c.stopped;
    fs.status = c.status;
    fs.bad = c.bad;
    return fs;
}

const double *fast_x(FastSolver *F) {
    Ctrl c;
    PF_CUDA(cudaMemcpy(&c, F->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost));
    return c.cur ? F->x1.p : F->x0.p;
}

const double *fast_root_sums(FastSolver *F) { return F->root_sums.p; }

void fast_export_state(FastSolver *F, double *x, double *y, double *dd, double *dc, double *dcon, double *dn,
                       cudaStream_t s) {
    const Index &I = *F->inst->idx;
    DevBuf<double> dy(I.NP ? I.NP : 1), ddc(I.NP ? I.NP : 1), tmp(std::max<int64_t>({I.C, I.E, I.P, 1}));
    if (I.NP) k_export_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(F->P, F->L->pair_tile.p, F->L->pair_slot.p, dy.p, ddc.p);
    PF_CHECK_LAUNCH();
    Ctrl c;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    if (x) d2h(x, c.cur ? F->x1.p : F->x0.p, I.P, s);
    if (y) d2h(y, dy.p, I.NP, s);
    if (dcon) d2h(dcon, ddc.p, I.NP, s);
    auto scaled = [&](const double *src, int64_t n, double *out) {
        if (!out || !n) return;
        k_scaled_copy<<<ceil_div(n, 256), 256, 0, s>>>(src, n, F->ctrl.p, tmp.p);
        PF_CHECK_LAUNCH();
        d2h(out, tmp.p, n, s);
        PF_CUDA(cudaStreamSynchronize(s));
    };
    PF_CUDA(cudaStreamSynchronize(s));
    scaled(F->dd.p, I.C, dd);
    scaled(F->dc.p, I.E, dc);
    scaled(F->dn.p, I.P, dn);
}

void fast_stats(FastSolver *F, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes) {
    const Index &I = *F->inst->idx;
    if (launches) *launches = F->launches;
    if (tiles) *tiles = F->L->ntiles;
    if (grid) *grid = F->G;
    // compulsory HBM bytes per iteration of this kernel's data layout:
    //  per slot: dcon r/w in A (16) + r in B (8) + slot_eid A,B (4) + pos A,B (4)
    //  per path: x_k (A,B 16) + x_{k-1} (A 8) + x_{k+1} write (8) + dn r/w A + r B (24) + pair_ptr A,B (8)
    //  per commodity: dd r/w A + r B (24) + demand A,B (16) + com_path_ptr A,B (8)
    //  per CTA: edge partials written and read back (2 x 2 x 8 B per edge)
    if (bytes) *bytes = 32 * F->L->nslots + 64 * I.P + 48 * I.C + (int64_t)F->G * I.E * 32;
}

}  // namespace pf
