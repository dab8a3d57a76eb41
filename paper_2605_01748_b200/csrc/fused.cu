// Fast mode: the whole GATE iteration (controller.py:225-273 with kernels.py's
// five steps) as ONE persistent, grid-synchronised kernel per run of iterations.
//
// Layout (built once per instance, TileLayout):
//   Commodities are cut into TILES of <= TP consecutive pairs (commodity-major,
//   the reference's own pair order).  Inside a tile the pairs are stored in
//   SLOTS sorted by edge id (stable), so every edge's pairs inside a tile form one
//   contiguous run.  Per pair we keep `pair_slot` (u16, tile-local slot of the
//   pair, path-major order); per slot `slot_eid` (u16 edge id).  Tiles start at a
//   64-slot boundary.  The only per-pair state is dual_consensus (fp64, slot order).
//   y is never stored: y_k = max0((x_{k-1} + dcon_k) - adj_k) is recomputed from
//   per-path x_{k-1}, per-slot dcon_k and per-edge adj_k (bitwise the value
//   _k_suggest produced), which removes 16 B/pair/iteration of HBM traffic.
//
// One iteration = 3 grid barriers:
//   ctrl   residual partials -> s, r -> EMA / beta / alpha / stop (every CTA
//          evaluates the same scalar logic redundantly; no host round trip)
//   A      per tile: S_c, dual_demand, dual_nonneg (per commodity / path), then per
//          slot: y_{k-1} recompute, dual_consensus update, T value (x + dcon');
//          edge runs reduced into a CTA-private smem accumulator (no atomics)
//   R      CTA partials -> per-edge totals in a fixed order; dual_capacity and the
//          suggestion adjustment per edge (kernels.py:94-96, :212)
//   B      per tile: y_k, path coefficients K/w (path order, kernels.py:110-119),
//          commodity coefficients + sum roots (thread per commodity), new rates;
//          y_k edge runs reduced for the next iteration's capacity dual.
// Reductions are deterministic (fixed tile->CTA map and orders); the per-edge
// sums differ in association from the reference's sequential sums, so fast mode
// is tolerance-matched (exact mode is the bitwise path).
//
// dual rescaling on a beta change (controller.py:255-266) is applied lazily: the
// factor is folded into the next read of each dual array.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "fused.cuh"

namespace cg = cooperative_groups;

namespace pf {

constexpr int NT = 512;        // threads per CTA
constexpr int TP = 2048;       // max pairs (slots) per tile
constexpr int TPATH = 512;     // max paths per tile
constexpr int SLOT_ALIGN = 64; // tile slot start alignment
constexpr int RGRP = 32;       // edges per reduction group (one lane per edge)

struct TileLayout {
    int32_t ntiles = 0;
    int64_t nslots = 0;
    DevBuf<int4> tiles;         // {com_begin, com_end, slot_begin, npairs}
    DevBuf<uint16_t> pair_slot; // [NP]
    DevBuf<uint16_t> slot_eid;  // [nslots]
    std::vector<int4> h_tiles;
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
    const int4 *tiles;
    const uint16_t *pair_slot, *slot_eid;
    double *dcon, *x0, *x1, *dn, *dd, *dc, *adj;
    double *partT, *partL;  // [G][E]
    double *sub;            // [nslices][E] x 2
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

// ------------------------------------------------------------------ smem layout
struct Smem {
    double *dcon, *v, *acc, *adj;
    double *px, *pxp, *pK, *pw;
    uint16_t *eid, *pos, *pidx;
    int32_t *poff;
    double *red;
};

__device__ __forceinline__ Smem carve(char *base, int E) {
    Smem s;
    double *d = (double *)base;
    s.dcon = d; d += TP;
    s.v = d; d += TP;
    s.acc = d; d += E;
    s.adj = d; d += E;
    s.px = d; d += TPATH;
    s.pxp = d; d += TPATH;  // aliases pK in sweep B
    s.pK = s.pxp;
    s.pw = d; d += TPATH;
    s.red = d; d += 32;
    uint16_t *u = (uint16_t *)d;
    s.eid = u; u += TP;
    s.pos = u; u += TP;
    s.pidx = u; u += TP;
    s.poff = (int32_t *)(((uintptr_t)u + 15) & ~(uintptr_t)15);
    return s;
}

static size_t smem_bytes(int E) {
    size_t b = sizeof(double) * (2 * TP + 2 * (size_t)E + 3 * TPATH + 32);
    b += sizeof(uint16_t) * 3 * TP + 16;
    b += sizeof(int32_t) * (TPATH + 1);
    return b;
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

struct TileRange {
    int32_t c0, c1, p0, p1, t0, np, npath, sb;
};

__device__ __forceinline__ TileRange tile_range(const Params &P, int tile) {
    int4 ti = P.tiles[tile];
    TileRange r;
    r.c0 = ti.x;
    r.c1 = ti.y;
    r.sb = ti.z;
    r.np = ti.w;
    r.p0 = P.I.com_path_ptr[r.c0];
    r.p1 = P.I.com_path_ptr[r.c1];
    r.t0 = P.I.pair_ptr[r.p0];
    r.npath = r.p1 - r.p0;
    return r;
}

// Common tile staging: slot eids, pair->slot map, path offsets, and the
// slot->path scatter.
__device__ __forceinline__ void stage_tile_index(const Params &P, const TileRange &R, Smem &S) {
    for (int i = threadIdx.x; i < R.np; i += NT) {
        S.eid[i] = P.slot_eid[R.sb + i];
        S.pos[i] = P.pair_slot[R.t0 + i];
    }
    for (int i = threadIdx.x; i <= R.npath; i += NT) S.poff[i] = P.I.pair_ptr[R.p0 + i] - R.t0;
}

// Segmented reduction of vals[] over the tile's edge runs into acc[eid]
// (each run is owned by the thread whose chunk contains its head: no races).
__device__ __forceinline__ void reduce_runs(const Smem &S, const double *vals, int np, double *acc) {
    int chunk = (np + NT - 1) / NT;
    int a = threadIdx.x * chunk;
    int b = a + chunk < np ? a + chunk : np;
    int s = a;
    if (s < b && s > 0) {
        uint16_t e0 = S.eid[s - 1];
        while (s < b && S.eid[s] == e0) ++s;
    }
    while (s < b) {
        uint16_t e = S.eid[s];
        double sum = 0.0;
        int t = s;
        while (t < np && S.eid[t] == e) sum += vals[t++];
        acc[e] += sum;
        s = t;
    }
}

// ------------------------------------------------------------------ controller

__device__ void controller_eval(const Params &P, Ctrl &c, double *red) {
    // Every CTA computes the same values in the same order.
    __shared__ double s_out[2];
    __shared__ int32_t s_err[2];
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
        if (threadIdx.x == 0) {
            s_out[0] = sqrt(acc[0]);
            s_out[1] = sqrt(((acc[1] + acc[2]) + acc[3]) + acc[4]);
            s_err[0] = __ldcg(&P.err[0]);
            s_err[1] = __ldcg(&P.err[1]);
        }
    }
    __syncthreads();
    double s = s_out[0], r = s_out[1];
    int32_t ec = s_err[0], er = s_err[1];
    __syncthreads();
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

// ------------------------------------------------------------------ sweep A

__device__ void sweep_A(const Params &P, const Ctrl &c, Smem &S, int g) {
    const InstView &I = P.I;
    const double f = c.f;
    const double *xk = c.cur ? P.x1 : P.x0;
    const double *xp = c.cur ? P.x0 : P.x1;
    for (int e = threadIdx.x; e < I.E; e += NT) {
        S.acc[e] = 0.0;
        S.adj[e] = __ldcg(&P.adj[e]);
    }
    double r_dd = 0.0, r_dn = 0.0, r_dcon = 0.0;
    for (int tile = g; tile < P.ntiles; tile += P.G) {
        TileRange R = tile_range(P, tile);
        stage_tile_index(P, R, S);
        for (int i = threadIdx.x; i < R.np; i += NT) S.dcon[i] = P.dcon[R.sb + i];
        for (int i = threadIdx.x; i < R.npath; i += NT) {
            S.px[i] = xk[R.p0 + i];
            S.pxp[i] = xp[R.p0 + i];
        }
        __syncthreads();
        // per path: dual_nonneg (kernels.py:215) and the slot -> path scatter
        for (int i = threadIdx.x; i < R.npath; i += NT) {
            double dold = P.dn[R.p0 + i] * f;
            double dnew = npmax0(dold - S.px[i]);
            P.dn[R.p0 + i] = dnew;
            double d = dnew - dold;
            r_dn += d * d;
            for (int l = S.poff[i]; l < S.poff[i + 1]; ++l) S.pidx[S.pos[l]] = (uint16_t)i;
        }
        // per commodity: S_c (model.py:297-302 order) and dual_demand (kernels.py:211)
        for (int cc = R.c0 + threadIdx.x; cc < R.c1; cc += NT) {
            int32_t lo = I.com_path_ptr[cc] - R.p0, hi = I.com_path_ptr[cc + 1] - R.p0;
            double total = 0.0;
            for (int i = lo; i < hi;) {
                int j = i + 32 < hi ? i + 32 : hi;
                double part = 0.0;
                for (int t = i; t < j; ++t) part += S.px[t];
                total += part;
                i = j;
            }
            double dold = P.dd[cc] * f;
            double dnew = npmax0(dold + (total - I.demand[cc]));
            P.dd[cc] = dnew;
            double d = dnew - dold;
            r_dd += d * d;
        }
        __syncthreads();
        // per slot: y_{k-1}, dual_consensus (kernels.py:72), T value (kernels.py:91)
        for (int sl = threadIdx.x; sl < R.np; sl += NT) {
            int i = S.pidx[sl];
            double dk = S.dcon[sl];
            double y = c.first ? S.pxp[i] : max0(S.pxp[i] + dk - S.adj[S.eid[sl]]);
            double dks = dk * f;
            double dnew = max0(dks + S.px[i] - y);
            P.dcon[R.sb + sl] = dnew;
            double d = dnew - dks;
            r_dcon += d * d;
            S.v[sl] = S.px[i] + dnew;
        }
        __syncthreads();
        reduce_runs(S, S.v, R.np, S.acc);
        __syncthreads();
    }
    for (int e = threadIdx.x; e < I.E; e += NT) P.partT[(size_t)g * I.E + e] = S.acc[e];
    double t;
    t = block_sum(r_dd, S.red);
    if (threadIdx.x == 0) P.res[g * 8 + 1] = t;
    t = block_sum(r_dcon, S.red);
    if (threadIdx.x == 0) P.res[g * 8 + 3] = t;
    t = block_sum(r_dn, S.red);
    if (threadIdx.x == 0) P.res[g * 8 + 4] = t;
}

// ------------------------------------------------------------------ edge phase

// Work item (group, slice): lanes = 32 edges of the group, sum CTA partials of
// the slice in CTA order; the last item of a group combines slices in order and
// applies kernels.py:212 (dual_capacity) and :94-96 (adjustment).
__device__ void edge_phase(const Params &P, const Ctrl &c, int g) {
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

// ------------------------------------------------------------------ sweep B

__device__ void sweep_B(const Params &P, const Ctrl &c, Smem &S, int g) {
    const InstView &I = P.I;
    const double *xk = c.cur ? P.x1 : P.x0;
    double *xn = c.cur ? P.x0 : P.x1;
    const double beta = c.beta;
    const int64_t alpha = c.alpha;
    for (int e = threadIdx.x; e < I.E; e += NT) {
        S.acc[e] = 0.0;
        S.adj[e] = __ldcg(&P.adj[e]);
    }
    double r_x = 0.0;
    int my = 0;
    for (int tile = g; tile < P.ntiles; tile += P.G) ++my;
    // reverse tile order: re-read first what sweep A wrote last (L2 reuse)
    for (int k = my - 1; k >= 0; --k) {
        int tile = g + k * P.G;
        TileRange R = tile_range(P, tile);
        stage_tile_index(P, R, S);
        for (int i = threadIdx.x; i < R.np; i += NT) S.dcon[i] = P.dcon[R.sb + i];
        for (int i = threadIdx.x; i < R.npath; i += NT) S.px[i] = xk[R.p0 + i];
        __syncthreads();
        // per path: y_k and K_p in path order (kernels.py:98-100, :110-119)
        for (int i = threadIdx.x; i < R.npath; i += NT) {
            double x = S.px[i];
            double acc = 0.0;
            for (int l = S.poff[i]; l < S.poff[i + 1]; ++l) {
                int sl = S.pos[l];
                double dk = S.dcon[sl];
                double y = max0(x + dk - S.adj[S.eid[sl]]);
                S.v[sl] = y;
                acc += y - dk;
            }
            int p = R.p0 + i;
            double dn = P.dn[p];
            double h = (double)(S.poff[i + 1] - S.poff[i]);
            if (x < dn) {
                S.pK[i] = acc + dn;
                S.pw[i] = 1.0 / (h + 1.0);
            } else {
                S.pK[i] = acc;
                S.pw[i] = 1.0 / h;
            }
        }
        __syncthreads();
        // per commodity: W, Q, root, rates (kernels.py:122-131, 176-195, 285-296)
        for (int cc = R.c0 + threadIdx.x; cc < R.c1; cc += NT) {
            int32_t lo = I.com_path_ptr[cc] - R.p0, hi = I.com_path_ptr[cc + 1] - R.p0;
            double ws = 0.0, qw = 0.0;
            for (int i = lo; i < hi; ++i) {
                ws += S.pw[i];
                qw += S.pw[i] * S.pK[i];
            }
            if (!(isfinite(ws) && isfinite(qw))) {
                atomicMin(&P.err[0], cc);
                continue;
            }
            double D = I.demand[cc], dd = P.dd[cc];
            double Sc = commodity_root(ws, qw, D - dd, beta, alpha);
            if (!isfinite(Sc)) atomicMin(&P.err[1], cc);
            if (P.root_sums) P.root_sums[cc] = Sc;
            double ct = commodity_term(Sc, D, dd, beta, alpha);
            for (int i = lo; i < hi; ++i) {
                double xv = S.pw[i] * (S.pK[i] + ct);
                xn[R.p0 + i] = xv;
                double d = xv - S.px[i];
                r_x += d * d;
            }
        }
        reduce_runs(S, S.v, R.np, S.acc);
        __syncthreads();
    }
    for (int e = threadIdx.x; e < I.E; e += NT) P.partL[(size_t)g * I.E + e] = S.acc[e];
    double t = block_sum(r_x, S.red);
    if (threadIdx.x == 0) P.res[g * 8 + 0] = t;
}

// Initial capacity-dual load: L(y_0) with y_0 = x_0[pair_path] (controller.py:118).
__device__ void sweep_L0(const Params &P, const Ctrl &c, Smem &S, int g) {
    const double *xk = c.cur ? P.x1 : P.x0;
    for (int e = threadIdx.x; e < P.I.E; e += NT) S.acc[e] = 0.0;
    for (int tile = g; tile < P.ntiles; tile += P.G) {
        TileRange R = tile_range(P, tile);
        stage_tile_index(P, R, S);
        for (int i = threadIdx.x; i < R.npath; i += NT) S.px[i] = xk[R.p0 + i];
        __syncthreads();
        for (int i = threadIdx.x; i < R.npath; i += NT)
            for (int l = S.poff[i]; l < S.poff[i + 1]; ++l) S.v[S.pos[l]] = S.px[i];
        __syncthreads();
        reduce_runs(S, S.v, R.np, S.acc);
        __syncthreads();
    }
    for (int e = threadIdx.x; e < P.I.E; e += NT) P.partL[(size_t)g * P.I.E + e] = S.acc[e];
}

// ------------------------------------------------------------------ kernels

__global__ void __launch_bounds__(NT, 1) k_fused(Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem S = carve(smem_raw, P.I.E);
    cg::grid_group grid = cg::this_grid();
    const int g = blockIdx.x;
    Ctrl c = *P.ctrl;
    for (;;) {
        if (c.iteration > c.evaluated) controller_eval(P, c, S.red);
        if (c.stopped || c.status || c.iteration >= c.target || c.iteration >= P.max_iterations) break;
        c.alpha_used = c.alpha;
        c.beta_used = c.beta;
        sweep_A(P, c, S, g);
        grid.sync();
        edge_phase(P, c, g);
        grid.sync();
        sweep_B(P, c, S, g);
        c.f = 1.0;
        c.first = 0;
        c.cur ^= 1;
        c.iteration += 1;
        grid.sync();
    }
    if (g == 0 && threadIdx.x == 0) *P.ctrl = c;
}

__global__ void __launch_bounds__(NT, 1) k_init_L0(Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem S = carve(smem_raw, P.I.E);
    Ctrl c = *P.ctrl;
    for (int g = blockIdx.x; g < P.G; g += gridDim.x) sweep_L0(P, c, S, g);
}

// Export helpers: reference pair order <- slot order.
__global__ void k_export_pairs(Params P, const int32_t *pair_tile, double *y_out, double *dcon_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.I.NP) return;
    Ctrl c = *P.ctrl;
    int4 ti = P.tiles[pair_tile[t]];
    int sl = ti.z + P.pair_slot[t];
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
    std::vector<int4> tiles;
    int64_t slot = 0;
    int32_t c = 0;
    while (c < I.C) {
        int32_t c0 = c;
        int32_t p0 = cpp[c0];
        int32_t t0 = pptr[p0];
        while (c < I.C) {
            int32_t np_ = pptr[cpp[c + 1]] - t0;
            int32_t npath = cpp[c + 1] - p0;
            if (c > c0 && (np_ > TP || npath > TPATH)) break;
            require(np_ <= TP && npath <= TPATH,
                    "commodity " + std::to_string(c) + " has more pairs/paths than a fast-mode tile holds");
            ++c;
        }
        int32_t np_ = pptr[cpp[c]] - t0;
        tiles.push_back(make_int4(c0, c, (int)slot, np_));
        L->max_pairs = std::max(L->max_pairs, np_);
        L->max_paths = std::max(L->max_paths, cpp[c] - p0);
        slot += (np_ + SLOT_ALIGN - 1) / SLOT_ALIGN * SLOT_ALIGN;
    }
    require(slot < INT_MAX, "too many slots");
    L->ntiles = (int32_t)tiles.size();
    L->nslots = slot;
    std::vector<uint16_t> pair_slot(I.NP), slot_eid(slot ? slot : 1, (uint16_t)0xFFFF);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t ti = 0; ti < (int64_t)tiles.size(); ++ti) {
        int4 T = tiles[ti];
        int32_t t0 = pptr[cpp[T.x]];
        std::vector<int32_t> ord(T.w);
        for (int32_t l = 0; l < T.w; ++l) ord[l] = l;
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return pedge[t0 + a] < pedge[t0 + b]; });
        for (int32_t sl = 0; sl < T.w; ++sl) {
            pair_slot[t0 + ord[sl]] = (uint16_t)sl;
            slot_eid[T.z + sl] = (uint16_t)pedge[t0 + ord[sl]];
        }
    }
    L->tiles.alloc(tiles.size() ? tiles.size() : 1);
    L->pair_slot.alloc(I.NP ? I.NP : 1);
    L->slot_eid.alloc(slot ? slot : 1);
    h2d(L->tiles.p, tiles.data(), tiles.size(), s);
    h2d(L->pair_slot.p, pair_slot.data(), I.NP, s);
    h2d(L->slot_eid.p, slot_eid.data(), slot, s);
    PF_CUDA(cudaStreamSynchronize(s));
    L->h_tiles = std::move(tiles);
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
    DevBuf<int32_t> pair_tile;  // export only
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
    P.tiles = F->L->tiles.p;
    P.pair_slot = F->L->pair_slot.p;
    P.slot_eid = F->L->slot_eid.p;
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
    if (!F->pair_tile.p && I.NP) {
        std::vector<int32_t> pt(I.NP);
        std::vector<int32_t> cpp(I.C + 1), pptr(I.P + 1);
        d2h(cpp.data(), I.com_path_ptr.p, I.C + 1, s);
        d2h(pptr.data(), I.pair_ptr.p, I.P + 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        for (int32_t ti = 0; ti < F->L->ntiles; ++ti) {
            int4 T = F->L->h_tiles[ti];
            int32_t t0 = pptr[cpp[T.x]];
            for (int32_t l = 0; l < T.w; ++l) pt[t0 + l] = ti;
        }
        F->pair_tile.alloc(I.NP);
        h2d(F->pair_tile.p, pt.data(), I.NP, s);
    }
    DevBuf<double> dy(I.NP ? I.NP : 1), ddc(I.NP ? I.NP : 1), tmp(std::max<int64_t>({I.C, I.E, I.P, 1}));
    if (I.NP) k_export_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(F->P, F->pair_tile.p, dy.p, ddc.p);
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
    //  per slot: dcon r/w in A (16) + r in B (8) + slot_eid A,B (4) + pair_slot A,B (4)
    //  per path: x_k (A,B 16) + x_{k-1} (A 8) + x_{k+1} write (8) + dn r/w A + r B (24) + pair_ptr (8)
    //  per commodity: dd r/w + r (24) + demand (16) + com_path_ptr (8)
    if (bytes) *bytes = 32 * I.NP + 64 * I.P + 48 * I.C + (int64_t)F->G * I.E * 16;
}

}  // namespace pf
