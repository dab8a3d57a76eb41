// Fast mode: the GATE iteration (controller.py:225-273 with kernels.py's five
// steps) as ONE persistent, grid-synchronised kernel per run of iterations.
//
// Layout (TileLayout, built once per instance):
//   Commodities are cut into TILES of <= TP consecutive pairs (commodity-major,
//   the reference's own pair order).  Inside a tile the pairs are stored in
//   SLOTS sorted by edge id (stable), so every edge's pairs form one contiguous
//   run per tile.  Per slot: `slot_eid` (u16); per tile-local pair (path-major,
//   stored at the tile's slot base): `pos` (u16 slot of that pair).  Tiles start
//   on a 64-slot boundary.  The only per-pair STATE is dual_consensus (fp64, slot
//   order, double buffered); y is never stored.
//
// One pass per iteration.  Iteration k+1 of the reference is
//   A(k+1): duals_{k+1} from (x_k, y_k, duals_k * f_k)        kernels.py:206-216
//   E(k+1): dual_capacity_{k+1}, adjustment_{k+1} per edge    kernels.py:88-96, 212
//   B(k+1): y_{k+1}, coefficients, sum roots, x_{k+1}         kernels.py:235-296
// and the pass M(k+1) fuses B(k+1) with A(k+2): y_{k+1} and x_{k+1} never leave
// shared memory before they are consumed by the next dual update, so each pair
// costs one fp64 read + one fp64 write of dual_consensus per iteration (~20 B
// with its two u16 indices).  A(k+2) needs the rescale factor f_{k+1} of the
// controller step that follows B(k+1) (controller.py:251-266); the pass
// speculates f = 1 (certain during the post-change cooldown and when adapt is
// off) and a ROLLBACK pass recomputes A(k+2) from the still-intact duals_{k+1}
// buffers on the rare iterations where beta changes.
//
// Per iteration: M pass -> grid barrier -> controller (every CTA evaluates the
// same scalar logic from the residual partials) [-> rollback pass -> barrier]
// -> edge phase -> barrier.  Edge sums are reduced deterministically: a block
// segmented scan over each tile's edge runs into CTA-private shared-memory
// accumulators, then CTA partials in a fixed order.  The association differs
// from the reference's sequential per-edge sums, so fast mode is
// tolerance-matched (PF_MODE_EXACT is the bitwise path).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "fused.cuh"

namespace cg = cooperative_groups;

namespace pf {

constexpr int NT = 256;        // threads per CTA (3 CTAs per SM)
constexpr int TP = 1024;       // max pairs (slots) per tile
constexpr int ITEMS = TP / NT; // slots per thread in the segmented scan
constexpr int TPATH = 256;     // max paths per tile (u8 local path index)
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
    DevBuf<uint8_t> spath;      // [nslots] tile-local path index of each slot
    DevBuf<uint16_t> pair_slot; // [NP] tile-local slot of pair t (export only)
    DevBuf<int32_t> pair_tile;  // [NP] tile of pair t (export only)
    std::vector<TileDesc> h_desc;
    int32_t max_pairs = 0, max_paths = 0;
};

struct Ctrl {
    double beta, beta_used, ema_s, ema_r, f, s, r;
    int64_t alpha, alpha_used, iteration, cooldown, target;
    int32_t just_incremented, stopped, status, xc, db, need_a1, need_edge, pad;
    int64_t bad;
};

struct Params {
    InstView I;
    int32_t ntiles, G, nslices, pad;
    const TileDesc *desc;
    const uint16_t *slot_eid, *pos;
    const uint8_t *spath;
    double *dcon[2], *dn[2], *dd[2], *x[2];
    double *dc, *adj;
    const double *ne;       // [E] paths per edge (global across ranks when sharded)
    double *tot;            // [2E + 16] rank totals (multi-GPU): T, L, residual sums, error counts
    double *partT, *partL;  // [G][E]
    double *sub;            // [2][nslices][E]
    double *res;            // [G][8]: 0 dx | 1..3 (dd, dcon, dn) parity 0 | 4..6 parity 1
    double *res_dc;         // [ngroups]
    int32_t *grp_count;     // [ngroups]
    double *root_sums;      // [C] or null
    Ctrl *ctrl;
    int32_t *err;           // [2]: bad_coef, bad_root (INT_MAX = none)
    double gamma, residual_ratio, beta_scale, beta_min, beta_max;
    int64_t alpha_target, max_iterations;
    int32_t adapt;
};

// ------------------------------------------------------------------ shared memory

struct Stage {
    TileDesc d;
    double dcon[TP];  // duals_k dual_consensus; reused for the T values
    double xk[TPATH], xo[TPATH], dn[TPATH];
    double D[TCOM], dd[TCOM];
    uint16_t eid[TP], pos[TP];
    uint8_t spath[TP];        // tile-local path of each slot
    int32_t poff[TPATH + 4];  // raw pair_ptr[p0 .. p1]
    int32_t cpp[TCOM + 4];    // raw com_path_ptr[c0 .. c1]
};

struct Work {
    double y[TP];
    double pK[TPATH], pw[TPATH], xn[TPATH];
    double ct[TCOM];
    uint8_t pcom[TPATH];
    double wv1[NT / 32], wv2[NT / 32];
    int32_t wflag[NT / 32];
    double red[NT / 32];
};

struct Smem {
    Stage *st;
    Work *w;
    double *accT, *accL, *adj;
};

__device__ __forceinline__ Smem carve(char *base, int E) {
    Smem s;
    char *p = base;
    s.st = (Stage *)p;
    p += sizeof(Stage);
    s.w = (Work *)p;
    p += sizeof(Work);
    s.accT = (double *)p;
    p += sizeof(double) * E;
    s.accL = (double *)p;
    p += sizeof(double) * E;
    s.adj = (double *)p;
    return s;
}

static size_t smem_bytes(int E) { return sizeof(Stage) + sizeof(Work) + 3 * sizeof(double) * (size_t)E; }

// ------------------------------------------------------------------ cp.async staging

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
__device__ __forceinline__ void cp_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

enum { MODE_M = 0, MODE_RB = 1, MODE_A1 = 2 };

// Buffers a pass reads/writes (selected from the controller state).
struct PassIO {
    const double *dcon_in, *dn_in, *dd_in, *xk, *xo;
    double *dcon_out, *dn_out, *dd_out, *x_out;
    double f;
    int par;  // residual parity of the A-part iteration
};

// Issue the copies of one tile's inputs, then wait (other CTAs on the SM overlap).
template <int MODE>
__device__ __forceinline__ void stage_tile(const Params &P, const TileDesc &d, Stage &st, const PassIO &io) {
    const int tid = threadIdx.x;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    for (int i = tid; i < (np + 1) / 2; i += NT) cp16(&st.dcon[2 * i], &io.dcon_in[d.sb + 2 * i]);
    for (int i = tid; i < (np + 7) / 8; i += NT) {
        cp16(&st.eid[8 * i], &P.slot_eid[d.sb + 8 * i]);
        cp16(&st.pos[8 * i], &P.pos[d.sb + 8 * i]);
    }
    for (int i = tid; i < (np + 15) / 16; i += NT) cp16(&st.spath[16 * i], &P.spath[d.sb + 16 * i]);
    for (int i = tid; i < npath; i += NT) {
        cp8(&st.xk[i], &io.xk[d.p0 + i]);
        if (MODE == MODE_RB) cp8(&st.xo[i], &io.xo[d.p0 + i]);
        cp8(&st.dn[i], &io.dn_in[d.p0 + i]);
    }
    for (int i = tid; i <= npath; i += NT) cp4(&st.poff[i], &P.I.pair_ptr[d.p0 + i]);
    for (int i = tid; i <= nc; i += NT) cp4(&st.cpp[i], &P.I.com_path_ptr[d.c0 + i]);
    for (int i = tid; i < nc; i += NT) {
        cp8(&st.D[i], &P.I.demand[d.c0 + i]);
        cp8(&st.dd[i], &io.dd_in[d.c0 + i]);
    }
    cp_commit_wait_all();
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

// Segmented-sum operator on (head flag, value pair): (f1,a1) (+) (f2,a2).
__device__ __forceinline__ void seg_op2(int f1, double a1, double b1, int &f2, double &a2, double &b2) {
    if (!f2) {
        a2 = a1 + a2;
        b2 = b1 + b2;
    }
    f2 |= f1;
}

// Block-wide segmented inclusive scan over the tile's slots (ITEMS consecutive
// slots per thread) keyed by edge id, for two value streams at once.  The value
// at the last slot of each edge run is that run's total; the thread owning it
// adds it to acc[eid] (one run per edge per tile: no write conflicts).  Fixed
// operator tree, so the result is deterministic.
template <bool TWO>
__device__ void seg_reduce_runs(const double *v1, const double *v2, const uint16_t *eid, int np, double *acc1,
                                double *acc2, Work &W) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = ITEMS * tid;
    int key[ITEMS + 1];
    double a[ITEMS], b[ITEMS];
    int h[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        int sl = base + i;
        bool ok = sl < np;
        key[i] = ok ? (int)eid[sl] : -1 - i;
        a[i] = ok ? v1[sl] : 0.0;
        b[i] = (TWO && ok) ? v2[sl] : 0.0;
    }
    key[ITEMS] = base + ITEMS < np ? (int)eid[base + ITEMS] : -100;
    const int kprev = (base > 0 && base - 1 < np) ? (int)eid[base - 1] : -200;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) h[i] = (i == 0 ? key[0] != kprev : key[i] != key[i - 1]);
    int f = h[0];
    double x = a[0], z = b[0];
#pragma unroll
    for (int i = 1; i < ITEMS; ++i) {
        int fi = h[i];
        double xi = a[i], zi = b[i];
        seg_op2(f, x, z, fi, xi, zi);
        f = fi;
        x = xi;
        z = zi;
    }
    for (int o = 1; o < 32; o <<= 1) {
        int fo = __shfl_up_sync(0xffffffffu, f, o);
        double xo = __shfl_up_sync(0xffffffffu, x, o);
        double zo = TWO ? __shfl_up_sync(0xffffffffu, z, o) : 0.0;
        if (lane >= o) seg_op2(fo, xo, zo, f, x, z);
    }
    if (lane == 31) {
        W.wflag[warp] = f;
        W.wv1[warp] = x;
        W.wv2[warp] = z;
    }
    int fe = __shfl_up_sync(0xffffffffu, f, 1);
    double xe = __shfl_up_sync(0xffffffffu, x, 1);
    double ze = TWO ? __shfl_up_sync(0xffffffffu, z, 1) : 0.0;
    if (lane == 0) {
        fe = 0;
        xe = 0.0;
        ze = 0.0;
    }
    __syncthreads();
    if (warp == 0) {
        const bool in = lane < NT / 32;
        int wf = in ? W.wflag[lane] : 0;
        double wx = in ? W.wv1[lane] : 0.0, wz = in ? W.wv2[lane] : 0.0;
        for (int o = 1; o < NT / 32; o <<= 1) {
            int fo = __shfl_up_sync(0xffffffffu, wf, o);
            double xo = __shfl_up_sync(0xffffffffu, wx, o);
            double zo = __shfl_up_sync(0xffffffffu, wz, o);
            if (lane >= o) seg_op2(fo, xo, zo, wf, wx, wz);
        }
        int pf_ = __shfl_up_sync(0xffffffffu, wf, 1);
        double px = __shfl_up_sync(0xffffffffu, wx, 1);
        double pz = __shfl_up_sync(0xffffffffu, wz, 1);
        if (in) {
            W.wflag[lane] = lane ? pf_ : 0;
            W.wv1[lane] = lane ? px : 0.0;
            W.wv2[lane] = lane ? pz : 0.0;
        }
    }
    __syncthreads();
    int fp = fe;
    double xr = xe, zr = ze;
    seg_op2(W.wflag[warp], W.wv1[warp], W.wv2[warp], fp, xr, zr);  // exclusive prefix of this thread
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        int fi = h[i];
        double xi = a[i], zi = b[i];
        seg_op2(fp, xr, zr, fi, xi, zi);
        fp = fi;
        xr = xi;
        zr = zi;
        if (base + i < np && key[i + 1] != key[i]) {
            acc1[key[i]] += xi;
            if (TWO) acc2[key[i]] += zi;
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ controller

// controller.py:237-273 on the residuals of the iteration just completed.
__device__ __noinline__ void controller_step(const Params &P, Ctrl &c, double s, double r, int32_t ec, int32_t er) {
    c.s = s;
    c.r = r;
    c.f = 1.0;
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

// Every CTA reduces the residual partials in the same fixed order and runs the
// same scalar controller step on its shared-memory copy of the state.
__device__ void controller_eval(const Params &P, Ctrl &c) {
    if (threadIdx.x < 32) {
        const int par = (int)(c.iteration & 1);
        double acc[4] = {0, 0, 0, 0};  // dx, dd, dcon, dn
        for (int g = threadIdx.x; g < P.G; g += 32) {
            const double *r = P.res + g * 8;
            acc[0] += __ldcg(&r[0]);
            acc[1] += __ldcg(&r[1 + 3 * par]);
            acc[2] += __ldcg(&r[2 + 3 * par]);
            acc[3] += __ldcg(&r[3 + 3 * par]);
        }
        double dcs = 0.0;
        int ngroups = (P.I.E + RGRP - 1) / RGRP;
        for (int g = threadIdx.x; g < ngroups; g += 32) dcs += __ldcg(&P.res_dc[g]);
        for (int j = 0; j < 4; ++j)
            for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_down_sync(0xffffffffu, acc[j], o);
        for (int o = 16; o > 0; o >>= 1) dcs += __shfl_down_sync(0xffffffffu, dcs, o);
        if (threadIdx.x == 0)
            controller_step(P, c, sqrt(acc[0]), sqrt(((acc[1] + dcs) + acc[2]) + acc[3]), __ldcg(&P.err[0]),
                            __ldcg(&P.err[1]));
    }
    __syncthreads();
}

// ------------------------------------------------------------------ edge phase

// Work item (group, slice): lanes = 32 edges of the group, sum the CTA partials
// of the slice in CTA order; the last item of a group combines the slices in
// order and applies kernels.py:212 (dual_capacity) and :94-96 (adjustment).
__device__ __noinline__ void edge_phase(const Params &P, double f) {
    const InstView &I = P.I;
    const int g = blockIdx.x;
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
                double dold = __ldcg(&P.dc[e]) * f;
                double dnew = npmax0(dold + (L - cap));
                double adj = (T + dnew - cap) / (P.ne[e] + 1.0);
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

// ------------------------------------------------------------------ tile compute

// MODE_M : B(k+1) [y, K/w, roots, x_{k+1}] fused with A(k+2) [duals_{k+2}, T/L]
// MODE_RB: A(k+2) only, recomputing y_{k+1} from x_k, dcon_{k+1}, adj_{k+1}
// MODE_A1: A(1) with y_0 = x_0[pair_path] (controller.py:118)
// Every phase is parallel over slots or paths; only the sum-root runs one thread
// per commodity.
template <int MODE>
__device__ __forceinline__ void tile_compute(const Params &P, const Ctrl &c, const PassIO &io, Smem &S, double &r_x,
                                             double &r_dd, double &r_dcon, double &r_dn) {
    Stage &st = *S.st;
    Work &W = *S.w;
    const TileDesc &d = st.d;
    const int tid = threadIdx.x;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    const double f = io.f;
    // (1) slots: y (kernels.py:98-100) and y - dcon (kernels.py:114); path -> commodity map
    for (int sl = tid; sl < np; sl += NT) {
        const int i = st.spath[sl];
        const double dk = st.dcon[sl];
        double y;
        if (MODE == MODE_A1)
            y = st.xk[i];
        else
            y = max0((MODE == MODE_RB ? st.xo[i] : st.xk[i]) + dk - S.adj[st.eid[sl]]);
        W.y[sl] = y;
    }
    if (MODE == MODE_M)
        for (int j = tid; j < nc; j += NT)
            for (int i = st.cpp[j] - d.p0; i < st.cpp[j + 1] - d.p0; ++i) W.pcom[i] = (uint8_t)j;
    __syncthreads();
    if (MODE == MODE_M) {
        // (2) paths: K_p in path order, frozen non-negativity activity (kernels.py:110-119)
        for (int i = tid; i < npath; i += NT) {
            const int lo = st.poff[i] - d.t0, hi = st.poff[i + 1] - d.t0;
            double acc = 0.0;
            for (int l = lo; l < hi; ++l) {
                const int sl = st.pos[l];
                acc += W.y[sl] - st.dcon[sl];
            }
            const double x = st.xk[i], dn = st.dn[i];
            const double h = (double)(hi - lo);
            if (x < dn) {
                W.pK[i] = acc + dn;
                W.pw[i] = 1.0 / (h + 1.0);
            } else {
                W.pK[i] = acc;
                W.pw[i] = 1.0 / h;
            }
        }
        __syncthreads();
        // (3) commodities: W, Q (kernels.py:122-131), sum root (kernels.py:176-189), rate term (:289-294)
        for (int j = tid; j < nc; j += NT) {
            const int lo = st.cpp[j] - d.p0, hi = st.cpp[j + 1] - d.p0;
            const int cc = d.c0 + j;
            double ws = 0.0, qw = 0.0;
            for (int i = lo; i < hi; ++i) {
                ws += W.pw[i];
                qw += W.pw[i] * W.pK[i];
            }
            double ct = NAN;
            if (!(isfinite(ws) && isfinite(qw))) {
                atomicMin(&P.err[0], cc);
            } else {
                const double D = st.D[j], ddk = st.dd[j];
                const double Sc = commodity_root(ws, qw, D - ddk, c.beta, c.alpha);
                if (!isfinite(Sc)) atomicMin(&P.err[1], cc);
                if (P.root_sums) P.root_sums[cc] = Sc;
                ct = commodity_term(Sc, D, ddk, c.beta, c.alpha);
            }
            W.ct[j] = ct;
        }
        __syncthreads();
    }
    // (4) paths: new rate (kernels.py:195) and dual_nonneg (kernels.py:215)
    for (int i = tid; i < npath; i += NT) {
        double xv;
        if (MODE == MODE_M) {
            xv = W.pw[i] * (W.pK[i] + W.ct[W.pcom[i]]);
            io.x_out[d.p0 + i] = xv;
            const double df = xv - st.xk[i];
            r_x += df * df;
        } else {
            xv = st.xk[i];
        }
        W.xn[i] = xv;
        const double o = st.dn[i] * f;
        const double n = npmax0(o - xv);
        io.dn_out[d.p0 + i] = n;
        const double dg = n - o;
        r_dn += dg * dg;
    }
    __syncthreads();
    // (5) slots: dual_consensus (kernels.py:72), T value x + dcon' (kernels.py:91);
    //     commodities: S_c in model.py:297-302 order and dual_demand (kernels.py:211)
    for (int sl = tid; sl < np; sl += NT) {
        const double dks = st.dcon[sl] * f;
        const double xn = W.xn[st.spath[sl]];
        const double dnew = max0(dks + xn - W.y[sl]);
        io.dcon_out[d.sb + sl] = dnew;
        const double df = dnew - dks;
        r_dcon += df * df;
        st.dcon[sl] = xn + dnew;
    }
    for (int j = tid; j < nc; j += NT) {
        const int lo = st.cpp[j] - d.p0, hi = st.cpp[j + 1] - d.p0;
        double total = 0.0;
        for (int i = lo; i < hi;) {
            const int k2 = i + 32 < hi ? i + 32 : hi;
            double part = 0.0;
            for (int t = i; t < k2; ++t) part += W.xn[t];
            total += part;
            i = k2;
        }
        const double dold = st.dd[j] * f;
        const double dnew = npmax0(dold + (total - st.D[j]));
        io.dd_out[d.c0 + j] = dnew;
        const double df = dnew - dold;
        r_dd += df * df;
    }
    __syncthreads();
    if (MODE == MODE_RB)
        seg_reduce_runs<false>(st.dcon, nullptr, st.eid, np, S.accT, nullptr, W);
    else
        seg_reduce_runs<true>(st.dcon, W.y, st.eid, np, S.accT, S.accL, W);
}

template <int MODE>
__device__ PassIO pass_io(const Params &P, const Ctrl &c) {
    PassIO io;
    if (MODE == MODE_M) {  // reads duals_{k+1} (db), x_k (xc); writes the other buffers
        io.dcon_in = P.dcon[c.db];
        io.dn_in = P.dn[c.db];
        io.dd_in = P.dd[c.db];
        io.xk = P.x[c.xc];
        io.xo = nullptr;
        io.dcon_out = P.dcon[c.db ^ 1];
        io.dn_out = P.dn[c.db ^ 1];
        io.dd_out = P.dd[c.db ^ 1];
        io.x_out = P.x[c.xc ^ 1];
        io.f = 1.0;  // speculative f_{k+1}
        io.par = (int)((c.iteration + 2) & 1);
    } else if (MODE == MODE_RB) {  // after the M pass flipped xc/db: duals_{k+1} in db^1, x_{k+1} in xc
        io.dcon_in = P.dcon[c.db ^ 1];
        io.dn_in = P.dn[c.db ^ 1];
        io.dd_in = P.dd[c.db ^ 1];
        io.xk = P.x[c.xc];
        io.xo = P.x[c.xc ^ 1];
        io.dcon_out = P.dcon[c.db];
        io.dn_out = P.dn[c.db];
        io.dd_out = P.dd[c.db];
        io.x_out = nullptr;
        io.f = c.f;
        io.par = (int)((c.iteration + 1) & 1);
    } else {  // A(1): duals_0 in db, x_0 in xc
        io.dcon_in = P.dcon[c.db];
        io.dn_in = P.dn[c.db];
        io.dd_in = P.dd[c.db];
        io.xk = P.x[c.xc];
        io.xo = nullptr;
        io.dcon_out = P.dcon[c.db ^ 1];
        io.dn_out = P.dn[c.db ^ 1];
        io.dd_out = P.dd[c.db ^ 1];
        io.x_out = nullptr;
        io.f = 1.0;
        io.par = 1;
    }
    return io;
}

// One pass over this CTA's tiles.  Odd iterations walk the tiles in reverse so a
// pass first re-reads what the previous pass wrote last (L2 reuse).
template <int MODE>
__device__ __noinline__ void pass_tiles(const Params &P, const Ctrl &c, Smem &S) {
    const int g = blockIdx.x;
    const int E = P.I.E;
    __shared__ PassIO io;  // kept in shared memory: frees ~20 registers per thread
    if (threadIdx.x == 0) io = pass_io<MODE>(P, c);
    for (int e = threadIdx.x; e < E; e += NT) {
        S.accT[e] = 0.0;
        S.accL[e] = 0.0;
        S.adj[e] = MODE == MODE_A1 ? 0.0 : __ldcg(&P.adj[e]);
    }
    const int my = g < P.ntiles ? (P.ntiles - 1 - g) / P.G + 1 : 0;
    const bool rev = (c.iteration & 1) != 0;
    double r_x = 0.0, r_dd = 0.0, r_dcon = 0.0, r_dn = 0.0;
    for (int k = 0; k < my; ++k) {
        const int tile = g + (rev ? my - 1 - k : k) * P.G;
        const TileDesc d = P.desc[tile];
        __syncthreads();  // previous tile finished with the stage buffer
        if (threadIdx.x == 0) S.st->d = d;
        stage_tile<MODE>(P, d, *S.st, io);
        __syncthreads();
        tile_compute<MODE>(P, c, io, S, r_x, r_dd, r_dcon, r_dn);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += NT) {
        P.partT[(size_t)g * E + e] = S.accT[e];
        if (MODE != MODE_RB) P.partL[(size_t)g * E + e] = S.accL[e];
    }
    double *r = P.res + g * 8;
    double t;
    if (MODE == MODE_M) {
        t = block_sum(r_x, S.w->red);
        if (threadIdx.x == 0) r[0] = t;
    }
    t = block_sum(r_dd, S.w->red);
    if (threadIdx.x == 0) r[1 + 3 * io.par] = t;
    t = block_sum(r_dcon, S.w->red);
    if (threadIdx.x == 0) r[2 + 3 * io.par] = t;
    t = block_sum(r_dn, S.w->red);
    if (threadIdx.x == 0) r[3 + 3 * io.par] = t;
}

// ------------------------------------------------------------------ kernels

__global__ void __launch_bounds__(NT, 3) k_fused(const __grid_constant__ Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ Ctrl c;
    Smem S = carve(smem_raw, P.I.E);
    cg::grid_group grid = cg::this_grid();
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    if (c.need_a1) {
        pass_tiles<MODE_A1>(P, c, S);
        grid.sync();
        if (threadIdx.x == 0) {
            c.need_a1 = 0;
            c.db ^= 1;
            c.need_edge = 1;
            c.f = 1.0;
        }
        __syncthreads();
    }
    for (;;) {
        // the pending edge phase belongs to the next iteration: run it only when
        // continuing, so a stopped / paused state keeps adj_k for export
        if (c.stopped || c.status || c.iteration >= c.target || c.iteration >= P.max_iterations) break;
        if (c.need_edge) {
            edge_phase(P, c.f);
            grid.sync();
            __syncthreads();
            if (threadIdx.x == 0) {
                c.need_edge = 0;
                c.f = 1.0;
            }
            __syncthreads();
        }
        pass_tiles<MODE_M>(P, c, S);
        grid.sync();
        __syncthreads();
        if (threadIdx.x == 0) {
            c.iteration += 1;
            c.alpha_used = c.alpha;
            c.beta_used = c.beta;
            c.xc ^= 1;
            c.db ^= 1;
        }
        __syncthreads();
        controller_eval(P, c);
        if (!c.stopped && !c.status && c.f != 1.0) {
            pass_tiles<MODE_RB>(P, c, S);
            grid.sync();
        }
        __syncthreads();
        if (threadIdx.x == 0) c.need_edge = 1;
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.ctrl = c;
}

// ------------------------------------------------------------------ multi-GPU split kernels
//
// With a communicator attached (one process per GPU, commodities sharded), the
// iteration runs as separate launches around ONE ncclAllReduce of
// [T_e, L_e, residual sums] (2E + 16 doubles) per iteration (a second one only
// on the rare rollback iterations):
//   k_pass<M> -> k_local_reduce -> allreduce -> k_ctrl_dist -> [k_pass<RB> ->
//   k_local_reduce -> allreduce] -> k_edge_dist (next iteration) -> ...
// Every rank evaluates the same controller on the same totals, so all ranks take
// the same branch and issue matching collectives.

template <int MODE>
__global__ void __launch_bounds__(NT, 3) k_pass(const __grid_constant__ Params P) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ Ctrl c;
    Smem S = carve(smem_raw, P.I.E);
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    pass_tiles<MODE>(P, c, S);
}

// CTA partials -> rank totals in a fixed order: tot[0:E] = T, tot[E:2E] = L,
// tot[2E + 0..6] = residual slots summed over CTAs, tot[2E + 7/8] = error flags.
__global__ void k_local_reduce(const __grid_constant__ Params P) {
    const int E = P.I.E;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        double t = 0.0, l = 0.0;
        for (int g = 0; g < P.G; ++g) {
            t += __ldcg(&P.partT[(size_t)g * E + e]);
            l += __ldcg(&P.partL[(size_t)g * E + e]);
        }
        P.tot[e] = t;
        P.tot[E + e] = l;
    }
    if (blockIdx.x == 0 && threadIdx.x < 7) {
        double r = 0.0;
        for (int g = 0; g < P.G; ++g) r += __ldcg(&P.res[g * 8 + threadIdx.x]);
        P.tot[2 * E + threadIdx.x] = r;
    }
    if (blockIdx.x == 0 && threadIdx.x == 7) {
        P.tot[2 * E + 7] = __ldcg(&P.err[0]) != INT_MAX ? 1.0 : 0.0;
        P.tot[2 * E + 8] = __ldcg(&P.err[1]) != INT_MAX ? 1.0 : 0.0;
    }
}

// controller step from the allreduced totals (one thread)
__global__ void k_ctrl_dist(const __grid_constant__ Params P) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Ctrl c = *P.ctrl;
    c.iteration += 1;
    c.alpha_used = c.alpha;
    c.beta_used = c.beta;
    c.xc ^= 1;
    c.db ^= 1;
    const int E = P.I.E;
    const int par = (int)(c.iteration & 1);
    const double *t = P.tot + 2 * E;
    double dcs = 0.0;  // dual_capacity is replicated: its residual is rank-local and identical
    const int ngroups = (E + RGRP - 1) / RGRP;
    for (int g = 0; g < ngroups; ++g) dcs += P.res_dc[g];
    const int32_t ec = t[7] > 0.0 ? (P.err[0] != INT_MAX ? P.err[0] : -1) : INT_MAX;
    const int32_t er = t[8] > 0.0 ? (P.err[1] != INT_MAX ? P.err[1] : -1) : INT_MAX;
    controller_step(P, c, sqrt(t[0]), sqrt(((t[1 + 3 * par] + dcs) + t[2 + 3 * par]) + t[3 + 3 * par]), ec, er);
    c.need_edge = 1;
    *P.ctrl = c;
}

// kernels.py:212 and :94-96 from the allreduced per-edge totals (one warp per 32 edges)
__global__ void k_edge_dist(const __grid_constant__ Params P) {
    const int E = P.I.E;
    const int grp = blockIdx.x;
    const int e = grp * RGRP + threadIdx.x;
    const double f = P.ctrl->f;
    double rdc = 0.0;
    if (e < E) {
        const double T = P.tot[e], L = P.tot[E + e];
        const double cap = P.I.capacity[e];
        const double dold = P.dc[e] * f;
        const double dnew = npmax0(dold + (L - cap));
        double adj = (T + dnew - cap) / (P.ne[e] + 1.0);
        if (adj < 0.0) adj = 0.0;
        P.dc[e] = dnew;
        P.adj[e] = adj;
        const double d = dnew - dold;
        rdc = d * d;
    }
    for (int o = 16; o > 0; o >>= 1) rdc += __shfl_down_sync(0xffffffffu, rdc, o);
    if (threadIdx.x == 0) P.res_dc[grp] = rdc;
}

enum { CU_AFTER_A1 = 0, CU_AFTER_EDGE = 1 };
__global__ void k_ctrl_update(Ctrl *ctrl, int op) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (op == CU_AFTER_A1) {
        ctrl->need_a1 = 0;
        ctrl->db ^= 1;
        ctrl->need_edge = 1;
        ctrl->f = 1.0;
    } else {
        ctrl->need_edge = 0;
        ctrl->f = 1.0;
    }
}

// Export helpers (reference pair order <- slot order), for the state of the last
// completed iteration k: x_k in x[xc], x_{k-1} in x[xc^1], duals_k in buffer db^1
// (db holds the speculative duals_{k+1}), adj_k, rescale factor f_k pending.
__global__ void k_export_pairs(const __grid_constant__ Params P, const int32_t *pair_tile,
                               const uint16_t *pair_slot, double *y_out, double *dcon_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.I.NP) return;
    const Ctrl c = *P.ctrl;
    const TileDesc d = P.desc[pair_tile[t]];
    const int sl = d.sb + pair_slot[t];
    const int p = P.I.pair_path[t];
    if (c.iteration == 0) {
        if (y_out) y_out[t] = P.x[c.xc][p];
        if (dcon_out) dcon_out[t] = 0.0;
        return;
    }
    const double dk = P.dcon[c.db ^ 1][sl];
    if (y_out) y_out[t] = max0(P.x[c.xc ^ 1][p] + dk - P.adj[P.slot_eid[sl]]);
    if (dcon_out) dcon_out[t] = dk * c.f;
}

__global__ void k_scaled_copy(const double *a, int64_t n, const Ctrl *ctrl, double *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = ctrl->iteration == 0 ? a[i] : a[i] * ctrl->f;
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
    std::vector<uint8_t> spath(slot ? slot : 1, (uint8_t)0);
    std::vector<int32_t> pair_tile(I.NP);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t ti = 0; ti < (int64_t)tiles.size(); ++ti) {
        const TileDesc &T = tiles[ti];
        std::vector<int32_t> ord(T.np);
        for (int32_t l = 0; l < T.np; ++l) ord[l] = l;
        std::stable_sort(ord.begin(), ord.end(),
                         [&](int32_t a, int32_t b) { return pedge[T.t0 + a] < pedge[T.t0 + b]; });
        std::vector<uint8_t> lpath(T.np);
        for (int32_t p = T.p0; p < T.p1; ++p)
            for (int32_t t = pptr[p]; t < pptr[p + 1]; ++t) lpath[t - T.t0] = (uint8_t)(p - T.p0);
        for (int32_t sl = 0; sl < T.np; ++sl) {
            int32_t l = ord[sl];
            pair_slot[T.t0 + l] = (uint16_t)sl;
            pair_tile[T.t0 + l] = (int32_t)ti;
            slot_eid[T.sb + sl] = (uint16_t)pedge[T.t0 + l];
            pos[T.sb + l] = (uint16_t)sl;
            spath[T.sb + sl] = lpath[l];
        }
    }
    L->desc.alloc(tiles.size() ? tiles.size() : 1);
    L->slot_eid.alloc(slot ? slot : 1);
    L->pos.alloc(slot ? slot : 1);
    L->spath.alloc(slot ? slot : 1);
    L->pair_slot.alloc(I.NP ? I.NP : 1);
    L->pair_tile.alloc(I.NP ? I.NP : 1);
    h2d(L->desc.p, tiles.data(), tiles.size(), s);
    h2d(L->slot_eid.p, slot_eid.data(), slot, s);
    h2d(L->pos.p, pos.data(), slot, s);
    h2d(L->spath.p, spath.data(), slot, s);
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
    DevBuf<double> dcon[2], dn[2], dd[2], x[2];
    DevBuf<double> dc, adj, ne, tot, partT, partL, sub, res, res_dc, root_sums;
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
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_A1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
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
    for (int b = 0; b < 2; ++b) {
        F->dcon[b].alloc(F->L->nslots ? F->L->nslots : 1);
        F->dn[b].alloc(I.P ? I.P : 1);
        F->dd[b].alloc(I.C ? I.C : 1);
        F->x[b].alloc(I.P ? I.P : 1);
    }
    F->dc.alloc(E);
    F->adj.alloc(E);
    F->ne.alloc(E);
    F->tot.alloc(2 * E + 16);
    {
        std::vector<int32_t> cnt(I.E);
        std::vector<double> ned(E, 0.0);
        d2h(cnt.data(), I.edge_path_count.p, I.E, s);
        PF_CUDA(cudaStreamSynchronize(s));
        for (int64_t e = 0; e < I.E; ++e) ned[e] = (double)cnt[e];
        h2d(F->ne.p, ned.data(), E, s);
    }
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
    P.spath = F->L->spath.p;
    for (int b = 0; b < 2; ++b) {
        P.dcon[b] = F->dcon[b].p;
        P.dn[b] = F->dn[b].p;
        P.dd[b] = F->dd[b].p;
        P.x[b] = F->x[b].p;
    }
    P.dc = F->dc.p;
    P.adj = F->adj.p;
    P.ne = F->ne.p;
    P.tot = F->tot.p;
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

void fast_set_comm(FastSolver *F, const CommOps *ops) {
    F->comm = ops;
    if (!ops) return;
    // the suggestion divisor n_e + 1 counts paths of ALL ranks (kernels.py:94)
    cudaStream_t s = nullptr;
    PF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int64_t E = F->inst->idx->E;
    if (E) ops->allreduce_sum(ops->ctx, F->ne.p, E, s);
    PF_CUDA(cudaStreamSynchronize(s));
    PF_CUDA(cudaStreamDestroy(s));
}

// Host-driven iteration for sharded solves (see the split kernels above).
static int64_t fast_run_dist(FastSolver *F, int64_t max_steps, cudaStream_t s, float *ms) {
    const Index &I = *F->inst->idx;
    const int64_t E = I.E;
    const int nred = (int)std::max<int64_t>(1, (E + 255) / 256);
    const int ngroups = (int)((E + RGRP - 1) / RGRP);
    auto read = [&]() {
        Ctrl c;
        d2h(&c, F->ctrl.p, 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        return c;
    };
    auto reduce_allreduce = [&]() {
        k_local_reduce<<<nred, 256, 0, s>>>(F->P);
        PF_CHECK_LAUNCH();
        F->comm->allreduce_sum(F->comm->ctx, F->tot.p, 2 * E + 16, s);
    };
    Ctrl c = read();
    const int64_t start = c.iteration;
    if (I.P == 0 || max_steps <= 0 || c.stopped || c.status) {
        if (ms) *ms = 0.f;
        return 0;
    }
    const int64_t target = std::min<int64_t>(start + max_steps, F->cfg.max_iterations);
    PF_CUDA(cudaEventRecord(F->e0, s));
    if (c.need_a1) {
        k_pass<MODE_A1><<<F->G, NT, F->smem, s>>>(F->P);
        PF_CHECK_LAUNCH();
        reduce_allreduce();
        k_ctrl_update<<<1, 1, 0, s>>>(F->ctrl.p, CU_AFTER_A1);
        F->launches += 3;
        c = read();
    }
    while (!c.stopped && !c.status && c.iteration < target) {
        if (c.need_edge) {
            if (ngroups) k_edge_dist<<<ngroups, RGRP, 0, s>>>(F->P);
            k_ctrl_update<<<1, 1, 0, s>>>(F->ctrl.p, CU_AFTER_EDGE);
        }
        k_pass<MODE_M><<<F->G, NT, F->smem, s>>>(F->P);
        PF_CHECK_LAUNCH();
        reduce_allreduce();
        k_ctrl_dist<<<1, 32, 0, s>>>(F->P);
        PF_CHECK_LAUNCH();
        F->launches += 5;
        c = read();
        if (!c.stopped && !c.status && c.f != 1.0) {
            k_pass<MODE_RB><<<F->G, NT, F->smem, s>>>(F->P);
            PF_CHECK_LAUNCH();
            reduce_allreduce();
            F->launches += 2;
        }
    }
    PF_CUDA(cudaEventRecord(F->e1, s));
    PF_CUDA(cudaEventSynchronize(F->e1));
    float t = 0.f;
    PF_CUDA(cudaEventElapsedTime(&t, F->e0, F->e1));
    if (ms) *ms = t;
    c = read();
    return c.iteration - start;
}

void fast_init(FastSolver *F, const double *d_x0, int64_t alpha0, double beta0, cudaStream_t s) {
    const Index &I = *F->inst->idx;
    for (int b = 0; b < 2; ++b) {
        PF_CUDA(cudaMemcpyAsync(F->x[b].p, d_x0, sizeof(double) * I.P, cudaMemcpyDeviceToDevice, s));
        PF_CUDA(cudaMemsetAsync(F->dcon[b].p, 0, F->dcon[b].bytes(), s));
        PF_CUDA(cudaMemsetAsync(F->dn[b].p, 0, F->dn[b].bytes(), s));
        PF_CUDA(cudaMemsetAsync(F->dd[b].p, 0, F->dd[b].bytes(), s));
    }
    PF_CUDA(cudaMemsetAsync(F->dc.p, 0, F->dc.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->adj.p, 0, F->adj.bytes(), s));
    PF_CUDA(cudaMemsetAsync(F->partT.p, 0, F->partT.bytes(), s));
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
    c.s = c.r = NAN;
    c.bad = -1;
    c.xc = 0;
    c.db = 0;
    c.need_a1 = 1;
    c.need_edge = 0;
    h2d(F->ctrl.p, &c, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
}

int64_t fast_run(FastSolver *F, int64_t max_steps, cudaStream_t s, float *ms) {
    if (F->comm) return fast_run_dist(F, max_steps, s, ms);
    Ctrl c;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    int64_t start = c.iteration;
    if (F->inst->idx->P == 0 || max_steps <= 0 || c.stopped || c.status) {
        if (ms) *ms = 0.f;
        return 0;
    }
    int64_t target = start + max_steps;
    PF_CUDA(cudaMemcpyAsync((char *)F->ctrl.p + offsetof(Ctrl, target), &target, sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
    void *args[] = {(void *)&F->P};
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
    return F->x[c.xc].p;
}

const double *fast_root_sums(FastSolver *F) { return F->root_sums.p; }

void fast_export_state(FastSolver *F, double *x, double *y, double *dd, double *dc, double *dcon, double *dn,
                       cudaStream_t s) {
    const Index &I = *F->inst->idx;
    Ctrl c;
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    const int dcur = c.iteration == 0 ? c.db : (c.db ^ 1);
    DevBuf<double> dy(I.NP ? I.NP : 1), ddc(I.NP ? I.NP : 1), tmp(std::max<int64_t>({I.C, I.E, I.P, 1}));
    if (I.NP)
        k_export_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(F->P, F->L->pair_tile.p, F->L->pair_slot.p, dy.p,
                                                           ddc.p);
    PF_CHECK_LAUNCH();
    if (x) d2h(x, F->x[c.xc].p, I.P, s);
    if (y) d2h(y, dy.p, I.NP, s);
    if (dcon) d2h(dcon, ddc.p, I.NP, s);
    PF_CUDA(cudaStreamSynchronize(s));
    auto scaled = [&](const double *src, int64_t n, double *out) {
        if (!out || !n) return;
        k_scaled_copy<<<ceil_div(n, 256), 256, 0, s>>>(src, n, F->ctrl.p, tmp.p);
        PF_CHECK_LAUNCH();
        d2h(out, tmp.p, n, s);
        PF_CUDA(cudaStreamSynchronize(s));
    };
    scaled(F->dd[dcur].p, I.C, dd);
    scaled(F->dc.p, I.E, dc);
    scaled(F->dn[dcur].p, I.P, dn);
}

void fast_stats(FastSolver *F, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes) {
    const Index &I = *F->inst->idx;
    if (launches) *launches = F->launches;
    if (tiles) *tiles = F->L->ntiles;
    if (grid) *grid = F->G;
    // compulsory HBM bytes per iteration of this layout (one fused pass):
    //  per slot: dual_consensus read + write (16) + slot_eid (2) + pos (2) + spath (1)
    //  per path: x_k read + x_{k+1} write (16) + dual_nonneg read + write (16) + pair_ptr (4)
    //  per commodity: dual_demand read + write (16) + demand (8) + com_path_ptr (4)
    //  per CTA: edge partials T and L written and read back (4 x 8 B per edge)
    if (bytes) *bytes = 21 * F->L->nslots + 36 * I.P + 28 * I.C + (int64_t)F->G * I.E * 32;
}

}  // namespace pf
