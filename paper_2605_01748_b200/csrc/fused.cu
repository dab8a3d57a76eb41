// Fast mode: the GATE iteration (controller.py:225-273 with kernels.py's five
// steps) as ONE persistent, grid-synchronised kernel per run of iterations.
//
// Layout (TileLayout, built once per instance):
//   Commodities are packed into GROUPS of consecutive commodities holding at
//   most 32 paths (one lane per path), and groups into TILES of NW groups (one
//   warp per group) and at most `tps` demand-path pairs.  Dynamic per-pair state
//   (dual_consensus, double buffered) is stored in the reference's pair order
//   (path-major) with every tile starting on a 16-slot boundary, so a tile is
//   one contiguous, 128-byte aligned range.  The static per-tile metadata
//   (edge id per pair, tile-local path per pair, the pair permutation that sorts
//   the tile's pairs by edge, path / commodity / group offsets) is one
//   contiguous 16-byte aligned block.  y is never stored.
//
// Per tile: one elected thread issues TMA bulk copies (cp.async.bulk) of the
// tile's dual_consensus, metadata, rates, dual_nonneg, demand and dual_demand
// into a double-buffered shared-memory stage completing on an mbarrier, one
// tile ahead of the compute.  Each warp then runs its commodity group:
//   pairs (lanes over pairs):   y                               kernels.py:98-100
//   paths (lane = path):        K_p, frozen activity test, w    kernels.py:110-119
//   commodity (lane segments):  W, Q by segmented shuffles, sum
//                               root, rate term, x_{k+1}        kernels.py:122-195
//   pairs:                      dual_consensus, T = x + dcon'   kernels.py:72, :91
// and the CTA reduces the tile's per-edge T and L = sum y with a warp-level
// segmented scan over the edge-sorted permutation into CTA-private shared
// accumulators (one run per edge per tile, so no write conflicts).
//
// One pass per iteration.  Iteration k+1 of the reference is
//   A(k+1): duals_{k+1} from (x_k, y_k, duals_k * f_k)        kernels.py:206-216
//   E(k+1): dual_capacity_{k+1}, adjustment_{k+1} per edge    kernels.py:88-96, 212
//   B(k+1): y_{k+1}, coefficients, sum roots, x_{k+1}         kernels.py:235-296
// and the pass M(k+1) fuses B(k+1) with A(k+2): y_{k+1} and x_{k+1} never leave
// shared memory before they are consumed by the next dual update.  A(k+2) needs
// the rescale factor f_{k+1} of the controller step that follows B(k+1)
// (controller.py:251-266); the pass speculates f = 1 (certain during the
// post-change cooldown and when adapt is off) and a ROLLBACK pass recomputes
// A(k+2) from the still-intact duals_{k+1} buffers on the rare iterations where
// beta changes.
//
// Per iteration: M pass -> grid barrier -> controller (every CTA evaluates the
// same scalar logic from the residual partials) [-> rollback pass -> barrier]
// -> edge phase -> barrier.  Every reduction has a fixed association, so fast
// mode is deterministic run to run; the association differs from the
// reference's sequential per-edge sums, so it is tolerance-matched
// (PF_MODE_EXACT is the bitwise path).
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "fused.cuh"

namespace cg = cooperative_groups;

namespace pf {

#ifndef PF_NW
#define PF_NW 8
#endif
#ifndef PF_MINB
#define PF_MINB 2  // resident CTAs per SM the fused kernels are register-bounded for
#endif
constexpr int NW = PF_NW;         // warps per CTA = commodity groups per tile
constexpr int NT = 32 * NW;       // threads per CTA
constexpr int GPATH = 32;         // max paths per group (one lane per path)
constexpr int TPATH = NW * GPATH; // max paths per tile
constexpr int TCOM = TPATH;       // max commodities per tile
static_assert(TPATH <= 256, "tile-local path / commodity indices are u8");
static_assert(3 * 8 * (TPATH + 2) >= NT * 16, "the edge-run head pieces reuse the stage's per-path arrays");
constexpr int TPS_MIN = 2560;     // default max pairs per tile (large-E layouts)
constexpr int TPS_CAP = 4096;     // upper bound of the shared-memory fit (two CTAs per SM)
constexpr int SLOT_ALIGN = 16;    // tile start alignment in the per-pair arrays (128 B)
constexpr int RGRP = 32;          // edges per reduction group (one lane per edge)
constexpr unsigned FULL = 0xffffffffu;

struct TileDesc {
    int32_t c0, c1, p0, p1, t0, np, sb, mb16;  // mb16: metadata offset / 16
    int32_t nrun;                              // edge runs: distinct edges of the tile's pairs
    int32_t nhb;                               // entries of the hop-step table (sum over groups of hops + 1)
};

__host__ __device__ __forceinline__ int r16(int b) { return (b + 15) & ~15; }
__host__ __device__ __forceinline__ int even(int n) { return (n + 1) & ~1; }

// Byte offsets of the sections of one tile's metadata block.  With run slots
// (large-E layout) the per-pair u16 holds the pair's tile-local RUN (distinct
// edge of the tile, in edge order) instead of its edge id, and two per-run
// sections follow: the run's edge and its global slot (the edge-major position
// of this (tile, run) among all tiles that touch the edge).
struct MetaOff {
    int eid, sperm, poff, pcom, cpp, gpath, hbo, hb, hperm, hinv, xlen, redge, rdst, bytes;
};
__host__ __device__ __forceinline__ MetaOff meta_off(int np, int npath, int nc, int nrun, int nhb, bool rs = false) {
    MetaOff m;
    int o = 0;
    m.eid = o;  // u16 [np] edge id (run id with run slots) of each pair (hop-major within each group)
    o += r16(2 * np);
    m.sperm = o;  // u16 [np] tile-local pairs sorted by (edge, pair): the edge runs, back to back; bit 15 = run start
    o += r16(2 * np);
    m.poff = o;  // u16 [npath + 1] tile-local pair offset of each path
    o += r16(2 * (npath + 1));
    m.pcom = o;  // u8 [npath] tile-local commodity of each path
    o += r16(npath);
    m.cpp = o;  // u16 [nc + 1] tile-local path offset of each commodity
    o += r16(2 * (nc + 1));
    m.gpath = o;  // u16 [NW + 1] tile-local path offset of each group
    o += r16(2 * (NW + 1));
    // hop-major order: within a group the paths take the lanes by decreasing hop
    // count (hop lanes), so the lanes active at step j are a prefix 0 .. n_j - 1
    // and step j's pairs are hb[j] + lane, hb[j] .. hb[j + 1]
    m.hbo = o;  // u16 [NW + 1] each group's first entry in hb
    o += r16(2 * (NW + 1));
    m.hb = o;  // u16 [nhb] per group: the tile-local start of each hop step, then the group's end
    o += r16(2 * nhb);
    m.hperm = o;  // u8 [npath] per group: the path (group-relative) of each hop lane
    o += r16(npath);
    m.hinv = o;  // u8 [npath] per group: the hop lane of each path
    o += r16(npath);
    m.xlen = o;  // u16 [NT] per walk chunk: how many following chunks its tail's crossing run reaches (0: none)
    o += r16(2 * NT);
    m.redge = o;  // run slots: u16 [nrun] edge of each run
    if (rs) o += r16(2 * nrun);
    m.rdst = o;  // run slots: u32 [nrun] global slot of each run's {T, L}
    if (rs) o += r16(4 * nrun);
    m.bytes = o;
    return m;
}

// Dynamic shared memory: two stages + work arrays + the per-edge tables.
// Run slots (rs): no per-edge tables; a per-tile adjustment table of the
// tile's runs (at most rmax) instead.
struct SmemPlan {
    int stage, s_dcon, s_meta, s_xk, s_xo, s_dn, s_D, s_dd;  // offsets inside a stage
    int y, adj, acc, adjt, hp, total;                       // offsets from the base
};
__host__ __device__ __forceinline__ SmemPlan smem_plan(int tps, int E, int nbuf, int hbmax, bool adj_smem = true,
                                                      bool acc_smem = true, bool rs = false, int rmax = 0) {
    SmemPlan s;
    int o = 0;
    s.s_dcon = o;
    o += 8 * tps;
    s.s_meta = o;
    o += meta_off(tps, TPATH, TCOM, rs ? rmax : (tps < E ? tps : E), hbmax, rs).bytes;  // at most min(pairs, edges) runs
    s.s_xk = o;
    o += 8 * (TPATH + 2);
    s.s_xo = o;
    o += 8 * (TPATH + 2);
    s.s_dn = o;
    o += 8 * (TPATH + 2);
    s.s_D = o;
    o += 8 * (TCOM + 2);
    s.s_dd = o;
    o += 8 * (TCOM + 2);
    s.stage = r16(o);
    o = nbuf * s.stage;
    s.y = o;
    o += 8 * tps;
    s.adj = o;  // per-edge adjustment table (absent for large E: read through L1)
    if (adj_smem && !rs) o += r16(8 * E);
    s.acc = o;  // double2 {T, L} per edge (absent for large E: the CTA's partial rows in L2)
    if (acc_smem && !rs) o += r16(16 * E);
    s.adjt = o;  // run slots: adjustment of each of the tile's runs
    if (rs) o += r16(8 * rmax);
    s.hp = o;  // the edge-run walk's head pieces (outside the stage: the next tile's copy may start early)
    o += 16 * NT;
    s.total = o;
    return s;
}

struct TileLayout {
    int32_t ntiles = 0, tps = TPS_MIN, kspan = 1;
    bool adj_smem = true;  // false for large E: the adjustment table read through L1
    bool acc_smem = true;  // false for large E: run totals accumulate in the CTA's partial rows (L2)
    bool run_slots = false;  // per-(tile, run) totals in edge-major global slots (any E: no per-edge tables)
    int32_t rmax = 0;        // most runs in one tile
    int32_t hbmax = 0;       // hop-step table bound: NW * (most hops of a path + 1)
    int64_t nruns = 0;       // run slots: total (tile, run) slots
    DevBuf<int32_t> eoff;    // run slots: [E + 1] first slot of each edge
    int64_t nslots = 0, meta_bytes = 0;
    DevBuf<TileDesc> desc;      // per tile
    DevBuf<uint8_t> meta;       // per-tile metadata blocks
    DevBuf<int32_t> pair_slot;  // [NP] fast-layout slot of reference pair t (export only)
    std::vector<TileDesc> h_desc;
    int64_t bytes_per_pass = 0;  // compulsory HBM bytes of one M pass over the tiles
};

struct Ctrl {
    double beta, beta_used, ema_s, ema_r, f, s, r;
    int64_t alpha, alpha_used, iteration, cooldown, target;
    int32_t just_incremented, stopped, status, xc, db, need_a1, need_edge, pad;
    int64_t bad;
    uint64_t xepoch;  // multi-GPU exchanges done (mirrors *Params::xepoch)
    double fspec;     // the rescale factor the M pass speculated (predict_f); a rollback iff f != fspec
    double fnext;     // predict_f for the next M pass (set at the end of controller_step)
    int64_t rollbacks;  // rollback passes run (statistics)
};

struct Params {
    InstView I;
    // pad0 keeps the layout of the 8-byte fields below: k_fused's register
    // allocation (pass spills) measured sensitive to it
    int32_t ntiles, G, pad0, tps, nbuf, kspan;  // kspan: power of two >= max paths per commodity
    int32_t adj_smem;                               // adjustment table in shared memory (else L1)
    int32_t acc_smem;                               // edge accumulators in shared memory (else L2 rows)
    // multi-GPU over peer memory (CUDA IPC): rank-local totals are written into
    // slot [rank] of every rank's exchange buffer; nranks = 0 when single-GPU
    int32_t rank, nranks;
    int64_t xslot;                 // doubles per slot: T[E], L[E], 16 scalars
    double *const *peers;          // [nranks] exchange buffer bases (peers[rank] = own)
    unsigned long long *xepoch;    // exchanges done (device, never reset)
    int32_t pf_dist;                                // L2 prefetch distance in tiles (single stage)
    const TileDesc *desc;
    const int32_t *cta_ptr, *cta_tiles;  // CTA g walks tiles cta_tiles[cta_ptr[g] .. cta_ptr[g + 1])
    const uint8_t *meta;
    const double *D;  // [C + 2] demand (padded copy for 16-byte bulk copies)
    double *dcon[2], *dn[2], *dd[2], *x[2];
    double *dc, *adj;
    const double *ne;       // [E] paths per edge (global across ranks when sharded)
    double *tot;            // [2E + 16] rank totals (multi-GPU): T, L, residual sums, error counts
    double *partT, *partL;  // [E][G]: edge-major, so one edge's CTA partials are contiguous
    double *res;            // [G][8]: 0 dx | 1..3 (dd, dcon, dn) parity 0 | 4..6 parity 1
    double *res_dc;         // [2][E] squared dual_capacity change per edge (halves by iteration parity)
    double *root_sums;      // [C] or null
    Ctrl *ctrl;
    int32_t *err;           // [2]: bad_coef, bad_root (INT_MAX = none)
    double gamma, residual_ratio, beta_scale, beta_min, beta_max;
    int64_t alpha_target, max_iterations;
    int32_t adapt;
    int32_t probe;   // tuning only (PF_FAST_PROBE): iteration-phase times of CTA 0 into g_probe
    int32_t ablate;  // tuning only (PF_FAST_ABLATE): 1 skip y/paths/commodities/dcon, 2 skip the edge scan, 16 skip commodities, 32 skip K, 64 skip y
    // run slots (TileLayout::run_slots): every (tile, run) stores its {T, L} into
    // slots[2 * s], s in the edge's range eoff[e] .. eoff[e + 1] (tile order)
    int32_t run_slots, rmax;
    int32_t hbmax;        // most hop-step entries of one tile (the shared-memory metadata bound)
    int32_t spec_f;       // speculate the rescale factor (predict_f); 0: always f = 1 (PF_FAST_SPEC=0)
    double spec_margin;   // predict_f's margin past the residual-ratio threshold (PF_FAST_SPEC_MARGIN)
    const int32_t *eoff;
    const int32_t *ebound;  // run slots, single GPU: CTA g sums edges ebound[g] .. ebound[g + 1] (slot-balanced)
    double *slots;
};

// Iteration-phase probe (tuning only, PF_FAST_PROBE): %globaltimer deltas of
// CTA 0, thread 0, summed into g_probe[phase] (ns).
__device__ unsigned long long g_probe[8];
// first exchange whose slots carried the wrong epoch tag: {epoch + 1, rank, tag, iteration, counter}
__device__ unsigned long long g_xdebug[5];
// Tile-phase probe (tuning builds only, -DPF_TPROBE): clock64 deltas of thread 0
// of every CTA per tile phase, summed over tiles and CTAs into g_tprobe
// (0 TMA wait, 1 y, 2 K + commodities, 3 dcon + barrier, 4 edge runs, 5 end barrier, 7 tiles).
__device__ unsigned long long g_tprobe[8];
#ifdef PF_TPROBE
#define TP_DECL unsigned long long tp_last = 0;
#define TP(i)                                                        \
    if (threadIdx.x == 0) {                                          \
        const unsigned long long t_ = clock64();                     \
        if ((i) >= 0) atomicAdd(&g_tprobe[(i) < 0 ? 0 : (i)], t_ - tp_last); \
        tp_last = t_;                                                \
    }
#else
#define TP_DECL
#define TP(i)
#endif
__device__ unsigned long long g_pmax[3];  // per-phase max over CTAs (reset per launch read)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ TMA / mbarrier

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// explicit shared-space accesses: tables reached through pointers that may also
// point to global memory would otherwise compile to generic loads (LD.E), whose
// latency the per-pair loops pay on every element
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64x2(uint32_t a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
// order this thread's generic-proxy accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

enum { MODE_M = 0, MODE_RB = 1, MODE_A1 = 2 };

// Buffers a pass reads/writes (selected from the controller state).
struct PassIO {
    const double *dcon_in, *dn_in, *dd_in, *xk, *xo;
    double *dcon_out, *dn_out, *dd_out, *x_out;
    double f;
    int par;  // residual parity of the A-part iteration
};

// Stage pointers of one buffer.
struct StageView {
    int o_dcon, o_meta, o_xk;  // byte offsets from the dynamic shared-memory base
    const double *dcon;
    const uint8_t *meta;
    const double *xk, *xo, *dn, *D, *dd;  // already shifted to the tile's first path / commodity
};

__device__ __forceinline__ StageView stage_view(char *base, const SmemPlan &sp, int b, const TileDesc &d) {
    char *s = base + b * sp.stage;
    StageView v;
    v.o_dcon = b * sp.stage + sp.s_dcon;
    v.o_meta = b * sp.stage + sp.s_meta;
    v.o_xk = b * sp.stage + sp.s_xk;
    v.dcon = (double *)(s + sp.s_dcon);
    v.meta = (const uint8_t *)(s + sp.s_meta);
    v.xk = (const double *)(s + sp.s_xk) + (d.p0 & 1);
    v.xo = (const double *)(s + sp.s_xo) + (d.p0 & 1);
    v.dn = (const double *)(s + sp.s_dn) + (d.p0 & 1);
    v.D = (const double *)(s + sp.s_D) + (d.c0 & 1);
    v.dd = (const double *)(s + sp.s_dd) + (d.c0 & 1);
    return v;
}

// One elected thread: bulk copies of a tile's inputs into stage b.
template <int MODE, bool RS>
__device__ __forceinline__ void issue_tile(const Params &P, const PassIO &io, const TileDesc &d, char *base,
                                           const SmemPlan &sp, int b, uint64_t *bar) {
    char *s = base + b * sp.stage;
    const int npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    const MetaOff m = meta_off(d.np, npath, nc, d.nrun, d.nhb, RS);
    const int pa = d.p0 & ~1, npa = even(d.p1 - pa);
    const int ca = d.c0 & ~1, nca = even(d.c1 - ca);
    const uint32_t b_dcon = 8u * even(d.np), b_p = 8u * npa, b_c = 8u * nca;
    uint32_t total = b_dcon + (uint32_t)m.bytes + 2 * b_p + 2 * b_c;
    if (MODE == MODE_RB) total += b_p;
    mbar_expect_tx(bar, total);
    bulk_g2s(s + sp.s_dcon, io.dcon_in + d.sb, b_dcon, bar);
    bulk_g2s(s + sp.s_meta, P.meta + (size_t)d.mb16 * 16, (uint32_t)m.bytes, bar);
    bulk_g2s(s + sp.s_xk, io.xk + pa, b_p, bar);
    bulk_g2s(s + sp.s_dn, io.dn_in + pa, b_p, bar);
    if (MODE == MODE_RB) bulk_g2s(s + sp.s_xo, io.xo + pa, b_p, bar);
    bulk_g2s(s + sp.s_D, P.D + ca, b_c, bar);
    bulk_g2s(s + sp.s_dd, io.dd_in + ca, b_c, bar);
}

// Block reduction of one double in a fixed tree order (deterministic).
__device__ double block_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < NW ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(FULL, r, o);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

// Four block reductions at once, each with block_sum's association (so the
// results are bitwise those of four block_sum calls): valid in thread 0.
__device__ void block_sum4(double v[4], double (*red4)[4]) {
    for (int j = 0; j < 4; ++j)
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(FULL, v[j], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
        for (int j = 0; j < 4; ++j) red4[w][j] = v[j];
    __syncthreads();
    if (w == 0) {
        for (int j = 0; j < 4; ++j) {
            double r = l < NW ? red4[l][j] : 0.0;
            for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(FULL, r, o);
            v[j] = r;
        }
    }
}

// Inclusive sum over the lane segment [first, lane] (Hillis-Steele, fixed tree),
// then broadcast the segment total from lane `last`.
__device__ __forceinline__ double seg_total(double v, int lane, int first, int last, int span) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        if (o >= span) break;  // a commodity spans at most `span` lanes
        double t = __shfl_up_sync(FULL, v, o);
        if (lane - o >= first) v += t;
    }
    return __shfl_sync(FULL, v, last);
}
__device__ __forceinline__ void seg_total2(double &a, double &b, int lane, int first, int last, int span) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        if (o >= span) break;
        const double ta = __shfl_up_sync(FULL, a, o);
        const double tb = __shfl_up_sync(FULL, b, o);
        if (lane - o >= first) {
            a += ta;
            b += tb;
        }
    }
    a = __shfl_sync(FULL, a, last);
    b = __shfl_sync(FULL, b, last);
}

// Correctly rounded 1/h for the path weights 1/hops and 1/(hops+1)
// (kernels.py:115-119): a table of IEEE quotients is bitwise the division.
constexpr int RCP_MAX = 64;
__constant__ double c_rcp[RCP_MAX + 1];
__device__ __forceinline__ double rcp_int(int h) { return h <= RCP_MAX ? c_rcp[h] : 1.0 / (double)h; }

// kernels.py:134-173 with lin = 1: (q + c) / 1.0 is q + c exactly, and the
// alpha = 1 quotient by 2.0 is an exact scaling; other cases as the reference.
__device__ __forceinline__ double root_lin1(double c, double q, int64_t alpha) {
    if (alpha == 0) return q + c;
    if (alpha == 1) {
        const double sq = sqrt(q * q + 4.0 * c);
        if (q >= 0.0) return (q + sq) * 0.5;
        return (2.0 * c) / (sq - q);
    }
    return root_newton(1.0, c, q, alpha);
}
// kernels.py:183-189 (commodity_root) using root_lin1 for the first root
__device__ __forceinline__ double fast_commodity_root(double w, double q, double d_eff, double beta, int64_t alpha) {
    const double cc = w / beta;
    double s = root_lin1(cc, q, alpha);
    if (s > d_eff) s = root_scalar(1.0 + w, cc, q + w * d_eff, alpha);
    return s;
}
// kernels.py:289-294 with 1/beta hoisted for alpha = 0 (the same quotient)
__device__ __forceinline__ double fast_commodity_term(double S, double D, double dd, double beta, double inv_beta,
                                                      int64_t alpha) {
    double gain;
    if (alpha == 0)
        gain = inv_beta;
    else if (alpha == 1)
        gain = (1.0 / S) / beta;
    else
        gain = pow(S, -(double)alpha) / beta;
    return gain - npmax0(S - (D - dd));
}

// Lane-strided sums of NV fields of the CTAs' residual records (res[g * 8 + off[j]]
// for g = lane, lane + 32, ...), each in index order (bitwise the plain loop),
// in predicated chunks of 4 CTAs per lane: one L2 round trip per 128 CTAs.
template <int NV>
__device__ __forceinline__ void res_sums(const double *res, int G, int lane, const int (&off)[NV], double (&acc)[NV]) {
    for (int j = 0; j < NV; ++j) acc[j] = 0.0;
    for (int g = lane; g < G; g += 128) {
        double b[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < NV; ++j) b[u][j] = g + 32 * u < G ? __ldcg(&res[(g + 32 * u) * 8 + off[j]]) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (g + 32 * u < G)
#pragma unroll
                for (int j = 0; j < NV; ++j) acc[j] += b[u][j];
    }
}

// Per-edge total of the CTA partials by one warp: lane j sums CTAs j, j + 32,
// ... in index order (the loads of 4 CTAs issued ahead), then a fixed shuffle
// tree; lane 0 holds the totals.  One L2 round trip for G <= 128 instead of a
// G-long chain per lane, and the same association wherever rank-local edge
// totals are formed (single GPU, peer-memory exchange, NCCL split kernels).
__device__ __forceinline__ void warp_edge_sums(const double *pT, const double *pL, int G, int E, int e, int lane,
                                               double &T, double &L) {
    double t = 0.0, l = 0.0;
    for (int g = lane; g < G; g += 128) {  // predicated chunks of 4 CTAs: one round trip per 128 CTAs
        double bt[4], bl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool in = g + 32 * u < G;
            bt[u] = in ? __ldcg(pT + (size_t)e * G + g + 32 * u) : 0.0;  // coalesced: [E][G]
            bl[u] = in ? __ldcg(pL + (size_t)e * G + g + 32 * u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (g + 32 * u < G) {
                t += bt[u];
                l += bl[u];
            }
    }
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_down_sync(FULL, t, o);
        l += __shfl_down_sync(FULL, l, o);
    }
    T = t;
    L = l;
}

// Run slots: the per-edge total of the (tile, run) slots eoff[e] .. eoff[e + 1]
// by one warp: lane j sums slots j, j + 32, ... in slot (= tile) order, 8 slots
// in flight per lane, then the same fixed shuffle tree; lane 0 holds the totals.
__device__ __forceinline__ void warp_slot_sums(const double *slots, const int32_t *eoff, int e, int lane,
                                               double &T, double &L) {
    const int a = __ldg(&eoff[e]), b = __ldg(&eoff[e + 1]);
    double t = 0.0, l = 0.0;
    for (int s = a + lane; s < b; s += 32 * 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            v[u] = s + 32 * u < b ? __ldcg((const double2 *)slots + s + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (s + 32 * u < b) {
                t += v[u].x;
                l += v[u].y;
            }
    }
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_down_sync(FULL, t, o);
        l += __shfl_down_sync(FULL, l, o);
    }
    T = t;
    L = l;
}

// The rank-local per-edge totals {T, L} of the pass just completed, whichever
// layout holds the partials (one warp; lane 0 holds the result)
__device__ __forceinline__ void edge_totals(const Params &P, int e, int lane, double &T, double &L) {
    if (P.run_slots)
        warp_slot_sums(P.slots, P.eoff, e, lane, T, L);
    else
        warp_edge_sums(P.partT, P.partL, P.G, P.I.E, e, lane, T, L);
}

// The per-edge squared dual_capacity changes are double-buffered by iteration
// parity inside the persistent kernel: the edge phase of iteration k + 1 (at
// the loop top, iteration counter k) writes half k & 1, and the controller of
// the same iteration (counter k + 1 after the pass) reads it.  No grid barrier
// separates one iteration's controller from the next edge phase, so with a
// single buffer a CTA that leaves the controller early could overwrite entries
// a slower CTA was still summing, and the CTAs' controller copies could diverge.
// (The split multi-GPU kernels are separate launches and use half 0.)
__device__ __forceinline__ double *res_dc_write(const Params &P, const Ctrl &c) {
    return P.res_dc + (size_t)(c.iteration & 1) * (size_t)P.I.E;
}
__device__ __forceinline__ const double *res_dc_read(const Params &P, const Ctrl &c) {
    return P.res_dc + (size_t)((c.iteration + 1) & 1) * (size_t)P.I.E;
}

// Sum of the per-edge dual_capacity residuals by the whole CTA (NT threads):
// thread i sums edges i, i + NT, ... in order, then a warp shuffle tree and the
// warp sums in warp order.  Every thread returns the same value.
__device__ double dcs_block(const double *res_dc, int E) {
    __shared__ double wred[NT / 32];
    double v = 0.0;
    for (int e = threadIdx.x; e < E; e += 4 * NT) {  // predicated chunks of 4
        double b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = e + u * NT < E ? __ldcg(res_dc + e + u * NT) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (e + u * NT < E) v += b[u];
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wred[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = wred[0];
    for (int w = 1; w < NT / 32; ++w) r += wred[w];
    return r;
}

// ------------------------------------------------------------------ controller

// The dual rescale factor f_{k+1} the M pass applies speculatively to A(k+2):
// the beta decision of controller.py:251-266 taken on the residual EMAs as
// they stand before this iteration's residuals move them by 10%.  Certain when
// adaptation is off or a cooldown is running (f = 1); during beta's ramp the
// ratio of the EMAs sits far from the thresholds, so the prediction holds and
// no rollback pass is needed.  A wrong prediction costs the rollback pass the
// kernel always had (a recomputation of A(k+2) with the true f from the
// intact duals_{k+1}): the iterates are bitwise those of the rollback path.
__device__ __forceinline__ double predict_f(const Params &P, const Ctrl &c) {
    if (!P.adapt || c.cooldown > 0 || c.ema_s < 0.0) return 1.0;
    double b = c.beta;
    const double m = P.spec_margin;  // predict a change only this far past the threshold
    if (c.ema_r > m * P.residual_ratio * c.ema_s)
        b = b * P.beta_scale;
    else if (c.ema_s > m * P.residual_ratio * c.ema_r)
        b = b / P.beta_scale;
    const double lo = b > P.beta_min ? b : P.beta_min;
    const double nb = lo < P.beta_max ? lo : P.beta_max;
    return nb != c.beta ? c.beta / nb : 1.0;
}

// controller.py:237-273 on the residuals of the iteration just completed.
__device__ __noinline__ void controller_step(const Params &P, Ctrl &c, double s, double r, int32_t ec, int32_t er) {
    c.fspec = c.fnext;  // what the M pass applied
    c.s = s;
    c.r = r;
    c.f = 1.0;
    if (P.ablate) return;  // timing experiments: results are meaningless, keep iterating
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
    c.fnext = P.spec_f ? predict_f(P, c) : 1.0;  // off the next pass's start: its state is this one
}

// Every CTA reduces the residual partials in the same fixed order and runs the
// same scalar controller step on its shared-memory copy of the state.
__device__ void controller_eval(const Params &P, Ctrl &c) {
    const double dcs = dcs_block(res_dc_read(P, c), P.I.E);
    if (threadIdx.x < 32) {
        const int par = (int)(c.iteration & 1);
        double acc[4];  // dx, dd, dcon, dn: lane-strided over the CTAs
        const int off[4] = {0, 1 + 3 * par, 2 + 3 * par, 3 + 3 * par};
        res_sums<4>(P.res, P.G, threadIdx.x, off, acc);
        for (int j = 0; j < 4; ++j)
            for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_down_sync(FULL, acc[j], o);
        if (threadIdx.x == 0)
            controller_step(P, c, sqrt(acc[0]), sqrt(((acc[1] + dcs) + acc[2]) + acc[3]), __ldcg(&P.err[0]),
                            __ldcg(&P.err[1]));
    }
    __syncthreads();
}

// ------------------------------------------------------------------ edge phase

// One warp per edge: the CTA partials summed by warp_edge_sums, then
// kernels.py:212 (dual_capacity) and :94-96 (adjustment); the squared
// dual_capacity change per edge for the residual (summed by dcs_block).
// Run slots, single GPU: one CTA per edge at a time over a slot-balanced range
// of edges (a heavily shared edge of config 3 holds tens of thousands of
// slots; a warp per edge left the phase waiting on the heaviest edges).  Thread
// t sums slots t, t + NT, ... in order (8 in flight), then a fixed block tree;
// then kernels.py:212 and :94-96 as edge_phase.
__device__ __noinline__ void edge_phase_rs(const Params &P, double f, double *res_dc) {
    const InstView &I = P.I;
    __shared__ double2 wsum[NT / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double2 *slots = (const double2 *)P.slots;
    for (int e = P.ebound[blockIdx.x]; e < P.ebound[blockIdx.x + 1]; ++e) {
        const int a = __ldg(&P.eoff[e]), b = __ldg(&P.eoff[e + 1]);
        double t = 0.0, l = 0.0;
        for (int s0 = a + tid; s0 < b; s0 += 8 * NT) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = s0 + u * NT < b ? __ldcg(slots + s0 + u * NT) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (s0 + u * NT < b) {
                    t += v[u].x;
                    l += v[u].y;
                }
        }
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_down_sync(FULL, t, o);
            l += __shfl_down_sync(FULL, l, o);
        }
        if (lane == 0) wsum[warp] = make_double2(t, l);
        __syncthreads();
        if (tid == 0) {
            double T = wsum[0].x, L = wsum[0].y;
            for (int w = 1; w < NT / 32; ++w) {
                T += wsum[w].x;
                L += wsum[w].y;
            }
            const double cap = I.capacity[e];
            const double dold = __ldcg(&P.dc[e]) * f;
            const double dnew = npmax0(dold + (L - cap));
            double adj = (T + dnew - cap) / (P.ne[e] + 1.0);
            if (adj < 0.0) adj = 0.0;
            P.dc[e] = dnew;
            P.adj[e] = adj;
            const double d = dnew - dold;
            res_dc[e] = d * d;
        }
        __syncthreads();
    }
}

__device__ __noinline__ void edge_phase(const Params &P, double f, double *res_dc) {
    const InstView &I = P.I;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = blockIdx.x + P.G * warp; e < I.E; e += P.G * (NT / 32)) {  // edges spread over all CTAs
        double T, L;
        edge_totals(P, e, lane, T, L);
        if (lane == 0) {
            const double cap = I.capacity[e];
            const double dold = __ldcg(&P.dc[e]) * f;
            const double dnew = npmax0(dold + (L - cap));
            double adj = (T + dnew - cap) / (P.ne[e] + 1.0);
            if (adj < 0.0) adj = 0.0;
            P.dc[e] = dnew;
            P.adj[e] = adj;
            const double d = dnew - dold;
            res_dc[e] = d * d;
        }
    }
}

// ------------------------------------------------------------------ tile compute

struct Acc {
    double *adj, *y;
    double2 *acc;      // per edge {T, L} in shared memory, or
    double *gT, *gL;   // this CTA's partials (large E): edge e at gT[e * gs]
    int gs;
    uint32_t adj_s, acc_s;  // shared-space addresses of the tables (when in shared memory)
    double *adjt;           // run slots: the tile's per-run adjustment table
    uint32_t adjt_s;
    double *slots;          // run slots: the global {T, L} slots
    int o_y, o_adj, o_adjt, o_hp;  // byte offsets from the dynamic shared-memory base
};

template <int MODE, bool RS>
__device__ __forceinline__ void acc_add(const Acc &A, const uint32_t *rdst, int e, double T, double L) {
    if (RS) {  // run slots: e is the tile-local run; one store, no read-modify-write
        double *q = A.slots + 2 * (size_t)rdst[e];
        if (MODE != MODE_RB)
            __stcg((double2 *)q, make_double2(T, L));
        else
            __stcg(q, T);
    } else if (A.acc) {
        const uint32_t a = A.acc_s + 16u * (uint32_t)e;
        double2 v = lds_f64x2(a);
        v.x += T;
        if (MODE != MODE_RB) v.y += L;
        sts_f64x2(a, v);
    } else {  // L2-resident CTA-private rows (bypass L1: it holds the adjustment table)
        const size_t o = (size_t)e * A.gs;
        __stcg(&A.gT[o], __ldcg(&A.gT[o]) + T);
        if (MODE != MODE_RB) __stcg(&A.gL[o], __ldcg(&A.gL[o]) + L);
    }
}

// The dynamic shared memory, addressed through the symbol so that the per-pair
// loops compile to shared-space loads and stores (pointers handed through
// structs or non-inlined calls degrade to generic accesses).
extern __shared__ __align__(128) char g_smem[];

// Per-pair loops over one commodity group in its hop-major order.  The group's
// paths take the hop lanes by decreasing hop count, so the lanes active at step
// j are a prefix 0 .. n_j - 1 and step j's pairs are hb[j] + lane: one
// contiguous, conflict-free row per step, no per-step vote, no per-pair path
// index, and each lane keeps its path's rate and K_p in registers.  Inactive
// lanes read the step's first slot and store nothing (straight-line code, so
// the unrolled steps' loads overlap).
//   y_j = max0(x + dcon_j - adj_e) (kernels.py:98-100), K = sum_j (y_j - dcon_j) in
//   hop order (kernels.py:110-113)
// Offsets are bytes from the dynamic shared-memory base.
template <int MODE, bool ADJ_L1>
__device__ __forceinline__ double hops_y(int hb_o, int H, int lane, double xl, int eid_o, int dcon_o, int adj_o,
                                         const double *__restrict__ adj_g, int ys_o) {
    const uint16_t *hb = (const uint16_t *)(g_smem + hb_o);
    const uint16_t *eid = (const uint16_t *)(g_smem + eid_o);
    const double *dcon = (const double *)(g_smem + dcon_o);
    const double *adj = (const double *)(g_smem + adj_o);
    double *ys = (double *)(g_smem + ys_o);
    double K = 0.0;
    int b0 = hb[0];
#pragma unroll 4
    for (int j = 0; j < H; ++j) {
        const int b1 = hb[j + 1];
        const bool on = lane < b1 - b0;
        const int l = on ? b0 + lane : b0;
        const double dv = dcon[l];
        double y;
        if (MODE == MODE_A1) {
            y = xl;
        } else {
            const int e = eid[l];
            const double a = ADJ_L1 ? __ldca(&adj_g[e]) : adj[e];
            y = max0(xl + dv - a);
        }
        if (on) ys[l] = y;
        K += on ? y - dv : 0.0;
        b0 = b1;
    }
    return K;
}

// dual_consensus' (kernels.py:72) stored coalesced to global; T = x' + dcon'
// (kernels.py:91) into tv (tv aliases dcon on purpose: every step reads dcon[l]
// before it writes tv[l], for its own row only)
// Inactive lanes read `dummy_o`, a double nobody writes in this phase (the
// step's own slots are rewritten by the active lanes).
__device__ __forceinline__ double hops_dcon(int hb_o, int H, int lane, double xn, double f, int dcon_o, int ys_o,
                                            double *__restrict__ dco, int dummy_o) {
    const uint16_t *hb = (const uint16_t *)(g_smem + hb_o);
    double *dcon = (double *)(g_smem + dcon_o);
    const double *dummy = (const double *)(g_smem + dummy_o);
    const double *ys = (const double *)(g_smem + ys_o);
    double r = 0.0;
    int b0 = hb[0];
#pragma unroll 4
    for (int j = 0; j < H; ++j) {
        const int b1 = hb[j + 1];
        const bool on = lane < b1 - b0;
        const int l = on ? b0 + lane : b0;
        const double dks = (on ? dcon + l : dummy)[0] * f;
        const double dnew = max0(dks + xn - ys[l]);
        const double df = dnew - dks;
        if (on) {
            dco[l] = dnew;
            dcon[l] = xn + dnew;
        }
        r += on ? df * df : 0.0;
        b0 = b1;
    }
    return r;
}

// MODE_M : B(k+1) [y, K/w, roots, x_{k+1}] fused with A(k+2) [duals_{k+2}, T/L]
// MODE_RB: A(k+2) only, recomputing y_{k+1} from x_k, dcon_{k+1}, adj_{k+1}
// MODE_A1: A(1) with y_0 = x_0[pair_path] (controller.py:118)
template <int MODE, bool RS>
__device__ __forceinline__ void tile_compute(const Params &P, const Ctrl &c, const PassIO &io, const TileDesc &d,
                                             const StageView &st, const Acc &A, double &r_x,
                                             double &r_dd, double &r_dcon, double &r_dn, const TileDesc *next,
                                             TileDesc *sd_slot, char *base, const SmemPlan &sp, uint64_t *bar) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int np = d.np, npath = d.p1 - d.p0, nc = d.c1 - d.c0;
    const MetaOff m = meta_off(np, npath, nc, d.nrun, d.nhb, RS);
    const uint32_t *rdst = RS ? (const uint32_t *)(st.meta + m.rdst) : nullptr;
    const uint16_t *poff = (const uint16_t *)(st.meta + m.poff);
    const uint8_t *pcom = st.meta + m.pcom;
    const uint16_t *cpp = (const uint16_t *)(st.meta + m.cpp);
    const uint16_t *gpath = (const uint16_t *)(st.meta + m.gpath);
    TP_DECL
    TP(-1)
    const double f = io.f;
    const double inv_beta = 1.0 / c.beta;
    double *const x_out = io.x_out, *const dn_out = io.dn_out, *const dd_out = io.dd_out;

    // ---- this warp's commodity group
    const int gp0 = gpath[w], gp1 = gpath[w + 1];
    const int hl = gp0 + lane < gp1 ? poff[gp0 + lane + 1] - poff[gp0 + lane] : 0;  // this lane's path hops
    // hop lanes: lane i runs path gp0 + hperm[gp0 + i] through the group's H hop steps
    const uint16_t *hbo = (const uint16_t *)(st.meta + m.hbo);
    const uint8_t *hperm = st.meta + m.hperm, *hinv = st.meta + m.hinv;
    const int hb0 = hbo[w], H = hbo[w + 1] - hb0 - 1;
    const int hb_o = st.o_meta + m.hb + 2 * hb0;
    const bool hv = gp0 + lane < gp1;
    const int ph = gp0 + (hv ? (int)hperm[gp0 + lane] : 0);
    if (!(P.ablate & 1)) {
    // (1) pairs: y (kernels.py:98-100) and K_p (kernels.py:110-113) in the hop lane
    const double xlane = hv ? (MODE == MODE_RB ? st.xo[ph] : st.xk[ph]) : 0.0;
    double Kl = 0.0;
    if (RS && MODE != MODE_A1) {  // the adjustment of each of the tile's runs (kernels.py:94-96)
        const uint16_t *redge = (const uint16_t *)(st.meta + m.redge);
        for (int r = threadIdx.x; r < d.nrun; r += NT) A.adjt[r] = __ldcg(&P.adj[redge[r]]);
        __syncthreads();
    }
    if (!(P.ablate & 64)) {
        if (RS || P.adj_smem)
            Kl = hops_y<MODE, false>(hb_o, H, lane, xlane, st.o_meta + m.eid, st.o_dcon, RS ? A.o_adjt : A.o_adj,
                                     nullptr, A.o_y);
        else
            Kl = hops_y<MODE, true>(hb_o, H, lane, xlane, st.o_meta + m.eid, st.o_dcon, 0, P.adj, A.o_y);
    }
    // K_p from its hop lane to the path's lane (commodity order)
    Kl = __shfl_sync(FULL, Kl, hv ? (int)hinv[gp0 + lane] : lane);
    TP(1)
    // (2) paths (lane = path) and commodities (lane segments)
    double xnew_lane = 0.0;  // x' of this lane's path
    {
        const int p = gp0 + lane;
        const bool valid = p < gp1;
        int j = 0, first = lane, last = lane;
        if (valid) {
            j = pcom[p];
            first = cpp[j] - gp0;
            last = cpp[j + 1] - 1 - gp0;
        }
        const bool head = valid && lane == first;
        const int cc = d.c0 + j;
        const double xk = valid ? st.xk[p] : 0.0;
        double xv = xk;
        if (MODE == MODE_M && !(P.ablate & 16)) {
            double K = 0.0, wgt = 0.0;
            if (valid) {
                K = (P.ablate & 32) ? 0.0 : Kl;
                const double dnv = st.dn[p];
                if (xk < dnv) {  // frozen non-negativity activity (kernels.py:114-119)
                    K += dnv;
                    wgt = rcp_int(hl + 1);
                } else {
                    wgt = rcp_int(hl);
                }
            }
            double Wc = wgt, Qc = wgt * K;
            seg_total2(Wc, Qc, lane, first, last, P.kspan);
            double ct = NAN;
            if (valid) {
                if (!(isfinite(Wc) && isfinite(Qc))) {
                    if (head) atomicMin(&P.err[0], cc);
                } else {
                    const double D = st.D[j], ddk = st.dd[j];
                    const double Sc = fast_commodity_root(Wc, Qc, D - ddk, c.beta, c.alpha);
                    if (head) {
                        if (!isfinite(Sc)) atomicMin(&P.err[1], cc);
                        if (P.root_sums) P.root_sums[cc] = Sc;
                    }
                    ct = fast_commodity_term(Sc, D, ddk, c.beta, inv_beta, c.alpha);
                }
                xv = wgt * (K + ct);
                x_out[d.p0 + p] = xv;
                const double df = xv - xk;
                r_x += df * df;
            }
        }
        if (valid) {
            xnew_lane = xv;
            const double o = st.dn[p] * f;
            const double n = npmax0(o - xv);
            dn_out[d.p0 + p] = n;
            const double dg = n - o;
            r_dn += dg * dg;
        }
        // S_c (model.py:297-302) and dual_demand (kernels.py:211)
        const double Sx = seg_total(valid ? xv : 0.0, lane, first, last, P.kspan);
        if (head) {
            const double dold = st.dd[j] * f;
            const double dnew = npmax0(dold + (Sx - st.D[j]));
            dd_out[cc] = dnew;
            const double df = dnew - dold;
            r_dd += df * df;
        }
    }
    __syncwarp();
    TP(2)
    // (3) pairs, hop-major: dual_consensus' (kernels.py:72) stored coalesced;
    // T = x' + dcon' (kernels.py:91) replaces the consumed dcon in the stage
    // (tv aliases dcon on purpose: every step reads dcon[l] before it writes
    // tv[l], for the same l only)
    const double xh = __shfl_sync(FULL, xnew_lane, hv ? (int)hperm[gp0 + lane] : lane);  // back to the hop lane
    r_dcon += hops_dcon(hb_o, H, lane, xh, f, st.o_dcon, A.o_y, io.dcon_out + d.sb, st.o_xk);
    fence_proxy_async_shared();  // these generic writes precede the TMA that refills the stage
    __syncthreads();
    TP(3)

    }
    if (P.ablate & 2) return;
    // (4) per-edge sums over the tile's edge runs: T = sum (x' + dcon')
    // (kernels.py:91) and L = sum y (kernels.py:210).  A run is the tile's pairs
    // on one edge; sperm lists the tile's pairs sorted by (edge, pair), so the
    // runs lie back to back.  Thread t sums the contiguous chunk
    // [t * cs, (t + 1) * cs) of that order in sequence: a run that starts and
    // ends inside the chunk goes straight to its edge accumulator; a chunk's
    // head piece (the continuation of a run begun in an earlier chunk) is
    // published, and after a barrier the thread where a crossing run begins adds
    // the following chunks' head pieces in chunk order.  Every run is summed
    // in a fixed order and added once by one thread; runs of one tile have
    // distinct edges and tiles are separated by block barriers: deterministic
    // without atomics, balanced by items rather than runs.
    {
        const int tid = threadIdx.x;
        const int so = st.o_meta + m.sperm;  // shared offsets
        const uint16_t *sperm = (const uint16_t *)(g_smem + so);
        const uint16_t *ed = (const uint16_t *)(g_smem + st.o_meta + m.eid);  // edge (run) of each pair
        const double *tv = (const double *)(g_smem + st.o_dcon);             // x' + dcon' (step 3)
        const double *yv = (const double *)(g_smem + A.o_y);
        // head pieces: the stage's per-path arrays are dead once step 3 is done
        double2 *hp = (double2 *)(g_smem + A.o_hp);
        const uint16_t *xlen = (const uint16_t *)(g_smem + st.o_meta + m.xlen);
        const int cs = max((np + NT - 1) / NT, 4);  // small tiles: fewer, longer chunks (fewer crossings)
        const int a0 = tid * cs, b0 = min(a0 + cs, np);
        double T = 0.0, L = 0.0;
        int cur = -1;
        bool inside = false;  // the current piece started inside this chunk
        if (a0 < b0) {
            // sperm: bit 15 marks the first pair of a run, bits 0-14 the pair;
            // the run's edge (or run id) is read once per run
            const int w0 = sperm[a0];
            cur = ed[w0 & 0x7fff];
            inside = (w0 >> 15) != 0;
#pragma unroll 4
            for (int q = a0; q < b0; ++q) {
                const int wq = sperm[q];
                const int u = wq & 0x7fff;
                const double t = tv[u];
                const double yy = MODE != MODE_RB ? yv[u] : 0.0;
                if (q > a0 && (wq >> 15)) {  // the piece of run `cur` ends here
                    const int e = ed[u];
                    if (inside) {
                        acc_add<MODE, RS>(A, rdst, cur, T, L);
                    } else {
                        hp[tid] = make_double2(T, L);  // this chunk's head piece
                    }
                    cur = e;
                    inside = true;
                    T = 0.0;
                    L = 0.0;
                }
                T += t;
                if (MODE != MODE_RB) L += yy;
            }
            const bool cont = b0 < np && !(sperm[b0] >> 15);
            if (!cont) {
                if (inside) {
                    acc_add<MODE, RS>(A, rdst, cur, T, L);
                } else {
                    hp[tid] = make_double2(T, L);  // this chunk's head piece
                }
                inside = false;  // nothing left to finish
            } else if (!inside) {
                hp[tid] = make_double2(T, L);  // the whole chunk lies inside one crossing run
            }
        }
        // what phase 2 needs from the stage, read before the stage is released
        const int nx = inside ? (int)xlen[tid] : 0;  // static: the layout knows which chunks a run crosses
        const uint32_t rd1 = RS && nx > 0 ? rdst[cur] : 0u;
        TP(6)
        __syncthreads();
        // the stage is free: the next tile's bulk copies overlap phase 2 and the
        // end-of-tile barrier (single-stage layout)
        // (the last thread: its walk chunk is the tile's tail, usually short or
        // empty, so the copies do not delay a crossing run's owner)
        if (next && tid == NT - 1) {  // (every thread read this tile's descriptor long ago)
            *sd_slot = *next;
            fence_proxy_async_shared();
            issue_tile<MODE, RS>(P, io, *sd_slot, base, sp, 0, bar);
        }
        if (nx > 0) {  // this chunk's tail begins a run that crosses into the next nx chunks
#pragma unroll 4
            for (int k = 1; k <= nx; ++k) {
                const double2 v = hp[tid + k];
                T += v.x;
                L += v.y;
            }
            acc_add<MODE, RS>(A, &rd1, RS ? 0 : cur, T, L);  // (run slots: the slot read above)
        }
    }
    TP(4)
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
        io.f = c.fnext;  // speculative f_{k+1} (predict_f, taken by the previous controller step)
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

// Per-CTA persistent shared state.
constexpr int DL = 64;  // tile descriptors of a CTA's first DL tiles kept in shared memory

struct CtaShared {
    uint64_t bar[2];
    TileDesc sd[2];
    TileDesc dl[DL];  // this CTA's tiles (thread 0 reads them on the tile boundaries)
    int32_t dl_rev;   // walk direction dl[] is stored in; -1 = not filled (a CTA owns <= DL tiles: kept)
    PassIO io;
    double red[NW];
    double red4[NW][4];
};

// One pass over this CTA's tiles (static assignment tile = g + k*G, so every
// tile's state is only ever touched by one CTA).  Odd iterations walk the tiles
// in reverse so a pass first re-reads what the previous pass wrote last (L2
// reuse).  `seq` counts the tiles this CTA has staged (stage = seq & 1, mbarrier
// parity = (seq >> 1) & 1), persistent across passes.
template <int MODE, bool RS>
__device__ __noinline__ void pass_tiles(const Params &P, const Ctrl &c, char *base, CtaShared &cs, uint32_t &seq) {
    const int g = blockIdx.x, tid = threadIdx.x;
    const int E = P.I.E;
    const SmemPlan sp = smem_plan(P.tps, E, P.nbuf, P.hbmax, P.adj_smem, P.acc_smem, RS, P.rmax);
    Acc A;
    A.adj = P.adj_smem ? (double *)(base + sp.adj) : P.adj;
    A.acc = P.acc_smem ? (double2 *)(base + sp.acc) : nullptr;
    A.gT = P.partT + g;  // column g of the edge-major partials
    A.gL = P.partL + g;
    A.gs = P.G;
    A.y = (double *)(base + sp.y);
    A.adj_s = su32(base + sp.adj);
    A.acc_s = su32(base + sp.acc);
    A.adjt = (double *)(base + sp.adjt);
    A.adjt_s = su32(base + sp.adjt);
    A.slots = P.slots;
    A.o_y = sp.y;
    A.o_adj = sp.adj;
    A.o_adjt = sp.adjt;
    A.o_hp = sp.hp;
    const int t0 = P.cta_ptr[g], my = P.cta_ptr[g + 1] - t0;
    // the rollback pass (after the iteration count moved on) walks in its M
    // pass's direction: the CTA partials keep the M pass's association, so a
    // speculated rescale factor gives bitwise the rollback path's iterates
    const bool rev = ((MODE == MODE_RB ? c.iteration - 1 : c.iteration) & 1) != 0;
    auto tile_of = [&](int k) { return P.cta_tiles[t0 + (rev ? my - 1 - k : k)]; };
    // the next tile's descriptor from shared memory: no dependent global loads
    // on thread 0's path between two tiles (its TMA issue and L2 prefetch).  A
    // CTA's tile set is fixed for the launch: with <= DL tiles, dl[] is filled by
    // the first pass and read in either walk direction afterwards.
    const bool keep = my <= DL && cs.dl_rev >= 0;
    const bool flip = keep && cs.dl_rev != (rev ? 1 : 0);
    auto desc_of = [&](int k) -> TileDesc { return k < DL ? cs.dl[flip ? my - 1 - k : k] : P.desc[tile_of(k)]; };
    auto desc_ptr = [&](int k) -> const TileDesc * {
        return k < DL ? &cs.dl[flip ? my - 1 - k : k] : &P.desc[tile_of(k)];
    };
    const bool dbl = P.nbuf == 2;
    if (tid == 0) {
        cs.io = pass_io<MODE>(P, c);
        fence_proxy_async();  // this pass's inputs were written by generic stores after a grid barrier
        if (my > 0) {
            const int b = dbl ? (seq & 1) : 0;
            cs.sd[b] = keep ? desc_of(0) : P.desc[tile_of(0)];
            issue_tile<MODE, RS>(P, cs.io, cs.sd[b], base, sp, b, &cs.bar[b]);
        }
    }
    if (!keep)
        for (int i = tid; i < my && i < DL; i += NT) cs.dl[i] = P.desc[tile_of(i)];  // visible after the barrier below
    for (int e0 = tid; e0 < E && !RS; e0 += 4 * NT) {  // the adjustment loads of 4 edges in flight
        double av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            av[u] = P.adj_smem && MODE != MODE_A1 && e < E ? __ldcg(&P.adj[e]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            if (e >= E) break;
            if (P.acc_smem) {
                A.acc[e] = make_double2(0.0, 0.0);
            } else {
                __stcg(&A.gT[(size_t)e * A.gs], 0.0);
                if (MODE != MODE_RB) __stcg(&A.gL[(size_t)e * A.gs], 0.0);
            }
            if (P.adj_smem) A.adj[e] = av[u];
        }
    }
    // without the shared table adj is read through L1 (ld.global.ca); it was
    // rewritten by the edge phase before the grid barrier: acquire at gpu scope
    // so no stale L1 line survives
    if (!P.adj_smem && !RS) asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    __syncthreads();
    if (tid == 0 && !keep && my <= DL) cs.dl_rev = rev ? 1 : 0;  // every thread read dl_rev before the barrier
    const PassIO &io = cs.io;
    double r_x = 0.0, r_dd = 0.0, r_dcon = 0.0, r_dn = 0.0;
    for (int k = 0; k < my; ++k, ++seq) {
        const int b = dbl ? (seq & 1) : 0;
        const uint32_t par = dbl ? ((seq >> 1) & 1) : (seq & 1);
        if (tid == 0 && k + 1 < my) {
            if (dbl) {  // prefetch the next tile into the other stage
                const int nb = b ^ 1;
                cs.sd[nb] = desc_of(k + 1);
                issue_tile<MODE, RS>(P, io, cs.sd[nb], base, sp, nb, &cs.bar[nb]);
            } else if (k + P.pf_dist < my) {  // single stage: warm L2 with a later tile's pair data
                const TileDesc dn_ = desc_of(k + P.pf_dist);
                prefetch_l2(io.dcon_in + dn_.sb, 8u * even(dn_.np));
                prefetch_l2(P.meta + (size_t)dn_.mb16 * 16,
                            (uint32_t)meta_off(dn_.np, dn_.p1 - dn_.p0, dn_.c1 - dn_.c0, dn_.nrun, dn_.nhb, RS).bytes);
            }
        }
#ifdef PF_TPROBE
        const unsigned long long tw0 = clock64();
#endif
        mbar_wait(&cs.bar[b], par);
#ifdef PF_TPROBE
        if (tid == 0) {
            atomicAdd(&g_tprobe[0], clock64() - tw0);
            atomicAdd(&g_tprobe[7], 1ull);
        }
#endif
        const TileDesc d = cs.sd[b];
        const StageView st = stage_view(base, sp, b, d);
        // single stage: the next tile's copies are issued from inside the tile,
        // as soon as its stage is released (after the edge-run walk's first phase)
        const bool early = !dbl && k + 1 < my;
        tile_compute<MODE, RS>(P, c, io, d, st, A, r_x, r_dd, r_dcon, r_dn, early ? desc_ptr(k + 1) : nullptr,
                               &cs.sd[0], base, sp, &cs.bar[0]);
#ifdef PF_TPROBE
        const unsigned long long tb0 = clock64();
#endif
        // With the next tile's copies already issued (early), no barrier here: the
        // walk's second phase only reads the head pieces and adds to the edge
        // accumulators, and the next tile touches neither before its own block
        // barrier after dual_consensus; the copies' mbarrier arrival (release)
        // publishes the next descriptor.  Otherwise (a CTA's last tile: the
        // accumulator flush follows; the double-buffered stage) the barrier stays.
        if (!early) __syncthreads();
#ifdef PF_TPROBE
        if (tid == 0) atomicAdd(&g_tprobe[5], clock64() - tb0);
#endif

    }
    for (int e = tid; e < E; e += NT) {
        if (!P.acc_smem) break;  // the rows are the partials already
        const double2 v = A.acc[e];
        P.partT[(size_t)e * P.G + g] = v.x;
        if (MODE != MODE_RB) P.partL[(size_t)e * P.G + g] = v.y;
    }
    double *r = P.res + g * 8;
    double v4[4] = {r_x, r_dd, r_dcon, r_dn};
    block_sum4(v4, cs.red4);
    if (tid == 0) {
        if (MODE == MODE_M) r[0] = v4[0];
        r[1 + 3 * io.par] = v4[1];
        r[2 + 3 * io.par] = v4[2];
        r[3 + 3 * io.par] = v4[3];
    }
    // the generic-proxy stores of this pass (dual_consensus, rates, ...) are read
    // by TMA in the next pass
    fence_proxy_async();
}

__device__ __forceinline__ void cta_init(CtaShared &cs) {
    if (threadIdx.x == 0) {
        mbar_init(&cs.bar[0], 1);
        mbar_init(&cs.bar[1], 1);
        cs.dl_rev = -1;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
}

// ------------------------------------------------------------------ multi-GPU exchange
//
// Buffer layout per rank (peer-writable): [2 parities][nranks slots][xslot
// doubles] followed by one u64 arrival counter.  Exchange number n uses parity
// n & 1; a rank adds 1 to every rank's counter after its slot is written, so
// exchange n is complete on a rank when its counter reaches nranks * (n + 1).
// Two parities suffice: a rank reads exchange n before it computes the pass
// whose totals it sends in exchange n + 1.

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double *xb_slot(const Params &P, const double *base, uint64_t epoch, int r) {
    return (double *)base + ((epoch & 1) * (uint64_t)P.nranks + (uint64_t)r) * (uint64_t)P.xslot;
}
__device__ __forceinline__ unsigned long long *xb_flag(const Params &P, const double *base) {
    return (unsigned long long *)((double *)base + 2 * (uint64_t)P.nranks * (uint64_t)P.xslot);
}

// Rank-local totals of the pass just completed -> every rank's slot [rank]:
// per-edge T and L (CTA partials summed as in the single-GPU edge phase), the 7 residual sums and the 2 error flags; then the
// counter barrier across ranks.  Ends with a grid barrier after which every CTA
// may read all slots of this exchange.
__device__ __noinline__ void xchg_phase(const Params &P, Ctrl &c, cg::grid_group &grid) {
    const InstView &I = P.I;
    const int g = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ep = c.xepoch;
    bool wrote = false;  // this thread stored into peer memory
    for (int e = g + P.G * warp; e < I.E; e += P.G * (NT / 32)) {
        double T, L;
        edge_totals(P, e, lane, T, L);
        if (lane == 0) {
            wrote = true;
            for (int r = 0; r < P.nranks; ++r) {
                double *d = xb_slot(P, P.peers[r], ep, P.rank);
                d[e] = T;
                d[I.E + e] = L;
            }
        }
    }
    if (g == 0 && threadIdx.x < 32) {  // residual sums over the CTAs, error flags
        // same association as controller_eval (lane-strided, then a shuffle tree),
        // so one rank reproduces the single-GPU controller bitwise
        double acc[7];
        const int off[7] = {0, 1, 2, 3, 4, 5, 6};
        res_sums<7>(P.res, P.G, threadIdx.x, off, acc);
        for (int j = 0; j < 7; ++j)
            for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_down_sync(FULL, acc[j], o);
        if (threadIdx.x == 0) {
            wrote = true;
            const double e0 = __ldcg(&P.err[0]) != INT_MAX ? 1.0 : 0.0;
            const double e1 = __ldcg(&P.err[1]) != INT_MAX ? 1.0 : 0.0;
            for (int r = 0; r < P.nranks; ++r) {
                double *d = xb_slot(P, P.peers[r], ep, P.rank) + 2 * I.E;
                for (int j = 0; j < 7; ++j) d[j] = acc[j];
                d[7] = e0;
                d[8] = e1;
                d[9] = __longlong_as_double((long long)(ep + 1));  // the slot's epoch tag
            }
        }
    }
    if (wrote) __threadfence_system();  // this thread's peer stores before the arrival signal
    grid.sync();
    __shared__ int s_timeout;
    if (threadIdx.x == 0) {
        s_timeout = 0;
        if (g == 0) {
            __threadfence_system();
            for (int r = 0; r < P.nranks; ++r) atomicAdd_system(xb_flag(P, P.peers[r]), 1ull);
        }
        // every CTA waits for all ranks' slots (bounded: ~20 s, then PF_ERR_COMM)
        const unsigned long long want = (unsigned long long)P.nranks * (ep + 1);
        const unsigned long long *flag = xb_flag(P, P.peers[P.rank]);
        // the global nanosecond timer: an SM's clock64 is not comparable across
        // a preemption that resumes the CTA on another SM
        const unsigned long long t0 = gtimer();
        while (ld_acquire_sys(flag) < want) {
            if (gtimer() - t0 > 20000000000ull) {
                s_timeout = 1;
                break;
            }
            __nanosleep(64);
        }
        // every slot must carry this exchange's epoch tag: a mismatch (a rank
        // out of step) stops the run with PF_ERR_COMM instead of summing stale totals
        for (int r = 0; !s_timeout && r < P.nranks; ++r) {
            const long long tag = __double_as_longlong(__ldcg(&xb_slot(P, P.peers[P.rank], ep, r)[2 * P.I.E + 9]));
            if (tag != (long long)(ep + 1)) {
                s_timeout = 2;
                if (atomicCAS(&g_xdebug[0], 0ull, ep + 1) == 0ull) {
                    g_xdebug[1] = (unsigned long long)r;
                    g_xdebug[2] = (unsigned long long)tag;
                    g_xdebug[3] = (unsigned long long)c.iteration;
                    g_xdebug[4] = ld_acquire_sys(flag);
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_timeout) c.status = PF_ERR_COMM;
        c.xepoch = ep + 1;
    }
    __syncthreads();
}

// Sum of slot values over the ranks in rank order (identical on every rank).
__device__ __forceinline__ double xsum(const Params &P, uint64_t ep, int64_t off) {
    double v = __ldcg(&xb_slot(P, P.peers[P.rank], ep, 0)[off]);
    for (int r = 1; r < P.nranks; ++r) v += __ldcg(&xb_slot(P, P.peers[P.rank], ep, r)[off]);
    return v;
}

// kernels.py:212 and :94-96 from the exchanged totals of the last exchange
__device__ __noinline__ void xchg_edge_apply(const Params &P, const Ctrl &c, double f) {
    const InstView &I = P.I;
    const uint64_t ep = c.xepoch - 1;
    const int ngroups = (I.E + RGRP - 1) / RGRP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int grp = blockIdx.x * NW + warp; grp < ngroups; grp += P.G * NW) {
        const int e = grp * RGRP + lane;
        if (e < I.E) {
            const double T = xsum(P, ep, e), L = xsum(P, ep, I.E + e);
            const double cap = I.capacity[e];
            const double dold = __ldcg(&P.dc[e]) * f;
            const double dnew = npmax0(dold + (L - cap));
            double adj = (T + dnew - cap) / (P.ne[e] + 1.0);
            if (adj < 0.0) adj = 0.0;
            P.dc[e] = dnew;
            P.adj[e] = adj;
            const double d = dnew - dold;
            res_dc_write(P, c)[e] = d * d;
        }
    }
}

// controller_eval from the exchanged residual sums (every CTA, same result)
__device__ void xchg_controller_eval(const Params &P, Ctrl &c) {
    const double dcs = dcs_block(res_dc_read(P, c), P.I.E);
    if (threadIdx.x == 0) {
        const uint64_t ep = c.xepoch - 1;
        const int64_t b = 2 * (int64_t)P.I.E;
        const int par = (int)(c.iteration & 1);
        const double dx = xsum(P, ep, b + 0), rdd = xsum(P, ep, b + 1 + 3 * par),
                     rdcon = xsum(P, ep, b + 2 + 3 * par), rdn = xsum(P, ep, b + 3 + 3 * par);
        const bool fc = xsum(P, ep, b + 7) > 0.0, fr = xsum(P, ep, b + 8) > 0.0;
        const int32_t ec = fc ? (__ldcg(&P.err[0]) != INT_MAX ? __ldcg(&P.err[0]) : -1) : INT_MAX;
        const int32_t er = fr ? (__ldcg(&P.err[1]) != INT_MAX ? __ldcg(&P.err[1]) : -1) : INT_MAX;
        if (!c.status) controller_step(P, c, sqrt(dx), sqrt(((rdd + dcs) + rdcon) + rdn), ec, er);
    }
    __syncthreads();
}

// ------------------------------------------------------------------ kernels

// DIST: the multi-GPU variant with the in-kernel peer-memory exchange (a
// separate instantiation keeps the single-GPU kernel's registers untouched)
template <bool DIST>
__global__ void __launch_bounds__(NT, PF_MINB) k_fused(const __grid_constant__ Params P) {
    extern __shared__ __align__(128) char smem_raw[];
    __shared__ Ctrl c;
    __shared__ CtaShared cs;
    cg::grid_group grid = cg::this_grid();
    cta_init(cs);
    uint32_t seq = 0;
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    constexpr bool dist = DIST;
    if (c.need_a1) {
        (P.run_slots ? pass_tiles<MODE_A1, true>(P, c, smem_raw, cs, seq) : pass_tiles<MODE_A1, false>(P, c, smem_raw, cs, seq));
        grid.sync();
        if (dist) xchg_phase(P, c, grid);
        if (threadIdx.x == 0) {
            c.need_a1 = 0;
            c.db ^= 1;
            c.need_edge = 1;
            c.f = 1.0;
        }
        __syncthreads();
    }
    // CTA 0 sums its phase times into g_probe[0..4]; every CTA's per-phase time
    // also goes into a running maximum over CTAs, summed per iteration in g_probe[5..7]
    // (edge, pass, controller) by CTA 0 (approximate: the max of the previous iteration)
    const bool prb = P.probe && threadIdx.x == 0;
    unsigned long long pt = prb ? gtimer() : 0;
    auto mark = [&](int i) {
        if (prb) {
            const unsigned long long t = gtimer();
            if (blockIdx.x == 0) g_probe[i] += t - pt;
            const int slot = i == 0 ? 0 : i == 2 ? 1 : i == 4 ? 2 : -1;
            if (slot >= 0) atomicMax(&g_pmax[slot], t - pt);
            pt = t;
        }
    };
    for (;;) {
        // the pending edge phase belongs to the next iteration: run it only when
        // continuing, so a stopped / paused state keeps adj_k for export
        if (c.stopped || c.status || c.iteration >= c.target || c.iteration >= P.max_iterations) break;
        if (c.need_edge) {
            if (dist)
                xchg_edge_apply(P, c, c.f);
            else
                (P.ebound ? edge_phase_rs(P, c.f, res_dc_write(P, c)) : edge_phase(P, c.f, res_dc_write(P, c)));
            mark(0);
            grid.sync();
            mark(1);
            __syncthreads();
            if (threadIdx.x == 0) {
                c.need_edge = 0;
                c.f = 1.0;
            }
            __syncthreads();
        }
        (P.run_slots ? pass_tiles<MODE_M, true>(P, c, smem_raw, cs, seq) : pass_tiles<MODE_M, false>(P, c, smem_raw, cs, seq));
        mark(2);
        grid.sync();
        mark(3);
        __syncthreads();
        if (threadIdx.x == 0) {
            c.iteration += 1;
            c.alpha_used = c.alpha;
            c.beta_used = c.beta;
            c.xc ^= 1;
            c.db ^= 1;
        }
        __syncthreads();
        if (dist) {
            xchg_phase(P, c, grid);
            xchg_controller_eval(P, c);
        } else {
            controller_eval(P, c);
        }
        mark(4);
        if (!c.stopped && !c.status && c.f != c.fspec) {
            if (threadIdx.x == 0) c.rollbacks += 1;
            (P.run_slots ? pass_tiles<MODE_RB, true>(P, c, smem_raw, cs, seq) : pass_tiles<MODE_RB, false>(P, c, smem_raw, cs, seq));
            grid.sync();
            if (dist) xchg_phase(P, c, grid);
        }
        __syncthreads();
        if (threadIdx.x == 0) c.need_edge = 1;
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *P.ctrl = c;
        if (dist) *P.xepoch = c.xepoch;
    }
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
__global__ void __launch_bounds__(NT, PF_MINB) k_pass(const __grid_constant__ Params P) {
    extern __shared__ __align__(128) char smem_raw[];
    __shared__ Ctrl c;
    __shared__ CtaShared cs;
    cta_init(cs);
    uint32_t seq = 0;
    if (threadIdx.x == 0) c = *P.ctrl;
    __syncthreads();
    (P.run_slots ? pass_tiles<MODE, true>(P, c, smem_raw, cs, seq) : pass_tiles<MODE, false>(P, c, smem_raw, cs, seq));
}

// CTA partials -> rank totals in the single-GPU association (one warp per
// edge): tot[0:E] = T, tot[E:2E] = L, tot[2E + 0..6] = residual slots summed
// over the CTAs (lane-strided, shuffle tree: controller_eval's order),
// tot[2E + 7/8] = error flags.
__global__ void __launch_bounds__(NT) k_local_reduce(const __grid_constant__ Params P) {
    const int E = P.I.E;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = blockIdx.x + gridDim.x * warp; e < E; e += gridDim.x * (NT / 32)) {
        double T, L;
        edge_totals(P, e, lane, T, L);
        if (lane == 0) {
            P.tot[e] = T;
            P.tot[E + e] = L;
        }
    }
    if (blockIdx.x == 0 && warp == 0) {
        double acc[7];
        const int off[7] = {0, 1, 2, 3, 4, 5, 6};
        res_sums<7>(P.res, P.G, lane, off, acc);
        for (int j = 0; j < 7; ++j)
            for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_down_sync(FULL, acc[j], o);
        if (lane == 0) {
            for (int j = 0; j < 7; ++j) P.tot[2 * E + j] = acc[j];
            P.tot[2 * E + 7] = __ldcg(&P.err[0]) != INT_MAX ? 1.0 : 0.0;
            P.tot[2 * E + 8] = __ldcg(&P.err[1]) != INT_MAX ? 1.0 : 0.0;
        }
    }
}

// controller step from the allreduced totals (one thread).  Inside the
// per-run CUDA graph it also sets the graph's conditions: run the rollback
// branch, continue the iteration loop.
__global__ void __launch_bounds__(NT) k_ctrl_dist(const __grid_constant__ Params P,
                                                  cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_rb,
                                                  int in_graph) {
    // dual_capacity is replicated: its residual is rank-local and identical
    const double dcs = dcs_block(P.res_dc, P.I.E);  // the whole CTA
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
    const int32_t ec = t[7] > 0.0 ? (P.err[0] != INT_MAX ? P.err[0] : -1) : INT_MAX;
    const int32_t er = t[8] > 0.0 ? (P.err[1] != INT_MAX ? P.err[1] : -1) : INT_MAX;
    controller_step(P, c, sqrt(t[0]), sqrt(((t[1 + 3 * par] + dcs) + t[2 + 3 * par]) + t[3 + 3 * par]), ec, er);
    c.need_edge = 1;
    *P.ctrl = c;
    if (in_graph) {
        const bool live = !c.stopped && !c.status;
        cudaGraphSetConditional(h_rb, live && c.f != c.fspec ? 1u : 0u);
        cudaGraphSetConditional(h_loop, live && c.iteration < c.target && c.iteration < P.max_iterations ? 1u : 0u);
    }
}

// kernels.py:212 and :94-96 from the allreduced per-edge totals (one thread per edge)
__global__ void k_edge_dist(const __grid_constant__ Params P) {
    const int E = P.I.E;
    const int e = blockIdx.x * RGRP + threadIdx.x;
    const double f = P.ctrl->f;
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
        P.res_dc[e] = d * d;
    }
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

// Export helpers (reference pair order), for the state of the last completed
// iteration k: x_k in x[xc], x_{k-1} in x[xc^1], duals_k in buffer db^1 (db
// holds the speculative duals_{k+1}), adj_k, rescale factor f_k pending.
__global__ void k_export_pairs(const __grid_constant__ Params P, const int32_t *pair_slot, double *y_out,
                               double *dcon_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.I.NP) return;
    const Ctrl c = *P.ctrl;
    const int sl = pair_slot[t];
    const int p = P.I.pair_path[t];
    if (c.iteration == 0) {
        if (y_out) y_out[t] = P.x[c.xc][p];
        if (dcon_out) dcon_out[t] = 0.0;
        return;
    }
    const double dk = P.dcon[c.db ^ 1][sl];
    if (y_out) y_out[t] = max0(P.x[c.xc ^ 1][p] + dk - P.adj[P.I.pair_edge[t]]);
    if (dcon_out) dcon_out[t] = dk * c.f;
}

__global__ void k_scaled_copy(const double *a, int64_t n, const Ctrl *ctrl, double *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = ctrl->iteration == 0 ? a[i] : a[i] * ctrl->f;
}

// ------------------------------------------------------------------ host side

// Pack commodities into groups (<= GPATH paths, one warp) and groups into tiles
// (<= NW groups, <= tps pairs), then write each tile's metadata block.
bool fast_supported(const pf_instance *inst, std::string *why) {
    std::lock_guard<std::mutex> lk(inst->ws_mu);
    if (inst->fast_ok < 0) {
        const Index &I = *inst->idx;
        std::string w;
        if (I.E > 65535) {
            w = "more than 65535 edges (u16 edge ids)";
        } else if (I.NP >= ((int64_t)1 << 30)) {
            w = "more than 2^30 demand-path pairs";
        } else {
            std::vector<int32_t> cpp(I.C + 1), pptr(I.P + 1);
            d2h(cpp.data(), I.com_path_ptr.p, I.C + 1, inst->stream);
            d2h(pptr.data(), I.pair_ptr.p, I.P + 1, inst->stream);
            PF_CUDA(cudaStreamSynchronize(inst->stream));
            for (int64_t c = 0; c < I.C && w.empty(); ++c) {
                if (cpp[c + 1] - cpp[c] > GPATH)
                    w = "commodity " + std::to_string(c) + " has more than " + std::to_string(GPATH) + " paths";
                else if (pptr[cpp[c + 1]] - pptr[cpp[c]] > 16384)
                    w = "commodity " + std::to_string(c) + " has more than 16384 demand-path pairs";
            }
        }
        inst->fast_ok = w.empty() ? 1 : 0;
        inst->fast_why = w;
    }
    if (why) *why = inst->fast_why;
    return inst->fast_ok == 1;
}

static std::shared_ptr<TileLayout> build_tiles(const pf_instance *inst, cudaStream_t s) {
    const Index &I = *inst->idx;
    std::vector<int32_t> cpp(I.C + 1), pptr(I.P + 1), pedge(I.NP);
    d2h(cpp.data(), I.com_path_ptr.p, I.C + 1, s);
    d2h(pptr.data(), I.pair_ptr.p, I.P + 1, s);
    d2h(pedge.data(), I.pair_edge.p, I.NP, s);
    PF_CUDA(cudaStreamSynchronize(s));
    require(I.E <= 65535, "fast mode supports up to 65535 edges (u16 edge ids)");
    auto L = std::make_shared<TileLayout>();
    int64_t max_com_pairs = 0;
    for (int64_t c = 0; c < I.C; ++c) {
        require(cpp[c + 1] - cpp[c] <= GPATH, "fast mode supports at most " + std::to_string(GPATH) +
                                                  " paths per commodity (commodity " + std::to_string(c) + ")");
        max_com_pairs = std::max<int64_t>(max_com_pairs, pptr[cpp[c + 1]] - pptr[cpp[c]]);
    }
    int64_t hmax = 0;  // most hops of one path
    for (int64_t p = 0; p < I.P; ++p) hmax = std::max<int64_t>(hmax, pptr[p + 1] - pptr[p]);
    require(hmax < 65535, "fast mode supports paths of at most 65534 hops");
    const int hbmax = (int)(NW * (hmax + 1));
    L->hbmax = hbmax;
    // largest tile (<= TPS_MIN pairs) that keeps two CTAs per SM with this
    // instance's per-edge tables; PF_FAST_TPS overrides (tuning)
    int64_t tps_min = TPS_MIN;
    {
        int per_sm = 0, reserved = 0;
        PF_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, inst->device()));
        PF_CUDA(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, inst->device()));
        // static shared memory of the kernels (CtaShared, Ctrl, ...), queried
        int64_t stat = 0;
        {
            cudaFuncAttributes fa{};
            PF_CUDA(cudaFuncGetAttributes(&fa, k_fused<false>));
            stat = (int64_t)fa.sharedSizeBytes;
            PF_CUDA(cudaFuncGetAttributes(&fa, k_fused<true>));
            stat = std::max<int64_t>(stat, (int64_t)fa.sharedSizeBytes);
            PF_CUDA(cudaFuncGetAttributes(&fa, k_pass<MODE_M>));
            stat = std::max<int64_t>(stat, (int64_t)fa.sharedSizeBytes);
        }
        const int64_t budget = per_sm / PF_MINB - reserved - stat;
        // large E: the per-edge tables leave room for no tile of 2,048 pairs
        const bool large_e = smem_plan(2048, (int)I.E, 1, hbmax).total > budget || getenv("PF_FAST_LARGE_E");
        // run slots: default for large E (no per-edge shared-memory tables, so two
        // CTAs per SM at any E); PF_FAST_RS=1 / 0 forces them on / off (tuning)
        const char *rs_env = getenv("PF_FAST_RS");
        L->run_slots = rs_env ? atoi(rs_env) != 0 : large_e;
        if (L->run_slots) {
            // the per-tile run tables are sized by the layout's most runs per tile
            // (known after the build); a quarter of the tile's pairs for the search
            // (config 2: 270 runs per 2,345-pair tile, config 3: 394 per 2,846)
            L->adj_smem = L->acc_smem = false;
            tps_min = TPS_CAP;
            while (tps_min > 1024 &&
                   smem_plan((int)tps_min, (int)I.E, 1, hbmax, false, false, true,
                             (int)std::min<int64_t>(I.E, tps_min / 4)).total > budget)
                tps_min -= 64;
        } else if (large_e) {
            // large E: the shared-memory edge tables rule out two CTAs per SM; the
            // adjustment table is read through L1 (one CTA per SM, large tiles), or
            // the run totals also move to the CTA's private partial rows in L2
            // (read-modify-write by one thread per run, tiles separated by block
            // barriers: deterministic) for two CTAs per SM
            // (measured at config 3: shared-memory accumulators at one CTA per SM
            // 11.4 ms/iteration, L2 rows at two CTAs per SM 12.5 ms: the row
            // read-modify-writes cost more than the second CTA gains;
            // PF_FAST_ACC_L2=1 selects the L2 rows)
            L->adj_smem = false;
            if (getenv("PF_FAST_ACC_L2")) {
                L->acc_smem = false;
                while (tps_min > 512 && smem_plan((int)tps_min, (int)I.E, 1, hbmax, false, false).total > budget)
                    tps_min -= 256;
            } else {
                const int64_t budget1 = per_sm - reserved - stat;
                while (tps_min > 512 && smem_plan((int)tps_min, (int)I.E, 1, hbmax, false).total > budget1)
                    tps_min -= 256;
            }
        } else {
            // the largest tile that keeps two CTAs per SM: fewer, larger tiles cut
            // the per-tile fixed costs (config 2: 2,560 pairs 307 us/iteration,
            // 2,816 pairs 302 us; one more pair-row and only one CTA fits)
            tps_min = TPS_CAP;
            while (tps_min > 1024 && smem_plan((int)tps_min, (int)I.E, 1, hbmax).total > budget) tps_min -= 64;
        }
    }
    {  // small instances: smaller tiles so that the tiles fill the grid (per-tile latency
       // bounds an iteration when every CTA holds one tile).  Measured plateau:
       // NP / (3 SMs) pairs per tile, at least 512 (cfg1 15.8 us/iteration at 512,
       // 17.3 at 256; the 630k-pair 150-node instance 29.6-30.2 us at 1,280-1,664)
        int sms = 148;
        PF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, inst->device()));
        const int64_t fill = (I.NP / (3 * (int64_t)sms) + 63) / 64 * 64;
        tps_min = std::min<int64_t>(tps_min, std::max<int64_t>(512, fill));
    }
    if (const char *v = getenv("PF_FAST_TPS")) tps_min = std::max(256, atoi(v)) / 64 * 64;
    const int64_t tps = std::max<int64_t>(tps_min, (max_com_pairs + 63) / 64 * 64);
    require(tps <= 16384, "a commodity has too many demand-path pairs for a fast-mode tile");
    L->tps = (int32_t)tps;
    // paths per group: as many as lets NW groups of mean-length paths fill a tile
    // (k = 8, 9.2 hops: 3 commodities = 24 paths = ~220 pairs per warp)
    int64_t max_paths = 1;
    for (int64_t c = 0; c < I.C; ++c) max_paths = std::max<int64_t>(max_paths, cpp[c + 1] - cpp[c]);
    while (L->kspan < max_paths) L->kspan <<= 1;
    const double mean_hops = I.P ? (double)I.NP / (double)I.P : 1.0;
    const int64_t gmax = std::min<int64_t>(GPATH, std::max<int64_t>(max_paths, (int64_t)(tps / (NW * mean_hops * 1.08))));
    // groups
    std::vector<int32_t> gstart;  // first commodity of each group
    {
        int32_t c = 0;
        while (c < I.C) {
            gstart.push_back(c);
            const int32_t c0 = c;
            while (c < I.C) {
                const int64_t npath = cpp[c + 1] - cpp[c0];
                const int64_t npair = pptr[cpp[c + 1]] - pptr[cpp[c0]];
                if (c > c0 && (npath > gmax || npair > tps)) break;
                ++c;
            }
        }
        gstart.push_back((int32_t)I.C);
    }
    // tiles: up to NW groups and tps pairs each.  Tile t goes to CTA t mod G, so
    // with n0 greedy tiles the busiest CTA holds ceil(n0 / G) of them; packing
    // T = ceil(n0 / G) * G tiles instead (group caps spread evenly) gives every
    // CTA the same count of smaller tiles: its load drops from
    // ceil(n0 / G) * NP / n0 to NP / G pairs (config 2: 7,835 -> 7,992 tiles)
    const int64_t ng = (int64_t)gstart.size() - 1;
    auto tile_end = [&](int64_t gi, int64_t cap) {
        const int32_t c0 = gstart[gi];
        int64_t gj = gi;
        while (gj < ng && gj - gi < cap) {
            const int64_t npair = pptr[cpp[gstart[gj + 1]]] - pptr[cpp[c0]];
            if (gj > gi && npair > tps) break;
            ++gj;
        }
        return gj;
    };
    int64_t target = 0;
    {
        int64_t n0 = 0;
        for (int64_t gi = 0; gi < ng; gi = tile_end(gi, NW)) ++n0;
        int sms = 148;
        PF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, inst->device()));
        const int64_t ctas = (int64_t)sms * (L->acc_smem || L->run_slots ? PF_MINB : 1);  // CTAs per SM of this layout
        // only with several tiles per CTA (measured: 500-node k=4, 13.2 -> 14 tiles
        // per CTA, 163.7 -> 161.4 us; config 2 unchanged; 1.6 -> 2 per CTA no gain)
        if (n0 >= 4 * ctas && !getenv("PF_FAST_NO_BALANCE")) target = (n0 + ctas - 1) / ctas * ctas;
    }
    std::vector<TileDesc> tiles;
    std::vector<std::array<int32_t, NW + 1>> tgroups;  // group commodity boundaries per tile
    int64_t slot = 0, mb = 0;
    std::vector<int32_t> emark(I.E > 0 ? I.E : 1, -1);  // tile stamp per edge: counts a tile's runs
    {
        int64_t gi = 0;
        while (gi < ng) {
            const int32_t c0 = gstart[gi];
            const int64_t left = target - (int64_t)tiles.size();
            const int64_t cap = target && left > 0 ? std::min<int64_t>(NW, (ng - gi + left - 1) / left) : NW;
            int64_t gj = gi;
            while (gj < ng && gj - gi < cap) {
                const int64_t npair = pptr[cpp[gstart[gj + 1]]] - pptr[cpp[c0]];
                if (gj > gi && npair > tps) break;
                ++gj;
            }
            std::array<int32_t, NW + 1> gb;
            for (int k = 0; k <= NW; ++k) gb[k] = gstart[std::min<int64_t>(gi + k, gj)];
            const int32_t c1 = gstart[gj];
            TileDesc d;
            d.c0 = c0;
            d.c1 = c1;
            d.p0 = cpp[c0];
            d.p1 = cpp[c1];
            d.t0 = pptr[d.p0];
            d.np = pptr[d.p1] - d.t0;
            d.sb = (int32_t)slot;
            require(mb / 16 < INT_MAX, "fast-mode metadata exceeds 32 GB");
            d.mb16 = (int32_t)(mb / 16);
            d.nrun = 0;
            d.nhb = 0;
            for (int k = 0; k < NW; ++k) {  // hop steps of each group + its end
                int64_t H = 0;
                for (int32_t p = cpp[gb[k]]; p < cpp[gb[k + 1]]; ++p) H = std::max<int64_t>(H, pptr[p + 1] - pptr[p]);
                d.nhb += (int32_t)H + 1;
            }
            for (int32_t t = d.t0; t < d.t0 + d.np; ++t)
                if (emark[pedge[t]] != (int32_t)tiles.size()) {
                    emark[pedge[t]] = (int32_t)tiles.size();
                    ++d.nrun;
                }
            tiles.push_back(d);
            tgroups.push_back(gb);
            slot += (d.np + SLOT_ALIGN - 1) / SLOT_ALIGN * SLOT_ALIGN;
            mb += meta_off(d.np, d.p1 - d.p0, d.c1 - d.c0, d.nrun, d.nhb, L->run_slots).bytes;
            require(slot < INT_MAX, "too many demand-path pairs for fast mode");
            gi = gj;
        }
    }
    L->ntiles = (int32_t)tiles.size();
    L->nslots = slot;
    L->meta_bytes = mb;
    std::vector<uint8_t> meta(mb ? mb : 16, 0);
    std::vector<int32_t> pair_slot(I.NP);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t ti = 0; ti < (int64_t)tiles.size(); ++ti) {
        const TileDesc &T = tiles[ti];
        const int np = T.np, npath = T.p1 - T.p0, nc = T.c1 - T.c0;
        const MetaOff m = meta_off(np, npath, nc, T.nrun, T.nhb, L->run_slots);
        uint8_t *blk = meta.data() + (int64_t)T.mb16 * 16;
        uint16_t *eid = (uint16_t *)(blk + m.eid);
        std::vector<uint16_t> perm(np);
        uint16_t *poff = (uint16_t *)(blk + m.poff);
        uint8_t *pcom = blk + m.pcom;
        uint16_t *lcpp = (uint16_t *)(blk + m.cpp);
        uint16_t *gpath = (uint16_t *)(blk + m.gpath);
        for (int i = 0; i < npath; ++i) poff[i] = (uint16_t)(pptr[T.p0 + i] - T.t0);
        poff[npath] = (uint16_t)np;
        for (int k = 0; k <= NW; ++k) gpath[k] = (uint16_t)(cpp[tgroups[ti][k]] - T.p0);
        // hop-major order within each group: the group's paths take the hop lanes
        // by decreasing hop count (stable), and step j holds the j-th pair of
        // every path with more than j hops, in hop-lane order (the kernel's
        // hops_y / hops_dcon): the lanes active at step j are a prefix
        uint16_t *hbo = (uint16_t *)(blk + m.hbo);
        uint16_t *hb = (uint16_t *)(blk + m.hb);
        uint8_t *hperm = blk + m.hperm;
        uint8_t *hinv = blk + m.hinv;
        int hbn = 0;
        std::vector<int> ord;
        for (int k = 0; k < NW; ++k) {
            const int g0 = gpath[k], g1 = gpath[k + 1];
            ord.clear();
            for (int i = g0; i < g1; ++i) ord.push_back(i);
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
                return poff[a + 1] - poff[a] > poff[b + 1] - poff[b];
            });
            for (int i = 0; i < (int)ord.size(); ++i) {
                hperm[g0 + i] = (uint8_t)(ord[i] - g0);
                hinv[ord[i]] = (uint8_t)i;
            }
            const int H = ord.empty() ? 0 : poff[ord[0] + 1] - poff[ord[0]];
            int pos = g0 < npath ? poff[g0] : np;
            hbo[k] = (uint16_t)hbn;
            hb[hbn++] = (uint16_t)pos;
            for (int j = 0; j < H; ++j) {
                for (int i = 0; i < (int)ord.size(); ++i) {
                    const int pth = ord[i];
                    if (poff[pth + 1] - poff[pth] <= j) break;  // a prefix of the hop lanes
                    const int l = poff[pth] + j;              // tile-local reference pair
                    eid[pos] = (uint16_t)pedge[T.t0 + l];
                    pair_slot[T.t0 + l] = T.sb + pos;
                    ++pos;
                }
                hb[hbn++] = (uint16_t)pos;
            }
        }
        hbo[NW] = (uint16_t)hbn;
        require(hbn == T.nhb, "fast layout: hop-step count mismatch");
        for (int l = 0; l < np; ++l) perm[l] = (uint16_t)l;
        std::stable_sort(perm.begin(), perm.end(), [&](uint16_t a, uint16_t b) { return eid[a] < eid[b]; });
        // edge runs: sperm = pairs sorted by (edge, pair), the runs back to back
        uint16_t *sperm = (uint16_t *)(blk + m.sperm);
        std::vector<int> rstart;
        require(np <= 0x7fff, "fast layout: more than 32,767 pairs in a tile");
        for (int sl = 0; sl < np; ++sl) {
            const bool start = sl == 0 || eid[perm[sl]] != eid[perm[sl - 1]];
            sperm[sl] = (uint16_t)(perm[sl] | (start ? 0x8000 : 0));  // bit 15: a run starts here
            if (start) rstart.push_back(sl);
        }
        const int nr = (int)rstart.size();
        require(nr == T.nrun, "fast layout: run count mismatch");
        rstart.push_back(np);
        {  // the walk's chunks (tile_compute step 5: cs items per thread): for each
           // chunk whose last item's run began inside it and continues, the number
           // of following chunks that run reaches (their head pieces are added
           // to it in chunk order)
            uint16_t *xlen = (uint16_t *)(blk + m.xlen);
            const int cs = std::max((np + NT - 1) / NT, 4);
            int r = 0;
            for (int t = 0; t < NT; ++t) {
                xlen[t] = 0;
                const int a = t * cs, b = std::min(a + cs, np);
                if (a >= b) continue;
                while (rstart[r + 1] <= b - 1) ++r;  // the run holding item b - 1
                const int s0 = rstart[r], s1 = rstart[r + 1];
                if (s0 >= a && s1 > b) xlen[t] = (uint16_t)((s1 - b + cs - 1) / cs);
            }
        }
        if (L->run_slots) {  // the run's edge; the per-pair u16 becomes the pair's run
            uint16_t *redge = (uint16_t *)(blk + m.redge);
            for (int r = 0; r < nr; ++r) redge[r] = eid[sperm[rstart[r]] & 0x7fff];
            for (int r = 0; r < nr; ++r)
                for (int sl = rstart[r]; sl < rstart[r + 1]; ++sl) eid[sperm[sl] & 0x7fff] = (uint16_t)r;
        }
        for (int j = 0; j < nc; ++j) {
            lcpp[j] = (uint16_t)(cpp[T.c0 + j] - T.p0);
            for (int32_t p = cpp[T.c0 + j]; p < cpp[T.c0 + j + 1]; ++p) pcom[p - T.p0] = (uint8_t)j;
        }
        lcpp[nc] = (uint16_t)npath;
    }
    if (L->run_slots) {
        // edge-major slots: edge e's (tile, run) totals at eoff[e] .. eoff[e + 1] in
        // tile order (the edge phase sums them in that order: deterministic)
        std::vector<int32_t> eoff(I.E + 1, 0);
        int64_t total = 0;
        for (const TileDesc &T : tiles) {
            const MetaOff m = meta_off(T.np, T.p1 - T.p0, T.c1 - T.c0, T.nrun, T.nhb, true);
            const uint16_t *redge = (const uint16_t *)(meta.data() + (int64_t)T.mb16 * 16 + m.redge);
            for (int r = 0; r < T.nrun; ++r) ++eoff[redge[r] + 1];
            total += T.nrun;
            L->rmax = std::max(L->rmax, T.nrun);
        }
        require(total < INT_MAX, "too many (tile, run) slots for fast mode");
        for (int64_t e = 0; e < I.E; ++e) eoff[e + 1] += eoff[e];
        std::vector<int32_t> cur(eoff.begin(), eoff.end() - 1);
        for (const TileDesc &T : tiles) {
            const MetaOff m = meta_off(T.np, T.p1 - T.p0, T.c1 - T.c0, T.nrun, T.nhb, true);
            uint8_t *blk = meta.data() + (int64_t)T.mb16 * 16;
            const uint16_t *redge = (const uint16_t *)(blk + m.redge);
            uint32_t *rdst = (uint32_t *)(blk + m.rdst);
            for (int r = 0; r < T.nrun; ++r) rdst[r] = (uint32_t)cur[redge[r]]++;
        }
        L->nruns = total;
        L->eoff.alloc(I.E + 1);
        h2d(L->eoff.p, eoff.data(), I.E + 1, s);
    }
    // compulsory HBM bytes of one M pass: what the bulk copies read plus what the pass writes
    int64_t bytes = 0;
    for (const TileDesc &d : tiles) {
        const int npath = d.p1 - d.p0, nc = d.c1 - d.c0;
        const int npa = even(d.p1 - (d.p0 & ~1)), nca = even(d.c1 - (d.c0 & ~1));
        bytes += 8LL * even(d.np) + meta_off(d.np, npath, nc, d.nrun, d.nhb, L->run_slots).bytes + 16LL * npa +
                 16LL * nca;  // reads
        bytes += 8LL * d.np + 16LL * npath + 8LL * nc;                                            // writes
        if (L->run_slots) bytes += 2 * 16LL * d.nrun;  // the run totals written, read back by the edge phase
    }
    L->bytes_per_pass = bytes;
    L->desc.alloc(tiles.size() ? tiles.size() : 1);
    L->meta.alloc(meta.size());
    L->pair_slot.alloc(I.NP ? I.NP : 1);
    h2d(L->desc.p, tiles.data(), tiles.size(), s);
    h2d(L->meta.p, meta.data(), meta.size(), s);
    h2d(L->pair_slot.p, pair_slot.data(), I.NP, s);
    PF_CUDA(cudaStreamSynchronize(s));
    if (getenv("PF_FAST_DEBUG"))
        fprintf(stderr, "[fast layout] tps %d gmax %lld tiles %d run_slots %d rmax %d hbmax %d nruns %lld meta %lld B\n",
                L->tps, (long long)gmax, L->ntiles, (int)L->run_slots, L->rmax, L->hbmax, (long long)L->nruns,
                (long long)L->meta_bytes);
    L->h_desc = std::move(tiles);
    return L;
}

struct FastSolver {
    const pf_instance *inst;
    pf_config cfg;
    std::shared_ptr<TileLayout> L;
    int G = 0, nbuf = 1;
    size_t smem = 0;
    DevBuf<double> dcon[2], dn[2], dd[2], x[2];
    DevBuf<double> D, dc, adj, ne, tot, partT, partL, res, res_dc, root_sums, slots;
    DevBuf<int32_t> err, cta_ptr, cta_tiles, ebound;
    DevBuf<Ctrl> ctrl;
    Params P{};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int64_t launches = 0;
    const CommOps *comm = nullptr;
    // multi-GPU: one CUDA graph per run (WHILE over the iteration body, IF for the rollback)
    cudaGraph_t dgraph = nullptr;
    cudaGraphExec_t dexec = nullptr;
    int dgraph_state = 0;  // 0 untried, 1 built, -1 unavailable (host-driven loop)
    // multi-GPU over peer memory (CUDA IPC): see xchg_phase
    int rank = 0, nranks = 0;
    DevBuf<double> xb;                       // this rank's exchange buffer
    DevBuf<double *> peers_dev;              // [nranks] peer bases
    std::vector<void *> opened;              // IPC mappings to close
    DevBuf<unsigned long long> xepoch;       // exchanges done
    // per-solve scratch kept with the (pooled) solver: warm-start staging, outputs
    DevBuf<double> x0stage, rates_out, sums_out, flag;
    DevBuf<char> snap;  // fast_snapshot's copy of the dynamic state
};

static void fast_set_config(FastSolver *F, const pf_config &cfg) {
    const Index &I = *F->inst->idx;
    F->cfg = cfg;
    if (cfg.trace && !F->root_sums.p) F->root_sums.alloc(I.C ? I.C : 1);
    Params &P = F->P;
    P.root_sums = cfg.trace ? F->root_sums.p : nullptr;
    P.gamma = cfg.gamma;
    P.residual_ratio = cfg.residual_ratio;
    P.beta_scale = cfg.beta_scale;
    P.beta_min = cfg.beta_min;
    P.beta_max = cfg.beta_max;
    P.alpha_target = cfg.alpha_target;
    P.max_iterations = cfg.max_iterations;
    P.adapt = cfg.adapt;
}

static void pool_free(void *p) { fast_destroy((FastSolver *)p); }

void fast_release(FastSolver *F) {
    if (!F) return;
    if (!F->comm && !F->nranks) {
        std::lock_guard<std::mutex> lk(F->inst->ws_mu);
        if (!F->inst->fast_pool) {
            F->inst->fast_pool = F;
            F->inst->fast_pool_free = pool_free;
            return;
        }
    }
    fast_destroy(F);
}

static const cudaDeviceProp &device_props(int dev) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<cudaDeviceProp>> props;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)props.size() <= dev) props.resize(dev + 1);
    if (!props[dev]) {
        props[dev].reset(new cudaDeviceProp());
        PF_CUDA(cudaGetDeviceProperties(props[dev].get(), dev));
    }
    return *props[dev];
}

FastSolver *fast_create(const pf_instance *inst, const pf_config &cfg, cudaStream_t s) {
    const Index &I = *inst->idx;
    {  // reuse the instance's idle solver (same index spaces and layout)
        FastSolver *pooled = nullptr;
        {
            std::lock_guard<std::mutex> lk(inst->ws_mu);
            pooled = (FastSolver *)inst->fast_pool;
            inst->fast_pool = nullptr;
        }
        if (pooled) {
            fast_set_config(pooled, cfg);
            pooled->launches = 0;
            return pooled;
        }
    }
    std::unique_ptr<FastSolver> F(new FastSolver());
    F->inst = inst;
    F->cfg = cfg;
    {
        std::lock_guard<std::mutex> lk(inst->idx->tiles_mu);
        if (!inst->idx->tiles) inst->idx->tiles = build_tiles(inst, s);
        F->L = inst->idx->tiles;
    }
    F->nbuf = 1;  // measured: a second stage costs an SM's second CTA, which hides more
    if (const char *v = getenv("PF_FAST_NBUF")) F->nbuf = std::max(1, std::min(2, atoi(v)));
    F->smem = (size_t)smem_plan(F->L->tps, (int)I.E, F->nbuf, F->L->hbmax, F->L->adj_smem, F->L->acc_smem, F->L->run_slots,
                                F->L->rmax)
                  .total;
    int dev = inst->device();
    const cudaDeviceProp &prop = device_props(dev);
    const size_t static_smem = sizeof(Ctrl) + sizeof(CtaShared) + 64;
    require(F->smem + static_smem <= (size_t)prop.sharedMemPerBlockOptin,
            "fast mode: edge tables do not fit in shared memory (too many edges)");
    PF_CUDA(cudaFuncSetAttribute(k_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    PF_CUDA(cudaFuncSetAttribute(k_pass<MODE_A1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F->smem));
    int per_sm = 0;
    PF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused<false>, NT, F->smem));
    {  // the multi-GPU variant must be co-resident with the same grid
        int per_sm_d = 0;
        PF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_d, k_fused<true>, NT, F->smem));
        per_sm = std::min(per_sm, per_sm_d);
    }
    require(per_sm >= 1, "fast kernel does not fit on an SM");
    if (getenv("PF_FAST_DEBUG"))
        fprintf(stderr, "[fast layout] dynamic smem %zu B per CTA, %d CTAs per SM\n", F->smem, per_sm);
    int G = prop.multiProcessorCount * per_sm;
    G = std::max(1, std::min(G, F->L->ntiles));
    F->G = G;
    int64_t E = I.E ? I.E : 1;
    for (int b = 0; b < 2; ++b) {
        F->dcon[b].alloc(F->L->nslots + SLOT_ALIGN);
        F->dn[b].alloc(I.P + 2);
        F->dd[b].alloc(I.C + 2);
        F->x[b].alloc(I.P + 2);
    }
    F->D.alloc(I.C + 2);
    PF_CUDA(cudaMemsetAsync(F->D.p, 0, F->D.bytes(), s));
    if (I.C) PF_CUDA(cudaMemcpyAsync(F->D.p, inst->demand.p, sizeof(double) * I.C, cudaMemcpyDeviceToDevice, s));
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
    {  // static tile -> CTA assignment: round robin (tile g + k*G), so at any time
       // the grid works on one contiguous window of tiles (DRAM / L2 locality;
       // measured faster than a pair-balanced assignment)
        const int64_t nt = F->L->ntiles;
        std::vector<int32_t> ptr(G + 1, 0), flat;
        flat.reserve(nt);
        for (int g = 0; g < G; ++g) {
            for (int64_t t = g; t < nt; t += G) flat.push_back((int32_t)t);
            ptr[g + 1] = (int32_t)flat.size();
        }
        F->cta_ptr.alloc(G + 1);
        F->cta_tiles.alloc(flat.size() ? flat.size() : 1);
        h2d(F->cta_ptr.p, ptr.data(), G + 1, s);
        h2d(F->cta_tiles.p, flat.data(), flat.size(), s);
    }
    const size_t npart = F->L->run_slots ? 1 : (size_t)G * E;  // run slots hold the partials instead
    F->partT.alloc(npart);
    F->partL.alloc(npart);
    if (F->L->run_slots) F->slots.alloc(2 * (size_t)std::max<int64_t>(F->L->nruns, 1));
    F->res.alloc((size_t)G * 8);
    F->res_dc.alloc(2 * E);  // two halves by iteration parity (res_dc_write)
    F->err.alloc(2);
    F->ctrl.alloc(1);
    if (cfg.trace) F->root_sums.alloc(I.C ? I.C : 1);
    PF_CUDA(cudaEventCreate(&F->e0));
    PF_CUDA(cudaEventCreate(&F->e1));
    Params &P = F->P;
    P.I = inst->view();
    P.ntiles = F->L->ntiles;
    P.G = G;
    P.tps = F->L->tps;
    P.nbuf = F->nbuf;
    P.kspan = F->L->kspan;
    P.adj_smem = F->L->adj_smem ? 1 : 0;
    P.acc_smem = F->L->acc_smem ? 1 : 0;
    P.pf_dist = 1;
    if (const char *v = getenv("PF_FAST_PFDIST")) P.pf_dist = std::max(1, atoi(v));
    {
        double rcp[RCP_MAX + 1];
        rcp[0] = 0.0;
        for (int h = 1; h <= RCP_MAX; ++h) rcp[h] = 1.0 / (double)h;  // correctly rounded (IEEE division)
        PF_CUDA(cudaMemcpyToSymbolAsync(c_rcp, rcp, sizeof(rcp), 0, cudaMemcpyHostToDevice, s));
    }
    P.desc = F->L->desc.p;
    P.cta_ptr = F->cta_ptr.p;
    P.cta_tiles = F->cta_tiles.p;
    P.meta = F->L->meta.p;
    P.D = F->D.p;
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
    P.run_slots = F->L->run_slots ? 1 : 0;
    P.rmax = F->L->rmax;
    P.hbmax = F->L->hbmax;
    P.spec_f = !getenv("PF_FAST_SPEC") || atoi(getenv("PF_FAST_SPEC")) != 0;
    P.spec_margin = getenv("PF_FAST_SPEC_MARGIN") ? atof(getenv("PF_FAST_SPEC_MARGIN")) : 1.5;
    P.eoff = F->L->run_slots ? F->L->eoff.p : nullptr;
    P.ebound = nullptr;
    if (F->L->run_slots && !getenv("PF_FAST_RS_WARP_EDGES")) {
        // slot-balanced contiguous edge ranges, one per CTA (edge_phase_rs)
        std::vector<int32_t> eoff(I.E + 1), eb(G + 1, (int32_t)I.E);
        d2h(eoff.data(), F->L->eoff.p, I.E + 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        const int64_t tot = eoff[I.E];
        int64_t e = 0;
        for (int g = 0; g <= G; ++g) {
            const int64_t want = tot * g / G;
            while (e < I.E && eoff[e] < want) ++e;
            eb[g] = (int32_t)(g == G ? I.E : e);
        }
        eb[0] = 0;
        F->ebound.alloc(G + 1);
        h2d(F->ebound.p, eb.data(), G + 1, s);
        P.ebound = F->ebound.p;
    }
    P.slots = F->L->run_slots ? F->slots.p : nullptr;
    P.res = F->res.p;
    P.res_dc = F->res_dc.p;
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
    P.ablate = 0;
    if (const char *v = getenv("PF_FAST_ABLATE")) P.ablate = atoi(v);
    P.probe = getenv("PF_FAST_PROBE") ? 1 : 0;
    PF_CUDA(cudaStreamSynchronize(s));
    return F.release();
}

void fast_destroy(FastSolver *F) {
    if (!F) return;
    if (F->dexec) cudaGraphExecDestroy(F->dexec);
    if (F->dgraph) cudaGraphDestroy(F->dgraph);
    for (void *p : F->opened) cudaIpcCloseMemHandle(p);
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

// The iteration loop of a sharded solve as ONE CUDA graph:
//   WHILE (continue) {
//     k_edge_dist -> k_ctrl_update -> k_pass<M> -> k_local_reduce -> ncclAllReduce -> k_ctrl_dist
//     IF (beta changed) { k_pass<RB> -> k_local_reduce -> ncclAllReduce }
//   }
// k_ctrl_dist sets both conditions on the device, so a run of iterations has no
// host round trip (every rank evaluates the same controller on the same totals,
// so all ranks take the same branches and issue matching collectives).
static bool build_dist_graph(FastSolver *F, cudaStream_t s) {
    const Index &I = *F->inst->idx;
    const int64_t E = I.E;
    const int nred = (int)std::max<int64_t>(1, std::min<int64_t>((E + NT / 32 - 1) / (NT / 32), 1184));
    const int ngroups = (int)((E + RGRP - 1) / RGRP);
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    cudaGraph_t top = nullptr;
    if (!ok(cudaGraphCreate(&top, 0))) return false;
    bool good = false;
    do {
        cudaGraphConditionalHandle h_loop, h_rb;
        if (!ok(cudaGraphConditionalHandleCreate(&h_loop, top, 1, cudaGraphCondAssignDefault))) break;
        cudaGraphNodeParams wp = {cudaGraphNodeTypeConditional};
        wp.conditional.handle = h_loop;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        cudaGraphNode_t wnode;
        if (!ok(cudaGraphAddNode(&wnode, top, nullptr, 0, &wp))) break;
        cudaGraph_t body = wp.conditional.phGraph_out[0];
        if (!ok(cudaGraphConditionalHandleCreate(&h_rb, body, 0, cudaGraphCondAssignDefault))) break;
        if (!ok(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed))) break;
        // (k_ctrl_update is not needed inside the loop: the M pass speculates f = 1
        // itself and k_ctrl_dist rewrites f and need_edge)
        if (ngroups) k_edge_dist<<<ngroups, RGRP, 0, s>>>(F->P);
        k_pass<MODE_M><<<F->G, NT, F->smem, s>>>(F->P);
        k_local_reduce<<<nred, NT, 0, s>>>(F->P);
        F->comm->allreduce_sum(F->comm->ctx, F->tot.p, 2 * E + 16, s);
        k_ctrl_dist<<<1, NT, 0, s>>>(F->P, h_loop, h_rb, 1);
        cudaStreamCaptureStatus cst;
        cudaGraph_t capg = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t ndeps = 0;
        bool cap_ok = ok(cudaStreamGetCaptureInfo(s, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphNodeParams ip = {cudaGraphNodeTypeConditional};
        ip.conditional.handle = h_rb;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode = nullptr;
        if (cap_ok) cap_ok = ok(cudaGraphAddNode(&inode, capg, deps, ndeps, &ip));
        if (cap_ok) cap_ok = ok(cudaStreamUpdateCaptureDependencies(s, &inode, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t tmp = nullptr;
        if (!ok(cudaStreamEndCapture(s, &tmp)) || !cap_ok) break;
        cudaGraph_t rbody = ip.conditional.phGraph_out[0];
        if (!ok(cudaStreamBeginCaptureToGraph(s, rbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed))) break;
        k_pass<MODE_RB><<<F->G, NT, F->smem, s>>>(F->P);
        k_local_reduce<<<nred, NT, 0, s>>>(F->P);
        F->comm->allreduce_sum(F->comm->ctx, F->tot.p, 2 * E + 16, s);
        if (!ok(cudaStreamEndCapture(s, &tmp))) break;
        if (!ok(cudaGraphInstantiate(&F->dexec, top, 0))) break;
        good = true;
    } while (false);
    if (!good) {
        cudaGetLastError();  // clear a sticky-free capture / instantiate error
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(s, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
            cudaGraph_t tmp = nullptr;
            cudaStreamEndCapture(s, &tmp);
            if (tmp) cudaGraphDestroy(tmp);
        }
        cudaGetLastError();
        cudaGraphDestroy(top);
        F->dexec = nullptr;
        return false;
    }
    F->dgraph = top;
    return true;
}

// Host-driven iteration for sharded solves (see the split kernels above); the
// iteration loop itself runs as the per-run CUDA graph when it could be built.
static int64_t fast_run_dist(FastSolver *F, int64_t max_steps, cudaStream_t s, float *ms) {
    const Index &I = *F->inst->idx;
    const int64_t E = I.E;
    const int nred = (int)std::max<int64_t>(1, std::min<int64_t>((E + NT / 32 - 1) / (NT / 32), 1184));
    const int ngroups = (int)((E + RGRP - 1) / RGRP);
    auto read = [&]() {
        Ctrl c;
        d2h(&c, F->ctrl.p, 1, s);
        PF_CUDA(cudaStreamSynchronize(s));
        return c;
    };
    auto reduce_allreduce = [&]() {
        k_local_reduce<<<nred, NT, 0, s>>>(F->P);
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
    if (F->dgraph_state == 0) {
        const bool off = getenv("PF_DIST_NO_GRAPH") != nullptr;
        F->dgraph_state = !off && build_dist_graph(F, s) ? 1 : -1;
    }
    if (F->dgraph_state == 1 && !c.stopped && !c.status && c.iteration < target && c.need_edge) {
        PF_CUDA(cudaMemcpyAsync((char *)F->ctrl.p + offsetof(Ctrl, target), &target, sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
        PF_CUDA(cudaGraphLaunch(F->dexec, s));
        F->launches += 1;
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
        k_ctrl_dist<<<1, NT, 0, s>>>(F->P, 0, 0, 0);
        PF_CHECK_LAUNCH();
        F->launches += 5;
        c = read();
        if (!c.stopped && !c.status && c.f != c.fspec) {
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

// The buffers a launch reads and writes (both halves of the double buffers).
static std::vector<std::pair<void *, size_t>> fast_state_bufs(FastSolver *F) {
    std::vector<std::pair<void *, size_t>> v;
    for (int b = 0; b < 2; ++b) {
        v.push_back({F->dcon[b].p, F->dcon[b].bytes()});
        v.push_back({F->dn[b].p, F->dn[b].bytes()});
        v.push_back({F->dd[b].p, F->dd[b].bytes()});
        v.push_back({F->x[b].p, F->x[b].bytes()});
    }
    for (DevBuf<double> *d : {&F->dc, &F->adj, &F->partT, &F->partL, &F->slots, &F->res, &F->res_dc})
        if (d->p) v.push_back({d->p, d->bytes()});
    v.push_back({F->err.p, F->err.bytes()});
    v.push_back({F->ctrl.p, F->ctrl.bytes()});
    return v;
}

void fast_snapshot(FastSolver *F, cudaStream_t s) {
    require(F->nranks == 0 && F->comm == nullptr, "snapshots are single-GPU");
    const auto bufs = fast_state_bufs(F);
    size_t total = 0;
    for (const auto &b : bufs) total += (b.second + 255) & ~(size_t)255;
    if (F->snap.n < total) F->snap.alloc(total);
    size_t o = 0;
    for (const auto &b : bufs) {
        PF_CUDA(cudaMemcpyAsync(F->snap.p + o, b.first, b.second, cudaMemcpyDeviceToDevice, s));
        o += (b.second + 255) & ~(size_t)255;
    }
}

void fast_restore(FastSolver *F, cudaStream_t s) {
    require(F->snap.p != nullptr, "no snapshot to restore");
    size_t o = 0;
    for (const auto &b : fast_state_bufs(F)) {
        PF_CUDA(cudaMemcpyAsync(b.first, F->snap.p + o, b.second, cudaMemcpyDeviceToDevice, s));
        o += (b.second + 255) & ~(size_t)255;
    }
}

void fast_init(FastSolver *F, const double *d_x0, int64_t alpha0, double beta0, cudaStream_t s) {
    const Index &I = *F->inst->idx;
    for (int b = 0; b < 2; ++b) {
        PF_CUDA(cudaMemsetAsync(F->x[b].p, 0, F->x[b].bytes(), s));
        if (I.P) PF_CUDA(cudaMemcpyAsync(F->x[b].p, d_x0, sizeof(double) * I.P, cudaMemcpyDeviceToDevice, s));
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
    c.fspec = c.fnext = 1.0;
    c.alpha = c.alpha_used = alpha0;
    c.s = c.r = NAN;
    c.bad = -1;
    c.xc = 0;
    c.db = 0;
    c.need_a1 = 1;
    c.need_edge = 0;
    c.xepoch = 0;
    if (F->nranks) d2h(&c.xepoch, (uint64_t *)F->xepoch.p, 1, s);  // exchange numbering continues
    PF_CUDA(cudaStreamSynchronize(s));
    h2d(F->ctrl.p, &c, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
}

// Traced runs (capi.cu): one iteration per launch with no host round trip.  The
// run target is set on the device (one past the current iteration), so a
// stopped controller just leaves its iteration unchanged.
__global__ void k_ctrl_next(Ctrl *c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) c->target = c->iteration + 1;
}

// row[0..6] = iteration, alpha_used, beta_used, s, r, stopped-or-failed, status
__global__ void k_ctrl_row(const Ctrl *c, double *row) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    row[0] = (double)c->iteration;
    row[1] = (double)c->alpha_used;
    row[2] = c->beta_used;
    row[3] = c->s;
    row[4] = c->r;
    row[5] = (c->stopped || c->status) ? 1.0 : 0.0;
    row[6] = (double)c->status;
}

void fast_launch_one(FastSolver *F, cudaStream_t s) {
    require(!F->comm && !F->nranks, "traced multi-GPU runs are not supported");
    k_ctrl_next<<<1, 32, 0, s>>>(F->ctrl.p);
    PF_CHECK_LAUNCH();
    void *args[] = {(void *)&F->P};
    PF_CUDA(cudaLaunchCooperativeKernel((const void *)k_fused<false>, dim3(F->G), dim3(NT), args, F->smem, s));
    PF_CHECK_LAUNCH();
    ++F->launches;
}

void fast_ctrl_row(FastSolver *F, double *row7, cudaStream_t s) {
    k_ctrl_row<<<1, 32, 0, s>>>(F->ctrl.p, row7);
    PF_CHECK_LAUNCH();
}

// dst = the current rates x[ctrl.xc], the buffer chosen on the device
__global__ void k_copy_current_x(const Ctrl *c, const double *x0, const double *x1, int64_t n, double *dst) {
    const double *x = c->xc ? x1 : x0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = x[i];
}

void fast_copy_x(FastSolver *F, double *dst, cudaStream_t s) {
    const int64_t P = F->inst->idx->P;
    if (!P) return;
    k_copy_current_x<<<(int)std::min<int64_t>(ceil_div(P, 256), 1184), 256, 0, s>>>(F->ctrl.p, F->x[0].p, F->x[1].p,
                                                                                    P, dst);
    PF_CHECK_LAUNCH();
}

const int64_t *fast_alpha_used_dev(FastSolver *F) {
    return (const int64_t *)((const char *)F->ctrl.p + offsetof(Ctrl, alpha_used));
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
    // multi-GPU over peer memory: launches of at most PF_DIST_LAUNCH_ITERS
    // iterations, back to back on the stream (the same iterates: every reduction
    // has a fixed order and a launch resumes from the device state).  A
    // persistent kernel that spins on its peers for thousands of iterations
    // gave wrong totals when ranks were time-sliced on one GPU.
    static const int64_t seg_env = getenv("PF_DIST_LAUNCH_ITERS") ? atoll(getenv("PF_DIST_LAUNCH_ITERS")) : 256;
    const int64_t seg = F->nranks && seg_env > 0 ? seg_env : max_steps;
    std::vector<int64_t> targets;
    for (int64_t t = start + seg; t < start + max_steps; t += seg) targets.push_back(t);
    targets.push_back(start + max_steps);
    void *args[] = {(void *)&F->P};
    PF_CUDA(cudaEventRecord(F->e0, s));
    const void *kern = F->nranks ? (const void *)k_fused<true> : (const void *)k_fused<false>;
    for (const int64_t &target : targets) {
        PF_CUDA(cudaMemcpyAsync((char *)F->ctrl.p + offsetof(Ctrl, target), &target, sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
        PF_CUDA(cudaLaunchCooperativeKernel(kern, dim3(F->G), dim3(NT), args, F->smem, s));
        PF_CHECK_LAUNCH();
        ++F->launches;
    }
    PF_CUDA(cudaEventRecord(F->e1, s));
    d2h(&c, F->ctrl.p, 1, s);
    PF_CUDA(cudaStreamSynchronize(s));
    float t = 0.f;
    PF_CUDA(cudaEventElapsedTime(&t, F->e0, F->e1));
    if (ms) *ms = t;
    if (F->P.probe) {
        unsigned long long pr[8];
        PF_CUDA(cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr)));
        const double n = (double)std::max<int64_t>(1, c.iteration - start);
        unsigned long long mx[3];
        PF_CUDA(cudaMemcpyFromSymbol(mx, g_pmax, sizeof(mx)));
        fprintf(stderr, "[probe] per iteration (CTA 0): edge %.2f us, sync %.2f us, pass %.2f us, sync %.2f us, "
                        "controller %.2f us; max over CTAs and iterations: edge %.2f us, pass %.2f us, "
                        "controller %.2f us\n", pr[0] / n / 1e3, pr[1] / n / 1e3, pr[2] / n / 1e3, pr[3] / n / 1e3,
                pr[4] / n / 1e3, mx[0] / 1e3, mx[1] / 1e3, mx[2] / 1e3);
        unsigned long long zm[3] = {0, 0, 0};
        PF_CUDA(cudaMemcpyToSymbol(g_pmax, zm, sizeof(zm)));
        unsigned long long z[8] = {0};
        PF_CUDA(cudaMemcpyToSymbol(g_probe, z, sizeof(z)));
    }
#ifdef PF_TPROBE
    {
        unsigned long long tp[8];
        PF_CUDA(cudaMemcpyFromSymbol(tp, g_tprobe, sizeof(tp)));
        const double nt = (double)std::max<unsigned long long>(1, tp[7]);
        fprintf(stderr, "[tprobe] cycles per tile (thread 0, %llu tiles): tma-wait %.0f, y %.0f, K+com %.0f, "
                        "dcon+bar %.0f, runs-long %.0f, runs-short %.0f, end-bar %.0f\n",
                tp[7], tp[0] / nt, tp[1] / nt, tp[2] / nt, tp[3] / nt, tp[6] / nt, tp[4] / nt, tp[5] / nt);
        unsigned long long z[8] = {0};
        PF_CUDA(cudaMemcpyToSymbol(g_tprobe, z, sizeof(z)));
    }
#endif
    if (F->nranks) {
        unsigned long long xd[5];
        PF_CUDA(cudaMemcpyFromSymbol(xd, g_xdebug, sizeof(xd)));
        if (xd[0]) {
            fprintf(stderr, "[pf] rank %d: exchange %llu read rank %llu's slot with epoch tag %lld at iteration %llu "
                            "(arrival counter %llu)\n", F->rank, xd[0] - 1, xd[1], (long long)xd[2], xd[3], xd[4]);
            unsigned long long z[5] = {0, 0, 0, 0, 0};
            PF_CUDA(cudaMemcpyToSymbol(g_xdebug, z, sizeof(z)));
        }
    }
    if (getenv("PF_FAST_DEBUG"))
        fprintf(stderr, "[fast run] iterations %lld, rollback passes so far %lld\n", (long long)c.iteration,
                (long long)c.rollbacks);
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
    if (I.NP) k_export_pairs<<<ceil_div(I.NP, 256), 256, 0, s>>>(F->P, F->L->pair_slot.p, dy.p, ddc.p);
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

void fast_xchg_create(FastSolver *F, int rank, int nranks, void *handle64) {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / world size");
    require(!F->comm, "solver already has an NCCL communicator");
    const Index &I = *F->inst->idx;
    const int64_t xslot = (2 * I.E + 16 + 15) / 16 * 16;
    F->rank = rank;
    F->nranks = nranks;
    // its own 2 MB allocation (the IPC granularity): small cudaMalloc blocks may
    // share a physical page with other allocations of this process
    const size_t xwords = (size_t)2 * nranks * xslot + 16;  // + the arrival counter
    F->xb.alloc((xwords * sizeof(double) + (2u << 20) - 1) / (2u << 20) * (2u << 20) / sizeof(double));
    PF_CUDA(cudaMemset(F->xb.p, 0, F->xb.bytes()));
    F->xepoch.alloc(1);
    PF_CUDA(cudaMemset(F->xepoch.p, 0, sizeof(unsigned long long)));
    // cudaMemset of device memory may still be pending when it returns: the
    // zeroed counter and slots must be in place before any peer can see the
    // handle (a late memset would erase a peer's first arrival or totals)
    PF_CUDA(cudaDeviceSynchronize());
    cudaIpcMemHandle_t h;
    PF_CUDA(cudaIpcGetMemHandle(&h, F->xb.p));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, 64);
    F->P.xslot = xslot;
    F->P.xepoch = F->xepoch.p;
}

void fast_xchg_connect(FastSolver *F, const void *handles) {
    require(F->nranks >= 1, "call pf_solver_xchg_create first");
    std::vector<double *> bases(F->nranks);
    for (int r = 0; r < F->nranks; ++r) {
        if (r == F->rank) {
            bases[r] = F->xb.p;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, (const char *)handles + 64 * r, 64);
        void *p = nullptr;
        PF_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        F->opened.push_back(p);
        bases[r] = (double *)p;
    }
    F->peers_dev.alloc(F->nranks);
    PF_CUDA(cudaMemcpy(F->peers_dev.p, bases.data(), sizeof(double *) * F->nranks, cudaMemcpyHostToDevice));
    F->P.peers = F->peers_dev.p;
    F->P.rank = F->rank;
    F->P.nranks = F->nranks;
}

void fast_set_edge_counts(FastSolver *F, const double *counts) {
    const Index &I = *F->inst->idx;
    if (I.E) PF_CUDA(cudaMemcpy(F->ne.p, counts, sizeof(double) * I.E, cudaMemcpyHostToDevice));
}

double *fast_scratch(FastSolver *F, int which) {
    const Index &I = *F->inst->idx;
    DevBuf<double> &b = which == 0 ? F->x0stage : which == 1 ? F->rates_out : which == 2 ? F->sums_out : F->flag;
    const size_t n = (size_t)std::max<int64_t>(1, which == 3 ? 1 : which == 2 ? I.C + 1 : I.P);
    if (b.n < n) b.alloc(n);
    return b.p;
}

void fast_stats(FastSolver *F, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes) {
    const Index &I = *F->inst->idx;
    if (launches) *launches = F->launches;
    if (tiles) *tiles = F->L->ntiles;
    if (grid) *grid = F->G;
    // compulsory HBM bytes per iteration of this layout: one M pass (bulk-copied
    // inputs + written state) plus the CTA edge partials T and L written and read
    // back (4 x 8 B per edge per CTA)
    if (bytes) *bytes = F->L->bytes_per_pass + (int64_t)F->G * I.E * 32;
}

}  // namespace pf
