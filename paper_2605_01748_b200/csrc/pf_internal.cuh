// Internal declarations shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "pf_b200.h"

namespace pf {

// ----------------------------------------------------------------- errors

struct Error : std::exception {
    int status;
    std::string msg;
    Error(int s, std::string m) : status(s), msg(std::move(m)) {}
    const char *what() const noexcept override { return msg.c_str(); }
};

void set_error(const std::string &m);
const std::string &get_error();

#define PF_CUDA(call)                                                                                  \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess)                                                                         \
            throw ::pf::Error(PF_ERR_CUDA, std::string(#call) + " failed: " + cudaGetErrorString(e_)); \
    } while (0)

#define PF_CHECK_LAUNCH() PF_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string &msg, int status = PF_ERR_INPUT) {
    if (!ok) throw Error(status, msg);
}

// Translate exceptions to a C status.
template <class F>
int guard(F &&f) {
    try {
        f();
        return PF_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc &) {
        set_error("host out of memory");
        return PF_ERR_NOMEM;
    } catch (const std::exception &e) {
        set_error(e.what());
        return PF_ERR_CUDA;
    }
}

// ----------------------------------------------------------------- device memory

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) {
            cudaError_t e = cudaMalloc(&p, sizeof(T) * count);
            if (e != cudaSuccess) {
                p = nullptr;
                n = 0;
                throw Error(PF_ERR_NOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
            }
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    T *get() const { return p; }
};

template <class T>
void h2d(T *dst, const T *src, size_t n, cudaStream_t s) {
    if (n) PF_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
void d2h(T *dst, const T *src, size_t n, cudaStream_t s) {
    if (n) PF_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) PF_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void ensure_device(int device);

// ----------------------------------------------------------------- instance

struct TileLayout;  // fused.cu

// Index spaces of model.py:135-180, int32 on device (every config fits: NP < 2^31).
struct Index {
    int device = 0;
    int64_t C0 = 0, C = 0, P = 0, E = 0, NP = 0;
    DevBuf<int64_t> kept_rows;
    DevBuf<int32_t> com_path_ptr, path_com, hops, pair_ptr, pair_edge, pair_path;
    DevBuf<int32_t> edge_path_count, edge_pair_ptr, edge_pairs;
    std::mutex tiles_mu;
    std::shared_ptr<TileLayout> tiles;  // fast-mode layout, built lazily
};

struct InstView {
    int32_t C, P, E, NP;
    const int32_t *com_path_ptr, *path_com, *hops, *pair_ptr, *pair_edge, *pair_path;
    const int32_t *edge_path_count, *edge_pair_ptr, *edge_pairs;
    const double *demand, *capacity;
};

}  // namespace pf

struct pf_instance {
    std::shared_ptr<pf::Index> idx;
    pf::DevBuf<double> demand, capacity;
    cudaStream_t stream = nullptr;
    mutable std::mutex ws_mu;
    mutable std::shared_ptr<void> proj_ws;  // projection scratch (projection.cu)
    mutable std::shared_ptr<void> val_ws;   // validate_allocation scratch (capi.cu), under ws_mu
    // the handle plus every solver created from it: the instance is freed with
    // the last of them (pf_instance_destroy may come first, e.g. from a garbage
    // collector finalising a cycle in arbitrary order)
    mutable std::atomic<int> refs{1};
    mutable int fast_ok = -1;               // the fused kernel's layout limits hold (-1: not checked)
    mutable std::string fast_why;
    // one idle fast-mode solver kept for the next solve on this instance (fused.cu):
    // its device buffers are reused instead of re-allocated per solve
    mutable void *fast_pool = nullptr;
    mutable void (*fast_pool_free)(void *) = nullptr;
    ~pf_instance() {
        if (fast_pool && fast_pool_free) fast_pool_free(fast_pool);
    }
    pf::InstView view() const {
        pf::InstView v;
        v.C = (int32_t)idx->C;
        v.P = (int32_t)idx->P;
        v.E = (int32_t)idx->E;
        v.NP = (int32_t)idx->NP;
        v.com_path_ptr = idx->com_path_ptr.p;
        v.path_com = idx->path_com.p;
        v.hops = idx->hops.p;
        v.pair_ptr = idx->pair_ptr.p;
        v.pair_edge = idx->pair_edge.p;
        v.pair_path = idx->pair_path.p;
        v.edge_path_count = idx->edge_path_count.p;
        v.edge_pair_ptr = idx->edge_pair_ptr.p;
        v.edge_pairs = idx->edge_pairs.p;
        v.demand = demand.p;
        v.capacity = capacity.p;
        return v;
    }
    int device() const { return idx->device; }
};

namespace pf {

// ----------------------------------------------------------------- exact-order helpers (exact.cu)

// Device-resident SolverState in the reference's index spaces.
struct DevState {
    DevBuf<double> x, y, dd, dc, dcon, dn;
    void alloc(const Index &I) {
        x.alloc(I.P);
        y.alloc(I.NP);
        dd.alloc(I.C);
        dc.alloc(I.E);
        dcon.alloc(I.NP);
        dn.alloc(I.P);
    }
};

struct StatePtrs {
    const double *x, *y, *dd, *dc, *dcon, *dn;
};

// Status flags written by kernels (first offending commodity via atomicMin).
struct Flags {
    int32_t bad_coef;  // INT_MAX if none
    int32_t bad_root;
    int32_t bad_edge;  // input validation
    int32_t pad;
};

void exact_commodity_sums(const InstView &I, const double *x, double *out, cudaStream_t s);
void exact_edge_loads_from_pairs(const InstView &I, const double *pair_vals, double *out, cudaStream_t s);
// drops one reference of the instance (the handle's or a solver's); frees it with the last
void instance_release(const pf_instance *inst);
void exact_edge_loads_of_rates(const InstView &I, const double *rates, double *out, cudaStream_t s);
// Same sums through an edge-major copy gathered via the incidence (scratch: NP doubles).
void exact_edge_loads_of_rates_em_pairs(const InstView &I, const double *rates, double *scratch, double *out,
                                        cudaStream_t s);
// oracles.py:262-287 dao_carry_rates on the device rates x (in place); returns
// the number of edge passes that scaled (dao.cu).
int64_t dao_carry_device(const pf_instance *inst, double *x, double tol, cudaStream_t s);
// Same sums (same association) through an edge-major copy: epath[t] =
// pair_path[edge_pairs[t]], scratch holds NP doubles.
void exact_edge_loads_of_rates_em(const InstView &I, const double *rates, const int32_t *epath, double *scratch,
                                  double *out, cudaStream_t s);
void exact_update_duals(const InstView &I, const StatePtrs &st, double *sums_tmp, double *loads_tmp, double *dd,
                        double *dc, double *dcon, double *dn, cudaStream_t s, double *scratch = nullptr);
void exact_update_slacks(const InstView &I, const StatePtrs &st, double beta, double *sums_tmp, double *loads_tmp,
                         double *sd, double *sc, cudaStream_t s);
// scratch: optional [NP] doubles (edge-major values; faster sequential chains)
void exact_suggest(const InstView &I, const StatePtrs &st, double *y_out, cudaStream_t s,
                   double *scratch = nullptr);
void exact_coefficients(const InstView &I, const StatePtrs &st, double *pk, double *pw, double *wsum, double *q,
                        cudaStream_t s);
void exact_roots(const InstView &I, const double *wsum, const double *q, const double *dd, double beta,
                 int64_t alpha, double *sums, Flags *flags, cudaStream_t s);
void exact_rates(const InstView &I, const double *pk, const double *pw, const double *sums, const double *dd,
                 double beta, int64_t alpha, double *x_out, cudaStream_t s);
// Squared-norm partial of det_diff_norm (returns sum of squares via `out_sumsq`, device scalar).
void exact_sqdiff_sum(const double *a, const double *b, int64_t n, double *block_tmp, double *out_sumsq,
                      cudaStream_t s);
size_t sqdiff_tmp_len(int64_t n);
void scale_inplace(double *a, int64_t n, double f, cudaStream_t s);
void reset_flags(Flags *f, cudaStream_t s);

// Trace helpers (model.py:335-369, kernels.py:47-66 summed with numpy pairwise order).
struct TraceScratch {
    DevBuf<double> loads, sums, rel, tmp, leaf_sum;
    DevBuf<double> em;  // [NP] edge-major copy of the rates (exact-order edge loads)
    DevBuf<int64_t> leaf_lo;
    DevBuf<int32_t> cnt;
    DevBuf<double> out;  // [4]: objective, pct, mean_rel, n_viol
};
void trace_stats(const InstView &I, const double *x, const double *root_sums, int64_t alpha, TraceScratch &ts,
                 double tol, double *host_out4, cudaStream_t s);
void trace_stats_dev(const InstView &I, const double *x, const double *root_sums, const int64_t *d_alpha,
                     TraceScratch &ts, double tol, double *row4, cudaStream_t s);
void optimality_sum_dev(const InstView &I, const double *sums, const double *ref, double theta, TraceScratch &ts,
                        double *d_sum, cudaStream_t s);
void violation_stats(const InstView &I, const double *x, double tol, double *d_overload, double *d_excess,
                     TraceScratch &ts, pf_violation *rep, cudaStream_t s);

// Projection (projection.cu).
// fast = true (fast-mode solves): tolerance-matched parallel trims in phase 3
void project_device(const pf_instance *inst, const double *d_rates, int64_t alpha, double *d_out, cudaStream_t s,
                    bool fast = false);
void score_paths_device(const pf_instance *inst, const double *d_rates, int64_t alpha, double *d_scores,
                        cudaStream_t s);

// ----------------------------------------------------------------- inline device math

// On the device both clamps are one compare + one select (setp/selp); the
// compiler's own max-pattern lowering adds NaN/-0 fix-ups that these exact
// semantics do not need.
__host__ __device__ __forceinline__ double npmax0(double v) {  // np.maximum(v, 0): NaN and -0.0 pass through
#ifdef __CUDA_ARCH__
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, 0d0000000000000000;\n\t"
        "selp.f64 %0, 0d0000000000000000, %1, p;\n\t}"
        : "=d"(r)
        : "d"(v));
    return r;
#else
    return v < 0.0 ? 0.0 : v;
#endif
}
__host__ __device__ __forceinline__ double max0(double v) {  // numba clamp `v if v > 0 else 0`: NaN -> 0
#ifdef __CUDA_ARCH__
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\t"
        "selp.f64 %0, %1, 0d0000000000000000, p;\n\t}"
        : "=d"(r)
        : "d"(v));
    return r;
#else
    return v > 0.0 ? v : 0.0;
#endif
}
__host__ __device__ __forceinline__ double pymax1(double v) { return v > 1.0 ? v : 1.0; }  // max(1.0, v)

// kernels.py:153-173: safeguarded Newton + bisection for alpha >= 2 (kept out of
// line so the fused kernel's register budget is not sized for it).
static __device__ __noinline__ double root_newton(double lin, double c, double q, int64_t alpha) {
    double a = (double)alpha;
    double tol_f = 1e-10 * pymax1(fabs(q));
    double lo = 1e-12;
    double hi = q / lin;
    if (hi < 1.0) hi = 1.0;
    double f_hi = lin * hi - c * pow(hi, -a) - q;
    while (f_hi < 0.0) {
        hi *= 2.0;
        f_hi = lin * hi - c * pow(hi, -a) - q;
    }
    double s = hi;
    for (int it = 0; it < 200; ++it) {
        double f = lin * s - c * pow(s, -a) - q;
        if (f >= 0.0)
            hi = s;
        else
            lo = s;
        double fp = lin + a * c * pow(s, -a - 1.0);
        double t = s - f / fp;
        if (!(lo < t && t < hi)) t = 0.5 * (lo + hi);
        if (fabs(f) <= tol_f && fabs(t - s) <= 1e-12 * pymax1(fabs(s))) return s;
        s = t;
    }
    return s;
}

// kernels.py:134-173 _root_scalar: root of lin*S - c*S^(-alpha) - q.
// Compiled with -fmad=false so every op rounds exactly as the reference's.
__device__ __forceinline__ double root_scalar(double lin, double c, double q, int64_t alpha) {
    if (alpha == 0) return (q + c) / lin;
    if (alpha == 1) {
        double disc = q * q + 4.0 * lin * c;
        double sq = sqrt(disc);
        if (q >= 0.0) return (q + sq) / (2.0 * lin);
        return (2.0 * c) / (sq - q);
    }
    return root_newton(lin, c, q, alpha);
}

// kernels.py:183-189 _k_roots body for one commodity.
__device__ __forceinline__ double commodity_root(double w, double q, double d_eff, double beta, int64_t alpha) {
    double cc = w / beta;
    double s = root_scalar(1.0, cc, q, alpha);
    if (s > d_eff) s = root_scalar(1.0 + w, cc, q + w * d_eff, alpha);
    return s;
}

// kernels.py:289-294 per-commodity rate term: gain - over.
__device__ __forceinline__ double commodity_term(double S, double D, double dd, double beta, int64_t alpha) {
    double gain;
    if (alpha == 0)
        gain = 1.0 / beta;
    else if (alpha == 1)
        gain = (1.0 / S) / beta;  // numpy s ** -1.0 is the exact reciprocal
    else
        gain = pow(S, -(double)alpha) / beta;
    double over = npmax0(S - (D - dd));
    return gain - over;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace pf
