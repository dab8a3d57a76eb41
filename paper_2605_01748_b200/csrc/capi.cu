#include <cstdio>
// C-ABI entry points: kernel-level functions, projection, and the solve loop.
//
// pf_solve / pf_solver_* reproduce pathfair/controller.py:197-284:
//   PF_MODE_EXACT  the reference's kernels one-to-one in exact operation order
//                  (exact.cu) with the scalar controller on the host (the only
//                  per-iteration host traffic is 5 norms + 2 flags); bitwise
//                  identical to the reference for alpha <= 1.
//   PF_MODE_FAST   the fused persistent kernel (fused.cu) with the controller
//                  evaluated on device; no host round trip per iteration.
// Both end with the GPU projection (projection.cu).
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>

#include "fused.cuh"
#include "pf_internal.cuh"

namespace pf {

const CommOps *comm_ops(pf_comm *c);  // dist.cu

// numpy pairwise sum on the host (np.mean in optimality_from_sums).
static double np_pairwise_h(const double *a, int64_t n) {
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
    return np_pairwise_h(a, n2) + np_pairwise_h(a + n2, n - n2);
}

// CPython `n ** 2` == libm pow(n, 2.0) (controller.py:133-138); keep the call.
static double py_sq(double v) {
    volatile double two = 2.0;
    return std::pow(v, two);
}

static double wall() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void k_init_cold(InstView I, double *x) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= I.P) return;
    int32_t c = I.path_com[p];
    x[p] = I.demand[c] / (double)(I.com_path_ptr[c + 1] - I.com_path_ptr[c]);  // controller.py:113-114
}
__global__ void k_gather_pairs(InstView I, const double *x, double *y) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < I.NP) y[t] = x[I.pair_path[t]];
}

struct HostCtrl {
    double beta = 1.0;
    int64_t alpha = 0, iteration = 0;
    double ema_s = -1.0, ema_r = -1.0;
    int64_t cooldown = 0;
    bool just_incremented = false, stopped = false;
};

}  // namespace pf

using namespace pf;

struct pf_solver {
    const pf_instance *inst = nullptr;
    pf_config cfg{};
    std::vector<double> ref_sums;
    std::vector<double> h_demand;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // exact mode
    DevState cur, nxt;
    DevBuf<double> sums_tmp, loads_tmp, pk, pw, wsum, q, root_sums, sqtmp, norms, svals;
    DevBuf<Flags> flags;
    HostCtrl ctrl;
    // fast mode
    FastSolver *fast = nullptr;
    // common
    TraceScratch ts;
    std::vector<pf_trace_row> trace;
    double t0 = 0.0;
    double loop_ms = 0.0, proj_ms = 0.0;
    int status = PF_OK;
    int64_t bad_commodity = -1;
    bool initialized = false, finished = false;
    bool exact_fallback = false;                // fast mode requested outside the fused layout limits
    DevBuf<double> rates_out, sums_out, trace_proj, trace_sums;
    DevBuf<double> trace_rows;                  // traced fast runs: a batch of device rows
    cudaEvent_t tev[64] = {};                   // per-launch timing of a traced batch
    pf_comm *comm = nullptr;
    int64_t global_C = 0;

    int64_t C() const { return inst->idx->C; }
    int64_t P() const { return inst->idx->P; }
    int64_t E() const { return inst->idx->E; }
    int64_t NP() const { return inst->idx->NP; }
};

namespace pf {

static void validate_config(const pf_config &c) {
    // controller.py:51-61
    require(c.gamma > 0, "gamma must be > 0");
    require(c.residual_ratio > 1 && c.beta_scale > 1, "residual_ratio and beta_scale must be > 1");
    require(0 < c.beta_min && c.beta_min <= c.beta_max, "beta bounds must satisfy 0 < beta_min <= beta_max");
    require(c.alpha_target >= -1, "alpha_target must be >= 0");
    require(c.max_iterations >= 1, "max_iterations must be >= 1");
    require(c.mode == PF_MODE_EXACT || c.mode == PF_MODE_FAST, "unknown mode");
}

static double adapt_beta(double beta, double s, double r, const pf_config &c) {  // controller.py:142-150
    if (r > c.residual_ratio * s)
        beta = beta * c.beta_scale;
    else if (s > c.residual_ratio * r)
        beta = beta / c.beta_scale;
    double lo = beta > c.beta_min ? beta : c.beta_min;
    return lo < c.beta_max ? lo : c.beta_max;
}

static double default_theta(const std::vector<double> &D) {  // oracles.py:51-53
    double dmax = 0.0;
    for (double d : D) dmax = d > dmax ? d : dmax;
    return 1e-6 * (dmax > 0 ? dmax : 1.0);
}

static double optimality_from_sums(const std::vector<double> &sums, const std::vector<double> &ref, double theta) {
    if (sums.empty()) return 1.0;  // oracles.py:244-254
    std::vector<double> r(sums.size());
    for (size_t i = 0; i < sums.size(); ++i) {
        double den = ref[i] > theta ? ref[i] : theta;
        double v = sums[i] / den;
        r[i] = v < 1.0 ? v : 1.0;
    }
    return np_pairwise_h(r.data(), (int64_t)r.size()) / (double)r.size();
}

static void solver_trace_row(pf_solver *S, const double *d_x, const double *d_root_sums, int64_t iteration,
                             int64_t alpha, double beta, double s, double r) {
    InstView I = S->inst->view();
    pf_trace_row row;
    row.iteration = iteration;
    row.alpha = alpha;
    row.beta = beta;
    row.s = s;
    row.r = r;
    double st[4];
    trace_stats(I, d_x, d_root_sums, alpha, S->ts, 1e-9, st, S->stream);
    row.objective = st[0];
    row.pct_violated = st[1];
    row.mean_relative_violation = st[2];
    row.optimality = NAN;
    if (!S->ref_sums.empty()) {
        // per-row scratch kept on the solver (no cudaMalloc / cudaFree per iteration)
        if (S->trace_proj.n < (size_t)S->P() + 1) S->trace_proj.alloc(S->P() + 1);
        if (S->trace_sums.n < (size_t)S->C() + 1) S->trace_sums.alloc(S->C() + 1);
        project_device(S->inst, d_x, alpha, S->trace_proj.p, S->stream, S->cfg.mode == PF_MODE_FAST);
        exact_commodity_sums(I, S->trace_proj.p, S->trace_sums.p, S->stream);
        std::vector<double> hs(S->C());
        d2h(hs.data(), S->trace_sums.p, S->C(), S->stream);
        PF_CUDA(cudaStreamSynchronize(S->stream));
        row.optimality = optimality_from_sums(hs, S->ref_sums, default_theta(S->h_demand));
    }
    S->trace.push_back(row);
}

// Sets *flag = 1 if any x[i] is NaN or infinite (benign same-value stores).
__global__ void k_flag_nonfinite(const double *__restrict__ x, int64_t n, double *flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1.0;
}

static void solver_init(pf_solver *S, const double *warm) {
    DeviceGuard g(S->inst->device());
    InstView I = S->inst->view();
    cudaStream_t st = S->stream;
    S->t0 = wall();
    static const bool timing = getenv("PF_TIMING") != nullptr;
    auto lap = [&](const char *what) {
        if (timing) fprintf(stderr, "[solver_init] %s at %.2f ms\n", what, 1e3 * (wall() - S->t0));
    };
    S->initialized = false;  // a failed init leaves no runnable state
    S->trace.clear();
    S->loop_ms = S->proj_ms = 0.0;
    S->status = PF_OK;
    S->bad_commodity = -1;
    S->finished = false;
    HostCtrl c;
    c.beta = S->cfg.beta0;
    if (warm) c.alpha = S->cfg.alpha_target >= 0 ? S->cfg.alpha_target : 0;  // controller.py:104-111
    S->ctrl = c;
    lap("checks");
    DevBuf<double> x0own;
    double *x0 = nullptr;
    if (S->cfg.mode == PF_MODE_FAST) {
        x0 = fast_scratch(S->fast, 0);  // pooled with the solver: no allocation per solve
    } else {
        x0own.alloc(S->P() ? S->P() : 1);
        x0 = x0own.p;
    }
    lap("x0 alloc");
    // the warm start's finiteness (controller.py:104-111) is checked on the
    // device copy: one read of x0 instead of a host pass over P doubles
    DevBuf<double> flagown;
    double *flag = nullptr;
    double hflag = 0.0;
    if (warm) {
        h2d(x0, warm, S->P(), st);
        if (S->cfg.mode == PF_MODE_FAST) {
            flag = fast_scratch(S->fast, 3);
        } else {
            flagown.alloc(1);
            flag = flagown.p;
        }
        PF_CUDA(cudaMemsetAsync(flag, 0, sizeof(double), st));
        if (I.P) k_flag_nonfinite<<<std::min<int64_t>(ceil_div(I.P, 256), 1184), 256, 0, st>>>(x0, I.P, flag);
        PF_CHECK_LAUNCH();
        d2h(&hflag, flag, 1, st);
    } else if (I.P)
        k_init_cold<<<ceil_div(I.P, 256), 256, 0, st>>>(I, x0);
    PF_CHECK_LAUNCH();
    if (S->cfg.mode == PF_MODE_EXACT) {
        PF_CUDA(cudaMemcpyAsync(S->cur.x.p, x0, sizeof(double) * S->P(), cudaMemcpyDeviceToDevice, st));
        if (I.NP) k_gather_pairs<<<ceil_div(I.NP, 256), 256, 0, st>>>(I, x0, S->cur.y.p);
        PF_CHECK_LAUNCH();
        PF_CUDA(cudaMemsetAsync(S->cur.dd.p, 0, sizeof(double) * S->C(), st));
        PF_CUDA(cudaMemsetAsync(S->cur.dc.p, 0, sizeof(double) * S->E(), st));
        PF_CUDA(cudaMemsetAsync(S->cur.dcon.p, 0, sizeof(double) * S->NP(), st));
        PF_CUDA(cudaMemsetAsync(S->cur.dn.p, 0, sizeof(double) * S->P(), st));
    } else {
        lap("h2d issued");
        fast_init(S->fast, x0, c.alpha, c.beta, st);
    }
    PF_CUDA(cudaStreamSynchronize(st));
    lap("fast_init + sync");
    require(hflag == 0.0, "warm start contains non-finite rates");
    S->initialized = true;
}

// One iteration of controller.py:225-273 in exact order.  Returns false when stopped.
static bool exact_step(pf_solver *S) {
    InstView I = S->inst->view();
    cudaStream_t st = S->stream;
    HostCtrl &c = S->ctrl;
    DevState &cur = S->cur, &nxt = S->nxt;
    StatePtrs s0{cur.x.p, cur.y.p, cur.dd.p, cur.dc.p, cur.dcon.p, cur.dn.p};
    exact_update_duals(I, s0, S->sums_tmp.p, S->loads_tmp.p, nxt.dd.p, nxt.dc.p, nxt.dcon.p, nxt.dn.p, st,
                       S->svals.p);
    // update_slacks (controller.py:228) is bookkeeping never read by the loop; skipped.
    StatePtrs s1{cur.x.p, cur.y.p, nxt.dd.p, nxt.dc.p, nxt.dcon.p, nxt.dn.p};
    exact_suggest(I, s1, nxt.y.p, st, S->svals.p);
    StatePtrs s2{cur.x.p, nxt.y.p, nxt.dd.p, nxt.dc.p, nxt.dcon.p, nxt.dn.p};
    exact_coefficients(I, s2, S->pk.p, S->pw.p, S->wsum.p, S->q.p, st);
    reset_flags(S->flags.p, st);
    exact_roots(I, S->wsum.p, S->q.p, nxt.dd.p, c.beta, c.alpha, S->root_sums.p, S->flags.p, st);
    exact_rates(I, S->pk.p, S->pw.p, S->root_sums.p, nxt.dd.p, c.beta, c.alpha, nxt.x.p, st);
    exact_sqdiff_sum(nxt.x.p, cur.x.p, S->P(), S->sqtmp.p, S->norms.p + 0, st);
    exact_sqdiff_sum(nxt.dd.p, cur.dd.p, S->C(), S->sqtmp.p, S->norms.p + 1, st);
    exact_sqdiff_sum(nxt.dc.p, cur.dc.p, S->E(), S->sqtmp.p, S->norms.p + 2, st);
    exact_sqdiff_sum(nxt.dcon.p, cur.dcon.p, S->NP(), S->sqtmp.p, S->norms.p + 3, st);
    exact_sqdiff_sum(nxt.dn.p, cur.dn.p, S->P(), S->sqtmp.p, S->norms.p + 4, st);
    double nrm[5];
    Flags fl;
    d2h(nrm, S->norms.p, 5, st);
    d2h(&fl, S->flags.p, 1, st);
    PF_CUDA(cudaStreamSynchronize(st));
    if (fl.bad_coef != INT_MAX) {
        S->bad_commodity = fl.bad_coef;
        throw Error(PF_ERR_KERNEL_COEF, "non-finite sum coefficients for commodity " + std::to_string(fl.bad_coef));
    }
    if (fl.bad_root != INT_MAX) {
        S->bad_commodity = fl.bad_root;
        throw Error(PF_ERR_KERNEL_ROOT, "non-finite sum root for commodity " + std::to_string(fl.bad_root));
    }
    std::swap(cur.x, nxt.x);
    std::swap(cur.y, nxt.y);
    std::swap(cur.dd, nxt.dd);
    std::swap(cur.dc, nxt.dc);
    std::swap(cur.dcon, nxt.dcon);
    std::swap(cur.dn, nxt.dn);
    int64_t it = ++c.iteration;
    // controller.py:131-139 (sqrt of each det_diff_norm, then CPython ** 2)
    double s = std::sqrt(nrm[0]);
    double n1 = std::sqrt(nrm[1]), n2 = std::sqrt(nrm[2]), n3 = std::sqrt(nrm[3]), n4 = std::sqrt(nrm[4]);
    double r = std::sqrt(py_sq(n1) + py_sq(n2) + py_sq(n3) + py_sq(n4));
    if (!(std::isfinite(s) && std::isfinite(r)))
        throw Error(PF_ERR_SOLVER, "non-finite iterates at iteration " + std::to_string(it));
    bool converged = r <= S->cfg.gamma && s <= S->cfg.gamma;
    if (S->cfg.trace) solver_trace_row(S, cur.x.p, S->root_sums.p, it, c.alpha, c.beta, s, r);
    int decision = 0;  // controller.py:157-170
    if (converged) {
        if (S->cfg.alpha_target >= 0 && c.alpha >= S->cfg.alpha_target)
            decision = 1;
        else if (c.just_incremented)
            decision = 1;
        else
            decision = 2;
    }
    if (S->cfg.adapt) {  // controller.py:245-266
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
            double nb = adapt_beta(c.beta, c.ema_s, c.ema_r, S->cfg);
            if (nb != c.beta) {
                double f = c.beta / nb;
                scale_inplace(cur.dd.p, S->C(), f, st);
                scale_inplace(cur.dc.p, S->E(), f, st);
                scale_inplace(cur.dcon.p, S->NP(), f, st);
                scale_inplace(cur.dn.p, S->P(), f, st);
                c.beta = nb;
                c.cooldown = 10;
            }
        }
    }
    c.just_incremented = false;
    if (decision == 1) {
        c.stopped = true;
        return false;
    }
    if (decision == 2) {
        c.alpha += 1;
        c.just_incremented = true;
    }
    return true;
}

static int64_t solver_run(pf_solver *S, int64_t max_steps) {
    DeviceGuard g(S->inst->device());
    require(S->initialized, "solver not initialized");
    int64_t done = 0;
    if (S->P() == 0) return 0;
    if (S->cfg.mode == PF_MODE_EXACT) {
        PF_CUDA(cudaEventRecord(S->ev0, S->stream));
        while (done < max_steps && !S->ctrl.stopped && S->ctrl.iteration < S->cfg.max_iterations) {
            exact_step(S);
            ++done;
        }
        PF_CUDA(cudaEventRecord(S->ev1, S->stream));
        PF_CUDA(cudaEventSynchronize(S->ev1));
        float ms = 0.f;
        PF_CUDA(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
        S->loop_ms += ms;
        return done;
    }
    // fast mode
    if (!S->cfg.trace) {
        float ms = 0.f;
        done = fast_run(S->fast, max_steps, S->stream, &ms);
        S->loop_ms += ms;
        return done;
    }
    // fast mode with trace, single GPU, no optimality column: batches of
    // iterations with their rows computed on the device (controller fields,
    // objective, % violated, mean relative violation), one host read per batch
    if (S->ref_sums.empty() && !S->comm) {
        constexpr int RB = 32, RW = 12;
        cudaStream_t st = S->stream;
        if (S->trace_rows.n < (size_t)RB * RW) S->trace_rows.alloc((size_t)RB * RW);
        if (!S->tev[0])
            for (cudaEvent_t &e : S->tev) PF_CUDA(cudaEventCreate(&e));
        const InstView I = S->inst->view();
        std::vector<double> h((size_t)RB * RW);
        int64_t last = fast_status(S->fast, st).iteration;
        bool stop = false;
        while (done < max_steps && !stop) {
            const int B = (int)std::min<int64_t>(RB, max_steps - done);
            for (int i = 0; i < B; ++i) {
                double *row = S->trace_rows.p + (size_t)i * RW;
                PF_CUDA(cudaEventRecord(S->tev[2 * i], st));
                fast_launch_one(S->fast, st);
                PF_CUDA(cudaEventRecord(S->tev[2 * i + 1], st));
                fast_ctrl_row(S->fast, row, st);
                double *xcur = fast_scratch(S->fast, 1);  // free until finish()
                fast_copy_x(S->fast, xcur, st);
                trace_stats_dev(I, xcur, fast_root_sums(S->fast), fast_alpha_used_dev(S->fast), S->ts, 1e-9, row + 7,
                                st);
            }
            d2h(h.data(), S->trace_rows.p, (size_t)B * RW, st);
            PF_CUDA(cudaStreamSynchronize(st));
            bool progressed = false;
            for (int i = 0; i < B && !stop; ++i) {
                const double *r = &h[(size_t)i * RW];
                const int64_t it = (int64_t)r[0];
                if (it > last) {  // a stopped controller leaves its iteration unchanged
                    float ms = 0.f;
                    PF_CUDA(cudaEventElapsedTime(&ms, S->tev[2 * i], S->tev[2 * i + 1]));
                    S->loop_ms += ms;
                    pf_trace_row row;
                    row.iteration = it;
                    row.alpha = (int64_t)r[1];
                    row.beta = r[2];
                    row.s = r[3];
                    row.r = r[4];
                    row.objective = r[7];
                    row.pct_violated = r[8];
                    row.mean_relative_violation = r[9];
                    row.optimality = NAN;
                    S->trace.push_back(row);
                    last = it;
                    ++done;
                    progressed = true;
                }
                if (r[5] != 0.0 || it >= S->cfg.max_iterations) stop = true;
            }
            if (!progressed) break;
        }
        return done;
    }
    // with the optimality column (a projection per row): one iteration at a time
    while (done < max_steps) {
        float ms = 0.f;
        int64_t k = fast_run(S->fast, 1, S->stream, &ms);
        S->loop_ms += ms;
        if (k == 0) break;
        done += k;
        FastStatus fs = fast_status(S->fast, S->stream);
        solver_trace_row(S, fast_x(S->fast), fast_root_sums(S->fast), fs.iteration, fs.alpha_used, fs.beta_used,
                         fs.s, fs.r);
        if (fs.stopped || fs.iteration >= S->cfg.max_iterations) break;
    }
    return done;
}

static void solver_status(pf_solver *S, pf_result *res) {
    std::memset(res, 0, sizeof(*res));
    if (S->cfg.mode == PF_MODE_EXACT || S->P() == 0) {
        res->iterations = S->ctrl.iteration;
        res->alpha = S->ctrl.alpha;
        res->converged = S->P() == 0 ? 1 : (S->ctrl.stopped ? 1 : 0);
        res->beta = S->ctrl.beta;
    } else {
        FastStatus fs = fast_status(S->fast, S->stream);
        res->iterations = fs.iteration;
        res->alpha = fs.alpha;
        res->converged = fs.stopped;
        res->beta = fs.beta;
        if (fs.status != PF_OK) {
            res->status = fs.status;
            res->bad_commodity = fs.bad;
        }
    }
    res->status = res->status ? res->status : S->status;
    if (S->bad_commodity >= 0) res->bad_commodity = S->bad_commodity;
    res->runtime_s = wall() - S->t0;
    res->exact_fallback = S->exact_fallback ? 1 : 0;
    res->loop_ms = S->loop_ms;
    res->projection_ms = S->proj_ms;
}

static const double *solver_x(pf_solver *S) {
    return S->cfg.mode == PF_MODE_EXACT ? S->cur.x.p : fast_x(S->fast);
}

static void solver_finish(pf_solver *S, double *rates, double *sums) {
    DeviceGuard g(S->inst->device());
    InstView I = S->inst->view();
    cudaStream_t st = S->stream;
    if (S->P() == 0) {
        if (sums)
            for (int64_t c = 0; c < S->C(); ++c) sums[c] = 0.0;
        S->finished = true;
        return;
    }
    if (S->cfg.mode == PF_MODE_FAST) {
        FastStatus fs = fast_status(S->fast, st);
        if (fs.status == PF_ERR_SOLVER)
            throw Error(PF_ERR_SOLVER, "non-finite iterates at iteration " + std::to_string(fs.iteration));
        if (fs.status == PF_ERR_KERNEL_COEF || fs.status == PF_ERR_KERNEL_ROOT) {
            S->bad_commodity = fs.bad;
            throw Error(fs.status, std::string(fs.status == PF_ERR_KERNEL_COEF ? "non-finite sum coefficients"
                                                                                : "non-finite sum root") +
                                       " for commodity " + std::to_string(fs.bad));
        }
    }
    int64_t alpha = S->cfg.mode == PF_MODE_EXACT ? S->ctrl.alpha : fast_status(S->fast, st).alpha;
    double *rates_d, *sums_d;
    if (S->cfg.mode == PF_MODE_FAST) {  // pooled with the solver
        rates_d = fast_scratch(S->fast, 1);
        sums_d = fast_scratch(S->fast, 2);
    } else {
        if (S->rates_out.n < (size_t)S->P()) S->rates_out.alloc(S->P());
        if (S->sums_out.n < (size_t)S->C() + 1) S->sums_out.alloc(S->C() + 1);
        rates_d = S->rates_out.p;
        sums_d = S->sums_out.p;
    }
    PF_CUDA(cudaEventRecord(S->ev0, st));
    if (S->cfg.project)
        project_device(S->inst, solver_x(S), alpha, rates_d, st,
                       S->cfg.mode == PF_MODE_FAST);  // controller.py:275
    else
        PF_CUDA(cudaMemcpyAsync(rates_d, solver_x(S), sizeof(double) * S->P(), cudaMemcpyDeviceToDevice, st));
    exact_commodity_sums(I, rates_d, sums_d, st);
    PF_CUDA(cudaEventRecord(S->ev1, st));
    if (rates) d2h(rates, rates_d, S->P(), st);
    if (sums) d2h(sums, sums_d, S->C(), st);
    PF_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    PF_CUDA(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
    S->proj_ms += ms;
    S->finished = true;
}

// the fused-kernel entry points need a fast solver; name the layout limit when
// the instance fell back to the exact-order kernels
static void require_fast(const pf_solver *S, const char *what) {
    require(S != nullptr, "null solver");
    if (S->fast) return;
    std::string why;
    fast_supported(S->inst, &why);
    throw Error(PF_ERR_INPUT, std::string(what) + " needs the fused fast-mode kernel" +
                                  (why.empty() ? std::string(" (PF_MODE_FAST)") : ": this instance has " + why));
}

static pf_solver *solver_create(const pf_instance *inst, const pf_config *cfg) {
    require(inst && cfg, "null argument");
    validate_config(*cfg);
    DeviceGuard g(inst->device());
    std::unique_ptr<pf_solver> S(new pf_solver());
    S->inst = inst;
    S->cfg = *cfg;
    const Index &I = *inst->idx;
    if (cfg->reference_sums) {
        S->ref_sums.assign(cfg->reference_sums, cfg->reference_sums + I.C);
        S->cfg.reference_sums = nullptr;
    }
    PF_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
    PF_CUDA(cudaEventCreate(&S->ev0));
    PF_CUDA(cudaEventCreate(&S->ev1));
    if (!S->ref_sums.empty()) {  // only the trace's optimality column needs the demands on the host
        S->h_demand.resize(I.C);
        d2h(S->h_demand.data(), inst->demand.p, I.C, S->stream);
        PF_CUDA(cudaStreamSynchronize(S->stream));
    }
    // fast mode on an instance outside the fused kernel's layout limits (more
    // than 65535 edges, 32 paths or 16384 pairs per commodity): the exact-order
    // kernels run instead -- the reference's own arithmetic, on the GPU
    if (cfg->mode == PF_MODE_FAST && !fast_supported(inst, nullptr)) {
        S->cfg.mode = PF_MODE_EXACT;
        S->exact_fallback = true;
    }
    if (S->cfg.mode == PF_MODE_EXACT) {
        S->cur.alloc(I);
        S->nxt.alloc(I);
        S->sums_tmp.alloc(I.C + 1);
        S->loads_tmp.alloc(I.E + 1);
        S->svals.alloc(I.NP + 1);
        S->pk.alloc(I.P + 1);
        S->pw.alloc(I.P + 1);
        S->wsum.alloc(I.C + 1);
        S->q.alloc(I.C + 1);
        S->root_sums.alloc(I.C + 1);
        int64_t mx = std::max(std::max(I.P, I.C), std::max(I.E, I.NP));
        S->sqtmp.alloc(sqdiff_tmp_len(mx));
        S->norms.alloc(8);
        S->flags.alloc(1);
    } else {
        S->fast = fast_create(inst, *cfg, S->stream);
    }
    inst->refs.fetch_add(1);  // released by solver_destroy
    return S.release();
}

static void solver_destroy(pf_solver *S) {
    if (!S) return;
    const pf_instance *inst = S->inst;
    {
        DeviceGuard g(inst->device());
        if (S->fast) fast_release(S->fast);
        if (S->ev0) cudaEventDestroy(S->ev0);
        if (S->ev1) cudaEventDestroy(S->ev1);
        for (cudaEvent_t e : S->tev)
            if (e) cudaEventDestroy(e);
        if (S->stream) cudaStreamDestroy(S->stream);
        delete S;
    }
    instance_release(inst);  // the solver's reference
}

// ---------------------------------------------------------------- kernel-level helpers

struct Upload {
    DevBuf<double> x, y, dd, dc, dcon, dn;
    StatePtrs ptrs{};
    Upload(const pf_instance *inst, const pf_state_view *v, cudaStream_t s) {
        const Index &I = *inst->idx;
        auto up = [&](DevBuf<double> &b, const double *h, int64_t n) {
            b.alloc(n ? n : 1);
            if (h) h2d(b.p, h, n, s);
            else PF_CUDA(cudaMemsetAsync(b.p, 0, sizeof(double) * (n ? n : 1), s));
        };
        up(x, v->x, I.P);
        up(y, v->y, I.NP);
        up(dd, v->dual_demand, I.C);
        up(dc, v->dual_capacity, I.E);
        up(dcon, v->dual_consensus, I.NP);
        up(dn, v->dual_nonneg, I.P);
        ptrs = StatePtrs{x.p, y.p, dd.p, dc.p, dcon.p, dn.p};
    }
};

}  // namespace pf

extern "C" {

int pf_commodity_sums(const pf_instance *inst, const double *rates, double *out) {
    return guard([&] {
        require(inst && rates && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> r(I.P + 1), o(I.C + 1);
        h2d(r.p, rates, I.P, s);
        exact_commodity_sums(inst->view(), r.p, o.p, s);
        d2h(out, o.p, I.C, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_edge_loads(const pf_instance *inst, const double *rates, double *out) {
    return guard([&] {
        require(inst && rates && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> r(I.P + 1), o(I.E + 1);
        h2d(r.p, rates, I.P, s);
        exact_edge_loads_of_rates(inst->view(), r.p, o.p, s);
        d2h(out, o.p, I.E, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_edge_loads_from_pairs(const pf_instance *inst, const double *pv, double *out) {
    return guard([&] {
        require(inst && pv && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> r(I.NP + 1), o(I.E + 1);
        h2d(r.p, pv, I.NP, s);
        exact_edge_loads_from_pairs(inst->view(), r.p, o.p, s);
        d2h(out, o.p, I.E, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_validate_allocation(const pf_instance *inst, const double *rates, double tol, pf_violation *rep,
                           double *edge_overload, double *commodity_excess) {
    return guard([&] {
        require(inst && rates && rep, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        // scratch cached on the instance (no per-call cudaMalloc / cudaFree)
        struct ValWS {
            DevBuf<double> r, ov, ex;
            TraceScratch ts;
        };
        std::lock_guard<std::mutex> lk(inst->ws_mu);
        if (!inst->val_ws) {
            auto w = std::make_shared<ValWS>();
            w->r.alloc(I.P + 1);
            w->ov.alloc(I.E + 1);
            w->ex.alloc(I.C + 1);
            inst->val_ws = w;
        }
        ValWS &w = *static_cast<ValWS *>(inst->val_ws.get());
        h2d(w.r.p, rates, I.P, s);
        violation_stats(inst->view(), w.r.p, tol, w.ov.p, w.ex.p, w.ts, rep, s);
        if (edge_overload) d2h(edge_overload, w.ov.p, I.E, s);
        if (commodity_excess) d2h(commodity_excess, w.ex.p, I.C, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_det_diff_norm(int device, const double *a, const double *b, int64_t n, double *out) {
    return guard([&] {
        require(out != nullptr, "null argument");
        ensure_device(device);
        DeviceGuard g(device);
        DevBuf<double> da(n + 1), db(n + 1), tmp(sqdiff_tmp_len(n)), o(1);
        h2d(da.p, a, n, 0);
        h2d(db.p, b, n, 0);
        exact_sqdiff_sum(da.p, db.p, n, tmp.p, o.p, 0);
        double v;
        d2h(&v, o.p, 1, 0);
        PF_CUDA(cudaStreamSynchronize(0));
        *out = std::sqrt(v);
    });
}

int pf_update_duals(const pf_instance *inst, const pf_state_view *v, double *dd, double *dc, double *dcon, double *dn) {
    return guard([&] {
        require(inst && v, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        Upload U(inst, v, s);
        DevBuf<double> sums(I.C + 1), loads(I.E + 1), odd(I.C + 1), odc(I.E + 1), odcon(I.NP + 1), odn(I.P + 1);
        exact_update_duals(inst->view(), U.ptrs, sums.p, loads.p, odd.p, odc.p, odcon.p, odn.p, s);
        if (dd) d2h(dd, odd.p, I.C, s);
        if (dc) d2h(dc, odc.p, I.E, s);
        if (dcon) d2h(dcon, odcon.p, I.NP, s);
        if (dn) d2h(dn, odn.p, I.P, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_update_slacks(const pf_instance *inst, const pf_state_view *v, double *sd, double *sc) {
    return guard([&] {
        require(inst && v, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        Upload U(inst, v, s);
        DevBuf<double> sums(I.C + 1), loads(I.E + 1), osd(I.C + 1), osc(I.E + 1);
        exact_update_slacks(inst->view(), U.ptrs, v->beta, sums.p, loads.p, osd.p, osc.p, s);
        if (sd) d2h(sd, osd.p, I.C, s);
        if (sc) d2h(sc, osc.p, I.E, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_update_rate_suggestions(const pf_instance *inst, const pf_state_view *v, double *y) {
    return guard([&] {
        require(inst && v && y, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        Upload U(inst, v, s);
        DevBuf<double> oy(I.NP + 1), sv(I.NP + 1);
        exact_suggest(inst->view(), U.ptrs, oy.p, s, sv.p);
        d2h(y, oy.p, I.NP, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_solve_commodity_sums(const pf_instance *inst, const pf_state_view *v, int64_t alpha, double *sums,
                            int64_t *bad) {
    return guard([&] {
        require(inst && v && sums, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        Upload U(inst, v, s);
        DevBuf<double> pk(I.P + 1), pw(I.P + 1), ws(I.C + 1), q(I.C + 1), out(I.C + 1);
        DevBuf<Flags> fl(1);
        exact_coefficients(inst->view(), U.ptrs, pk.p, pw.p, ws.p, q.p, s);
        reset_flags(fl.p, s);
        exact_roots(inst->view(), ws.p, q.p, U.dd.p, v->beta, alpha, out.p, fl.p, s);
        Flags hf;
        d2h(&hf, fl.p, 1, s);
        d2h(sums, out.p, I.C, s);
        PF_CUDA(cudaStreamSynchronize(s));
        if (bad) *bad = -1;
        if (hf.bad_coef != INT_MAX) {
            if (bad) *bad = hf.bad_coef;
            throw Error(PF_ERR_KERNEL_COEF, "non-finite sum coefficients for commodity " + std::to_string(hf.bad_coef));
        }
        if (hf.bad_root != INT_MAX) {
            if (bad) *bad = hf.bad_root;
            throw Error(PF_ERR_KERNEL_ROOT, "non-finite sum root for commodity " + std::to_string(hf.bad_root));
        }
    });
}

int pf_update_rates(const pf_instance *inst, const pf_state_view *v, const double *sums, int64_t alpha, double *x) {
    return guard([&] {
        require(inst && v && sums && x, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        Upload U(inst, v, s);
        DevBuf<double> pk(I.P + 1), pw(I.P + 1), ws(I.C + 1), q(I.C + 1), ds(I.C + 1), ox(I.P + 1);
        h2d(ds.p, sums, I.C, s);
        exact_coefficients(inst->view(), U.ptrs, pk.p, pw.p, ws.p, q.p, s);
        exact_rates(inst->view(), pk.p, pw.p, ds.p, U.dd.p, v->beta, alpha, ox.p, s);
        d2h(x, ox.p, I.P, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

__global__ void k_one_root(double w, double beta, double q, int64_t alpha, double *out) {
    *out = root_scalar(1.0 + w, w / beta, q, alpha);  // kernels.py:198-203
}

int pf_solve_sum_equation(double w, double beta, double q, int64_t alpha, double *out) {
    return guard([&] {
        require(out != nullptr, "null argument");
        ensure_device(0);
        DevBuf<double> o(1);
        k_one_root<<<1, 1>>>(w, beta, q, alpha, o.p);
        PF_CHECK_LAUNCH();
        PF_CUDA(cudaMemcpy(out, o.p, sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int pf_score_paths(const pf_instance *inst, const double *rates, int64_t alpha, double *scores) {
    return guard([&] {
        require(inst && rates && scores, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> r(I.P + 1), o(I.P + 1);
        h2d(r.p, rates, I.P, s);
        score_paths_device(inst, r.p, alpha, o.p, s);
        d2h(scores, o.p, I.P, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_dao_carry_rates(const pf_instance *inst, const double *rates, double tol, double *out, int64_t *passes) {
    return guard([&] {
        require(inst && rates && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> x(I.P + 1);
        h2d(x.p, rates, I.P, s);
        const int64_t n = dao_carry_device(inst, x.p, tol, s);
        d2h(out, x.p, I.P, s);
        PF_CUDA(cudaStreamSynchronize(s));
        if (passes) *passes = n;
    });
}

int pf_project(const pf_instance *inst, const double *rates, int64_t alpha, double *out) {
    return guard([&] {
        require(inst && rates && out, "null argument");
        DeviceGuard g(inst->device());
        const Index &I = *inst->idx;
        cudaStream_t s = inst->stream;
        DevBuf<double> r(I.P + 1), o(I.P + 1);
        h2d(r.p, rates, I.P, s);
        project_device(inst, r.p, alpha, o.p, s);
        d2h(out, o.p, I.P, s);
        PF_CUDA(cudaStreamSynchronize(s));
    });
}

int pf_solver_create(const pf_instance *inst, const pf_config *cfg, pf_solver **out) {
    return guard([&] {
        require(out != nullptr, "null output handle");
        *out = solver_create(inst, cfg);
    });
}

int pf_solver_init(pf_solver *S, const double *warm) {
    return guard([&] {
        require(S != nullptr, "null solver");
        solver_init(S, warm);
    });
}

int pf_solver_run(pf_solver *S, int64_t max_steps, int64_t *done) {
    int64_t d = 0;
    int st = guard([&] {
        require(S != nullptr, "null solver");
        d = solver_run(S, max_steps);
    });
    if (done) *done = d;
    if (S && st != PF_OK) S->status = st;
    return st;
}

int pf_solver_result(pf_solver *S, pf_result *res) {
    return guard([&] {
        require(S && res, "null argument");
        solver_status(S, res);
    });
}

int pf_solver_finish(pf_solver *S, double *rates, double *sums) {
    return guard([&] {
        require(S != nullptr, "null solver");
        solver_finish(S, rates, sums);
    });
}

int pf_solver_get_x(pf_solver *S, double *x) {
    return guard([&] {
        require(S && x, "null argument");
        DeviceGuard g(S->inst->device());
        d2h(x, solver_x(S), S->P(), S->stream);
        PF_CUDA(cudaStreamSynchronize(S->stream));
    });
}

int pf_solver_get_state(pf_solver *S, double *x, double *y, double *dd, double *dc, double *dcon, double *dn,
                        double *beta, int64_t *alpha, int64_t *iteration) {
    return guard([&] {
        require(S != nullptr, "null solver");
        DeviceGuard g(S->inst->device());
        cudaStream_t st = S->stream;
        if (S->cfg.mode == PF_MODE_EXACT) {
            if (x) d2h(x, S->cur.x.p, S->P(), st);
            if (y) d2h(y, S->cur.y.p, S->NP(), st);
            if (dd) d2h(dd, S->cur.dd.p, S->C(), st);
            if (dc) d2h(dc, S->cur.dc.p, S->E(), st);
            if (dcon) d2h(dcon, S->cur.dcon.p, S->NP(), st);
            if (dn) d2h(dn, S->cur.dn.p, S->P(), st);
            PF_CUDA(cudaStreamSynchronize(st));
            if (beta) *beta = S->ctrl.beta;
            if (alpha) *alpha = S->ctrl.alpha;
            if (iteration) *iteration = S->ctrl.iteration;
        } else {
            fast_export_state(S->fast, x, y, dd, dc, dcon, dn, st);
            FastStatus fs = fast_status(S->fast, st);
            if (beta) *beta = fs.beta;
            if (alpha) *alpha = fs.alpha;
            if (iteration) *iteration = fs.iteration;
        }
    });
}

int pf_solver_time_loop(pf_solver *S, int64_t iterations, float *ms_total, float *ms_per_iter) {
    return guard([&] {
        require(S != nullptr, "null solver");
        DeviceGuard g(S->inst->device());
        require_fast(S, "time_loop");
        float ms = 0.f;
        int64_t done = fast_run(S->fast, iterations, S->stream, &ms);
        S->loop_ms += ms;
        if (ms_total) *ms_total = ms;
        if (ms_per_iter) *ms_per_iter = done ? ms / (float)done : 0.f;
    });
}

int pf_solver_kernel_stats(pf_solver *S, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes) {
    return guard([&] {
        require(S != nullptr, "null solver");
        if (S->cfg.mode != PF_MODE_FAST) {
            if (launches) *launches = 0;
            return;
        }
        fast_stats(S->fast, launches, tiles, grid, bytes);
    });
}

int pf_solver_attach_comm(pf_solver *S, pf_comm *c, int64_t global_commodities) {
    return guard([&] {
        require_fast(S, "a multi-GPU solve");
        S->comm = c;
        S->global_C = global_commodities;
        fast_set_comm(S->fast, comm_ops(c));
    });
}

int pf_solver_xchg_create(pf_solver *S, int rank, int nranks, void *handle64) {
    return guard([&] {
        require(handle64 != nullptr, "null argument");
        require_fast(S, "a multi-GPU solve");
        DeviceGuard g(S->inst->device());
        fast_xchg_create(S->fast, rank, nranks, handle64);
    });
}

int pf_solver_xchg_connect(pf_solver *S, const void *handles) {
    return guard([&] {
        require(S != nullptr && handles != nullptr, "null argument");
        DeviceGuard g(S->inst->device());
        require_fast(S, "a multi-GPU solve");
        fast_xchg_connect(S->fast, handles);
    });
}

int pf_solver_set_edge_counts(pf_solver *S, const double *counts) {
    return guard([&] {
        require(S != nullptr && counts != nullptr, "null argument");
        require_fast(S, "edge counts");
        DeviceGuard g(S->inst->device());
        fast_set_edge_counts(S->fast, counts);
    });
}

int pf_instance_fast_supported(const pf_instance *inst, int *ok, char *why, size_t why_len) {
    return guard([&] {
        require(inst != nullptr && ok != nullptr, "null argument");
        DeviceGuard g(inst->device());
        std::string w;
        *ok = fast_supported(inst, &w) ? 1 : 0;
        if (why && why_len) {
            std::snprintf(why, why_len, "%s", w.c_str());
        }
    });
}

int pf_solver_trace(pf_solver *S, pf_trace_row *rows, int64_t cap, int64_t *total) {
    return guard([&] {
        require(S != nullptr && total != nullptr && (rows != nullptr || cap == 0), "null argument");
        const int64_t n = (int64_t)S->trace.size();
        *total = n;
        if (cap > 0) std::memcpy(rows, S->trace.data(), sizeof(pf_trace_row) * (size_t)(n < cap ? n : cap));
    });
}

// pf_solver_time_to_quality: see include/pf_b200.h
static void solver_time_to_quality(pf_solver *S, const double *ref, double target, int64_t every,
                                   pf_ttq_result *out, int64_t *si, double *sq, int64_t cap) {
    require(S->initialized, "solver not initialized");
    require(S->fast != nullptr && S->comm == nullptr, "time_to_quality needs a single-GPU fast-mode solver");
    require(every >= 1, "sample_every must be >= 1");
    DeviceGuard g(S->inst->device());
    const InstView I = S->inst->view();
    cudaStream_t st = S->stream;
    FastSolver *F = S->fast;
    std::memset(out, 0, sizeof(*out));
    out->k_star = -1;
    out->quality = NAN;
    if (S->P() == 0) return;
    std::vector<double> dem(S->C());
    d2h(dem.data(), S->inst->demand.p, S->C(), st);
    PF_CUDA(cudaStreamSynchronize(st));
    const double theta = default_theta(dem);
    DevBuf<double> ref_d(S->C() + 1), q_d(1);
    h2d(ref_d.p, ref, S->C(), st);
    if (S->trace_proj.n < (size_t)S->P() + 1) S->trace_proj.alloc(S->P() + 1);
    if (S->trace_sums.n < (size_t)S->C() + 1) S->trace_sums.alloc(S->C() + 1);
    double *xcur = fast_scratch(F, 1);  // free until finish()
    auto quality = [&](int64_t alpha) {
        PF_CUDA(cudaEventRecord(S->ev0, st));
        fast_copy_x(F, xcur, st);
        project_device(S->inst, xcur, alpha, S->trace_proj.p, st, true);  // as the trace row (solver_trace_row)
        exact_commodity_sums(I, S->trace_proj.p, S->trace_sums.p, st);
        optimality_sum_dev(I, S->trace_sums.p, ref_d.p, theta, S->ts, q_d.p, st);
        PF_CUDA(cudaEventRecord(S->ev1, st));
        double h = 0.0;
        d2h(&h, q_d.p, 1, st);
        PF_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        PF_CUDA(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
        out->quality_ms += ms;
        return S->C() ? h / (double)S->C() : 1.0;
    };
    auto record = [&](int64_t it, double q) {
        if (out->samples < cap) {
            if (si) si[out->samples] = it;
            if (sq) sq[out->samples] = q;
        }
        ++out->samples;
    };
    auto run = [&](int64_t n) {
        float ms = 0.f;
        const int64_t k = fast_run(F, n, st, &ms);
        out->loop_ms += ms;
        S->loop_ms += ms;
        return k;
    };
    for (;;) {
        FastStatus fs = fast_status(F, st);
        if (fs.stopped || fs.status || fs.iteration >= S->cfg.max_iterations) break;
        const int64_t it0 = fs.iteration;
        fast_snapshot(F, st);
        const int64_t n = run(every);
        if (n == 0) break;
        fs = fast_status(F, st);
        const double q = quality(fs.alpha_used);
        record(fs.iteration, q);
        out->quality = q;
        if (q >= target) {  // the first crossing lies in (it0, it0 + n]: replay it one iteration at a time
            fast_restore(F, st);
            for (int64_t j = 1; j <= n; ++j) {
                if (run(1) == 0) break;
                const FastStatus fj = fast_status(F, st);
                const double qj = j == n ? q : quality(fj.alpha_used);
                if (j < n) record(fj.iteration, qj);
                if (qj >= target) {
                    out->k_star = fj.iteration;
                    out->quality = qj;
                    break;
                }
            }
            break;
        }
    }
    out->iterations = fast_status(F, st).iteration;
}

int pf_solver_time_to_quality(pf_solver *S, const double *ref, double target, int64_t every, pf_ttq_result *out,
                              int64_t *si, double *sq, int64_t cap) {
    return guard([&] {
        require(S != nullptr && ref != nullptr && out != nullptr, "null argument");
        solver_time_to_quality(S, ref, target, every, out, si, sq, cap);
    });
}

int pf_solver_destroy(pf_solver *S) {
    return guard([&] { solver_destroy(S); });
}

int pf_solve(const pf_instance *inst, const pf_config *cfg, const double *warm, double *rates, double *sums,
             pf_result *res, pf_trace_row *trace, int64_t trace_cap, int64_t *trace_len) {
    pf_solver *S = nullptr;
    int st = guard([&] {
        require(inst && cfg && res, "null argument");
        static const bool timing = getenv("PF_TIMING") != nullptr;  // tuning: phase wall times
        const double t0 = wall();
        S = solver_create(inst, cfg);
        const double t1 = wall();
        solver_init(S, warm);
        const double t2 = wall();
        if (S->P() > 0) solver_run(S, cfg->max_iterations);
        const double t3 = wall();
        solver_finish(S, rates, sums);
        const double t4 = wall();
        solver_status(S, res);
        if (timing)
            fprintf(stderr, "[pf_solve] create %.2f ms, init %.2f ms, run %.2f ms, finish %.2f ms\n",
                    1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3));
        if (trace && trace_len) {
            int64_t n = (int64_t)S->trace.size() < trace_cap ? (int64_t)S->trace.size() : trace_cap;
            std::memcpy(trace, S->trace.data(), sizeof(pf_trace_row) * (size_t)n);
            *trace_len = n;
        }
    });
    if (st != PF_OK && S) {
        res->status = st;
        res->bad_commodity = S->bad_commodity;
        if (S->cfg.mode == PF_MODE_EXACT) res->iterations = S->ctrl.iteration;
    }
    if (S) {
        char keep[1024];
        pf_last_error(keep, sizeof keep);
        const double t5 = wall();
        solver_destroy(S);
        if (getenv("PF_TIMING")) fprintf(stderr, "[pf_solve] destroy %.2f ms\n", 1e3 * (wall() - t5));
        set_error(keep);
    }
    return st;
}

}  // extern "C"
