/*
 * pf_b200.h -- C ABI of the B200-native GATE max-min-fair TE solver.
 *
 * Plain pointers and sizes only (no torch / CUDA types).  Every entry point
 * returns a status (0 == PF_OK); pf_last_error() returns the message of the
 * last failure on the calling thread.  Host pointers are ordinary pageable or
 * pinned host memory; the library owns all device memory.
 *
 * Each entry point replaces one interface of the reference package `pathfair`
 * (paths relative to /root/reference/pkg/src/pathfair):
 *
 *   pf_instance_create          model.py:206-271  build_instance (index part)
 *   pf_instance_with_conditions model.py:274-294  with_conditions
 *   pf_instance_export_index    model.py:135-180  Instance index arrays
 *   pf_commodity_sums           model.py:297-302  commodity_sums
 *   pf_edge_loads               model.py:305-311  edge_loads
 *   pf_edge_loads_from_pairs    model.py:314-319  edge_loads_from_pairs
 *   pf_validate_allocation      model.py:335-369  validate_allocation
 *   pf_update_duals             kernels.py:206-216 update_duals
 *   pf_update_slacks            kernels.py:219-232 update_slacks
 *   pf_update_rate_suggestions  kernels.py:235-252 update_rate_suggestions
 *   pf_solve_commodity_sums     kernels.py:267-282 solve_commodity_sums
 *   pf_update_rates             kernels.py:285-296 update_rates
 *   pf_solve_sum_equation       kernels.py:198-203 solve_sum_equation
 *   pf_det_diff_norm            _reduce.py:118-128 det_diff_norm
 *   pf_score_paths              projection.py:22-32 score_paths
 *   pf_project                  projection.py:51-107 project
 *   pf_dao_carry_rates          oracles.py:262-287 dao_carry_rates (drift carry)
 *   pf_solve                    controller.py:197-284 solve
 *   pf_solver_*                 controller.py:197-284, split so the device loop can
 *                               be timed / sharded (no reference equivalent)
 *
 * Input generation (k shortest paths, path validation) is host-only code in a
 * separate library, libpf_gen.so (include/pf_gen.h).
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pf_status {
    PF_OK = 0,
    PF_ERR_INPUT = 1,       /* pathfair.model.InputError            */
    PF_ERR_KERNEL_COEF = 2, /* pathfair.kernels.KernelError (coefficients) */
    PF_ERR_KERNEL_ROOT = 3, /* pathfair.kernels.KernelError (root)  */
    PF_ERR_SOLVER = 4,      /* pathfair.controller.SolverError      */
    PF_ERR_CUDA = 5,
    PF_ERR_NOMEM = 6,
    PF_ERR_COMM = 7
};

enum pf_index_field {
    PF_KEPT_ROWS = 0,
    PF_COM_PATH_PTR = 1,
    PF_PATH_COM = 2,
    PF_HOPS = 3,
    PF_PAIR_PTR = 4,
    PF_PAIR_EDGE = 5,
    PF_PAIR_PATH = 6,
    PF_EDGE_PATH_COUNT = 7,
    PF_EDGE_PAIR_PTR = 8,
    PF_EDGE_PAIRS = 9
};

enum pf_value_field { PF_DEMAND = 0, PF_CAPACITY = 1 };

enum pf_mode {
    PF_MODE_EXACT = 0, /* reference operation order, bitwise for alpha <= 1 */
    PF_MODE_FAST = 1   /* fused persistent kernel, deterministic tile order   */
};

typedef struct pf_instance pf_instance;
typedef struct pf_solver pf_solver;
typedef struct pf_comm pf_comm;

/* SolverState view (kernels.py:24-44); all host arrays, sized by the instance. */
typedef struct {
    const double *x;              /* P  */
    const double *y;              /* NP */
    const double *dual_demand;    /* C  */
    const double *dual_capacity;  /* E  */
    const double *dual_consensus; /* NP */
    const double *dual_nonneg;    /* P  */
    double beta;
    int64_t alpha;
} pf_state_view;

/* SolverConfig (controller.py:29-61) + build-only knobs. */
typedef struct {
    int64_t alpha_target; /* -1 == None: continue until the stagnation stop (max-min) */
    double gamma;
    double beta0;
    double residual_ratio;
    double beta_scale;
    int64_t max_iterations;
    double beta_min;
    double beta_max;
    int32_t adapt;
    int32_t trace;
    int32_t mode;                 /* pf_mode */
    int32_t project;              /* 1: project the final iterate (solve() always does) */
    const double *reference_sums; /* nullable host [C]: trace optimality column */
} pf_config;

/* IterationTrace (controller.py:74-84); optimality is NaN when absent. */
typedef struct {
    int64_t iteration;
    int64_t alpha;
    double beta, s, r, objective, pct_violated, mean_relative_violation, optimality;
} pf_trace_row;

typedef struct {
    int64_t iterations;
    int64_t alpha;
    int32_t converged;
    int32_t status;
    int64_t bad_commodity; /* KernelError commodity index, else -1 */
    double beta;
    double runtime_s;      /* init .. projection, wall clock (controller.py:204,281) */
    double loop_ms;        /* device time of the iteration loop (CUDA events) */
    double projection_ms;  /* device time of the projection */
    int32_t exact_fallback; /* 1: mode FAST was requested outside the fused layout limits (more than 32
                               paths or 16,384 pairs per commodity, or 65,535 edges) and the exact-order
                               kernels ran instead */
    int32_t reserved;
} pf_result;

typedef struct {
    int64_t n_violated;
    int64_t negative_count;
    double worst_negative;
    double pct_violated;
    double mean_relative_violation;
} pf_violation;

/* ---- errors / device ---- */
int pf_last_error(char *buf, size_t cap);
int pf_device_info(int device, int *sm_count, int64_t *l2_bytes, int64_t *hbm_bytes, char *name, size_t name_cap);

/* ---- incidence store ---- */
int pf_instance_create(int device, int64_t n_commodities0, int64_t n_edges, const int64_t *com_path_ptr0,
                       const int64_t *path_edge_ptr0, const int64_t *path_edges0, const double *demand0,
                       const double *capacity, pf_instance **out);
int pf_instance_with_conditions(const pf_instance *base, const double *capacity /*nullable*/,
                                const double *demand /*nullable*/, pf_instance **out);
int pf_instance_destroy(pf_instance *inst);
int pf_instance_sizes(const pf_instance *inst, int64_t *C, int64_t *P, int64_t *E, int64_t *NP);
/* Whether fast mode's fused kernel can run this instance (at most 32 paths and
 * 16,384 pairs per commodity, 65,535 edges); otherwise `why` says which limit. */
int pf_instance_fast_supported(const pf_instance *inst, int *ok, char *why /*nullable*/, size_t why_len);
int pf_instance_export_index(const pf_instance *inst, int field, int64_t *out);
int pf_instance_export_values(const pf_instance *inst, int field, double *out);

/* ---- model-level reductions (exact reference order) ---- */
int pf_commodity_sums(const pf_instance *inst, const double *rates, double *out);
int pf_edge_loads(const pf_instance *inst, const double *rates, double *out);
int pf_edge_loads_from_pairs(const pf_instance *inst, const double *pair_values, double *out);
int pf_validate_allocation(const pf_instance *inst, const double *rates, double tol, pf_violation *report,
                           double *edge_overload /*nullable E*/, double *commodity_excess /*nullable C*/);
int pf_det_diff_norm(int device, const double *a, const double *b, int64_t n, double *out);

/* ---- iterate kernels (exact reference order; pure functions of the state) ---- */
int pf_update_duals(const pf_instance *inst, const pf_state_view *st, double *dd, double *dc, double *dcon,
                    double *dn);
int pf_update_slacks(const pf_instance *inst, const pf_state_view *st, double *sd, double *sc);
int pf_update_rate_suggestions(const pf_instance *inst, const pf_state_view *st, double *y);
int pf_solve_commodity_sums(const pf_instance *inst, const pf_state_view *st, int64_t alpha, double *sums,
                            int64_t *bad_commodity);
int pf_update_rates(const pf_instance *inst, const pf_state_view *st, const double *sums, int64_t alpha,
                    double *x);
int pf_solve_sum_equation(double w_sum, double beta, double q, int64_t alpha, double *out);

/* ---- projection ---- */
int pf_score_paths(const pf_instance *inst, const double *rates, int64_t alpha, double *scores);
int pf_project(const pf_instance *inst, const double *rates, int64_t alpha, double *out);

/* ---- drift carry (oracles.py:262-287): a stale allocation applied to the
 * instance's current conditions; bitwise equal to the reference.  `passes`
 * (nullable) = edge passes that scaled. ---- */
int pf_dao_carry_rates(const pf_instance *inst, const double *rates, double tol, double *out, int64_t *passes);

/* ---- full solve (controller.py:197-284) ---- */
int pf_solve(const pf_instance *inst, const pf_config *cfg, const double *warm_start /*nullable P*/,
             double *rates /*P*/, double *sums /*C*/, pf_result *res, pf_trace_row *trace, int64_t trace_cap,
             int64_t *trace_len);

/* ---- device-resident solver (bench / sharding) ---- */
int pf_solver_create(const pf_instance *inst, const pf_config *cfg, pf_solver **out);
int pf_solver_init(pf_solver *s, const double *warm_start /*nullable host P*/);
int pf_solver_run(pf_solver *s, int64_t max_steps, int64_t *iterations_done);
int pf_solver_result(pf_solver *s, pf_result *res);
int pf_solver_finish(pf_solver *s, double *rates /*nullable*/, double *sums /*nullable*/);
int pf_solver_get_x(pf_solver *s, double *x);
int pf_solver_get_state(pf_solver *s, double *x, double *y, double *dd, double *dc, double *dcon, double *dn,
                        double *beta, int64_t *alpha, int64_t *iteration);
int pf_solver_time_loop(pf_solver *s, int64_t iterations, float *ms_total, float *ms_kernel_per_iter);
int pf_solver_kernel_stats(pf_solver *s, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes_per_iter);
/* The IterationTrace rows recorded so far (controller.py:173-194): copies min(cap, total) rows,
 * *total = the number recorded (lets a caller size its buffer by the actual run, not max_iterations). */
int pf_solver_trace(pf_solver *s, pf_trace_row *rows /*nullable when cap == 0*/, int64_t cap, int64_t *total);
/* Time to quality, on the device in one pass (the optimality column of controller.py:173-194
 * used as a stopping instrument): from the solver's current state, run until the
 * first iteration k whose post-projection optimality_from_sums(S_k, reference_sums,
 * default_theta) (oracles.py:51-53, 244-254) is >= target, or the controller stops / reaches
 * max_iterations.  S_k = commodity sums of project(x_k, alpha_k) (the trace row's alpha).  The
 * quality is sampled every `sample_every` iterations (a device projection, a device metric, one
 * scalar read); the chunk where it first reaches the target is replayed from a device snapshot
 * one iteration at a time, so k* is exact without re-solving from the start.  On return the
 * solver stands at k* (or at the stop).  Fast mode, single GPU.  Each sample is a
 * (iteration, optimality) pair, bitwise the trace row's optimality at that iteration. */
typedef struct {
    int64_t k_star;      /* -1: target not reached */
    int64_t iterations;  /* the solver's iteration on return */
    double quality;      /* optimality at k* (or at the last sample) */
    double loop_ms;      /* device time of the iterations run (replays included) */
    double quality_ms;   /* device time of the projections + metrics */
    int64_t samples;     /* samples taken (may exceed sample_cap; min(cap, samples) are stored) */
} pf_ttq_result;
int pf_solver_time_to_quality(pf_solver *s, const double *reference_sums /*host C*/, double target,
                              int64_t sample_every, pf_ttq_result *out, int64_t *sample_iteration /*nullable*/,
                              double *sample_quality /*nullable*/, int64_t sample_cap);
int pf_solver_destroy(pf_solver *s);

/* ---- multi-GPU: one process per GPU, NCCL over NVLink (dlopen'ed libnccl) ---- */
int pf_comm_unique_id(void *id128);
int pf_comm_create(int nranks, int rank, const void *id128, int device, pf_comm **out);
int pf_comm_destroy(pf_comm *c);
int pf_solver_attach_comm(pf_solver *s, pf_comm *c, int64_t global_commodities);
/* Multi-GPU over NVLink peer memory (one process per GPU): the fused kernel
 * writes its rank-local per-edge totals into every rank's exchange buffer and
 * meets the other ranks at a counter barrier (no host round trip, no NCCL).
 * xchg_create returns this rank's 64-byte CUDA IPC handle; xchg_connect takes
 * all ranks' handles (rank order).  set_edge_counts: global paths per edge
 * (the divisor n_e + 1 of kernels.py:94) summed over the ranks' shards. */
int pf_solver_xchg_create(pf_solver *s, int rank, int nranks, void *handle64);
int pf_solver_xchg_connect(pf_solver *s, const void *handles);
int pf_solver_set_edge_counts(pf_solver *s, const double *counts);

#ifdef __cplusplus
}
#endif

#endif /* PF_B200_H */
