// Fast mode: fused persistent kernel for the GATE iteration (see fused.cu).
#pragma once

#include "pf_internal.cuh"

namespace pf {

struct FastSolver;

struct FastStatus {
    int64_t iteration;   // completed iterations
    int64_t alpha;       // alpha for the next iteration (after any increment)
    int64_t alpha_used;  // alpha used by the last completed iteration
    double beta;         // beta for the next iteration
    double beta_used;    // beta used by the last completed iteration
    double s, r;         // residuals of the last completed iteration
    int32_t stopped;
    int32_t status;
    int64_t bad;
};

// The fused kernel's layout limits: u16 edge ids (E <= 65535), one warp lane
// per path (<= 32 paths per commodity), a commodity within one tile (<= 16384
// pairs).  Cached on the instance; `why` names the first limit that fails.
bool fast_supported(const pf_instance *inst, std::string *why);
FastSolver *fast_create(const pf_instance *inst, const pf_config &cfg, cudaStream_t s);
void fast_destroy(FastSolver *f);
// Return a solver to its instance's pool (kept for the next solve), or destroy it.
void fast_release(FastSolver *f);
// Device scratch owned by the (pooled) solver, grown on demand: 0 warm-start
// staging [P], 1 projected rates [P], 2 commodity sums [C + 1], 3 one flag.
double *fast_scratch(FastSolver *f, int which);
void fast_init(FastSolver *f, const double *d_x0, int64_t alpha0, double beta0, cudaStream_t s);
// Runs up to max_steps iterations (fewer if the controller stops); returns the count.
int64_t fast_run(FastSolver *f, int64_t max_steps, cudaStream_t s, float *ms);
FastStatus fast_status(FastSolver *f, cudaStream_t s);
// Traced runs without host round trips: one iteration launched asynchronously
// (single GPU), the controller's row fields copied to a device row
// (iteration, alpha_used, beta_used, s, r, stopped-or-failed, status), and the
// device address of alpha_used.
void fast_launch_one(FastSolver *f, cudaStream_t s);
void fast_ctrl_row(FastSolver *f, double *row7, cudaStream_t s);
const int64_t *fast_alpha_used_dev(FastSolver *f);
// dst [P] = the current rates (buffer chosen on the device: no host read)
void fast_copy_x(FastSolver *f, double *dst, cudaStream_t s);
const double *fast_x(FastSolver *f);
const double *fast_root_sums(FastSolver *f);
void fast_export_state(FastSolver *f, double *x, double *y, double *dd, double *dc, double *dcon, double *dn,
                       cudaStream_t s);
void fast_stats(FastSolver *f, int64_t *launches, int64_t *tiles, int64_t *grid, int64_t *bytes_per_iter);
// A device copy of every buffer the next launch reads (iterates, duals, edge
// partials, controller): restoring it makes the following iterations bitwise
// those that followed the snapshot (every reduction has a fixed order).
void fast_snapshot(FastSolver *f, cudaStream_t s);
void fast_restore(FastSolver *f, cudaStream_t s);

// Multi-GPU hooks (dist.cu): reduce edge partial vectors / residual scalars across ranks.
struct CommOps {
    void *ctx;
    void (*allreduce_sum)(void *ctx, double *buf, int64_t n, cudaStream_t s);
};
void fast_set_comm(FastSolver *f, const CommOps *ops);

// Multi-GPU over peer memory (one process per GPU, CUDA IPC): allocate this
// rank's exchange buffer and return its 64-byte IPC handle; connect with the
// handles of all ranks (rank order); the suggestion divisor n_e + 1 counts the
// paths of all ranks (kernels.py:94), set from the host.
void fast_xchg_create(FastSolver *f, int rank, int nranks, void *handle64);
void fast_xchg_connect(FastSolver *f, const void *handles);
void fast_set_edge_counts(FastSolver *f, const double *counts);

}  // namespace pf
