/* pf_gen.h -- host-only input preparation for the GATE solver (libpf_gen.so).
 *
 * Not part of the GPU hot path: the reference builds its inputs with
 * networkx (pathfair/harness.py:138-176) and validates paths in pure Python
 * (pathfair/model.py:183-203).  These are native equivalents, kept in their
 * own CPU-only library (g++ -fopenmp, no CUDA) so that programs that only
 * need inputs -- e.g. bench.py's reference arm -- never map the solver.
 *
 *   pf_ksp_*            harness.py:138-176 k_shortest_paths (Yen, OpenMP)
 *   pf_validate_paths   model.py:183-203 _check_path over every path
 */
#ifndef PF_GEN_H
#define PF_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- host input preparation: k shortest paths (harness.py:138-176) ---- */
void *pf_ksp_run(int32_t n_nodes, int64_t n_edges, const int64_t *edge_src, const int64_t *edge_dst,
                 const double *weight, const double *capacity, int64_t n_coms, const int64_t *com_src,
                 const int64_t *com_dst, int32_t k, int32_t n_threads);
void pf_ksp_sizes(void *h, int64_t *n_paths, int64_t *n_pairs);
void pf_ksp_export(void *h, int64_t *com_path_ptr, int64_t *path_edge_ptr, int64_t *path_edges);
void pf_ksp_free(void *h);
/* model.py:183-203 _check_path over every path (host, OpenMP): first bad path
 * in commodity-major order, or -1 (build_instance's validation) */
int64_t pf_validate_paths(int64_t n_commodities, const int64_t *com_path_ptr, const int64_t *path_edge_ptr,
                          const int64_t *path_edges, int64_t n_edges, const int64_t *edge_src,
                          const int64_t *edge_dst, const int64_t *com_src, const int64_t *com_dst);

#ifdef __cplusplus
}
#endif

#endif /* PF_GEN_H */
