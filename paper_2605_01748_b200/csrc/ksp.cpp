// Native k-shortest loopless paths (Yen) reproducing the selection rule of the
// reference's harness.k_shortest_paths (pathfair/harness.py:138-176):
//
//   * the routing graph keeps only edges with capacity > 0 (harness.py:124-131);
//   * k == 1: one Dijkstra per commodity (harness.py:145-155);
//   * k >= 2: paths are generated in nondecreasing weight; generation stops at the
//     first path heavier than the k-th lightest seen so far, or after k+16
//     candidates (tie capture); candidates are sorted by (weight, edge-id tuple)
//     and the first k kept (harness.py:157-173).
//
// Path weight is the left-to-right fp64 sum of edge weights, which is what the
// reference's `float(sum(weights[e] for e in eids))` computes.  Host code: this
// is input preparation (a config-3 prerequisite), not the GPU
// hot path.  Commodities are processed in parallel with OpenMP.
#include "pf_gen.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct Graph {
    int n = 0;
    std::vector<int> ptr;          // CSR by source node
    std::vector<int> nbr;          // head node
    std::vector<int> eid;          // edge id
    std::vector<double> w;         // edge weight
    std::vector<int> esrc, edst;   // per edge id
    std::vector<double> ew;        // per edge id
    std::vector<int> rptr, rnbr, reid;  // reverse CSR (by head)
};

struct Path {
    double w;
    std::vector<int> edges;
    bool operator<(const Path &o) const {
        if (w != o.w) return w < o.w;
        return edges < o.edges;
    }
    bool operator==(const Path &o) const { return edges == o.edges; }
};

double path_weight(const Graph &g, const std::vector<int> &edges) {
    double s = 0.0;  // Python sum() starts from int 0: 0 + w0 == w0 exactly
    for (int e : edges) s += g.ew[e];
    return s;
}

struct Workspace {
    std::vector<double> dist;
    std::vector<int> pred_edge;
    std::vector<char> done, banned_node, banned_edge;
    std::vector<double> h;  // exact distance-to-target on the full graph (A* potential)
    void init(const Graph &g, int n_edges) {
        dist.assign(g.n, 0.0);
        pred_edge.assign(g.n, -1);
        done.assign(g.n, 0);
        banned_node.assign(g.n, 0);
        banned_edge.assign(n_edges, 0);
        h.assign(g.n, 0.0);
    }
};

// Reverse Dijkstra from t on the full routing graph: h[v] = dist(v -> t).
void reverse_dijkstra(const Graph &g, int t, std::vector<double> &h) {
    const double INF = INFINITY;
    std::fill(h.begin(), h.end(), INF);
    std::vector<char> done(g.n, 0);
    typedef std::pair<double, int> QE;
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
    h[t] = 0.0;
    pq.push({0.0, t});
    while (!pq.empty()) {
        QE top = pq.top();
        pq.pop();
        int u = top.second;
        if (done[u]) continue;
        done[u] = 1;
        for (int j = g.rptr[u]; j < g.rptr[u + 1]; ++j) {
            int v = g.rnbr[j];
            double nd = h[u] + g.ew[g.reid[j]];
            if (nd < h[v]) {
                h[v] = nd;
                pq.push({nd, v});
            }
        }
    }
}

// Shortest s->t path avoiding banned nodes/edges.  Plain Dijkstra ordered by
// (distance, push order), strictly-smaller relaxation, adjacency in edge-id
// order (networkx's insertion order).  Returns false if unreachable.
bool dijkstra(const Graph &g, Workspace &ws, int s, int t, std::vector<int> &out_edges) {
    const double INF = INFINITY;
    std::fill(ws.dist.begin(), ws.dist.end(), INF);
    std::fill(ws.done.begin(), ws.done.end(), 0);
    std::fill(ws.pred_edge.begin(), ws.pred_edge.end(), -1);
    struct QE {
        double d;
        long c;
        int v;
        bool operator>(const QE &o) const { return d != o.d ? d > o.d : c > o.c; }
    };
    // A* with the exact unconstrained distance-to-target as potential: bans only
    // remove edges/nodes, so the potential stays admissible and consistent and
    // the search returns the same shortest path as plain Dijkstra (up to exact
    // weight ties), while settling a handful of nodes instead of the graph.
    const double *h = ws.h.data();
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
    long counter = 0;
    ws.dist[s] = 0.0;
    if (!(h[s] < INF)) return false;
    pq.push({h[s], counter++, s});
    while (!pq.empty()) {
        QE top = pq.top();
        pq.pop();
        int u = top.v;
        if (ws.done[u]) continue;
        ws.done[u] = 1;
        if (u == t) break;
        for (int j = g.ptr[u]; j < g.ptr[u + 1]; ++j) {
            int v = g.nbr[j];
            int e = g.eid[j];
            if (ws.banned_node[v] || ws.banned_edge[e] || ws.done[v]) continue;
            double nd = ws.dist[u] + g.w[j];
            if (nd < ws.dist[v] && h[v] < INF) {
                ws.dist[v] = nd;
                ws.pred_edge[v] = e;
                pq.push({nd + h[v], counter++, v});
            }
        }
    }
    if (!(ws.dist[t] < INF)) return false;
    out_edges.clear();
    for (int v = t; v != s;) {
        int e = ws.pred_edge[v];
        out_edges.push_back(e);
        v = g.esrc[e];
    }
    std::reverse(out_edges.begin(), out_edges.end());
    return true;
}

// Yen's algorithm as a generator of simple s->t paths in nondecreasing
// (weight, edge tuple) order.
struct Yen {
    const Graph &g;
    Workspace &ws;
    int s, t;
    std::vector<Path> A;
    std::vector<Path> B;  // candidate heap (min by Path::operator<)
    bool exhausted = false;

    Yen(const Graph &g_, Workspace &ws_, int s_, int t_) : g(g_), ws(ws_), s(s_), t(t_) {}

    static bool heap_cmp(const Path &a, const Path &b) { return b < a; }

    bool in_candidates(const std::vector<int> &edges) const {
        for (const Path &p : B)
            if (p.edges == edges) return true;
        for (const Path &p : A)
            if (p.edges == edges) return true;
        return false;
    }

    bool next(Path &out) {
        if (exhausted) return false;
        if (A.empty()) {
            std::vector<int> e;
            if (!dijkstra(g, ws, s, t, e)) {
                exhausted = true;
                return false;
            }
            A.push_back({path_weight(g, e), e});
            out = A.back();
            return true;
        }
        const Path &last = A.back();
        // nodes of the last path
        std::vector<int> nodes;
        nodes.push_back(s);
        for (int e : last.edges) nodes.push_back(g.edst[e]);
        std::vector<int> spur;
        for (size_t i = 0; i + 1 < nodes.size(); ++i) {
            int spur_node = nodes[i];
            // ban the next edge of every accepted path sharing this root
            for (const Path &p : A) {
                if (p.edges.size() > i && std::equal(last.edges.begin(), last.edges.begin() + i, p.edges.begin()))
                    ws.banned_edge[p.edges[i]] = 1;
            }
            for (size_t j = 0; j < i; ++j) ws.banned_node[nodes[j]] = 1;
            if (dijkstra(g, ws, spur_node, t, spur)) {
                std::vector<int> full(last.edges.begin(), last.edges.begin() + i);
                full.insert(full.end(), spur.begin(), spur.end());
                if (!in_candidates(full)) {
                    B.push_back({path_weight(g, full), full});
                    std::push_heap(B.begin(), B.end(), heap_cmp);
                }
            }
            for (size_t j = 0; j < i; ++j) ws.banned_node[nodes[j]] = 0;
            for (const Path &p : A)
                if (p.edges.size() > i) ws.banned_edge[p.edges[i]] = 0;
        }
        if (B.empty()) {
            exhausted = true;
            return false;
        }
        std::pop_heap(B.begin(), B.end(), heap_cmp);
        A.push_back(B.back());
        B.pop_back();
        out = A.back();
        return true;
    }
};

}  // namespace

struct pf_ksp_result {
    std::vector<std::vector<std::vector<int>>> paths;  // per commodity
};

extern "C" {

// Compute up to k paths per commodity.  Returns an opaque handle (nullptr on bad input).
void *pf_ksp_run(int32_t n_nodes, int64_t n_edges, const int64_t *edge_src, const int64_t *edge_dst,
                 const double *weight, const double *capacity, int64_t n_coms, const int64_t *com_src,
                 const int64_t *com_dst, int32_t k, int32_t n_threads) {
    if (k < 1 || n_nodes < 0 || n_edges < 0) return nullptr;
    Graph g;
    g.n = n_nodes;
    g.esrc.resize(n_edges);
    g.edst.resize(n_edges);
    g.ew.resize(n_edges);
    std::vector<int> deg(n_nodes + 1, 0), rdeg(n_nodes + 1, 0);
    for (int64_t e = 0; e < n_edges; ++e) {
        g.esrc[e] = (int)edge_src[e];
        g.edst[e] = (int)edge_dst[e];
        g.ew[e] = weight[e];
        if (capacity[e] > 0) {
            deg[edge_src[e] + 1]++;
            rdeg[edge_dst[e] + 1]++;
        }
    }
    for (int v = 0; v < n_nodes; ++v) {
        deg[v + 1] += deg[v];
        rdeg[v + 1] += rdeg[v];
    }
    g.ptr = deg;
    g.rptr = rdeg;
    g.nbr.resize(deg[n_nodes]);
    g.eid.resize(deg[n_nodes]);
    g.w.resize(deg[n_nodes]);
    g.rnbr.resize(rdeg[n_nodes]);
    g.reid.resize(rdeg[n_nodes]);
    std::vector<int> fill(deg.begin(), deg.end() - 1), rfill(rdeg.begin(), rdeg.end() - 1);
    for (int64_t e = 0; e < n_edges; ++e) {  // edge-id order == networkx insertion order
        if (!(capacity[e] > 0)) continue;
        int u = (int)edge_src[e], v = (int)edge_dst[e];
        int j = fill[u]++;
        g.nbr[j] = v;
        g.eid[j] = (int)e;
        g.w[j] = weight[e];
        int r = rfill[v]++;
        g.rnbr[r] = u;
        g.reid[r] = (int)e;
    }
    pf_ksp_result *res = new pf_ksp_result();
    res->paths.resize(n_coms);
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
    // Process commodities grouped by destination so the A* potential (one
    // reverse Dijkstra per destination) is shared across that group.
    std::vector<int64_t> order(n_coms);
    for (int64_t c = 0; c < n_coms; ++c) order[c] = c;
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return com_dst[a] < com_dst[b]; });
#pragma omp parallel
    {
        Workspace ws;
        ws.init(g, (int)n_edges);
        int h_target = -1;
#pragma omp for schedule(dynamic, 32)
        for (int64_t oc = 0; oc < n_coms; ++oc) {
            int64_t c = order[oc];
            int s = (int)com_src[c], t = (int)com_dst[c];
            if (t != h_target) {
                reverse_dijkstra(g, t, ws.h);
                h_target = t;
            }
            auto &out = res->paths[c];
            Yen yen(g, ws, s, t);
            Path p;
            if (k == 1) {
                if (yen.next(p)) out.push_back(p.edges);
                continue;
            }
            std::vector<Path> cand;
            while (yen.next(p)) {
                if ((int)cand.size() >= k) {
                    std::vector<double> ws_sorted;
                    for (auto &q : cand) ws_sorted.push_back(q.w);
                    std::sort(ws_sorted.begin(), ws_sorted.end());
                    if (p.w > ws_sorted[k - 1]) break;
                }
                cand.push_back(p);
                if ((int)cand.size() >= k + 16) break;
            }
            std::stable_sort(cand.begin(), cand.end());
            for (int i = 0; i < (int)cand.size() && i < k; ++i) out.push_back(cand[i].edges);
        }
    }
    return res;
}

void pf_ksp_sizes(void *h, int64_t *n_paths, int64_t *n_pairs) {
    pf_ksp_result *r = (pf_ksp_result *)h;
    int64_t P = 0, NP = 0;
    for (auto &pc : r->paths) {
        P += (int64_t)pc.size();
        for (auto &p : pc) NP += (int64_t)p.size();
    }
    *n_paths = P;
    *n_pairs = NP;
}

void pf_ksp_export(void *h, int64_t *com_path_ptr, int64_t *path_edge_ptr, int64_t *path_edges) {
    pf_ksp_result *r = (pf_ksp_result *)h;
    int64_t P = 0, NP = 0;
    com_path_ptr[0] = 0;
    path_edge_ptr[0] = 0;
    for (size_t c = 0; c < r->paths.size(); ++c) {
        for (auto &p : r->paths[c]) {
            for (int e : p) path_edges[NP++] = e;
            path_edge_ptr[++P] = NP;
        }
        com_path_ptr[c + 1] = P;
    }
}

void pf_ksp_free(void *h) { delete (pf_ksp_result *)h; }

// model.py:183-203 (_check_path) for every path, in parallel: returns the
// first (commodity-major) path that is empty, has an out-of-range edge id, does
// not start / end at its commodity's nodes, has non-adjacent consecutive edges
// or revisits a node; -1 when all paths are valid.
int64_t pf_validate_paths(int64_t n_commodities, const int64_t *com_path_ptr, const int64_t *path_edge_ptr,
                          const int64_t *path_edges, int64_t n_edges, const int64_t *edge_src,
                          const int64_t *edge_dst, const int64_t *com_src, const int64_t *com_dst) {
    const int64_t P = com_path_ptr[n_commodities];
    int64_t first = INT64_MAX;
#pragma omp parallel
    {
        int64_t mine = INT64_MAX;
        std::vector<int64_t> seen;
#pragma omp for schedule(dynamic, 4096)
        for (int64_t c = 0; c < n_commodities; ++c) {
            for (int64_t p = com_path_ptr[c]; p < com_path_ptr[c + 1] && p < mine; ++p) {
                const int64_t lo = path_edge_ptr[p], hi = path_edge_ptr[p + 1];
                bool bad = hi <= lo;
                for (int64_t t = lo; t < hi && !bad; ++t) bad = path_edges[t] < 0 || path_edges[t] >= n_edges;
                if (!bad) bad = edge_src[path_edges[lo]] != com_src[c] || edge_dst[path_edges[hi - 1]] != com_dst[c];
                for (int64_t t = lo; t + 1 < hi && !bad; ++t) bad = edge_dst[path_edges[t]] != edge_src[path_edges[t + 1]];
                if (!bad) {  // simple: src(first) and every dst distinct
                    seen.assign(1, edge_src[path_edges[lo]]);
                    for (int64_t t = lo; t < hi && !bad; ++t) {
                        const int64_t v = edge_dst[path_edges[t]];
                        for (int64_t u : seen) bad = bad || u == v;
                        seen.push_back(v);
                    }
                }
                if (bad) mine = std::min(mine, p);
            }
        }
#pragma omp critical
        first = std::min(first, mine);
    }
    (void)P;
    return first == INT64_MAX ? -1 : first;
}

}  // extern "C"
