/* pfsp_oracle — plain-C restatement of the reference PFSP Branch-and-Bound hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_2012_09511_b200/) never links or calls it.
 *
 * Restated from the reference (paths under /root/reference/proj):
 *   generate_taillard / taillard_named   src/instance.cpp:80-163
 *   makespan                              src/instance.cpp:165-183
 *   bound_tables / children_bounds / decompose (LB1, MinMin, prune)  src/bound.cpp:20-139
 *   Ivm init_at / select_next / branch / decode / prune_current       src/ivm.cpp:38-172
 *   explore_step                          src/explorer.cpp:37-63
 *   midpoint / compare                    src/factoradic.cpp:51-93
 *   neh                                   src/heuristic.cpp:24-103
 * LB2 (Johnson two-machine bound with lags over all machine pairs) has no reference
 * implementation; it follows SURVEY.md §8 row a22 (Lageweg et al. 1978 as cited at
 * PAPER.md:286-288). The reference cannot pin it, so LB2 is pinned to its DEFINITION:
 * or_children_bounds_lb2_exact computes every pair's two-machine relaxation optimum over all
 * job orders (subset DP, no Johnson order), and the tests require the restated order's
 * chains (and the GPU) to equal it; LB1 parity is pinned by oracle/_ref (the compiled
 * reference).
 */
#ifndef PFSP_ORACLE_H
#define PFSP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_LB1 = 1, OR_LB2 = 2 };
enum { OR_FORWARD = 0, OR_BACKWARD = 1 };

typedef struct {
  int n, m;
  int32_t* p;      /* job-major p[j*m+k] (owned copy) */
  int bound;       /* OR_LB1 | OR_LB2 */
  int npairs;      /* m(m-1)/2 */
  int* pk;         /* [npairs] first machine of pair (k < l, lexicographic) */
  int* pl;         /* [npairs] second machine */
  int* order;      /* [npairs*n] Johnson/Mitten job order per pair */
  int* lag;        /* [npairs*n] lag_j = sum_{k<i<l} p[j][i], indexed by job */
} or_problem;

typedef struct {
  uint64_t decomposed;   /* raw, as PoolStats.decomposed (explorer.hpp:46) */
  uint64_t unique;       /* raw - sum over init_at(a) of min(L, lnz(a)) */
  uint64_t leaves;
  uint64_t improvements;
  int64_t best;          /* min(initial ub, best found) */
  int32_t best_perm[512];
  int has_perm;
  double wall_s;
  int completed;
  uint64_t hist[513];    /* decomposed nodes by free-job count f (replays included) */
} or_stats;

/* instance */
int or_taillard(int n, int m, int32_t seed, int32_t* p_out);
int or_taillard_named(const char* name, int* n, int* m, int32_t* p_out /* >= 500*20 */);
int64_t or_makespan(int n, int m, const int32_t* p, const int* perm);
int64_t or_neh(int n, int m, const int32_t* p, int* perm_out);

/* problem (bounding data) */
int or_problem_init(or_problem* pr, int n, int m, const int32_t* p, int bound);
void or_problem_free(or_problem* pr);

/* one node: perm = sigma1 | free | sigma2 (bound.hpp:19-31); outputs have f entries */
int or_decompose(const or_problem* pr, const int* perm, int d1, int d2, int64_t incumbent,
                 int64_t* child_lb, int* direction, uint8_t* pruned);
/* both child sets before MinMin (bound.cpp:61-88 for LB1, row a22 for LB2) */
int or_children_bounds(const or_problem* pr, const int* perm, int d1, int d2, int64_t* lb_fwd,
                       int64_t* lb_bwd);
int64_t or_lb1_node(const or_problem* pr, const int* perm, int d1, int d2);
/* LB2 from its definition: per pair the exact optimum over all orders of the two-machine
 * time-lag relaxation (subset DP, no Johnson order); f <= 16. Pins the restated order. */
int or_children_bounds_lb2_exact(const or_problem* pr, const int* perm, int d1, int d2, int64_t* lb_fwd,
                                 int64_t* lb_bwd);

/* factoradic helpers (digits MSD first, radix n-l) */
int or_fact_compare(int n, const int* a, const int* b);
/* b == NULL means n!; returns 0 on success, -1 if a >= b */
int or_fact_midpoint(int n, const int* a, const int* b, int* out);

/* Solve over [0, n!) split into prefix_depth-level subtrees pulled by nthreads workers.
 * prefix_depth = 0 and nthreads = 1 reproduces pool_run with K = 1 exactly.
 * prune_disabled mirrors PoolConfig.disable_pruning; pinned != 0 means prune >= ub and never
 * improve (explore_step(prune = ub, improve = 0)). time_limit_s <= 0 means none. */
int or_solve(const or_problem* pr, int64_t ub, int nthreads, int prefix_depth, int pinned,
             int prune_disabled, double time_limit_s, or_stats* out);

#ifdef __cplusplus
}
#endif

#endif
