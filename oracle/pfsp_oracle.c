/* pfsp_oracle.c — CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 * See pfsp_oracle.h for the reference file:line each function follows. */
#define _POSIX_C_SOURCE 200809L
#include "pfsp_oracle.h"

#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OR_NO_INCUMBENT INT64_MAX

static double or_now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

/* ---------------------------------------------------------------- instance */

/* Park-Miller minimal standard generator via Schrage's factorisation, drawn
 * machine-major (src/instance.cpp:80-114). */
int or_taillard(int n, int m, int32_t seed, int32_t* p_out) {
  if (n < 1 || m < 1 || seed < 1 || seed > 2147483645) return -1;
  int64_t s = seed;
  for (int k = 0; k < m; ++k) {
    for (int j = 0; j < n; ++j) {
      int64_t hi = s / 127773, lo = s % 127773;
      s = 16807 * lo - 2836 * hi;
      if (s < 0) s += 2147483647;
      p_out[j * m + k] = (int32_t)(1 + (s * 99) / 2147483647);
    }
  }
  return 0;
}

/* Seed table of the 120 Taillard instances (src/instance.cpp:125-138; Taillard 1993). */
static const int32_t kTaSeeds[120] = {
    873654221,  379008056,  1866992158, 216771124,  495070989,  402959317,  1369363414, 2021925980,
    573109518,  88325120,   587595453,  1401007982, 873136276,  268827376,  1634173168, 691823909,
    73807235,   1273398721, 2065119309, 1672900551, 479340445,  268827376,  1958948863, 918272953,
    555010963,  2010851491, 1519833303, 1748670931, 1923497586, 1829909967, 1328042058, 200382020,
    496319842,  1203030903, 1730708564, 450926852,  1303135678, 1273398721, 587288402,  248421594,
    1958948863, 575633267,  655816003,  1977864101, 93805469,   1803345551, 49612559,   1899802599,
    2013025619, 578962478,  1539989115, 691823909,  655816003,  1315102446, 1949668355, 1923497586,
    1805594913, 1861070898, 715643788,  464843328,  896678084,  1179439976, 1122278347, 416756875,
    267829958,  1835213917, 1328833962, 1418570761, 161033112,  304212574,  1539989115, 655816003,
    960914243,  1915696806, 2013025619, 1168140026, 1923497586, 167698528,  1528387973, 993794175,
    450926852,  1462772409, 1021685265, 83696007,   508154254,  1861070898, 26482542,   444956424,
    2115448041, 118254244,  471503978,  1215892992, 135346136,  1602504050, 160037322,  551454346,
    519485142,  383947510,  1968171878, 540872513,  2013025619, 475051709,  914834335,  810642687,
    1019331795, 2056065863, 1342855162, 1325809384, 1988803007, 765656702,  1368624604, 450181436,
    1927888393, 1759567256, 606425239,  19268348,   1298201670, 2041736264, 379756761,  28837162};
static const int kTaN[12] = {20, 20, 20, 50, 50, 50, 100, 100, 100, 200, 200, 500};
static const int kTaM[12] = {5, 10, 20, 5, 10, 20, 5, 10, 20, 10, 20, 20};

int or_taillard_named(const char* name, int* n, int* m, int32_t* p_out) {
  if (!name || strlen(name) != 5 || (name[0] != 't' && name[0] != 'T') || name[1] != 'a') return -1;
  int idx = atoi(name + 2);
  if (idx < 1 || idx > 120) return -1;
  int cls = (idx - 1) / 10;
  *n = kTaN[cls];
  *m = kTaM[cls];
  return or_taillard(*n, *m, kTaSeeds[idx - 1], p_out);
}

/* Eq. (1) recursion (src/instance.cpp:165-183). */
int64_t or_makespan(int n, int m, const int32_t* p, const int* perm) {
  int64_t c[64];
  int64_t* cc = m <= 64 ? c : (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  for (int k = 0; k < m; ++k) cc[k] = 0;
  for (int i = 0; i < n; ++i) {
    const int32_t* row = p + (size_t)perm[i] * m;
    cc[0] += row[0];
    for (int k = 1; k < m; ++k) cc[k] = max64(cc[k], cc[k - 1]) + row[k];
  }
  int64_t r = cc[m - 1];
  if (cc != c) free(cc);
  return r;
}

/* NEH (src/heuristic.cpp:73-103): decreasing total time (ties: lower index), each job
 * inserted at the first position of minimal partial makespan. Plain O(n^3 m). */
int64_t or_neh(int n, int m, const int32_t* p, int* perm_out) {
  int* order = (int*)malloc(sizeof(int) * (size_t)n);
  int64_t* load = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  int* cur = (int*)malloc(sizeof(int) * (size_t)n);
  int* trial = (int*)malloc(sizeof(int) * (size_t)n);
  for (int j = 0; j < n; ++j) {
    order[j] = j;
    for (int k = 0; k < m; ++k) load[j] += p[j * m + k];
  }
  for (int i = 1; i < n; ++i) { /* stable insertion sort */
    int x = order[i], t = i;
    while (t > 0 && load[order[t - 1]] < load[x]) {
      order[t] = order[t - 1];
      --t;
    }
    order[t] = x;
  }
  int len = 0;
  int64_t last = 0;
  for (int s = 0; s < n; ++s) {
    int job = order[s], best_pos = 0;
    int64_t best = INT64_MAX;
    for (int pos = 0; pos <= len; ++pos) {
      int t = 0;
      for (int i = 0; i < pos; ++i) trial[t++] = cur[i];
      trial[t++] = job;
      for (int i = pos; i < len; ++i) trial[t++] = cur[i];
      int64_t v = or_makespan(len + 1, m, p, trial);
      if (v < best) {
        best = v;
        best_pos = pos;
      }
    }
    for (int i = len; i > best_pos; --i) cur[i] = cur[i - 1];
    cur[best_pos] = job;
    ++len;
    last = best;
  }
  memcpy(perm_out, cur, sizeof(int) * (size_t)n);
  free(order);
  free(load);
  free(cur);
  free(trial);
  return last;
}

/* ---------------------------------------------------------------- bounding data */

typedef struct {
  int job;
  int key;
  int first_set;
} or_jkey;

static int or_jkey_cmp(const void* x, const void* y) {
  const or_jkey* a = (const or_jkey*)x;
  const or_jkey* b = (const or_jkey*)y;
  if (a->first_set != b->first_set) return a->first_set ? -1 : 1;
  if (a->key != b->key) {
    if (a->first_set) return a->key < b->key ? -1 : 1; /* J1 ascending a+lag */
    return a->key > b->key ? -1 : 1;                    /* J2 descending b+lag */
  }
  return a->job < b->job ? -1 : (a->job > b->job);      /* ties: ascending job */
}

int or_problem_init(or_problem* pr, int n, int m, const int32_t* p, int bound) {
  memset(pr, 0, sizeof(*pr));
  if (n < 1 || m < 1 || (bound != OR_LB1 && bound != OR_LB2)) return -1;
  pr->n = n;
  pr->m = m;
  pr->bound = bound;
  pr->p = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * (size_t)m);
  memcpy(pr->p, p, sizeof(int32_t) * (size_t)n * (size_t)m);
  if (bound == OR_LB2 && m >= 2) {
    int P = m * (m - 1) / 2;
    pr->npairs = P;
    pr->pk = (int*)malloc(sizeof(int) * (size_t)P);
    pr->pl = (int*)malloc(sizeof(int) * (size_t)P);
    pr->order = (int*)malloc(sizeof(int) * (size_t)P * (size_t)n);
    pr->lag = (int*)malloc(sizeof(int) * (size_t)P * (size_t)n);
    or_jkey* keys = (or_jkey*)malloc(sizeof(or_jkey) * (size_t)n);
    int q = 0;
    for (int k = 0; k < m; ++k) {
      for (int l = k + 1; l < m; ++l, ++q) {
        pr->pk[q] = k;
        pr->pl[q] = l;
        for (int j = 0; j < n; ++j) {
          int lag = 0;
          for (int i = k + 1; i < l; ++i) lag += p[j * m + i];
          pr->lag[q * n + j] = lag;
          int a = p[j * m + k], b = p[j * m + l];
          keys[j].job = j;
          keys[j].first_set = a < b;
          keys[j].key = (a < b ? a : b) + lag;
        }
        qsort(keys, (size_t)n, sizeof(or_jkey), or_jkey_cmp);
        for (int t = 0; t < n; ++t) pr->order[q * n + t] = keys[t].job;
      }
    }
    free(keys);
  }
  return 0;
}

void or_problem_free(or_problem* pr) {
  free(pr->p);
  free(pr->pk);
  free(pr->pl);
  free(pr->order);
  free(pr->lag);
  memset(pr, 0, sizeof(*pr));
}

/* front / tail / remain tables of a node (src/bound.cpp:20-46) */
static void or_tables(const or_problem* pr, const int* perm, int d1, int d2, int64_t* front,
                      int64_t* tail, int64_t* remain) {
  const int m = pr->m, n = pr->n;
  for (int k = 0; k < m; ++k) front[k] = tail[k] = remain[k] = 0;
  for (int i = 0; i < d1; ++i) {
    const int32_t* row = pr->p + (size_t)perm[i] * m;
    front[0] += row[0];
    for (int k = 1; k < m; ++k) front[k] = max64(front[k], front[k - 1]) + row[k];
  }
  for (int i = n - 1; i >= n - d2; --i) {
    const int32_t* row = pr->p + (size_t)perm[i] * m;
    tail[m - 1] += row[m - 1];
    for (int k = m - 2; k >= 0; --k) tail[k] = max64(tail[k], tail[k + 1]) + row[k];
  }
  for (int i = d1; i < n - d2; ++i) {
    const int32_t* row = pr->p + (size_t)perm[i] * m;
    for (int k = 0; k < m; ++k) remain[k] += row[k];
  }
}

int64_t or_lb1_node(const or_problem* pr, const int* perm, int d1, int d2) {
  int64_t f[64], t[64], r[64];
  if (pr->m > 64) return -1;
  or_tables(pr, perm, d1, d2, f, t, r);
  int64_t best = 0;
  for (int k = 0; k < pr->m; ++k) best = max64(best, f[k] + r[k] + t[k]);
  return best;
}

int or_children_bounds(const or_problem* pr, const int* perm, int d1, int d2, int64_t* lb_fwd,
                       int64_t* lb_bwd) {
  const int n = pr->n, m = pr->m;
  const int f = n - d1 - d2;
  if (f < 1 || m > 64 || n > 512) return -1;
  int64_t front[64], tail[64], remain[64];
  or_tables(pr, perm, d1, d2, front, tail, remain);
  if (pr->bound == OR_LB1 || m < 2) {
    /* children_bounds (src/bound.cpp:61-88): O(m) per child, both directions */
    for (int c = 0; c < f; ++c) {
      const int32_t* row = pr->p + (size_t)perm[d1 + c] * m;
      int64_t prev = 0, best = 0;
      for (int k = 0; k < m; ++k) {
        prev = max64(prev, front[k]) + row[k];
        best = max64(best, prev + (remain[k] - row[k]) + tail[k]);
      }
      lb_fwd[c] = best;
      prev = 0;
      best = 0;
      for (int k = m - 1; k >= 0; --k) {
        prev = max64(prev, tail[k]) + row[k];
        best = max64(best, front[k] + (remain[k] - row[k]) + prev);
      }
      lb_bwd[c] = best;
    }
    return 0;
  }
  /* LB2. Child heads/tails first (forward child sigma1.j: extended
   * head, node tail; backward child j.sigma2: node head, extended tail), then per machine
   * pair the node's free jobs in that pair's Johnson order, shared by all 2f children. */
  uint8_t is_free[512];
  memset(is_free, 0, (size_t)n);
  for (int c = 0; c < f; ++c) is_free[perm[d1 + c]] = 1;
  int64_t* head = (int64_t*)malloc(sizeof(int64_t) * (size_t)f * (size_t)m * 2);
  int64_t* tl = head + (size_t)f * m;
  int* seq = (int*)malloc(sizeof(int) * (size_t)f * 4);
  int* sa = seq + f;
  int* sb = sa + f;
  int* slag = sb + f;
  for (int c = 0; c < f; ++c) {
    const int32_t* row = pr->p + (size_t)perm[d1 + c] * m;
    int64_t prev = 0;
    for (int k = 0; k < m; ++k) {
      prev = max64(prev, front[k]) + row[k];
      head[(size_t)c * m + k] = prev;
    }
    prev = 0;
    for (int k = m - 1; k >= 0; --k) {
      prev = max64(prev, tail[k]) + row[k];
      tl[(size_t)c * m + k] = prev;
    }
    lb_fwd[c] = 0;
    lb_bwd[c] = 0;
  }
  for (int pq = 0; pq < pr->npairs; ++pq) {
    const int k = pr->pk[pq], l = pr->pl[pq];
    const int* ord = pr->order + (size_t)pq * n;
    const int* lag = pr->lag + (size_t)pq * n;
    int len = 0;
    for (int t = 0; t < n; ++t) {
      const int j = ord[t];
      if (!is_free[j]) continue;
      seq[len] = j;
      sa[len] = pr->p[j * m + k];
      sb[len] = pr->p[j * m + l];
      slag[len] = lag[j];
      ++len;
    }
    for (int c = 0; c < 2 * f; ++c) {
      const int fwd = c < f, cc = fwd ? c : c - f;
      const int skip = perm[d1 + cc];
      const int64_t* r = fwd ? head + (size_t)cc * m : front;
      const int64_t* q = fwd ? tail : tl + (size_t)cc * m;
      int64_t t0 = r[k], t1 = r[l];
      for (int i = 0; i < len; ++i) {
        if (seq[i] == skip) continue;
        t0 += sa[i];
        t1 = max64(t1, t0 + slag[i]) + sb[i];
      }
      const int64_t v = max64(t0 + q[k], t1 + q[l]);
      int64_t* dst = fwd ? &lb_fwd[cc] : &lb_bwd[cc];
      if (v > *dst) *dst = v;
    }
  }
  free(head);
  free(seq);
  return 0;
}

/* LB2 pinned to its definition instead of to the restated order: for every machine pair
 * (k, l) the value is the OPTIMUM over all orders of the child's free jobs of the two-machine
 * time-lag relaxation (Lageweg et al. 1978; Mitten/Johnson):
 *     t0 = r_k + sum a,   t1 = chain  t1 <- max(t1, t0 + lag_j) + b_j  over the order,
 *     lb_kl = max(t0 + q_k, t1 + q_l)
 * t0 does not depend on the order and every chain step is nondecreasing in its input t1, so
 * the minimal final t1 over all orders is the subset DP
 *     D[S] = min_{j in S} max(D[S - j], r_k + a(S) + lag_j) + b_j,   D[{}] = r_l
 * (principle of optimality), exact for any tie structure. No Johnson order is used: this is
 * the independent check that the restated order (row a22) attains the relaxation's optimum.
 * Cost O(2^(f-1) (f-1)) per child and pair; f <= 16. */
int or_children_bounds_lb2_exact(const or_problem* pr, const int* perm, int d1, int d2, int64_t* lb_fwd,
                                 int64_t* lb_bwd) {
  const int n = pr->n, m = pr->m;
  const int f = n - d1 - d2;
  if (f < 1 || f > 16 || m < 2 || m > 64 || n > 512) return -1;
  int64_t front[64], tail[64], remain[64];
  or_tables(pr, perm, d1, d2, front, tail, remain);
  const int fm = f - 1;  /* jobs left in a child */
  int64_t* D = (int64_t*)malloc(sizeof(int64_t) << fm);
  int64_t* SA = (int64_t*)malloc(sizeof(int64_t) << fm);
  int jobs[16];
  for (int c = 0; c < 2 * f; ++c) {
    const int fwd = c < f, cc = fwd ? c : c - f;
    const int jc = perm[d1 + cc];
    const int32_t* rowc = pr->p + (size_t)jc * m;
    int64_t r[64], q[64];
    int64_t prev = 0;
    for (int k = 0; k < m; ++k) {  /* forward child: extended head, node tail */
      if (fwd) prev = max64(prev, front[k]) + rowc[k];
      r[k] = fwd ? prev : front[k];
    }
    prev = 0;
    for (int k = m - 1; k >= 0; --k) {  /* backward child: node head, extended tail */
      if (!fwd) prev = max64(prev, tail[k]) + rowc[k];
      q[k] = fwd ? tail[k] : prev;
    }
    int t = 0;
    for (int x = 0; x < f; ++x)
      if (x != cc) jobs[t++] = perm[d1 + x];
    int64_t best = 0;
    for (int k = 0; k < m; ++k) {
      for (int l = k + 1; l < m; ++l) {
        SA[0] = 0;
        D[0] = r[l];
        for (uint32_t S = 1; S < (1u << fm); ++S) {
          const int low = __builtin_ctz(S);
          SA[S] = SA[S & (S - 1)] + pr->p[(size_t)jobs[low] * m + k];
          int64_t v = INT64_MAX;
          for (uint32_t w = S; w; w &= w - 1) {
            const int i = __builtin_ctz(w);
            const int32_t* row = pr->p + (size_t)jobs[i] * m;
            int64_t lag = 0;
            for (int z = k + 1; z < l; ++z) lag += row[z];
            const int64_t e = max64(D[S & ~(1u << i)], r[k] + SA[S] + lag) + row[l];
            if (e < v) v = e;
          }
          D[S] = v;
        }
        const uint32_t all = (1u << fm) - 1u;
        const int64_t lb = max64(r[k] + SA[all] + q[k], D[all] + q[l]);
        if (lb > best) best = lb;
      }
    }
    if (fwd) lb_fwd[cc] = best;
    else lb_bwd[cc] = best;
  }
  free(D);
  free(SA);
  return 0;
}

/* decompose (src/bound.cpp:98-139): MinMin over the union minimum, ties to the larger
 * LB sum, then Forward; pruned = child_lb >= incumbent. */
int or_decompose(const or_problem* pr, const int* perm, int d1, int d2, int64_t incumbent,
                 int64_t* child_lb, int* direction, uint8_t* pruned) {
  const int f = pr->n - d1 - d2;
  if (f < 1 || incumbent <= 0) return -1;
  int64_t* fw = (int64_t*)malloc(sizeof(int64_t) * (size_t)f * 2);
  int64_t* bw = fw + f;
  if (or_children_bounds(pr, perm, d1, d2, fw, bw) != 0) {
    free(fw);
    return -1;
  }
  int64_t lo = INT64_MAX, sf = 0, sb = 0;
  int cf = 0, cb = 0;
  for (int c = 0; c < f; ++c) {
    if (fw[c] < lo) lo = fw[c];
    if (bw[c] < lo) lo = bw[c];
  }
  for (int c = 0; c < f; ++c) {
    cf += fw[c] == lo;
    cb += bw[c] == lo;
    sf += fw[c];
    sb += bw[c];
  }
  int dir;
  if (cf != cb) dir = cf < cb ? OR_FORWARD : OR_BACKWARD;
  else if (sf != sb) dir = sf > sb ? OR_FORWARD : OR_BACKWARD;
  else dir = OR_FORWARD;
  const int64_t* ch = dir == OR_FORWARD ? fw : bw;
  for (int c = 0; c < f; ++c) {
    child_lb[c] = ch[c];
    pruned[c] = ch[c] >= incumbent;
  }
  *direction = dir;
  free(fw);
  return 0;
}

/* ---------------------------------------------------------------- factoradic */

int or_fact_compare(int n, const int* a, const int* b) {
  for (int l = 0; l < n; ++l)
    if (a[l] != b[l]) return a[l] < b[l] ? -1 : 1;
  return 0;
}

/* floor((a+b)/2) on digit vectors (src/factoradic.cpp:59-93): mixed-radix sum from the
 * least significant digit, then halving from the most significant one. */
int or_fact_midpoint(int n, const int* a, const int* b, int* out) {
  int* sum = (int*)malloc(sizeof(int) * (size_t)n);
  int carry = 0;
  if (b) {
    if (or_fact_compare(n, a, b) >= 0) {
      free(sum);
      return -1;
    }
    for (int l = n - 1; l >= 0; --l) {
      int radix = n - l, s = a[l] + b[l] + carry;
      sum[l] = s % radix;
      carry = s / radix;
    }
  } else {
    for (int l = 0; l < n; ++l) sum[l] = a[l];
    carry = 1;
  }
  int rem = carry;
  for (int l = 0; l < n; ++l) {
    int cur = rem * (n - l) + sum[l];
    out[l] = cur / 2;
    rem = cur % 2;
  }
  free(sum);
  return 0;
}

/* ---------------------------------------------------------------- IVM */

enum { IVM_EMPTY = 0, IVM_ACTIVE = 1 };

typedef struct {
  int n, level, state, has_end;
  int *V, *M, *dir, *end; /* M row-major n*n, cell = job+1, negative = pruned/consumed */
  int* perm;              /* decode scratch */
  int d1, d2;
} or_ivm;

static void ivm_alloc(or_ivm* v, int n) {
  memset(v, 0, sizeof(*v));
  v->n = n;
  v->V = (int*)calloc((size_t)n, sizeof(int));
  v->M = (int*)calloc((size_t)n * (size_t)n, sizeof(int));
  v->dir = (int*)calloc((size_t)n, sizeof(int));
  v->end = (int*)calloc((size_t)n, sizeof(int));
  v->perm = (int*)calloc((size_t)n, sizeof(int));
}

static void ivm_free(or_ivm* v) {
  free(v->V);
  free(v->M);
  free(v->dir);
  free(v->end);
  free(v->perm);
}

#define CELL(v, r, c) ((v)->M[(size_t)(r) * (v)->n + (c)])

/* decode (src/ivm.cpp:152-172) */
static void ivm_decode(or_ivm* v) {
  const int n = v->n;
  int d1 = 0, d2 = 0;
  for (int l = 0; l <= v->level; ++l) {
    int job = abs(CELL(v, l, v->V[l])) - 1;
    if (v->dir[l] == OR_FORWARD) v->perm[d1++] = job;
    else v->perm[n - 1 - d2++] = job;
  }
  int pos = d1, len = n - v->level;
  for (int c = 0; c < len; ++c) {
    if (c == v->V[v->level]) continue;
    v->perm[pos++] = abs(CELL(v, v->level, c)) - 1;
  }
  v->d1 = d1;
  v->d2 = d2;
}

/* branch (src/ivm.cpp:124-145) */
static void ivm_branch(or_ivm* v, int direction, const uint8_t* pruned) {
  const int row = v->level, len = v->n - row, sel = v->V[row];
  int out = 0;
  for (int c = 0; c < len; ++c) {
    if (c == sel) continue;
    int job = abs(CELL(v, row, c));
    CELL(v, row + 1, out) = pruned[out] ? -job : job;
    ++out;
  }
  v->dir[row + 1] = direction;
  ++v->level;
  v->V[v->level] = 0;
}

/* position_reached_end (src/ivm.cpp:90-97) */
static int ivm_reached_end(const or_ivm* v) {
  for (int l = 0; l < v->n; ++l) {
    int pv = l <= v->level ? v->V[l] : 0;
    if (pv != v->end[l]) return pv > v->end[l];
  }
  return 1;
}

/* select_next (src/ivm.cpp:99-122) */
static int ivm_select_next(or_ivm* v) {
  if (v->state != IVM_ACTIVE) return 0;
  for (;;) {
    if (v->level < 0) {
      v->state = IVM_EMPTY;
      return 0;
    }
    int len = v->n - v->level, c = v->V[v->level];
    while (c < len && CELL(v, v->level, c) < 0) ++c;
    v->V[v->level] = c;
    if (c >= len) {
      v->V[v->level] = 0;
      --v->level;
      if (v->level >= 0) ++v->V[v->level];
      continue;
    }
    if (v->has_end && ivm_reached_end(v)) {
      v->state = IVM_EMPTY;
      return 0;
    }
    return 1;
  }
}

typedef struct {
  int64_t* child_lb;
  uint8_t* pruned;
} or_scratch;

/* init_at (src/ivm.cpp:48-88) with init_root (38-46); returns replay decompositions */
static uint64_t ivm_init_at(or_ivm* v, const or_problem* pr, const int* a, const int* b,
                            int64_t incumbent, or_scratch* s, uint64_t* hist) {
  const int n = v->n;
  for (int l = 0; l < n; ++l) {
    v->V[l] = 0;
    v->dir[l] = OR_FORWARD;
  }
  for (int c = 0; c < n; ++c) CELL(v, 0, c) = c + 1;
  v->level = 0;
  v->has_end = b != NULL;
  if (b) memcpy(v->end, b, sizeof(int) * (size_t)n);
  if (b && or_fact_compare(n, a, b) >= 0) {
    v->state = IVM_EMPTY;
    return 0;
  }
  uint64_t replayed = 0;
  for (int l = 0; l <= n - 2; ++l) {
    int digit = a[l];
    v->V[l] = digit;
    v->level = l;
    for (int c = 0; c < digit; ++c)
      if (CELL(v, l, c) > 0) CELL(v, l, c) = -CELL(v, l, c);
    if (CELL(v, l, digit) < 0) break;
    if (l == n - 2) break;
    ivm_decode(v);
    int dir;
    or_decompose(pr, v->perm, v->d1, v->d2, incumbent, s->child_lb, &dir, s->pruned);
    if (hist) ++hist[n - v->d1 - v->d2];
    ivm_branch(v, dir, s->pruned);
    ++replayed;
  }
  v->state = IVM_ACTIVE;
  return replayed;
}

enum { STEP_DECOMPOSED = 0, STEP_IMPROVED = 1, STEP_EXHAUSTED = 2 };

/* explore_step (src/explorer.cpp:37-63) */
static int explore_step(or_ivm* v, const or_problem* pr, int64_t prune, int64_t improve,
                        or_scratch* s, uint64_t* decomposed, uint64_t* leaves, uint64_t* hist,
                        int64_t* leaf_mk) {
  if (!ivm_select_next(v)) return STEP_EXHAUSTED;
  if (v->n - 1 - v->level <= 1) {
    ivm_decode(v);
    int64_t mk = or_makespan(v->n, pr->m, pr->p, v->perm);
    ++*leaves;
    int* x = &CELL(v, v->level, v->V[v->level]);
    if (*x > 0) *x = -*x;
    if (mk < improve) {
      *leaf_mk = mk;
      return STEP_IMPROVED;
    }
    return STEP_DECOMPOSED;
  }
  ivm_decode(v);
  int dir;
  or_decompose(pr, v->perm, v->d1, v->d2, prune, s->child_lb, &dir, s->pruned);
  if (hist) ++hist[pr->n - v->d1 - v->d2];
  ivm_branch(v, dir, s->pruned);
  ++*decomposed;
  return STEP_DECOMPOSED;
}

/* ---------------------------------------------------------------- solve */

/* Work queue of factoradic intervals [a, b) (b_nfact = b is n!). Workers pop intervals;
 * when the queue runs dry, busy workers donate the right half [mid, end) of their own
 * remaining interval [pos, end) (steal-right-half, src/explorer.cpp:265-281). Replay
 * duplicates are discounted with unique = raw - min(L, lnz(a)). */
typedef struct {
  int* a;
  int* b;
  int b_nfact;
} or_iv;

typedef struct {
  const or_problem* pr;
  int64_t ub;
  int pinned, prune_disabled, nthreads;
  double t0, limit;
  pthread_mutex_t mu;
  or_iv* q;
  int qlen, qcap;
  int idle;          /* workers waiting for work */
  _Atomic int hungry;
  _Atomic int64_t best;
  _Atomic int stop;
  int done;
  or_stats* out;
} or_solve_ctx;

static void q_push(or_solve_ctx* cx, const int* a, const int* b) {
  const int n = cx->pr->n;
  if (cx->qlen == cx->qcap) {
    cx->qcap = cx->qcap ? 2 * cx->qcap : 1024;
    cx->q = (or_iv*)realloc(cx->q, sizeof(or_iv) * (size_t)cx->qcap);
  }
  or_iv* iv = &cx->q[cx->qlen++];
  iv->a = (int*)malloc(sizeof(int) * (size_t)n * 2);
  iv->b = iv->a + n;
  memcpy(iv->a, a, sizeof(int) * (size_t)n);
  iv->b_nfact = b == NULL;
  if (b) memcpy(iv->b, b, sizeof(int) * (size_t)n);
}

static void piece_start(int n, int depth, uint64_t id, int* a) {
  for (int l = 0; l < n; ++l) a[l] = 0;
  for (int l = depth - 1; l >= 0; --l) {
    a[l] = (int)(id % (uint64_t)(n - l));
    id /= (uint64_t)(n - l);
  }
}

static void* solve_worker(void* arg) {
  or_solve_ctx* cx = (or_solve_ctx*)arg;
  const or_problem* pr = cx->pr;
  const int n = pr->n;
  or_ivm v;
  ivm_alloc(&v, n);
  or_scratch s;
  s.child_lb = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  s.pruned = (uint8_t*)malloc((size_t)n);
  int* a = (int*)malloc(sizeof(int) * (size_t)n * 3);
  int* b = a + n;
  int* mid = b + n;
  uint64_t* hist = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t raw = 0, dups = 0, leaves = 0, improvements = 0;
  int32_t best_perm[512];
  int has_perm = 0;
  int64_t my_best = INT64_MAX;
  for (;;) {
    /* take an interval, or wait for a donation */
    int have_b = 0;
    pthread_mutex_lock(&cx->mu);
    for (;;) {
      if (cx->done || atomic_load(&cx->stop)) break;
      if (cx->qlen > 0) {
        or_iv iv = cx->q[--cx->qlen];
        memcpy(a, iv.a, sizeof(int) * (size_t)n);
        have_b = !iv.b_nfact;
        if (have_b) memcpy(b, iv.b, sizeof(int) * (size_t)n);
        free(iv.a);
        break;
      }
      ++cx->idle;
      if (cx->idle == cx->nthreads) {
        cx->done = 1;
        break;
      }
      atomic_fetch_add(&cx->hungry, 1);
      pthread_mutex_unlock(&cx->mu);
      struct timespec ts = {0, 200000};
      nanosleep(&ts, NULL);
      pthread_mutex_lock(&cx->mu);
      --cx->idle;
      if (atomic_load(&cx->hungry) > 0) atomic_fetch_sub(&cx->hungry, 1);
    }
    const int finished = cx->done || atomic_load(&cx->stop);
    pthread_mutex_unlock(&cx->mu);
    if (finished) break;

    int64_t inc = cx->prune_disabled ? OR_NO_INCUMBENT : atomic_load(&cx->best);
    uint64_t L = ivm_init_at(&v, pr, a, have_b ? b : NULL, inc, &s, hist);
    int lnz = 0;
    for (int l = 0; l < n; ++l)
      if (a[l]) lnz = l;
    raw += L;
    const uint64_t dup = L < (uint64_t)lnz ? L : (uint64_t)lnz;
    dups += dup;
    for (uint64_t l = 0; l < dup; ++l) --hist[n - 1 - (int)l]; /* unique histogram */
    for (uint64_t it = 1;; ++it) {
      if ((it & 255) == 0) {
        if (cx->limit > 0 && or_now() - cx->t0 >= cx->limit) {
          atomic_store(&cx->stop, 1);
          break;
        }
        if (atomic_load_explicit(&cx->hungry, memory_order_relaxed) > 0 && v.state == IVM_ACTIVE &&
            v.level >= 0) {
          /* donate [mid, end) of the remaining [pos, end) */
          int* pos = a; /* reuse: a is no longer needed */
          for (int l = 0; l < n; ++l) pos[l] = l <= v.level ? v.V[l] : 0;
          if (or_fact_midpoint(n, pos, v.has_end ? v.end : NULL, mid) == 0 &&
              or_fact_compare(n, mid, pos) > 0) {
            pthread_mutex_lock(&cx->mu);
            if (atomic_load(&cx->hungry) > 0) {
              atomic_fetch_sub(&cx->hungry, 1);
              q_push(cx, mid, v.has_end ? v.end : NULL);
              memcpy(v.end, mid, sizeof(int) * (size_t)n);
              v.has_end = 1;
            }
            pthread_mutex_unlock(&cx->mu);
          }
        }
      }
      int64_t cur = atomic_load_explicit(&cx->best, memory_order_relaxed);
      int64_t prune = cx->prune_disabled ? OR_NO_INCUMBENT : (cx->pinned ? cx->ub : cur);
      int64_t improve = cx->pinned ? 0 : cur;
      int64_t mk = 0;
      int o = explore_step(&v, pr, prune, improve, &s, &raw, &leaves, hist, &mk);
      if (o == STEP_EXHAUSTED) break;
      if (o == STEP_IMPROVED) {
        pthread_mutex_lock(&cx->mu);
        if (mk < atomic_load(&cx->best)) {
          atomic_store(&cx->best, mk);
          ++improvements;
        }
        pthread_mutex_unlock(&cx->mu);
        if (mk < my_best) {
          my_best = mk;
          for (int i = 0; i < n; ++i) best_perm[i] = v.perm[i];
          has_perm = 1;
        }
      }
    }
  }
  pthread_mutex_lock(&cx->mu);
  or_stats* o = cx->out;
  o->decomposed += raw;
  o->unique += raw - dups;
  o->leaves += leaves;
  o->improvements += improvements;
  for (int f = 0; f <= n; ++f) o->hist[f] += hist[f];
  if (has_perm && (!o->has_perm || my_best < o->best)) {
    o->has_perm = 1;
    o->best = my_best;
    for (int i = 0; i < n; ++i) o->best_perm[i] = best_perm[i];
  }
  pthread_mutex_unlock(&cx->mu);
  ivm_free(&v);
  free(s.child_lb);
  free(s.pruned);
  free(a);
  free(hist);
  return NULL;
}

int or_solve(const or_problem* pr, int64_t ub, int nthreads, int prefix_depth, int pinned,
             int prune_disabled, double time_limit_s, or_stats* out) {
  const int n = pr->n;
  if (n > 512 || prefix_depth < 0 || prefix_depth > n || nthreads < 1) return -1;
  memset(out, 0, sizeof(*out));
  or_solve_ctx cx;
  memset(&cx, 0, sizeof(cx));
  cx.pr = pr;
  cx.ub = ub;
  cx.pinned = pinned;
  cx.prune_disabled = prune_disabled;
  cx.nthreads = nthreads;
  cx.limit = time_limit_s;
  uint64_t pieces = 1;
  for (int l = 0; l < prefix_depth; ++l) pieces *= (uint64_t)(n - l);
  int* a = (int*)malloc(sizeof(int) * (size_t)n * 2);
  int* b = a + n;
  /* pushed in reverse so that workers pop them in increasing order */
  for (uint64_t id = pieces; id-- > 0;) {
    piece_start(n, prefix_depth, id, a);
    if (id + 1 < pieces) piece_start(n, prefix_depth, id + 1, b);
    q_push(&cx, a, id + 1 < pieces ? b : NULL);
  }
  free(a);
  atomic_store(&cx.best, ub);
  atomic_store(&cx.stop, 0);
  atomic_store(&cx.hungry, 0);
  pthread_mutex_init(&cx.mu, NULL);
  cx.out = out;
  out->best = INT64_MAX;
  cx.t0 = or_now();
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, solve_worker, &cx);
  solve_worker(&cx);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  out->wall_s = or_now() - cx.t0;
  out->completed = !atomic_load(&cx.stop);
  int64_t bst = atomic_load(&cx.best);
  if (!out->has_perm || bst < out->best) out->best = bst;
  if (out->best > ub) out->best = ub;
  for (int i = 0; i < cx.qlen; ++i) free(cx.q[i].a);
  free(cx.q);
  pthread_mutex_destroy(&cx.mu);
  return 0;
}
