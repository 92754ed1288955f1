// Host driver of the B200 explorer pool + C-ABI (include/pbbgpu.h).
//
// Round structure (replaces ExplorerPool::run_round, src/explorer.cpp:224-257):
//   explore_kernel  persistent, all explorers resident, `steps` select/bound/branch cycles
//   steal_kernel    one CTA: activity count, steal-right-half pairing of idle explorers with
//                   the longest remaining intervals, factoradic midpoints, thief re-seating
//                   (src/explorer.cpp:265-340); thieves replay init_at inside the next
//                   explore launch
//   8-byte counter readback (the only per-round host<->device traffic)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pbbgpu.h"
#include "bound_big.cuh"
#include "explore.cuh"

using namespace pbbgpu;

namespace {

thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::logic_error {
  using std::logic_error::logic_error;
};
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ instance (host)

// Minimal-standard LCG (16807, 2^31-1) via Schrage, machine-major fill: reproduces the
// published Taillard matrices (generate_taillard, src/instance.cpp:80-114).
void taillard(int n, int m, int32_t seed, int32_t* p) {
  if (n < 1 || m < 1) throw std::invalid_argument("generate_taillard needs n >= 1 and m >= 1");
  if (seed < 1 || seed > 2147483645) throw std::invalid_argument("generator seed must be in [1, 2^31-3]");
  int64_t s = seed;
  for (int k = 0; k < m; ++k) {
    for (int j = 0; j < n; ++j) {
      const int64_t q = s / 127773, r = s % 127773;
      s = 16807 * r - 2836 * q;
      if (s < 0) s += 2147483647;
      p[static_cast<size_t>(j) * m + k] = static_cast<int32_t>(1 + s * 99 / 2147483647);
    }
  }
}

struct TaClass {
  int n, m;
  int32_t seeds[10];
};
// Taillard (1993) time seeds, classes ta001-010 ... ta111-120 (src/instance.cpp:125-138).
const TaClass kTa[12] = {
    {20, 5, {873654221, 379008056, 1866992158, 216771124, 495070989, 402959317, 1369363414, 2021925980, 573109518, 88325120}},
    {20, 10, {587595453, 1401007982, 873136276, 268827376, 1634173168, 691823909, 73807235, 1273398721, 2065119309, 1672900551}},
    {20, 20, {479340445, 268827376, 1958948863, 918272953, 555010963, 2010851491, 1519833303, 1748670931, 1923497586, 1829909967}},
    {50, 5, {1328042058, 200382020, 496319842, 1203030903, 1730708564, 450926852, 1303135678, 1273398721, 587288402, 248421594}},
    {50, 10, {1958948863, 575633267, 655816003, 1977864101, 93805469, 1803345551, 49612559, 1899802599, 2013025619, 578962478}},
    {50, 20, {1539989115, 691823909, 655816003, 1315102446, 1949668355, 1923497586, 1805594913, 1861070898, 715643788, 464843328}},
    {100, 5, {896678084, 1179439976, 1122278347, 416756875, 267829958, 1835213917, 1328833962, 1418570761, 161033112, 304212574}},
    {100, 10, {1539989115, 655816003, 960914243, 1915696806, 2013025619, 1168140026, 1923497586, 167698528, 1528387973, 993794175}},
    {100, 20, {450926852, 1462772409, 1021685265, 83696007, 508154254, 1861070898, 26482542, 444956424, 2115448041, 118254244}},
    {200, 10, {471503978, 1215892992, 135346136, 1602504050, 160037322, 551454346, 519485142, 383947510, 1968171878, 540872513}},
    {200, 20, {2013025619, 475051709, 914834335, 810642687, 1019331795, 2056065863, 1342855162, 1325809384, 1988803007, 765656702}},
    {500, 20, {1368624604, 450181436, 1927888393, 1759567256, 606425239, 19268348, 1298201670, 2041736264, 379756761, 28837162}},
};

int64_t makespan_host(int n, int m, const int32_t* p, const int32_t* perm) {
  std::vector<int64_t> c(static_cast<size_t>(m), 0);
  std::vector<char> seen(static_cast<size_t>(n), 0);
  for (int i = 0; i < n; ++i) {
    const int j = perm[i];
    if (j < 0 || j >= n || seen[static_cast<size_t>(j)]) throw std::invalid_argument("schedule is not a permutation of 0..n-1");
    seen[static_cast<size_t>(j)] = 1;
    const int32_t* row = p + static_cast<size_t>(j) * m;
    c[0] += row[0];
    for (int k = 1; k < m; ++k) c[k] = std::max(c[k], c[k - 1]) + row[k];
  }
  return c[static_cast<size_t>(m) - 1];
}

// NEH (src/heuristic.cpp:73-103) with Taillard's O(nm) insertion scan: e = prefix heads,
// q = suffix tails, best position = first minimum.
int64_t neh_host(int n, int m, const int32_t* p, int32_t* out) {
  std::vector<int> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::vector<int64_t> load(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < m; ++k) load[static_cast<size_t>(j)] += p[static_cast<size_t>(j) * m + k];
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return load[static_cast<size_t>(a)] > load[static_cast<size_t>(b)]; });
  std::vector<int> seq;
  std::vector<int64_t> e, q, f(static_cast<size_t>(m));
  int64_t last = 0;
  for (int s = 0; s < n; ++s) {
    const int job = order[static_cast<size_t>(s)];
    const int len = static_cast<int>(seq.size());
    e.assign(static_cast<size_t>(len + 1) * m, 0);
    q.assign(static_cast<size_t>(len + 2) * m, 0);
    for (int i = 1; i <= len; ++i) {
      const int32_t* row = p + static_cast<size_t>(seq[static_cast<size_t>(i - 1)]) * m;
      for (int k = 0; k < m; ++k) {
        const int64_t up = k ? e[static_cast<size_t>(i) * m + k - 1] : 0;
        e[static_cast<size_t>(i) * m + k] = std::max(up, e[static_cast<size_t>(i - 1) * m + k]) + row[k];
      }
    }
    for (int i = len; i >= 1; --i) {
      const int32_t* row = p + static_cast<size_t>(seq[static_cast<size_t>(i - 1)]) * m;
      for (int k = m - 1; k >= 0; --k) {
        const int64_t dn = k < m - 1 ? q[static_cast<size_t>(i) * m + k + 1] : 0;
        q[static_cast<size_t>(i) * m + k] = std::max(dn, q[static_cast<size_t>(i + 1) * m + k]) + row[k];
      }
    }
    const int32_t* jr = p + static_cast<size_t>(job) * m;
    int bp = 0;
    int64_t bv = INT64_MAX;
    for (int pos = 0; pos <= len; ++pos) {
      int64_t v = 0;
      for (int k = 0; k < m; ++k) {
        f[static_cast<size_t>(k)] = std::max(k ? f[static_cast<size_t>(k - 1)] : 0, e[static_cast<size_t>(pos) * m + k]) + jr[k];
        v = std::max(v, f[static_cast<size_t>(k)] + q[static_cast<size_t>(pos + 1) * m + k]);
      }
      if (v < bv) {
        bv = v;
        bp = pos;
      }
    }
    seq.insert(seq.begin() + bp, job);
    last = bv;
  }
  for (int i = 0; i < n; ++i) out[i] = seq[static_cast<size_t>(i)];
  return last;
}

// Makespans of inserting `job` at every position 0..len of `seq` in O(len*m) total
// (prefix heads e, suffix tails q; the scan of src/heuristic.cpp:24-69). Returns the values.
void insertion_scan(int m, const int32_t* p, const std::vector<int>& seq, int job, std::vector<int64_t>& vals,
                    std::vector<int64_t>& e, std::vector<int64_t>& q) {
  const int len = static_cast<int>(seq.size());
  e.assign(static_cast<size_t>(len + 1) * m, 0);
  q.assign(static_cast<size_t>(len + 2) * m, 0);
  for (int i = 1; i <= len; ++i) {
    const int32_t* row = p + static_cast<size_t>(seq[static_cast<size_t>(i - 1)]) * m;
    for (int k = 0; k < m; ++k) {
      const int64_t up = k ? e[static_cast<size_t>(i) * m + k - 1] : 0;
      e[static_cast<size_t>(i) * m + k] = std::max(up, e[static_cast<size_t>(i - 1) * m + k]) + row[k];
    }
  }
  for (int i = len; i >= 1; --i) {
    const int32_t* row = p + static_cast<size_t>(seq[static_cast<size_t>(i - 1)]) * m;
    for (int k = m - 1; k >= 0; --k) {
      const int64_t dn = k < m - 1 ? q[static_cast<size_t>(i) * m + k + 1] : 0;
      q[static_cast<size_t>(i) * m + k] = std::max(dn, q[static_cast<size_t>(i + 1) * m + k]) + row[k];
    }
  }
  const int32_t* jr = p + static_cast<size_t>(job) * m;
  vals.assign(static_cast<size_t>(len + 1), 0);
  std::vector<int64_t> f(static_cast<size_t>(m));
  for (int pos = 0; pos <= len; ++pos) {
    int64_t v = 0;
    for (int k = 0; k < m; ++k) {
      f[static_cast<size_t>(k)] = std::max(k ? f[static_cast<size_t>(k - 1)] : 0, e[static_cast<size_t>(pos) * m + k]) + jr[k];
      v = std::max(v, f[static_cast<size_t>(k)] + q[static_cast<size_t>(pos + 1) * m + k]);
    }
    vals[static_cast<size_t>(pos)] = v;
  }
}

// First-improvement remove-and-reinsert descent with seeded tie-breaking among equally good
// positions (insertion_local_search, src/heuristic.cpp:105-155): positions scanned left to
// right, until a local optimum or the budget (iterations / seconds) runs out.
int64_t insertion_ls_host(int n, int m, const int32_t* p, const int32_t* seed, uint64_t max_iter, double max_s,
                          uint64_t rng_seed, int32_t* out) {
  if (max_iter == 0 && max_s <= 0) throw std::invalid_argument("search budget needs an iteration or time bound");
  std::vector<int> cur(seed, seed + n);
  int64_t cmax = makespan_host(n, m, p, seed);
  std::mt19937_64 rng(rng_seed);
  std::vector<int64_t> vals, e, q;
  std::vector<int> reduced, ties;
  const auto t0 = std::chrono::steady_clock::now();
  uint64_t it = 0;
  auto spent = [&] {
    if (max_iter > 0 && it >= max_iter) return true;
    if (max_s > 0) {
      const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
      if (el.count() >= max_s) return true;
    }
    return false;
  };
  bool improved = true;
  while (improved && !spent()) {
    improved = false;
    for (int pos = 0; pos < n && !spent(); ++pos) {
      const int job = cur[static_cast<size_t>(pos)];
      reduced.assign(cur.begin(), cur.end());
      reduced.erase(reduced.begin() + pos);
      ++it;
      insertion_scan(m, p, reduced, job, vals, e, q);
      int64_t best = INT64_MAX;
      for (int64_t v : vals) best = std::min(best, v);
      if (best >= cmax) continue;
      ties.clear();
      for (int i = 0; i < n; ++i)
        if (vals[static_cast<size_t>(i)] == best) ties.push_back(i);
      const int choice = ties[std::uniform_int_distribution<std::size_t>(0, ties.size() - 1)(rng)];
      reduced.insert(reduced.begin() + choice, job);
      cur = reduced;
      cmax = best;
      improved = true;
    }
  }
  for (int i = 0; i < n; ++i) out[i] = cur[static_cast<size_t>(i)];
  return cmax;
}

// Johnson/Mitten order per machine pair for LB2: pairs (k<l)
// lexicographic; lag_j = sum_{k<i<l} p[j][i]; J1 = {a<b} ascending a+lag, then J2
// descending b+lag, ties by ascending job.
void lb2_tables(int n, int m, const int32_t* p, std::vector<uint8_t>& pk, std::vector<uint8_t>& pl,
                std::vector<uint8_t>& ord, std::vector<uint16_t>& lag, std::vector<uint32_t>& packed,
                bool& packable, std::vector<uint16_t>& ord16) {
  const int P = m * (m - 1) / 2;
  pk.resize(static_cast<size_t>(P));
  pl.resize(static_cast<size_t>(P));
  ord.resize(static_cast<size_t>(P) * n);
  ord16.resize(static_cast<size_t>(P) * n);
  lag.resize(static_cast<size_t>(P) * n);
  int q = 0;
  std::vector<int> idx(static_cast<size_t>(n));
  std::vector<int> key(static_cast<size_t>(n));
  std::vector<char> first(static_cast<size_t>(n));
  for (int k = 0; k < m; ++k) {
    for (int l = k + 1; l < m; ++l, ++q) {
      pk[static_cast<size_t>(q)] = static_cast<uint8_t>(k);
      pl[static_cast<size_t>(q)] = static_cast<uint8_t>(l);
      for (int j = 0; j < n; ++j) {
        int lg = 0;
        for (int i = k + 1; i < l; ++i) lg += p[static_cast<size_t>(j) * m + i];
        if (lg > 65535) throw std::invalid_argument("LB2 lag exceeds 16 bits");
        lag[static_cast<size_t>(q) * n + j] = static_cast<uint16_t>(lg);
        const int a = p[static_cast<size_t>(j) * m + k], b = p[static_cast<size_t>(j) * m + l];
        first[static_cast<size_t>(j)] = a < b;
        key[static_cast<size_t>(j)] = (a < b ? a : b) + lg;
        idx[static_cast<size_t>(j)] = j;
      }
      std::sort(idx.begin(), idx.end(), [&](int x, int y) {
        if (first[static_cast<size_t>(x)] != first[static_cast<size_t>(y)]) return first[static_cast<size_t>(x)] > first[static_cast<size_t>(y)];
        const int kx = key[static_cast<size_t>(x)], ky = key[static_cast<size_t>(y)];
        if (kx != ky) return first[static_cast<size_t>(x)] ? kx < ky : kx > ky;
        return x < y;
      });
      for (int t = 0; t < n; ++t) {
        ord[static_cast<size_t>(q) * n + t] = static_cast<uint8_t>(idx[static_cast<size_t>(t)]);  // n <= 64 kernels
        ord16[static_cast<size_t>(q) * n + t] = static_cast<uint16_t>(idx[static_cast<size_t>(t)]);
      }
    }
  }
  // transposed packed form [t][q] = job << 7 | u << 13 | v << 24 with u = a + lag (11 bits) and
  // v = a - b (8 bits, signed) for children_lb2_w: the job field is pre-shifted to the byte
  // offset of its row in the per-lane [job][32] int32 table
  const int PS = round_up(P, 32);  // row stride padded to 32 pairs (bank-conflict-free passes)
  packed.assign(static_cast<size_t>(PS) * n, 0);
  packable = n <= 64;
  for (int qq = 0; qq < P; ++qq) {
    for (int t = 0; t < n; ++t) {
      const int j = ord16[static_cast<size_t>(qq) * n + t];
      const int a = p[static_cast<size_t>(j) * m + pk[static_cast<size_t>(qq)]];
      const int b = p[static_cast<size_t>(j) * m + pl[static_cast<size_t>(qq)]];
      const int lg = lag[static_cast<size_t>(qq) * n + j];
      const int u = a + lg, v = a - b;
      if (u > 2047 || v < -128 || v > 127) packable = false;
      packed[static_cast<size_t>(t) * PS + qq] = static_cast<uint32_t>(j) << 7 | static_cast<uint32_t>(u & 0x7ff) << 13 |
                                                 static_cast<uint32_t>(v & 0xff) << 24;
    }
  }
}

// ------------------------------------------------------------------ small device kernels

__device__ void seat_explorer(unsigned char* blk, const IvmLayout& L, const int* ptot,
                              const int* a, const int* b, bool has_end) {
  const int n = L.n, m = L.m;
  IvmHdr* h = reinterpret_cast<IvmHdr*>(blk);
  int8_t* cells = reinterpret_cast<int8_t*>(blk + L.o_cells);
  int8_t* V = reinterpret_cast<int8_t*>(blk + L.o_v);
  uint8_t* dir = blk + L.o_dir;
  int8_t* endd = reinterpret_cast<int8_t*>(blk + L.o_end);
  int8_t* tgt = reinterpret_cast<int8_t*>(blk + L.o_tgt);
  uint16_t* ft = reinterpret_cast<uint16_t*>(blk + L.o_ft);
  uint16_t* R = reinterpret_cast<uint16_t*>(blk + L.o_r);
  uint32_t* ftw = reinterpret_cast<uint32_t*>(ft);
  uint32_t* Rw = reinterpret_cast<uint32_t*>(R);
  bool empty = false;
  if (has_end) {  // to_decimal(a) >= b -> Empty (src/ivm.cpp:61-64)
    int cmp = 0;
    for (int l = 0; l < n && !cmp; ++l) cmp = a[l] < b[l] ? -1 : (a[l] > b[l] ? 1 : 0);
    empty = cmp >= 0;
  }
  for (int c = 0; c < n; ++c) cells[c] = static_cast<int8_t>(c + 1);  // init_root (ivm.cpp:38-46)
  for (int l = 0; l < n; ++l) {
    V[l] = 0;
    dir[l] = kFwd;
    tgt[l] = static_cast<int8_t>(a[l]);
    endd[l] = static_cast<int8_t>(has_end ? b[l] : 0);
  }
  for (int k = 0; k < m; ++k) {
    if (L.ftb == 4) {
      ftw[k] = 0;
      ftw[n * m + k] = 0;
      Rw[k] = static_cast<uint32_t>(ptot[k]);
    } else {
      ft[k] = 0;                 // FS[0]
      ft[n * m + k] = 0;         // TS[0]
      R[k] = static_cast<uint16_t>(ptot[k]);
    }
  }
  h->level = 0;
  h->state = empty ? kEmpty : kInit;
  h->has_end = has_end ? 1 : 0;
  h->d1 = 1;
  h->d2 = 0;
  h->rlev = 0;
  h->nrep = 0;
}

__global__ void init_kernel(IvmLayout L, unsigned char* state, const int* ptot, const int* a,
                            const int* b, const uint8_t* b_nfact, const int* slots, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned char* blk = state + static_cast<size_t>(slots[i]) * L.gstride;
  seat_explorer(blk, L, ptot, a + static_cast<size_t>(i) * L.n, b + static_cast<size_t>(i) * L.n, !b_nfact[i]);
}

__global__ void clear_kernel(IvmLayout L, unsigned char* state, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  IvmHdr* h = reinterpret_cast<IvmHdr*>(state + static_cast<size_t>(i) * L.gstride);
  h->state = kEmpty;
  h->level = -1;
}

struct StealParams {
  IvmLayout L;
  unsigned char* state;
  int K;
  const int* ptot;
  DevCounters* ctr;
  int* thief;   // [K]
  int* victim;  // [K]
  float min_log2;
  const float* lgfact;  // [n+1] log2(k!)
  float trigger;        // steal when active < trigger * K (reference: 0.8, explorer.cpp:251)
  const float* lens;    // [K] per-explorer log2 remaining (written by explore_kernel)
  int max_split;        // thieves per victim in one steal phase (multi-way split), 1..63
  int* plan;            // [2] victims paired this phase, thieves per victim (split kernels)
  int split_mode;       // 0 live siblings, 1 factoradic midpoint
};

constexpr int kStealThreads = 1024;
constexpr int kBins = 2048;

// ---- live-sibling splitting (split_mode 0)
// An explorer's untouched work is the unexplored, unpruned cells right of its path: at level
// l, cells c > V[l] of row l with a positive entry (negative = pruned by bound or consumed),
// restricted to [pos, end): no level before the first digit where pos and end differ, and
// only cells below end[d] at that level d. The shallowest level l* holding any dominates (a
// cell there roots (n-1-l*)! leaves). Returns their count and positions (ascending).
__device__ int live_siblings(const unsigned char* vb, const IvmLayout& L, int& lstar, int* cells) {
  const int n = L.n;
  const IvmHdr* h = reinterpret_cast<const IvmHdr*>(vb);
  if (h->state != kActive) return 0;
  const int8_t* V = reinterpret_cast<const int8_t*>(vb + L.o_v);
  const int8_t* E = reinterpret_cast<const int8_t*>(vb + L.o_end);
  const int8_t* C = reinterpret_cast<const int8_t*>(vb + L.o_cells);
  const bool he = h->has_end != 0;
  const int level = h->level;
  int l = 0;
  if (he) {
    while (l <= level && V[l] == E[l]) ++l;
    if (l <= level && V[l] > E[l]) return 0;
  }
  const int d = he ? l : -1;
  for (; l <= level; ++l) {
    const int8_t* row = C + tri_off(l, n);
    const int lim = l == d ? E[l] : n - l;
    int cnt = 0;
    for (int c = V[l] + 1; c < lim; ++c)
      if (row[c] > 0) cells[cnt++] = c;
    if (cnt) {
      lstar = l;
      return cnt;
    }
  }
  return 0;
}

// Items of a live split: item 0 is the explorer's own path (the current cell at l* with
// everything below it), items 1..cnt the live siblings. g thieves cut the cnt + 1 items into
// g + 1 contiguous groups; the victim keeps group 0. Start cell of group i (1..g):
__device__ __forceinline__ int live_group_start(const int* cells, int cnt, int g, int i) {
  return cells[i * (cnt + 1) / (g + 1) - 1];
}

// digits of (prefix V[0..l*-1], cell at l*, zeros)
__device__ __forceinline__ void live_point(const int8_t* V, int lstar, int cell, int n, int* out) {
  for (int l = 0; l < n; ++l) out[l] = l < lstar ? V[l] : (l == lstar ? cell : 0);
}

// Remaining work of every explorer after a round (grid-wide, one thread per explorer), as
// log2 of leaves; -2 busy / unsplittable, -3 idle. mode 0: the live siblings of the
// shallowest level holding any, (cnt + 1) (n-1-l*)!; mode 1: the exact factoradic length of
// [effective position, end).
// One warp per explorer: the block is staged in shared memory with coalesced 16-byte loads, so
// the digit / row walks of explorer_lens run on shared memory instead of serialized global loads.
// (Evaluated inside the explore kernel's write-back instead, the code costs the explorer loop
// registers in every variant: 2-3 % on the ta021 / ta056 proofs.)
constexpr int kLensWarps = 8;
__global__ void __launch_bounds__(kLensWarps * 32) lens_kernel(IvmLayout L, const unsigned char* state, int K,
                                                               const float* lgfact, float* lens, int mode) {
  extern __shared__ __align__(16) unsigned char lbuf[];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  unsigned char* vb = lbuf + static_cast<size_t>(wi) * L.gstride;
  for (int i = blockIdx.x * kLensWarps + wi; i < K; i += gridDim.x * kLensWarps) {
    const uint4* src = reinterpret_cast<const uint4*>(state + static_cast<size_t>(i) * L.gstride);
    for (int w = lane; w < L.gstride / 16; w += 32) reinterpret_cast<uint4*>(vb)[w] = src[w];
    __syncwarp();
    if (lane == 0) lens[i] = explorer_lens(vb, L, lgfact, mode);
    __syncwarp();
  }
}

// ---- multi-way interval splitting (exact mixed-radix arithmetic, no big integers)
// D = end - pos as digits plus a top unit of weight n! (end = n! when !has_end).
template <typename T>
__device__ bool diff_digits(const int* pos, const T* E, bool has_end, int n, int* D, int& top) {
  top = 0;
  if (has_end) {
    int borrow = 0;
    for (int l = n - 1; l >= 0; --l) {
      int d = E[l] - pos[l] - borrow;
      borrow = d < 0;
      if (borrow) d += n - l;
      D[l] = d;
    }
    return !borrow;
  }
  int carry = 1;  // n! - pos = ((n! - 1) - pos) + 1
  for (int l = n - 1; l >= 0; --l) {
    int d = n - 1 - l - pos[l] + carry;
    carry = d > n - 1 - l;
    if (carry) d = 0;
    D[l] = d;
  }
  top = carry;
  return true;
}

// b = pos + floor(i * D / parts): long division from the most significant digit (the
// remainder converts into units of the next, smaller weight), quotient digits normalized
// from the least significant one, then a mixed-radix add.
__device__ void split_point(const int* pos, const int* D, int top, int i, int parts, int n, int* b) {
  int rem = i * top;
  for (int l = 0; l < n; ++l) {
    const int cur = rem * (n - l) + i * D[l];
    b[l] = cur / parts;
    rem = cur % parts;
  }
  for (int l = n - 1; l > 0; --l) {
    if (b[l] > n - 1 - l) {
      b[l - 1] += b[l] / (n - l);
      b[l] %= n - l;
    }
  }
  int carry = 0;
  for (int l = n - 1; l >= 0; --l) {
    const int s = pos[l] + b[l] + carry, radix = n - l;
    b[l] = s % radix;
    carry = s / radix;
  }
}

// Setup of an r-way split of a victim (shared by the grid-wide split kernels below, which
// re-derive it independently per thread from the unchanged victim state): the effective
// position, D = end - pos, and r shrunk so every part holds at least 2 leaves. 0 = no split.
__device__ int split_setup(const unsigned char* vb, const IvmLayout& L, int r, int* pos, int* D, int& top) {
  const int n = L.n;
  const IvmHdr* vh = reinterpret_cast<const IvmHdr*>(vb);
  if (vh->state != kActive) return 0;
  const int8_t* E = reinterpret_cast<const int8_t*>(vb + L.o_end);
  if (!effective_pos(reinterpret_cast<const int8_t*>(vb + L.o_v), vh->level,
                     reinterpret_cast<const int8_t*>(vb + L.o_cells), n, pos))
    return 0;
  if (!diff_digits(pos, E, vh->has_end != 0, n, D, top)) return 0;
  if (!top) {
    long long small = 0;
    bool big = false;
    for (int l = 0; l < n && !big; ++l) {
      small = small * (n - l) + D[l];
      if (small > (1ll << 40)) big = true;
    }
    if (!big) {
      if (small < 2) return 0;
      r = static_cast<int>(min(static_cast<long long>(r), max(small / 2 - 1, 1ll)));
    }
  }
  return r;
}

// Splits of a steal phase, one warp per victim: the victim's block is staged in shared memory
// with one coalesced read (the digit walks below then run on shared memory instead of
// serialized global loads); lane i in 1..r seats thief i - 1 with part i of the victim's work
// [pos, end) cut into r + 1 parts, and lane 0 cuts the victim's own end to the start of part 1
// (the thieves read the old end from the staged copy).
constexpr int kSplitWarps = 4;
__global__ void __launch_bounds__(kSplitWarps * 32) split_kernel(IvmLayout L, unsigned char* state, const int* ptot,
                                                                 const int* thief, const int* victim, const int* plan,
                                                                 DevCounters* ctr, int mode) {
  extern __shared__ __align__(16) unsigned char sbuf[];
  const int nv = plan[0], rs = plan[1];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int n = L.n;
  unsigned char* vb = sbuf + static_cast<size_t>(wi) * L.gstride;
  unsigned seated = 0;
  for (int v = blockIdx.x * kSplitWarps + wi; v < nv; v += gridDim.x * kSplitWarps) {
    unsigned char* gv = state + static_cast<size_t>(victim[v]) * L.gstride;
    for (int i = lane; i < L.gstride / 16; i += 32) reinterpret_cast<uint4*>(vb)[i] = reinterpret_cast<const uint4*>(gv)[i];
    __syncwarp();
    const IvmHdr* vh = reinterpret_cast<const IvmHdr*>(vb);
    const int8_t* V = reinterpret_cast<const int8_t*>(vb + L.o_v);
    const int8_t* E = reinterpret_cast<const int8_t*>(vb + L.o_end);
    int ok = 0;
    if (lane <= rs) {
      int b0[kMaxN], b1[kMaxN];
      int cells[kMaxN];
      int lstar = 0;
      int parts = 0;  // thieves this victim feeds
      const int cnt = mode == 1 ? 0 : live_siblings(vb, L, lstar, cells);
      const bool live = cnt > 0 || mode == 2;
      int pos[kMaxN], D[kMaxN];
      int top = 0;
      if (live) parts = min(rs, cnt);
      else parts = split_setup(vb, L, rs, pos, D, top);
      if (parts >= 1 && lane <= parts) {
        const int i = lane;
        if (live) live_point(V, lstar, live_group_start(cells, cnt, parts, max(i, 1)), n, b0);
        else split_point(pos, D, top, max(i, 1), parts + 1, n, b0);
        if (i == 0) {  // the victim keeps part 0: end <- start of part 1
          int8_t* gE = reinterpret_cast<int8_t*>(gv + L.o_end);
          for (int l = 0; l < n; ++l) gE[l] = static_cast<int8_t>(b0[l]);
          reinterpret_cast<IvmHdr*>(gv)->has_end = 1;
        } else {
          const bool last = i == parts;
          if (last) {
            for (int l = 0; l < n; ++l) b1[l] = E[l];
          } else if (live) {
            live_point(V, lstar, live_group_start(cells, cnt, parts, i + 1), n, b1);
          } else {
            split_point(pos, D, top, i + 1, parts + 1, n, b1);
          }
          seat_explorer(state + static_cast<size_t>(thief[v * rs + i - 1]) * L.gstride, L, ptot, b0, b1,
                        last ? vh->has_end != 0 : true);
          ok = 1;
        }
      }
    }
    seated += __popc(__ballot_sync(0xffffffffu, ok));
    __syncwarp();
  }
  if (lane == 0 && seated) {
    atomicAdd(&ctr->active, static_cast<int>(seated));
    atomicAdd(&ctr->steals, static_cast<unsigned long long>(seated));
    atomicAdd(&ctr->inits, static_cast<unsigned long long>(seated));
  }
}

#include "steal_ref.cuh"
#include "explore_big.cuh"

// Steal phase (src/explorer.cpp:283-340, B200 form). The explore kernel leaves one float per
// explorer in S.lens (log2 of its remaining leaves from the effective position, -2 busy /
// not splittable, -3 idle), so this single CTA only scans that array: idle explorers
// (thieves) are paired with the longest remaining intervals (log2 buckets, descending); the
// victim keeps [pos, mid), the thief is seated for an init_at replay of [mid, end).
__global__ void __launch_bounds__(kStealThreads) steal_kernel(StealParams S) {
  __shared__ int s_idle[kStealThreads];
  __shared__ int bins[kBins];
  __shared__ int s_tot[4];
  const int t = threadIdx.x;
  const int K = S.K;
  int idle = 0, active = 0;
  for (int i = t; i < K; i += kStealThreads) {
    if (S.lens[i] == -3.f) ++idle;
    else ++active;
  }
  s_idle[t] = idle;
  for (int b = t; b < kBins; b += kStealThreads) bins[b] = 0;
  if (t < 4) s_tot[t] = 0;
  __syncthreads();
  atomicAdd(&s_tot[0], active);
  for (int off = 1; off < kStealThreads; off <<= 1) {  // inclusive scan of idle counts
    const int v = t >= off ? s_idle[t - off] : 0;
    __syncthreads();
    s_idle[t] += v;
    __syncthreads();
  }
  const int total_idle = s_idle[kStealThreads - 1];
  const int total_active = s_tot[0];
  if (static_cast<float>(total_active) >= S.trigger * static_cast<float>(K) || total_idle == 0 || total_active == 0) {
    if (t == 0) {
      S.ctr->active = total_active;
      S.plan[0] = 0;
    }
    return;
  }
  int r = s_idle[t] - idle;
  for (int i = t; i < K; i += kStealThreads) {
    const float lg = S.lens[i];
    if (lg == -3.f) S.thief[r++] = i;
    else if (lg >= S.min_log2 && lg >= 1.f) atomicAdd(&bins[min(kBins - 1, static_cast<int>(lg * 4.f))], 1);
  }
  __syncthreads();
  if (t == 0) {  // descending exclusive offsets
    int acc = 0;
    for (int b = kBins - 1; b >= 0; --b) {
      const int c = bins[b];
      bins[b] = acc;
      acc += c;
    }
    s_tot[1] = acc;
  }
  __syncthreads();
  // thieves per victim: one when victims suffice, otherwise r-way splits of the longest
  const int nvict = s_tot[1];
  const int rs = nvict >= total_idle ? 1 : min(S.max_split, total_idle / max(nvict, 1));
  const int nv = min(nvict, total_idle / rs);
  for (int i = t; i < K; i += kStealThreads) {
    const float lg = S.lens[i];
    if (lg >= S.min_log2 && lg >= 1.f) {
      const int rank = atomicAdd(&bins[min(kBins - 1, static_cast<int>(lg * 4.f))], 1);
      if (rank < nv) S.victim[rank] = i;
    }
  }
  __syncthreads();
  if (t == 0) {  // the grid-wide split kernels that follow read the plan
    S.plan[0] = nv;
    S.plan[1] = rs;
    S.ctr->active = total_active;
    S.ctr->steal_phases += 1ull;
  }
}

// Export work to another GPU (inter-GPU interval stealing, the intra-box analogue of
// the coordinator's split_unit / steal_from_active, src/workunit.cpp:59-74,
// src/coordinator.cpp:170-187): the `want` active explorers with the longest remaining
// intervals keep [pos, mid) and hand [mid, end) out as factoradic digit vectors.
// Block-wide body (kStealThreads threads): returns the number of exported intervals (all
// threads), written as int digit pairs [a | b] (2n per interval) and end-is-n! flags.
__device__ int export_body(const StealParams& S, int want, int* out_digits, uint8_t* out_nf) {
  __shared__ int bins[kBins];
  __shared__ int s_tot[2];
  const int t = threadIdx.x, K = S.K, n = S.L.n;
  for (int b = t; b < kBins; b += kStealThreads) bins[b] = 0;
  if (t < 2) s_tot[t] = 0;
  __syncthreads();
  for (int i = t; i < K; i += kStealThreads) {
    const float lg = S.lens[i];
    if (lg >= S.min_log2 && lg >= 1.f) atomicAdd(&bins[min(kBins - 1, static_cast<int>(lg * 4.f))], 1);
  }
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int b = kBins - 1; b >= 0; --b) {
      const int c = bins[b];
      bins[b] = acc;
      acc += c;
    }
    s_tot[1] = acc;
  }
  __syncthreads();
  // r parts exported per victim: one when victims suffice, more when only a few hold work
  const int nvict = s_tot[1];
  const int r = nvict >= want ? 1 : min(63, (want + max(nvict, 1) - 1) / max(nvict, 1));  // export: up to 63
  const int nv = min(nvict, (want + r - 1) / r);
  for (int i = t; i < K; i += kStealThreads) {
    const float lg = S.lens[i];
    if (lg >= S.min_log2 && lg >= 1.f) {
      const int rank = atomicAdd(&bins[min(kBins - 1, static_cast<int>(lg * 4.f))], 1);
      if (rank < nv) S.victim[rank] = i;
    }
  }
  __syncthreads();
  int pos[kMaxN], D[kMaxN], b[kMaxN], pb[kMaxN], oend[kMaxN];
  for (int v = t; v < nv; v += kStealThreads) {
    unsigned char* vb = S.state + static_cast<size_t>(S.victim[v]) * S.L.gstride;
    IvmHdr* vh = reinterpret_cast<IvmHdr*>(vb);
    const int8_t* V = reinterpret_cast<const int8_t*>(vb + S.L.o_v);
    int8_t* E = reinterpret_cast<int8_t*>(vb + S.L.o_end);
    const bool had_end = vh->has_end != 0;
    int lstar = 0;
    const int cnt = S.split_mode == 1 ? 0 : live_siblings(vb, S.L, lstar, D);  // D holds the live cells here
    if (cnt > 0 || S.split_mode == 2) {
      int rv = min(r, cnt);
      if (rv < 1) continue;
      const int slot0 = atomicAdd(&s_tot[0], rv);
      if (slot0 >= want) continue;
      rv = min(rv, want - slot0);  // never more than the caller's buffer
      for (int l = 0; l < n; ++l) oend[l] = E[l];
      for (int i = 1; i <= rv; ++i) {
        const bool last = i == rv;
        live_point(V, lstar, live_group_start(D, cnt, rv, i), n, pb);
        if (!last) live_point(V, lstar, live_group_start(D, cnt, rv, i + 1), n, b);
        int* o = out_digits + static_cast<size_t>(slot0 + i - 1) * 2 * n;
        for (int l = 0; l < n; ++l) {
          o[l] = pb[l];
          o[n + l] = last ? (had_end ? oend[l] : 0) : b[l];
        }
        out_nf[slot0 + i - 1] = last ? (had_end ? 0 : 1) : 0;
      }
      live_point(V, lstar, live_group_start(D, cnt, rv, 1), n, pb);  // the victim keeps group 0
      for (int l = 0; l < n; ++l) E[l] = static_cast<int8_t>(pb[l]);
      vh->has_end = 1;
      continue;
    }
    if (!effective_pos(V, vh->level, reinterpret_cast<const int8_t*>(vb + S.L.o_cells), n, pos)) continue;
    int top = 0;
    if (!diff_digits(pos, E, had_end, n, D, top)) continue;
    int rv = r;
    if (!top) {
      long long small = 0;
      bool big = false;
      for (int l = 0; l < n && !big; ++l) {
        small = small * (n - l) + D[l];
        if (small > (1ll << 40)) big = true;
      }
      if (!big) {
        if (small < 2) continue;
        rv = static_cast<int>(min(static_cast<long long>(rv), max(small / 2 - 1, 1ll)));
      }
    }
    const int slot0 = atomicAdd(&s_tot[0], rv);
    if (slot0 >= want) continue;
    rv = min(rv, want - slot0);  // never more than the caller's buffer
    for (int l = 0; l < n; ++l) oend[l] = E[l];
    const int parts = rv + 1;
    split_point(pos, D, top, 1, parts, n, pb);
    for (int l = 0; l < n; ++l) E[l] = static_cast<int8_t>(pb[l]);
    vh->has_end = 1;
    for (int i = 1; i <= rv; ++i) {
      const bool last = i == rv;
      if (!last) split_point(pos, D, top, i + 1, parts, n, b);
      int* o = out_digits + static_cast<size_t>(slot0 + i - 1) * 2 * n;
      for (int l = 0; l < n; ++l) {
        o[l] = pb[l];
        o[n + l] = last ? (had_end ? oend[l] : 0) : b[l];
      }
      out_nf[slot0 + i - 1] = last ? (had_end ? 0 : 1) : 0;
      if (!last)
        for (int l = 0; l < n; ++l) pb[l] = b[l];
    }
  }
  __syncthreads();
  const int cnt = min(s_tot[0], want);
  __syncthreads();
  return cnt;
}

__global__ void __launch_bounds__(kStealThreads) export_kernel(StealParams S, int want, int* out_digits,
                                                              uint8_t* out_nf, int* out_count) {
  const int cnt = export_body(S, want, out_digits, out_nf);
  if (threadIdx.x == 0) *out_count = cnt;
}

// ---- multi-GPU group over NVLink peer memory (the intra-box analogue of the
// coordinator's WORK / BEST exchange, src/coordinator.cpp:170-306, src/workunit.cpp:59-74)
//
// Every rank (one process per GPU) owns one PeerWindow in its device memory, exported with
// cudaIpcGetMemHandle and mapped by every other rank. Per round, after the intra-GPU steal
// pipeline, two small kernels run on each rank's own stream, with no host involvement:
//   group_exchange_kernel  incumbent MIN (system-scope atomicMin into every window), import of
//                          intervals a donor deposited into this rank's inbox (seated on idle
//                          explorers), publication of the active count, a work request when
//                          below `low` active explorers, and the choice of one requesting peer
//                          to serve (claimed with a peer atomicCAS on its lock)
//   group_export_kernel    the claimed request served: the longest remaining intervals are split
//                          (export_body, right parts) and written straight into the peer's inbox
//                          over NVLink, then published with a system fence + ready flag
// The host only polls: termination = two consecutive identical waves of (active, sent, recv)
// over all windows with every active == 0 and sum(sent) == sum(recv) (double counting; in-flight
// deposits show as sent > recv).
constexpr int kMaxGroup = 8;

struct PeerWindow {
  int best;                  // group incumbent (system-scope atomicMin by every rank)
  int active;                // explorers not Empty after the owner's last round
  int req;                   // intervals wanted by the owner (0 = none)
  int lock;                  // 0 free, donor rank + 1 while a deposit is pending / being seated
  int count;                 // intervals left in the inbox
  int ready;                 // donor -> owner: inbox valid
  int pad[2];
  unsigned long long sent;   // intervals this rank deposited into peers
  unsigned long long recv;   // intervals this rank seated from its inbox
  // inbox: cap * 2n int digits, then cap uint8 end-is-n! flags
};
constexpr int kWindowHeader = 64;

struct GroupState {
  int serve, want;           // peer claimed this round (-1 none), intervals it asked for
  int act[kMaxGroup];        // the last wave over all windows (host termination check)
  unsigned long long sent[kMaxGroup], recv[kMaxGroup];
  unsigned long long exchanges, imported, exported;
};

struct GroupParams {
  unsigned char* win[kMaxGroup];  // mapped windows (own included, index = rank)
  int world, rank, K, cap, low, share_best;
  GroupState* gs;
};

__device__ __forceinline__ PeerWindow* pw(const GroupParams& G, int q) { return reinterpret_cast<PeerWindow*>(G.win[q]); }
__device__ __forceinline__ int* inbox_digits(const GroupParams& G, int q) {
  return reinterpret_cast<int*>(G.win[q] + kWindowHeader);
}
__device__ __forceinline__ uint8_t* inbox_nf(const GroupParams& G, int q, int n) {
  return G.win[q] + kWindowHeader + static_cast<size_t>(G.cap) * 2 * n * sizeof(int);
}
__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ unsigned long long vload64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__global__ void __launch_bounds__(kStealThreads) group_exchange_kernel(IvmLayout L, unsigned char* state, const int* ptot,
                                                                      DevCounters* ctr, GroupParams G) {
  __shared__ int s_idle[kStealThreads];
  __shared__ int s_take, s_cnt;
  const int t = threadIdx.x, K = G.K, n = L.n;
  PeerWindow* me = pw(G, G.rank);
  if (t == 0) {
    G.gs->serve = -1;
    G.gs->exchanges += 1ull;
    if (G.share_best) {  // incumbent MIN over the group
      const int b = vload(&ctr->best);
      for (int q = 0; q < G.world; ++q) atomicMin_system(&pw(G, q)->best, b);
      const int gb = vload(&me->best);
      if (gb < b) atomicMin(&ctr->best, gb);
    }
    s_cnt = vload(&me->ready) ? vload(&me->count) : 0;
    __threadfence_system();  // acquire: the inbox is read after the flag
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt > 0) {  // import: seat deposited intervals on idle explorers (list_idle_kernel's scan)
    const int CH = (K + kStealThreads - 1) / kStealThreads;
    const int lo = t * CH, hi = min(K, lo + CH);
    int idle = 0;
    for (int i = lo; i < hi; ++i) idle += reinterpret_cast<const IvmHdr*>(state + static_cast<size_t>(i) * L.gstride)->state == kEmpty;
    s_idle[t] = idle;
    __syncthreads();
    for (int off = 1; off < kStealThreads; off <<= 1) {
      const int v = t >= off ? s_idle[t - off] : 0;
      __syncthreads();
      s_idle[t] += v;
      __syncthreads();
    }
    const int take = min(cnt, s_idle[kStealThreads - 1]);
    int r = s_idle[t] - idle;
    const int* dig = inbox_digits(G, G.rank);
    const uint8_t* nf = inbox_nf(G, G.rank, n);
    for (int i = lo; i < hi && r < take; ++i) {
      unsigned char* blk = state + static_cast<size_t>(i) * L.gstride;
      if (reinterpret_cast<const IvmHdr*>(blk)->state != kEmpty) continue;
      const int e = cnt - 1 - r;  // consume the inbox from its end
      int a[kMaxN], b[kMaxN];
      for (int l = 0; l < n; ++l) {
        a[l] = dig[static_cast<size_t>(e) * 2 * n + l];
        b[l] = dig[static_cast<size_t>(e) * 2 * n + n + l];
      }
      seat_explorer(blk, L, ptot, a, b, !nf[e]);
      ++r;
    }
    if (t == 0) s_take = take;
    __syncthreads();
    if (t == 0 && s_take > 0) {
      me->recv += static_cast<unsigned long long>(s_take);
      ctr->active += s_take;
      ctr->inits += static_cast<unsigned long long>(s_take);
      G.gs->imported += static_cast<unsigned long long>(s_take);
      const int left = cnt - s_take;
      me->count = left;
      if (left == 0) {  // release: ready, request, then the lock (a donor claims only a free lock)
        me->ready = 0;
        me->req = 0;
        __threadfence_system();
        atomicExch_system(&me->lock, 0);
      }
    }
  }
  if (t == 0) {
    const int act = vload(&ctr->active);
    *reinterpret_cast<volatile int*>(&me->active) = act;
    // request work when running low (and nothing is pending)
    if (act < G.low && vload(&me->req) == 0 && vload(&me->lock) == 0 && !vload(&me->ready) && K - act > 0)
      *reinterpret_cast<volatile int*>(&me->req) = min(K - act, G.cap);
    // serve one requesting peer that is much less busy (round robin from the next rank)
    if (act > 0) {
      const unsigned long long rot = G.gs->exchanges;
      for (int i = 1; i < G.world; ++i) {
        const int q = static_cast<int>((static_cast<unsigned long long>(G.rank) + i + rot) % G.world);
        if (q == G.rank) continue;
        PeerWindow* w = pw(G, q);
        const int rq = vload(&w->req);
        if (rq <= 0 || vload(&w->lock) != 0 || 2 * vload(&w->active) + 1 >= act) continue;
        if (atomicCAS_system(&w->lock, 0, G.rank + 1) != 0) continue;
        __threadfence_system();
        G.gs->serve = q;
        G.gs->want = min(vload(&w->req), G.cap);
        break;
      }
    }
    // the wave the host checks for termination
    for (int q = 0; q < G.world; ++q) {
      PeerWindow* w = pw(G, q);
      G.gs->act[q] = vload(&w->active);
      G.gs->sent[q] = vload64(&w->sent);
      G.gs->recv[q] = vload64(&w->recv);
    }
  }
}

__global__ void __launch_bounds__(kStealThreads) group_export_kernel(StealParams S, GroupParams G) {
  const int q = G.gs->serve;
  if (q < 0) return;
  const int cnt = export_body(S, G.gs->want, inbox_digits(G, q), inbox_nf(G, q, S.L.n));
  if (threadIdx.x == 0) {
    PeerWindow* w = pw(G, q);
    if (cnt > 0) {
      pw(G, G.rank)->sent += static_cast<unsigned long long>(cnt);  // counted before it is visible
      G.gs->exported += static_cast<unsigned long long>(cnt);
      __threadfence_system();
      *reinterpret_cast<volatile int*>(&w->count) = cnt;
      __threadfence_system();
      *reinterpret_cast<volatile int*>(&w->ready) = 1;
    } else {
      atomicExch_system(&w->lock, 0);  // nothing to give: release
    }
    G.gs->serve = -1;
  }
}

// Idle explorers in index order (slots for assign / import) and their count.
__global__ void __launch_bounds__(kStealThreads) list_idle_kernel(size_t stride, int soff, const unsigned char* state, int K,
                                                                 int* slots, int* count) {
  __shared__ int s_idle[kStealThreads];
  const int t = threadIdx.x;
  const int CH = (K + kStealThreads - 1) / kStealThreads;
  const int lo = t * CH, hi = min(K, lo + CH);
  int idle = 0;
  for (int i = lo; i < hi; ++i)
    idle += state[static_cast<size_t>(i) * stride + soff] == kEmpty;
  s_idle[t] = idle;
  __syncthreads();
  for (int off = 1; off < kStealThreads; off <<= 1) {
    const int v = t >= off ? s_idle[t - off] : 0;
    __syncthreads();
    s_idle[t] += v;
    __syncthreads();
  }
  int r = s_idle[t] - idle;
  for (int i = lo; i < hi; ++i)
    if (state[static_cast<size_t>(i) * stride + soff] == kEmpty) slots[r++] = i;
  if (t == kStealThreads - 1) *count = s_idle[t];
}

// INT32 peak microbenchmark: 8 independent add+max chains per thread (IADD3 / IMNMX on
// the ALU pipe, the same mix as the LB1/LB2 chains).
__global__ void __launch_bounds__(256) int32_peak_kernel(const int* in, int* out, int iters) {
  int x[8];
  const int y = in[threadIdx.x & 7], z = in[8 + (threadIdx.x & 7)];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = in[16 + i] + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i] = max(x[i] + y, z);
      x[i] = max(x[i] + z, y);
    }
  }
  int acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 0x7fffffff) out[blockIdx.x] = acc;
}

// ------------------------------------------------------------------ kernel tables

using ExploreFn = void (*)(ExploreParams);
using BatchFn = void (*)(BatchParams);

template <int M, int B, bool W = false>
ExploreFn explore_for_group(int G, bool small) {
  switch (G) {
    case 4: return explore_kernel<M, 4, B, false, W>;
    case 8: return explore_kernel<M, 8, B, false, W>;
    case 16: return explore_kernel<M, 16, B, false, W>;
    case 32: return (B == kLB2 && small) ? explore_kernel<M, 32, B, true> : explore_kernel<M, 32, B, false, W>;
  }
  return nullptr;
}
template <int M, int B, bool W = false>
BatchFn batch_for_group(int G, bool small) {
  switch (G) {
    case 4: return decompose_batch_kernel<M, 4, B, false, W>;
    case 8: return decompose_batch_kernel<M, 8, B, false, W>;
    case 16: return decompose_batch_kernel<M, 16, B, false, W>;
    case 32: return (B == kLB2 && small) ? decompose_batch_kernel<M, 32, B, true> : decompose_batch_kernel<M, 32, B, false, W>;
  }
  return nullptr;
}

// SMALLN (n <= 32): LB2 passes iterate the set bits of a 32-bit free-position mask
// wide: 32-bit FT / R tables (LB1 only)
ExploreFn explore_fn(int m, int bound, int G, bool small, bool wide) {
  if (bound == kLB1 && wide) {
    switch (m) {
      case 5: return explore_for_group<5, kLB1, true>(G, false);
      case 10: return explore_for_group<10, kLB1, true>(G, false);
      case 20: return explore_for_group<20, kLB1, true>(G, false);
      case 40: return explore_for_group<40, kLB1, true>(G, false);
      case 60: return explore_for_group<60, kLB1, true>(G, false);
    }
  } else if (bound == kLB1) {
    switch (m) {
      case 5: return explore_for_group<5, kLB1>(G, false);
      case 10: return explore_for_group<10, kLB1>(G, false);
      case 20: return explore_for_group<20, kLB1>(G, false);
      case 40: return explore_for_group<40, kLB1>(G, false);
      case 60: return explore_for_group<60, kLB1>(G, false);
    }
  } else {
    switch (m) {
      case 5: return explore_for_group<5, kLB2>(G, small);
      case 10: return explore_for_group<10, kLB2>(G, small);
      case 20: return explore_for_group<20, kLB2>(G, small);
    }
  }
  return nullptr;
}

using BigFn = void (*)(BigBatchParams);
using Big1Fn = void (*)(BigBatchParams, const int*);
Big1Fn big1_fn(int m) {
  switch (m) {
    case 5: return decompose_big_lb1_kernel<5>;
    case 10: return decompose_big_lb1_kernel<10>;
    case 20: return decompose_big_lb1_kernel<20>;
  }
  return nullptr;
}

Big1Fn big1g_fn(int m) {
  switch (m) {
    case 5: return decompose_big_lb1g_kernel<5>;
    case 10: return decompose_big_lb1g_kernel<10>;
    case 20: return decompose_big_lb1g_kernel<20>;
  }
  return nullptr;
}

using Big2wFn = void (*)(BigBatchParams, const int*, const uint32_t*, int, int*);
Big2wFn big2w_fn(int m) {
  switch (m) {
    case 5: return decompose_big_lb2w_kernel<5>;
    case 10: return decompose_big_lb2w_kernel<10>;
    case 20: return decompose_big_lb2w_kernel<20>;
  }
  return nullptr;
}

BigFn big_fn(int m, int bound) {
  if (bound == kLB1) {
    switch (m) {
      case 5: return decompose_big_kernel<5, kLB1>;
      case 10: return decompose_big_kernel<10, kLB1>;
      case 20: return decompose_big_kernel<20, kLB1>;
    }
  } else {
    switch (m) {
      case 5: return decompose_big_kernel<5, kLB2>;
      case 10: return decompose_big_kernel<10, kLB2>;
      case 20: return decompose_big_kernel<20, kLB2>;
    }
  }
  return nullptr;
}

BatchFn batch_fn(int m, int bound, int G, bool small, bool wide) {
  if (bound == kLB1 && wide) {
    switch (m) {
      case 5: return batch_for_group<5, kLB1, true>(G, false);
      case 10: return batch_for_group<10, kLB1, true>(G, false);
      case 20: return batch_for_group<20, kLB1, true>(G, false);
      case 40: return batch_for_group<40, kLB1, true>(G, false);
      case 60: return batch_for_group<60, kLB1, true>(G, false);
    }
  } else if (bound == kLB1) {
    switch (m) {
      case 5: return batch_for_group<5, kLB1>(G, false);
      case 10: return batch_for_group<10, kLB1>(G, false);
      case 20: return batch_for_group<20, kLB1>(G, false);
      case 40: return batch_for_group<40, kLB1>(G, false);
      case 60: return batch_for_group<60, kLB1>(G, false);
    }
  } else {
    switch (m) {
      case 5: return batch_for_group<5, kLB2>(G, small);
      case 10: return batch_for_group<10, kLB2>(G, small);
      case 20: return batch_for_group<20, kLB2>(G, small);
    }
  }
  return nullptr;
}

}  // namespace

// ------------------------------------------------------------------ pool

// PBBGPU_TRACE=1: host-side timing of slow pool-management calls on stderr (diagnostics)
static bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("PBBGPU_TRACE");
    return e && *e && *e != '0';
  }();
  return on;
}
struct TraceScope {
  const char* what;
  std::chrono::steady_clock::time_point t0;
  explicit TraceScope(const char* w) : what(w), t0(std::chrono::steady_clock::now()) {}
  ~TraceScope() {
    if (!trace_on()) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms >= 5.0) std::fprintf(stderr, "[pbbgpu] %s: %.1f ms\n", what, ms);
  }
};

struct pbbgpu_pool {
  int n = 0, m = 0, mp = 0, bound = 0;  // m: compiled machine count (5, 10, 20)
  int m_real = 0;                        // the instance's machines (zero-time machines pad to m)
  bool wide = false;                     // 32-bit FT / R / prefix sums ((n+m)*max p >= 2^16, LB1)
  pbbgpu_config_t cfg{};
  std::vector<int32_t> p;
  int K = 0, G = 0, steps = 0, grid = 0, block = 128;
  double round_us = 0;
  size_t smem = 0;
  IvmLayout L{};
  InstLayout IL{};
  int npairs = 0;
  ExploreFn efn = nullptr;
  BatchFn bfn = nullptr;
  bool batch_only = false;  // n > 64: bounding (decompose_batch) only
  void (*big)(BigBatchParams) = nullptr;
  void (*big1)(BigBatchParams, const int*) = nullptr;   // LB1: warp per node (children-heavy batches)
  void (*big1g)(BigBatchParams, const int*) = nullptr;  // LB1: lane-per-node tables (table-heavy batches)
  int big1g_grid = 0;
  size_t big1g_smem = 0;
  uint2* d_packed64 = nullptr;
  uint32_t* d_packed32big = nullptr;   // LB2 warp-per-node order entries [n][PS]: job | u << 9 | v << 24
  bool packed32big = false;
  Big2wFn big2w = nullptr;
  int* d_pm_scratch = nullptr;         // per warp [kBig2wFmax][32] PM' ranks
  int big2w_grid = 0, big2w_warps = 0;
  size_t smem_optin = 0;               // cudaDevAttrMaxSharedMemoryPerBlockOptin
  int num_sms = 148;                   // cudaDeviceProp::multiProcessorCount
  int split_grid = 0;                  // split_kernel blocks (kSplitWarps victims each per pass)
  uint16_t* d_inv16 = nullptr;
  int* d_big_scratch = nullptr;
  int big_grid = 0;
  size_t big_smem = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evs[24] = {};  // per round: explore start, explore end, steal end
  double steal_ms = 0;
  int rounds_per_sync = 2;
  unsigned char* d_state = nullptr;
  int *d_p32 = nullptr, *d_ptot = nullptr, *d_wrk = nullptr;
  uint8_t *d_pk = nullptr, *d_pl = nullptr, *d_ord = nullptr;
  uint16_t* d_lag = nullptr;
  uint32_t* d_packed = nullptr;
  uint8_t* d_invord = nullptr;

  float* d_lgfact = nullptr;
  float* d_lens = nullptr;
  DevCounters* d_ctr = nullptr;
  DevCounters* h_ctr = nullptr;  // pinned
  unsigned long long *d_hist = nullptr, *d_dhist = nullptr;
  ImpRecord* d_imp = nullptr;
  std::mutex best_mu;
  std::atomic<int64_t> pending_offer{INT64_MAX};
  int64_t best_value = INT64_MAX;
  int64_t best_sched_value = INT64_MAX;
  int64_t pinned_ub = INT64_MAX;
  std::vector<int32_t> best_sched;
  uint64_t rounds = 0;
  uint64_t launches = 0;
  double batch_ms = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  double kernel_ms = 0;
  int last_active = 0;
  // grow-only device scratch for per-call staging (assign / export / decompose_batch): a
  // cudaMalloc + cudaFree pair per call synchronizes the device and occasionally stalls for
  // hundreds of milliseconds while the driver returns memory
  void* scr[8] = {};
  size_t scr_cap[8] = {};
  void* pin = nullptr;  // pinned host staging for table uploads (grow-only)
  size_t pin_cap = 0;
  // the reference steal policy (steal_policy = 1): exact lengths, flags, pairs
  u128* d_ref_len = nullptr;
  uint8_t* d_ref_flags = nullptr;
  int* d_ref_pairs = nullptr;
  u128 ref_min_steal = 0;
  // record_census
  unsigned long long* d_census = nullptr;
  int census_cap = 0;
  // activity timeline (explorer.cpp:71-85, 448-471)
  FILE* timeline = nullptr;
  std::chrono::steady_clock::time_point t_start{}, t_last_sample{};
  bool sampled = false;
  // explorer pool for n > 64 (explore_big.cuh): IVMs in HBM, bounded by the large-n kernels
  bool big_explore = false;
  BigIvmLayout BL{};
  int big_steps = 8;
  int *d_bperm = nullptr, *d_bd1 = nullptr, *d_bd2 = nullptr, *d_bfstat = nullptr;
  uint8_t *d_bkind = nullptr, *d_bdir = nullptr, *d_bpr = nullptr;
  int *d_blb = nullptr, *d_blf = nullptr, *d_blbw = nullptr;
  BigImp* d_bimp = nullptr;
  int* h_bfstat = nullptr;  // pinned
  // multi-GPU group over peer memory (pbbgpu_group_*)
  int g_world = 0, g_rank = 0, g_cap = 0;
  unsigned char* d_window = nullptr;       // own PeerWindow (IPC-exported)
  unsigned char* g_peer[kMaxGroup] = {};   // mapped windows (own at g_rank)
  bool g_open = false;
  GroupState* d_gs = nullptr;
  GroupState* h_gs = nullptr;              // pinned
  cudaEvent_t gev[8] = {};                 // per round: start of the exchange kernels
  double group_ms = 0;                     // device time of the exchange kernels
  uint64_t group_rounds = 0;
  // marks (explorer.hpp:94-96)
  int64_t improvement_mark = INT64_MAX;
  uint64_t steal_mark = 0;
  uint64_t host_improvements = 0;  // offer_schedule improvements of the bound (explorer.cpp:379-386)

  void release() {
    TraceScope ts("release");
    {
      TraceScope t1("release: stream sync");
      if (stream) cudaStreamSynchronize(stream);
    }
    TraceScope t2("release: frees");
    for (void* q : scr) cudaFree(q);
    cudaFree(d_state);
    cudaFree(d_p32);
    cudaFree(d_ptot);
    cudaFree(d_wrk);
    cudaFree(d_pk);
    cudaFree(d_pl);
    cudaFree(d_ord);
    cudaFree(d_lag);
    cudaFree(d_packed);
    cudaFree(d_invord);
    cudaFree(d_packed64);
    cudaFree(d_packed32big);
    cudaFree(d_pm_scratch);
    cudaFree(d_inv16);
    cudaFree(d_big_scratch);

    cudaFree(d_lgfact);
    cudaFree(d_lens);
    cudaFree(d_ctr);
    cudaFree(d_hist);
    cudaFree(d_dhist);
    cudaFree(d_imp);
    cudaFree(d_ref_len);
    cudaFree(d_ref_flags);
    cudaFree(d_ref_pairs);
    cudaFree(d_census);
    for (void* q : {static_cast<void*>(d_bperm), static_cast<void*>(d_bd1), static_cast<void*>(d_bd2),
                    static_cast<void*>(d_bfstat), static_cast<void*>(d_bkind), static_cast<void*>(d_bdir),
                    static_cast<void*>(d_bpr), static_cast<void*>(d_blb), static_cast<void*>(d_blf),
                    static_cast<void*>(d_blbw), static_cast<void*>(d_bimp)})
      cudaFree(q);
    if (h_bfstat) cudaFreeHost(h_bfstat);
    for (int q = 0; q < g_world; ++q)
      if (q != g_rank && g_peer[q]) cudaIpcCloseMemHandle(g_peer[q]);
    cudaFree(d_window);
    cudaFree(d_gs);
    if (h_gs) cudaFreeHost(h_gs);
    if (timeline) std::fclose(timeline);
    if (h_ctr) cudaFreeHost(h_ctr);
    if (pin) cudaFreeHost(pin);
    for (cudaEvent_t e : evs)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : gev)
      if (e) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// Every host<->device copy of a pool goes through here (counted for the e2e report).
void xfer(pbbgpu_pool* P, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) {
  ck(cudaMemcpyAsync(dst, src, bytes, kind, P->stream), what);
  ck(cudaStreamSynchronize(P->stream), what);
  if (kind == cudaMemcpyHostToDevice) P->h2d_bytes += bytes;
  else if (kind == cudaMemcpyDeviceToHost) P->d2h_bytes += bytes;
}

int pick_group(int n, int bound) {
  if (bound == kLB1) return 16;
  return 32;  // warp per explorer, lanes over machine pairs (children_lb2_w)
}

// Host-built instance tables (everything the kernels read about p), uploaded into the
// pool's device buffers at create time and again by pbbgpu_load_instance.
struct HostTables {
  std::vector<int> p32, ptot;
  std::vector<uint8_t> pk, pl, ord, inv;
  std::vector<uint16_t> lag, ord16, inv16;
  std::vector<uint32_t> packed;
  std::vector<uint2> pk64;
  std::vector<uint32_t> pk32big;  // [n][PS] job | u << 9 | v << 24 (decompose_big_lb2w_kernel)
  bool packable32big = false;
  bool packable = false;
};

// Returns whether the instance needs wide (32-bit) explorer tables: every front / tail /
// remain / bound is below (n+m)*max p, the 16-bit tables hold it when that is < 2^16. LB2's
// pair tables and SIMD combine stay 16-bit; LB1 goes up to n*(n+m)*max p < 2^31 (MinMin's sum
// of the children's bounds fits int32).
bool validate_times(int n, int m, const int32_t* p, int bound) {
  int pmax = 0;
  for (int i = 0; i < n * m; ++i) {
    if (p[i] < 0) throw std::invalid_argument("negative processing time");
    pmax = std::max(pmax, p[i]);
  }
  const int64_t span = static_cast<int64_t>(n + m) * pmax;
  if (span < 65536) return false;
  if (bound == kLB2) throw std::invalid_argument("pbbgpu: LB2 needs (n+m)*max(p) below 2^16 (use LB1 for wider times)");
  if (span * n >= (int64_t{1} << 31)) throw std::invalid_argument("pbbgpu: n*(n+m)*max(p) must stay below 2^31");
  return true;
}

// Compiled machine count for an instance with m machines: the instance is padded with
// zero-time machines after the last one. A trailing zero machine changes no makespan, no
// front / tail / remain of a real machine and no LB1 value (its chain term never exceeds the
// last real machine's), and LB2 pairs are built over the real machines only, so every value
// the reference defines is unchanged (tests/test_gpu.py::test_any_machine_count_*).
int compiled_m(int m) {
  if (m < 1 || m > 60) throw std::invalid_argument("pbbgpu: m must be in [1, 60] (padded to 5, 10, 20, 40 or 60 machines)");
  return m <= 5 ? 5 : (m <= 10 ? 10 : (m <= 20 ? 20 : (m <= 40 ? 40 : 60)));
}

std::vector<int32_t> pad_machines(int n, int m, int M, const int32_t* p) {
  std::vector<int32_t> q(static_cast<size_t>(n) * M, 0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < m; ++k) q[static_cast<size_t>(j) * M + k] = p[static_cast<size_t>(j) * m + k];
  return q;
}

// m: the instance's machines (p_real row stride, LB2 pairs); M: compiled (p32 / ptot width).
HostTables build_tables(int n, int m, int M, int bound, const int32_t* p_real, bool big) {
  HostTables T;
  const int mp = round_up(M, 4);
  const int npairs = m * (m - 1) / 2;
  const int32_t* p = p_real;
  T.p32.assign(static_cast<size_t>(n) * mp, 0);
  T.ptot.assign(static_cast<size_t>(M), 0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < m; ++k) {
      T.p32[static_cast<size_t>(j) * mp + k] = p[static_cast<size_t>(j) * m + k];
      T.ptot[static_cast<size_t>(k)] += p[static_cast<size_t>(j) * m + k];
    }
  if (bound != kLB2) return T;
  lb2_tables(n, m, p, T.pk, T.pl, T.ord, T.lag, T.packed, T.packable, T.ord16);
  if (big) {
    T.pk64.resize(static_cast<size_t>(n) * npairs);
    for (int q = 0; q < npairs; ++q)
      for (int t = 0; t < n; ++t) {
        const int j = T.ord16[static_cast<size_t>(q) * n + t];
        const int a = p[static_cast<size_t>(j) * m + T.pk[static_cast<size_t>(q)]];
        const int bb = p[static_cast<size_t>(j) * m + T.pl[static_cast<size_t>(q)]];
        const int lg = T.lag[static_cast<size_t>(q) * n + j];
        if (a > 65535 || bb > 65535) throw std::invalid_argument("processing time exceeds 16 bits");
        T.pk64[static_cast<size_t>(t) * npairs + q] =
            make_uint2(static_cast<unsigned>(j) | static_cast<unsigned>(a) << 16, static_cast<unsigned>(bb) | static_cast<unsigned>(lg) << 16);
      }
    {  // warp-per-node entries: u = a + lag (11 bits), v = a - b (8 bits, signed), job (9 bits)
      const int PS = round_up(npairs, 32);
      T.pk32big.assign(static_cast<size_t>(n) * PS, 0);
      T.packable32big = n <= 512;
      for (int q = 0; q < npairs; ++q)
        for (int t = 0; t < n; ++t) {
          const int j = T.ord16[static_cast<size_t>(q) * n + t];
          const int a = p[static_cast<size_t>(j) * m + T.pk[static_cast<size_t>(q)]];
          const int bb = p[static_cast<size_t>(j) * m + T.pl[static_cast<size_t>(q)]];
          const int u = a + T.lag[static_cast<size_t>(q) * n + j], v = a - bb;
          if (u > 2047 || v < -128 || v > 127) T.packable32big = false;
          T.pk32big[static_cast<size_t>(t) * PS + q] =
              static_cast<uint32_t>(j) | static_cast<uint32_t>(u & 0x7ff) << 9 | static_cast<uint32_t>(v & 0xff) << 24;
        }
    }
    T.inv16.assign(static_cast<size_t>(n) * npairs, 0);  // [job][pair] -> position
    for (int q = 0; q < npairs; ++q)
      for (int t = 0; t < n; ++t)
        T.inv16[static_cast<size_t>(T.ord16[static_cast<size_t>(q) * n + t]) * npairs + q] = static_cast<uint16_t>(t);
  } else {
    T.inv.assign(static_cast<size_t>(n) * npairs, 0);  // [job][pair] -> position
    for (int q = 0; q < npairs; ++q)
      for (int t = 0; t < n; ++t) T.inv[static_cast<size_t>(T.ord16[static_cast<size_t>(q) * n + t]) * npairs + q] = static_cast<uint8_t>(t);
  }
  return T;
}

// Table uploads: allocate on first use, stage through the pool's pinned host buffer and
// copy asynchronously; one stream sync at the end (counted host->device bytes).
struct Uploader {
  pbbgpu_pool* P;
  size_t off = 0;
  std::vector<std::pair<void*, std::pair<size_t, size_t>>> jobs;  // dst, (staging offset, bytes)
  std::vector<const void*> srcs;
  template <class D, class V>
  void put(D*& dptr, const V& v) {
    const size_t bytes = v.size() * sizeof(v[0]);
    if (!bytes) return;
    if (!dptr) ck(cudaMalloc(&dptr, bytes), "malloc");
    jobs.push_back({dptr, {off, bytes}});
    srcs.push_back(v.data());
    off += (bytes + 15) / 16 * 16;
  }
  void run() {
    if (P->pin_cap < off) {
      if (P->pin) cudaFreeHost(P->pin);
      P->pin = nullptr;
      P->pin_cap = 0;
      ck(cudaMallocHost(&P->pin, off), "malloc host");
      P->pin_cap = off;
    }
    unsigned char* st = static_cast<unsigned char*>(P->pin);
    for (size_t i = 0; i < jobs.size(); ++i) std::memcpy(st + jobs[i].second.first, srcs[i], jobs[i].second.second);
    for (const auto& jb : jobs) {
      ck(cudaMemcpyAsync(jb.first, st + jb.second.first, jb.second.second, cudaMemcpyHostToDevice, P->stream), "copy");
      P->h2d_bytes += jb.second.second;
    }
    ck(cudaStreamSynchronize(P->stream), "sync");
  }
};

template <class D, class V>
void put(pbbgpu_pool* P, D*& dptr, const V& v) {
  Uploader u{P};
  u.put(dptr, v);
  u.run();
}

void upload_tables(pbbgpu_pool* P, const HostTables& T) {
  Uploader u{P};
  u.put(P->d_p32, T.p32);
  u.put(P->d_ptot, T.ptot);
  if (P->bound == kLB2) {
    u.put(P->d_pk, T.pk);
    u.put(P->d_pl, T.pl);
    if (P->batch_only) {
      u.put(P->d_packed64, T.pk64);
      u.put(P->d_packed32big, T.pk32big);
      u.put(P->d_inv16, T.inv16);
    } else {
      u.put(P->d_ord, T.ord);
      u.put(P->d_lag, T.lag);
      u.put(P->d_packed, T.packed);
      u.put(P->d_invord, T.inv);
    }
  }
  u.run();
}

// counters, histograms, incumbent and explorer states back to a fresh pool's
void reset_search(pbbgpu_pool* P) {
  if (P->batch_only && !P->big_explore) return;  // bounding-only pools keep no search state
  DevCounters z{};
  z.best = INT_MAX;
  xfer(P, P->d_ctr, &z, sizeof(z), cudaMemcpyHostToDevice, "copy");
  ck(cudaMemsetAsync(P->d_hist, 0, (static_cast<size_t>(P->n) + 1) * sizeof(unsigned long long), P->stream), "memset");
  ck(cudaMemsetAsync(P->d_dhist, 0, (static_cast<size_t>(P->n) + 1) * sizeof(unsigned long long), P->stream), "memset");
  if (P->big_explore) big_clear_kernel<<<(P->K + 255) / 256, 256, 0, P->stream>>>(P->BL, P->d_state, P->K);
  else clear_kernel<<<(P->K + 255) / 256, 256, 0, P->stream>>>(P->L, P->d_state, P->K);
  ck(cudaGetLastError(), "clear_kernel");
  P->launches += 1;
  ck(cudaStreamSynchronize(P->stream), "sync");
  std::scoped_lock lk(P->best_mu);
  P->best_value = INT64_MAX;
  P->best_sched_value = INT64_MAX;
  P->pinned_ub = INT64_MAX;
  P->best_sched.clear();
  P->pending_offer.store(INT64_MAX);
  P->last_active = 0;
  P->improvement_mark = INT64_MAX;
  P->steal_mark = 0;
  P->host_improvements = 0;
}

void open_timeline(pbbgpu_pool* P);

void pool_init(pbbgpu_pool* P, int n, int m_real, const int32_t* p_real, int bound, const pbbgpu_config_t* cfg) {
  if (n < 2 || n > kBigMaxN) throw std::invalid_argument("pbbgpu: n must be in [2, 512]");
  if (bound != kLB1 && bound != kLB2) throw std::invalid_argument("pbbgpu: bound must be PBBGPU_LB1 or PBBGPU_LB2");
  const int m = compiled_m(m_real);
  if (bound == kLB2 && m_real < 2) bound = kLB1;  // no machine pair: LB2 is LB1
  if (m > 20 && (bound == kLB2 || n > kMaxN))
    throw std::invalid_argument("pbbgpu: m > 20 is supported for LB1 with n <= 64 (LB2 pair tables and the n > 64 "
                                "kernels are compiled for m <= 20)");
  P->wide = validate_times(n, m, pad_machines(n, m_real, m, p_real).data(), bound);
  P->m_real = m_real;
  if (cfg && cfg->record_census && n > 20) throw std::invalid_argument("record_census needs n <= 20 (position_u64)");
  if (cfg && cfg->steal_policy == 1 && n > 30) throw std::invalid_argument("the reference steal policy needs n <= 30");
  if (cfg && (cfg->steal_policy < 0 || cfg->steal_policy > 1)) throw std::invalid_argument("steal_policy must be 0 or 1");
  P->n = n;
  P->m = m;
  P->bound = bound;
  P->p = pad_machines(n, m_real, m, p_real);  // host makespans on the padded matrix are the instance's
  if (cfg) P->cfg = *cfg;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw CudaError("pbbgpu: no CUDA device (the product path has no CPU fallback)");
  cudaDeviceProp prop;
  {
    TraceScope ts("create: device, stream, events");
    ck(cudaSetDevice(P->cfg.device), "cudaSetDevice");
    ck(cudaGetDeviceProperties(&prop, P->cfg.device), "cudaGetDeviceProperties");
    if (prop.major < 10) throw CudaError("pbbgpu: kernels are built for sm_100a only");
    P->num_sms = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&P->ev0), "event");
    ck(cudaEventCreate(&P->ev1), "event");
    for (cudaEvent_t& e : P->evs) ck(cudaEventCreate(&e), "event");
  }
  P->rounds_per_sync = P->cfg.rounds_per_sync > 0 ? std::min(P->cfg.rounds_per_sync, 8) : 3;

  if (bound == kLB2) P->npairs = m_real * (m_real - 1) / 2;
  const HostTables T = build_tables(n, m_real, m, bound, p_real, n > kMaxN);
  const bool packable = T.packable;
  if (n > kMaxN) {  // batch-only pool: the large-n bounding kernel, no explorers
    P->batch_only = true;
    P->mp = round_up(m, 4);
    P->big = big_fn(m, bound);
    upload_tables(P, T);
    const void* kfn = reinterpret_cast<const void*>(P->big);
    int threads = kBigThreads;
    if (bound == kLB1) {  // warp per node
      P->big1 = big1_fn(m);
      kfn = reinterpret_cast<const void*>(P->big1);
      threads = kBig1Warps * 32;
      P->big_smem = static_cast<size_t>(big1_smem_bytes(n, P->mp, m));
      P->big1g = big1g_fn(m);
      P->big1g_smem = static_cast<size_t>(big1g_smem_bytes(n, P->mp));
      const void* gfn = reinterpret_cast<const void*>(P->big1g);
      ck(cudaFuncSetAttribute(gfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->big1g_smem)), "smem attr");
      int per_sm_g = 0;
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_g, gfn, kBig1gWarps * 32, P->big1g_smem), "occupancy");
      if (per_sm_g < 1) throw CapacityError("pbbgpu: large-n bounding kernel cannot be resident");
      P->big1g_grid = per_sm_g * prop.multiProcessorCount;
    } else {
      P->big_smem = static_cast<size_t>(big_smem_bytes(n, P->mp, m));
    }
    ck(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->big_smem)), "smem attr");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, P->big_smem), "occupancy");
    if (per_sm < 1) throw CapacityError("pbbgpu: large-n bounding kernel cannot be resident");
    P->big_grid = per_sm * prop.multiProcessorCount;
    if (bound == kLB2) {
      ck(cudaMalloc(&P->d_big_scratch, static_cast<size_t>(P->big_grid) * n * kBigThreads * sizeof(int)), "malloc scratch");
      // warp per node for batches of nodes with f <= kBig2wFmax: as many warps per SM as the
      // shared memory holds at the largest f (the launch sizes its dynamic smem per batch)
      P->packed32big = T.packable32big;
      P->big2w = big2w_fn(m);
      const void* wfn = reinterpret_cast<const void*>(P->big2w);
      const size_t cap = static_cast<size_t>(prop.sharedMemPerBlockOptin);
      P->smem_optin = cap;
      ck(cudaFuncSetAttribute(wfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cap)), "smem attr");
      int w = kBig2wMaxWarps;
      while (w > 1 && static_cast<size_t>(big2w_smem_bytes(n, P->mp, m, kBig2wFmax, w)) > cap) --w;
      P->big2w_warps = w;
      P->big2w_grid = prop.multiProcessorCount;
      ck(cudaMalloc(&P->d_pm_scratch, static_cast<size_t>(P->big2w_grid) * kBig2wMaxWarps * kBig2wFmax * 32 * sizeof(int)),
         "malloc scratch");
    }
    P->K = 0;
    if (P->cfg.explorers > 0) {  // explorer pool (explore_big.cuh)
      if (P->cfg.steal_policy == 1 || P->cfg.record_census)
        throw std::invalid_argument("pbbgpu: steal_policy 1 and census need n <= 64");
      P->big_explore = true;
      P->K = P->cfg.explorers;
      P->BL = big_ivm_layout(n);
      P->big_steps = P->cfg.steps_per_round > 0 ? P->cfg.steps_per_round : 8;
      const size_t K = static_cast<size_t>(P->K);
      ck(cudaMalloc(&P->d_state, K * P->BL.stride), "malloc explorers");
      ck(cudaMalloc(&P->d_bperm, K * n * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_bd1, K * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_bd2, K * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_bkind, K), "malloc");
      ck(cudaMalloc(&P->d_bfstat, 4 * sizeof(int)), "malloc");
      ck(cudaMallocHost(&P->h_bfstat, 4 * sizeof(int)), "malloc host");
      ck(cudaMalloc(&P->d_blb, K * n * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_blf, K * n * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_blbw, K * n * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_bdir, K), "malloc");
      ck(cudaMalloc(&P->d_bpr, K * n), "malloc");
      ck(cudaMalloc(&P->d_bimp, kBigImpCap * sizeof(BigImp)), "malloc");
      ck(cudaMalloc(&P->d_wrk, (K * 2 + 4) * sizeof(int)), "malloc");
      ck(cudaMalloc(&P->d_lens, K * sizeof(float)), "malloc");
      ck(cudaMalloc(&P->d_ctr, sizeof(DevCounters)), "malloc");
      ck(cudaMallocHost(&P->h_ctr, sizeof(DevCounters)), "malloc host");
      ck(cudaMalloc(&P->d_hist, (static_cast<size_t>(n) + 1) * sizeof(unsigned long long)), "malloc");
      ck(cudaMalloc(&P->d_dhist, (static_cast<size_t>(n) + 1) * sizeof(unsigned long long)), "malloc");
      std::vector<float> lgf(static_cast<size_t>(n) + 1, 0.f);
      for (int k = 2; k <= n; ++k) lgf[static_cast<size_t>(k)] = lgf[static_cast<size_t>(k - 1)] + std::log2(static_cast<float>(k));
      put(P, P->d_lgfact, lgf);
      reset_search(P);
      open_timeline(P);
    }
    P->cfg.timeline_path = nullptr;
    return;
  }
  P->G = P->cfg.group > 0 ? P->cfg.group : pick_group(n, bound);
  if (P->G != 4 && P->G != 8 && P->G != 16 && P->G != 32) throw std::invalid_argument("pbbgpu: group must be 4, 8, 16 or 32");
  if (bound == kLB2 && P->G == 32 && !packable) P->G = 16;  // packed (a, b, lag) do not fit 31 bits
  // CTA size: the instance tables are staged once per CTA, so larger CTAs amortize them;
  // pick the block size that keeps the most explorers resident per SM.
  auto size_for = [&](int G, int BS) {
    const IvmLayout L = ivm_layout(n, m, bound, G, P->wide);
    const InstLayout IL = inst_layout(n, L.mp, P->npairs, bound == kLB2 && G == 32, P->wide);
    return std::make_pair(static_cast<size_t>(IL.bytes) + static_cast<size_t>(BS / G) * L.sstride, std::make_pair(L, IL));
  };
  const size_t smem_cap = static_cast<size_t>(prop.sharedMemPerBlockOptin);
  // (block size, explorers resident per SM) for group size G
  auto choose = [&](int G) {
    // the occupancy calculator of this kernel variant (registers, smem, block limits) for
    // every warp-multiple block size: the most explorers resident per SM wins
    int bs = 0;
    long res = -1;
    const void* fn = reinterpret_cast<const void*>(explore_fn(m, bound, G, n <= 32, P->wide));
    cudaFuncAttributes fa{};
    ck(cudaFuncGetAttributes(&fa, fn), "func attrs");
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_cap)), "smem attr");
    for (int BS = 64; BS <= 1024; BS += 32) {
      if (BS > fa.maxThreadsPerBlock || BS % G) continue;
      const size_t need = size_for(G, BS).first;
      if (need > smem_cap) continue;
      int ctas = 0;
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, BS, need), "occupancy");
      if (static_cast<long>(ctas) * (BS / G) > res) {
        res = static_cast<long>(ctas) * (BS / G);
        bs = BS;
      }
    }
    return std::make_pair(bs, res);
  };
  TraceScope ts_choose("create: block choice");
  int best_bs = 0;
  for (;;) {
    best_bs = choose(P->G).first;
    if (best_bs || P->G >= 32) break;
    P->G *= 2;
  }
  // LB1: 8 lanes per explorer (4 explorers per warp amortize the single-lane table
  // extensions) when shared memory still seats >= 768 threads per SM; 16 otherwise
  if (bound == kLB1 && P->cfg.group <= 0 && P->G == 16) {
    const auto c8 = choose(8);
    if (c8.first && c8.second * 8 >= 768) {
      P->G = 8;
      best_bs = c8.first;
    }
  }
  if (!best_bs) throw CapacityError("pbbgpu: explorer state exceeds shared memory");
  if (P->cfg.block > 0) best_bs = P->cfg.block;
  P->block = best_bs;
  const auto sz = size_for(P->G, P->block);
  P->smem = sz.first;
  P->L = sz.second.first;
  P->IL = sz.second.second;
  P->mp = P->L.mp;
  P->efn = explore_fn(m, bound, P->G, n <= 32, P->wide);
  P->bfn = batch_fn(m, bound, P->G, n <= 32, P->wide);
  ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(P->efn), cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->smem)), "smem attr");
  ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(P->bfn), cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->smem)), "smem attr");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(P->efn), P->block, P->smem), "occupancy");
  if (per_sm < 1) throw CapacityError("pbbgpu: explore kernel cannot be resident");
  const int NGb = P->block / P->G;
  if (P->cfg.explorers > 0) {
    P->K = P->cfg.explorers;
  } else {
    P->K = per_sm * prop.multiProcessorCount * NGb;
  }
  P->grid = (P->K + NGb - 1) / NGb;
  if (P->cfg.steal_policy == 1 && P->cfg.steps_per_round <= 0) P->cfg.steps_per_round = 1024;  // batch_steps
  P->steps = P->cfg.steps_per_round > 0 ? P->cfg.steps_per_round : (1 << 30);
  // warp explorers (LB2) take tens of us per step: longer rounds amortize the round-end wait
  P->round_us = P->cfg.round_us > 0 ? P->cfg.round_us : (P->cfg.steps_per_round > 0 ? 0.0 : (P->G == 32 ? 2500.0 : 2000.0));

  // device buffers
  std::vector<float> lgf(static_cast<size_t>(n) + 1, 0.f);
  for (int k = 2; k <= n; ++k) lgf[static_cast<size_t>(k)] = lgf[static_cast<size_t>(k - 1)] + std::log2(static_cast<float>(k));
  ck(cudaMalloc(&P->d_state, static_cast<size_t>(P->K) * P->L.gstride), "malloc state");
  ck(cudaMalloc(&P->d_wrk, (static_cast<size_t>(P->K) * 2 + 4) * sizeof(int)), "malloc");
  ck(cudaMalloc(&P->d_lens, static_cast<size_t>(P->K) * sizeof(float)), "malloc");
  P->split_grid = std::max(1, std::min((P->K + kSplitWarps - 1) / kSplitWarps, 4 * P->num_sms));
  ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(split_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kSplitWarps * P->L.gstride), "smem attr");
  ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(lens_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kLensWarps * P->L.gstride), "smem attr");
  ck(cudaMalloc(&P->d_ctr, sizeof(DevCounters)), "malloc");
  ck(cudaMallocHost(&P->h_ctr, sizeof(DevCounters)), "malloc host");
  ck(cudaMalloc(&P->d_hist, (static_cast<size_t>(n) + 1) * sizeof(unsigned long long)), "malloc");
  ck(cudaMalloc(&P->d_dhist, (static_cast<size_t>(n) + 1) * sizeof(unsigned long long)), "malloc");
  ck(cudaMalloc(&P->d_imp, kImpCap * sizeof(ImpRecord)), "malloc");
  if (P->cfg.steal_policy == 1) {
    ck(cudaMalloc(&P->d_ref_len, static_cast<size_t>(P->K) * sizeof(u128)), "malloc");
    ck(cudaMalloc(&P->d_ref_flags, static_cast<size_t>(P->K)), "malloc");
    ck(cudaMalloc(&P->d_ref_pairs, static_cast<size_t>(P->K) * 3 * sizeof(int)), "malloc");
    // min_steal_len = min(8!, ceil(n!/4K)) (explorer.cpp:96-103), or the configured length
    u128 nf = 1;
    for (int i = 2; i <= n; ++i) nf *= static_cast<u128>(i);
    const u128 div = static_cast<u128>(4) * static_cast<u128>(P->K);
    const u128 quarter = (nf + div - 1) / div;
    P->ref_min_steal = quarter < static_cast<u128>(40320) ? quarter : static_cast<u128>(40320);
    if (P->cfg.min_steal_log2 > 0) P->ref_min_steal = static_cast<u128>(std::llround(std::exp2(P->cfg.min_steal_log2)));
  }
  if (P->cfg.record_census) {
    P->census_cap = P->cfg.census_cap > 0 ? P->cfg.census_cap : (1 << 20);
    ck(cudaMalloc(&P->d_census, static_cast<size_t>(P->census_cap) * sizeof(unsigned long long)), "malloc census");
  }
  open_timeline(P);
  P->cfg.timeline_path = nullptr;  // the caller's string is not kept
  put(P, P->d_lgfact, lgf);
  upload_tables(P, T);
  reset_search(P);
}

// pbbgpu_config_t.split_mode (0 factoradic = reference, 1 live siblings, 2 live else
// factoradic) -> the device kernels' mode (1 factoradic, 2 live only, 0 hybrid)
int split_kind(int cfg_mode) {
  switch (cfg_mode) {
    case 1: return 2;
    case 2: return 0;
    default: return 1;
  }
}

// Large-n bounding launch over `count` batch slots (dead slots have d1 < 0): LB1 lane-per-node
// tables when the fixed jobs dominate (measured crossover on ta111 near f = n/2), else warp per
// node; LB2 warp per node when every node has f <= kBig2wFmax (shared memory sized for the
// largest f), else CTA per node. nodes = live slots, fsum their free jobs.
void launch_big_bounding(pbbgpu_pool* P, const BigBatchParams& G, int count, int fmax, long long fsum, int nodes) {
  const int n = P->n;
  if (P->big1 && fsum * 2 < static_cast<long long>(nodes) * n)
    P->big1g<<<std::min((count + 31) / 32, P->big1g_grid), kBig1gWarps * 32, P->big1g_smem, P->stream>>>(G, P->d_ptot);
  else if (P->big1)
    P->big1<<<std::min((count + kBig1Warps - 1) / kBig1Warps, P->big_grid), kBig1Warps * 32, P->big_smem, P->stream>>>(
        G, P->d_ptot);
  else if (P->big2w && P->packed32big && fmax <= kBig2wFmax) {
    const int fm = round_up(std::max(fmax, 4), 4);
    int w = kBig2wMaxWarps;
    while (w > 1 && static_cast<size_t>(big2w_smem_bytes(n, P->mp, P->m, fm, w)) > P->smem_optin) --w;
    const int grid = std::min(P->big2w_grid, (count + w - 1) / w);
    P->big2w<<<grid, w * 32, big2w_smem_bytes(n, P->mp, P->m, fm, w), P->stream>>>(G, P->d_ptot, P->d_packed32big, fm,
                                                                                   P->d_pm_scratch);
  } else {
    P->big<<<std::min(count, P->big_grid), kBigThreads, P->big_smem, P->stream>>>(G);
  }
  ck(cudaGetLastError(), "decompose_big launch");
}

// remaining work of every explorer (lens_kernel) before a steal phase / export / census
void launch_lens(pbbgpu_pool* P, int mode) {
  const int grid = std::max(1, std::min((P->K + kLensWarps - 1) / kLensWarps, 4 * P->num_sms));
  lens_kernel<<<grid, kLensWarps * 32, kLensWarps * P->L.gstride, P->stream>>>(P->L, P->d_state, P->K, P->d_lgfact,
                                                                                P->d_lens, mode);
}

void read_counters(pbbgpu_pool* P) {
  xfer(P, P->h_ctr, P->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, "ctr copy");
}

void set_device_best(pbbgpu_pool* P, int64_t v) {
  const int b = v >= INT_MAX ? INT_MAX : static_cast<int>(std::max<int64_t>(v, 0));
  xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, best), &b, sizeof(int), cudaMemcpyHostToDevice, "best copy");
  ck(cudaStreamSynchronize(P->stream), "sync");
}

// Harvest leaf improvements recorded by the last round(s).
void harvest(pbbgpu_pool* P) {
  const int cnt = std::min(P->h_ctr->imp_count, kImpCap);  // ring: all slots valid once it wrapped
  if (cnt > 0) {
    std::vector<ImpRecord> recs(static_cast<size_t>(cnt));
    xfer(P, recs.data(), P->d_imp, recs.size() * sizeof(ImpRecord), cudaMemcpyDeviceToHost, "imp copy");
    std::scoped_lock lk(P->best_mu);
    std::vector<int32_t> perm(static_cast<size_t>(P->n));
    for (const ImpRecord& r : recs) {
      if (r.mk >= P->best_sched_value) continue;
      for (int i = 0; i < P->n; ++i) perm[static_cast<size_t>(i)] = r.perm[i];
      int64_t mk = -1;
      try {
        mk = makespan_host(P->n, P->m, P->p.data(), perm.data());
      } catch (const std::exception&) {
        continue;  // torn record (ring overwrite race): skip
      }
      if (mk != r.mk) continue;
      P->best_sched_value = r.mk;
      P->best_sched = perm;
    }
    const int zero = 0;
    xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, imp_count), &zero, sizeof(int), cudaMemcpyHostToDevice, "imp reset");
  }
  std::scoped_lock lk(P->best_mu);
  P->best_value = std::min<int64_t>(P->best_value, P->h_ctr->best);
}

ExploreParams explore_params(pbbgpu_pool* P) {
  ExploreParams E{};
  E.L = P->L;
  E.state = P->d_state;
  E.K = P->K;
  E.steps = P->steps;
  E.prune_mode = P->cfg.disable_pruning ? 2 : (P->cfg.pinned ? 1 : 0);
  E.pinned_ub = static_cast<int>(std::min<int64_t>(P->best_value, INT_MAX));
  E.p32 = P->d_p32;
  E.ptot = P->d_ptot;
  E.npairs = P->npairs;
  E.pk = P->d_pk;
  E.pl = P->d_pl;
  E.order = P->d_ord;
  E.lag = P->d_lag;
  E.packed = P->d_packed;
  E.invord = P->d_invord;
  E.ctr = P->d_ctr;
  E.hist = P->d_hist;
  E.dhist = P->d_dhist;
  E.imp = P->d_imp;
  E.smem_inst_bytes = P->IL.bytes;
  E.budget_ns = static_cast<unsigned long long>(P->round_us * 1000.0);
  E.free_replay = P->cfg.steal_policy == 1 ? 1 : 0;
  E.census = P->d_census;
  E.census_cap = P->census_cap;

  return E;
}

template <class T>
T* scratch(pbbgpu_pool* P, int slot, size_t count) {
  const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
  if (P->scr_cap[slot] < bytes) {
    if (P->scr[slot]) {
      ck(cudaStreamSynchronize(P->stream), "sync");
      cudaFree(P->scr[slot]);
      P->scr[slot] = nullptr;
      P->scr_cap[slot] = 0;
    }
    const size_t cap = std::max(bytes, 2 * P->scr_cap[slot]);
    ck(cudaMalloc(&P->scr[slot], cap), "malloc scratch");
    P->scr_cap[slot] = cap;
  }
  return static_cast<T*>(P->scr[slot]);
}

void clear_explorers(pbbgpu_pool* P) {
  if (P->big_explore) big_clear_kernel<<<(P->K + 255) / 256, 256, 0, P->stream>>>(P->BL, P->d_state, P->K);
  else clear_kernel<<<(P->K + 255) / 256, 256, 0, P->stream>>>(P->L, P->d_state, P->K);
  ck(cudaGetLastError(), "clear_kernel");
}

// activity timeline (PoolConfig.timeline_path, explorer.cpp:71-85): header row, clock start
void open_timeline(pbbgpu_pool* P) {
  if (P->cfg.timeline_path && *P->cfg.timeline_path) {
    P->timeline = std::fopen(P->cfg.timeline_path, "w");
    if (!P->timeline) throw std::runtime_error(std::string("cannot open timeline file: ") + P->cfg.timeline_path);
    std::fputs("timestamp_ms,explorer_id,active,interval_length_log2\n", P->timeline);
  }
  P->t_start = std::chrono::steady_clock::now();
}

size_t state_stride(const pbbgpu_pool* P) { return P->big_explore ? static_cast<size_t>(P->BL.stride) : static_cast<size_t>(P->L.gstride); }
int state_off(const pbbgpu_pool* P) { return P->big_explore ? static_cast<int>(offsetof(BigHdr, state)) : static_cast<int>(offsetof(IvmHdr, state)); }

void assign_digits(pbbgpu_pool* P, const std::vector<int>& a, const std::vector<int>& b, const std::vector<uint8_t>& nf, const std::vector<int>& slots) {
  if (P->batch_only && !P->big_explore)
    throw StateError("pbbgpu: this n > 64 pool is bounding-only (decompose_batch); create it with explorers > 0 to explore");
  const int cnt = static_cast<int>(slots.size());
  if (cnt == 0) return;
  int* da = scratch<int>(P, 0, a.size());
  int* db = scratch<int>(P, 1, b.size());
  int* ds = scratch<int>(P, 2, slots.size());
  uint8_t* dn = scratch<uint8_t>(P, 3, nf.size());
  xfer(P, da, a.data(), a.size() * sizeof(int), cudaMemcpyHostToDevice, "copy");
  xfer(P, db, b.data(), b.size() * sizeof(int), cudaMemcpyHostToDevice, "copy");
  xfer(P, ds, slots.data(), slots.size() * sizeof(int), cudaMemcpyHostToDevice, "copy");
  xfer(P, dn, nf.data(), nf.size(), cudaMemcpyHostToDevice, "copy");
  if (P->big_explore) big_init_kernel<<<(cnt + 7) / 8, 256, 0, P->stream>>>(P->BL, P->d_state, da, db, dn, ds, cnt);
  else init_kernel<<<(cnt + 127) / 128, 128, 0, P->stream>>>(P->L, P->d_state, P->d_ptot, da, db, dn, ds, cnt);
  ck(cudaGetLastError(), "init_kernel");
  P->launches += 1;
  read_counters(P);
  // inits counter
  unsigned long long inits = P->h_ctr->inits + static_cast<unsigned long long>(cnt);
  xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, inits), &inits, sizeof(inits), cudaMemcpyHostToDevice, "copy");
}

std::vector<int> idle_slots(pbbgpu_pool* P) {
  int* d_cnt = P->d_wrk + 2 * P->K;
  list_idle_kernel<<<1, kStealThreads, 0, P->stream>>>(state_stride(P), state_off(P), P->d_state, P->K, P->d_wrk, d_cnt);
  ck(cudaGetLastError(), "list_idle_kernel");
  P->launches += 1;
  int cnt = 0;
  xfer(P, &cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, "idle count");
  std::vector<int> slots(static_cast<size_t>(cnt));
  if (cnt) xfer(P, slots.data(), P->d_wrk, slots.size() * sizeof(int), cudaMemcpyDeviceToHost, "idle slots");
  return slots;
}

int count_active_host(pbbgpu_pool* P) {
  int* d_cnt = P->d_wrk + 2 * P->K;
  list_idle_kernel<<<1, kStealThreads, 0, P->stream>>>(state_stride(P), state_off(P), P->d_state, P->K, P->d_wrk, d_cnt);
  ck(cudaGetLastError(), "list_idle_kernel");
  P->launches += 1;
  int cnt = 0;
  xfer(P, &cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, "idle count");
  return P->K - cnt;
}

GroupParams group_params(const pbbgpu_pool* P) {
  GroupParams G{};
  for (int q = 0; q < P->g_world; ++q) G.win[q] = P->g_peer[q];
  G.world = P->g_world;
  G.rank = P->g_rank;
  G.K = P->K;
  G.cap = P->g_cap;
  G.low = P->K / 2;
  G.share_best = P->cfg.pinned || P->cfg.disable_pruning ? 0 : 1;
  G.gs = P->d_gs;
  return G;
}

// ---- host views of explorer blocks (snapshot, timeline, work updates)
std::vector<unsigned char> download_state(pbbgpu_pool* P) {
  std::vector<unsigned char> st(static_cast<size_t>(P->K) * state_stride(P));
  xfer(P, st.data(), P->d_state, st.size(), cudaMemcpyDeviceToHost, "state copy");
  return st;
}

// Host view of one explorer block of either layout (n <= 64: IvmHdr, int8 digits and cells;
// n > 64: BigHdr, int16) -- the IVM semantics are the same, so snapshot / work update / timeline
// code reads both through this.
struct BlockRef {
  const pbbgpu_pool* P;
  unsigned char* b;
  bool big() const { return P->big_explore; }
  template <typename T>
  T* at(int off) const { return reinterpret_cast<T*>(b + off); }
  int state() const { return big() ? at<BigHdr>(0)->state : at<IvmHdr>(0)->state; }
  int level() const { return big() ? at<BigHdr>(0)->level : at<IvmHdr>(0)->level; }
  int nrep() const { return big() ? at<BigHdr>(0)->nrep : at<IvmHdr>(0)->nrep; }
  bool has_end() const { return big() ? at<BigHdr>(0)->has_end != 0 : at<IvmHdr>(0)->has_end != 0; }
  void set_empty() const {
    if (big()) at<BigHdr>(0)->state = kEmpty, at<BigHdr>(0)->level = -1;
    else at<IvmHdr>(0)->state = kEmpty, at<IvmHdr>(0)->level = -1;
  }
  int digit(int o_big, int o_small, int l) const { return big() ? at<int16_t>(o_big)[l] : at<int8_t>(o_small)[l]; }
  int V(int l) const { return digit(P->BL.o_v, P->L.o_v, l); }
  int E(int l) const { return digit(P->BL.o_end, P->L.o_end, l); }
  int T(int l) const { return digit(P->BL.o_tgt, P->L.o_tgt, l); }
  int cell(int l, int c) const { return digit(P->BL.o_cells, P->L.o_cells, tri_off(l, P->n) + c); }
  int dir(int l) const { return at<uint8_t>(big() ? P->BL.o_dir : P->L.o_dir)[l]; }
  void set_end(const std::vector<int>& e) const {
    for (int l = 0; l < P->n; ++l) {
      if (big()) at<int16_t>(P->BL.o_end)[l] = static_cast<int16_t>(e[static_cast<size_t>(l)]);
      else at<int8_t>(P->L.o_end)[l] = static_cast<int8_t>(e[static_cast<size_t>(l)]);
    }
    if (big()) at<BigHdr>(0)->has_end = 1;
    else at<IvmHdr>(0)->has_end = 1;
  }
};
BlockRef block_ref(const pbbgpu_pool* P, std::vector<unsigned char>& st, int i) {
  return BlockRef{P, st.data() + static_cast<size_t>(i) * state_stride(P)};
}

// Remaining work of an explorer block: [pos, end), pos the effective position (a parked
// explorer's consumed cell excluded, as pbbgpu_snapshot reports it; kInit: the replay target).
// False when nothing remains.
// raw = the reference's position() (zero-padded V, ivm.cpp:180-184) instead of the effective one.
bool block_span(const BlockRef& h, std::vector<int>& pos, std::vector<int>& end, bool& end_nf, bool raw = false) {
  const int n = h.P->n;
  if (h.state() == kEmpty) return false;
  const int state = h.state(), level = h.level();
  pos.assign(static_cast<size_t>(n), 0);
  end.assign(static_cast<size_t>(n), 0);
  for (int l = 0; l < n; ++l) pos[static_cast<size_t>(l)] = state == kInit ? h.T(l) : (l <= level ? h.V(l) : 0);
  if (!raw && state == kActive && level >= 0 && h.cell(level, h.V(level)) <= 0) {
    int l = level;
    for (; l >= 0; --l) {
      if (++pos[static_cast<size_t>(l)] <= n - 1 - l) break;
      pos[static_cast<size_t>(l)] = 0;
    }
    if (l < 0) return false;
  }
  end_nf = !h.has_end();
  for (int l = 0; l < n; ++l) end[static_cast<size_t>(l)] = end_nf ? 0 : h.E(l);
  if (!end_nf) {
    int cmp = 0;
    for (int l = 0; l < n && !cmp; ++l) cmp = pos[static_cast<size_t>(l)] < end[static_cast<size_t>(l)] ? -1 : (pos[static_cast<size_t>(l)] > end[static_cast<size_t>(l)] ? 1 : 0);
    if (cmp >= 0) return false;
  }
  return true;
}

// floor(log2(end - pos)) exactly (multi-word): to_decimal by Horner in base 2^32 limbs.
long exact_log2_len(const std::vector<int>& pos, const std::vector<int>& end, bool end_nf, int n) {
  auto big = [n](const std::vector<int>* d, bool nfact) {
    std::vector<uint32_t> v(1, 0);
    auto mul_add = [&v](uint32_t mul, uint32_t add) {
      uint64_t carry = add;
      for (uint32_t& w : v) {
        const uint64_t x = static_cast<uint64_t>(w) * mul + carry;
        w = static_cast<uint32_t>(x);
        carry = x >> 32;
      }
      if (carry) v.push_back(static_cast<uint32_t>(carry));
    };
    if (nfact) {
      v[0] = 1;
      for (int i = 2; i <= n; ++i) mul_add(static_cast<uint32_t>(i), 0);
    } else {
      for (int l = 0; l < n; ++l) mul_add(static_cast<uint32_t>(n - l), static_cast<uint32_t>((*d)[static_cast<size_t>(l)]));
    }
    return v;
  };
  std::vector<uint32_t> e = big(&end, end_nf), p = big(&pos, false);
  p.resize(std::max(p.size(), e.size()), 0);
  e.resize(p.size(), 0);
  int64_t borrow = 0;
  for (size_t i = 0; i < e.size(); ++i) {
    int64_t x = static_cast<int64_t>(e[i]) - p[i] - borrow;
    borrow = x < 0;
    if (borrow) x += int64_t(1) << 32;
    e[i] = static_cast<uint32_t>(x);
  }
  if (borrow) return -1;
  for (size_t i = e.size(); i-- > 0;)
    if (e[i]) return static_cast<long>(32 * i + 31 - __builtin_clz(e[i]));
  return -1;
}

// Factoradic midpoint of [pos, end) (end = n! when end_nf): pos + floor((end - pos) / 2), digit
// l of radix n - l, exact mixed-radix arithmetic (the host counterpart of split_point).
std::vector<int> factoradic_mid(const std::vector<int>& pos, const std::vector<int>& end, bool end_nf, int n) {
  std::vector<int> d(static_cast<size_t>(n));
  int borrow = 0;
  for (int l = n - 1; l >= 0; --l) {  // end - pos
    int x = (end_nf ? 0 : end[static_cast<size_t>(l)]) - pos[static_cast<size_t>(l)] - borrow;
    borrow = x < 0;
    if (borrow) x += n - l;
    d[static_cast<size_t>(l)] = x;
  }
  int rem = end_nf ? 1 - borrow : 0;  // the n! unit above digit 0
  for (int l = 0; l < n; ++l) {  // halve, most significant digit first
    const int cur = rem * (n - l) + d[static_cast<size_t>(l)];
    d[static_cast<size_t>(l)] = cur / 2;
    rem = cur % 2;
  }
  std::vector<int> m(static_cast<size_t>(n));
  int carry = 0;
  for (int l = n - 1; l >= 0; --l) {  // pos + half
    int x = pos[static_cast<size_t>(l)] + d[static_cast<size_t>(l)] + carry;
    carry = x >= n - l;
    if (carry) x -= n - l;
    m[static_cast<size_t>(l)] = x;
  }
  return m;
}

// sample_timeline (src/explorer.cpp:448-464): one row per explorer, >= 50 ms apart unless forced.
void sample_timeline(pbbgpu_pool* P, bool force) {
  const auto now = std::chrono::steady_clock::now();
  if (!force && P->sampled && now - P->t_last_sample < std::chrono::milliseconds(50)) return;
  P->sampled = true;
  P->t_last_sample = now;
  const long long ts = std::chrono::duration_cast<std::chrono::milliseconds>(now - P->t_start).count();
  std::vector<unsigned char> st = download_state(P);
  std::vector<int> pos, end;
  for (int i = 0; i < P->K; ++i) {
    const BlockRef h = block_ref(P, st, i);
    const bool active = h.state() != kEmpty;
    bool nf = false;
    long lg = -1;
    if (active && block_span(h, pos, end, nf, true)) lg = exact_log2_len(pos, end, nf, P->n);
    std::fprintf(P->timeline, "%lld,%d,%d,%ld\n", ts, i, active ? 1 : 0, lg);
  }
}

// Leaf improvements of the large-n explorers (BigImp ring), validated by makespan.
void harvest_big(pbbgpu_pool* P) {
  const int cnt = std::min(P->h_ctr->imp_count, kBigImpCap);
  if (cnt > 0) {
    std::vector<BigImp> recs(static_cast<size_t>(cnt));
    xfer(P, recs.data(), P->d_bimp, recs.size() * sizeof(BigImp), cudaMemcpyDeviceToHost, "imp copy");
    std::scoped_lock lk(P->best_mu);
    std::vector<int32_t> perm(static_cast<size_t>(P->n));
    for (const BigImp& r : recs) {
      if (r.mk >= P->best_sched_value) continue;
      for (int i = 0; i < P->n; ++i) perm[static_cast<size_t>(i)] = r.perm[i];
      int64_t mk = -1;
      try {
        mk = makespan_host(P->n, P->m, P->p.data(), perm.data());
      } catch (const std::exception&) {
        continue;  // torn record
      }
      if (mk != r.mk) continue;
      P->best_sched_value = r.mk;
      P->best_sched = perm;
    }
    const int zero = 0;
    xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, imp_count), &zero, sizeof(int), cudaMemcpyHostToDevice, "imp reset");
  }
  std::scoped_lock lk(P->best_mu);
  P->best_value = std::min<int64_t>(P->best_value, P->h_ctr->best);
}

// run_round of the n > 64 explorer pool: rounds of big_steps select -> bound -> branch steps,
// then the steal pipeline (explore_big.cuh). Each step reads back 16 bytes (the batch's largest
// and total free-job counts) to pick the bounding kernel.
int big_run_round(pbbgpu_pool* P) {
  const int64_t offer = P->pending_offer.exchange(INT64_MAX);
  if (offer < P->best_value) {
    {
      std::scoped_lock lk(P->best_mu);
      P->best_value = offer;
    }
    if (!P->cfg.pinned) set_device_best(P, offer);
  }
  const int n = P->n;
  const int prune_mode = P->cfg.disable_pruning ? 2 : (P->cfg.pinned ? 1 : 0);
  BigStepParams BS{};
  BS.L = P->BL;
  BS.state = P->d_state;
  BS.K = P->K;
  BS.perms = P->d_bperm;
  BS.d1 = P->d_bd1;
  BS.d2 = P->d_bd2;
  BS.kind = P->d_bkind;
  BS.fstat = P->d_bfstat;
  BS.ctr = P->d_ctr;
  BS.hist = P->d_hist;
  BS.dhist = P->d_dhist;
  BS.dir = P->d_bdir;
  BS.pruned = P->d_bpr;
  BS.lb_fwd = P->d_blf;
  BS.prune_mode = prune_mode;
  BS.imp = P->d_bimp;
  BigBatchParams G{};
  G.n = n;
  G.m = P->m;
  G.mp = P->mp;
  G.npairs = P->npairs;
  G.perms = P->d_bperm;
  G.d1 = P->d_bd1;
  G.d2 = P->d_bd2;
  G.count = P->K;
  G.p32 = P->d_p32;
  G.pk = P->d_pk;
  G.pl = P->d_pl;
  G.packed = P->d_packed64;
  G.inv16 = P->d_inv16;
  G.scratch = P->d_big_scratch;
  G.child_lb = P->d_blb;
  G.lb_fwd = P->d_blf;
  G.lb_bwd = P->d_blbw;
  G.dir = P->d_bdir;
  G.pruned = P->d_bpr;
  StealParams S{};
  S.K = P->K;
  S.ctr = P->d_ctr;
  S.thief = P->d_wrk;
  S.victim = P->d_wrk + P->K;
  S.plan = P->d_wrk + 2 * P->K + 2;
  S.min_log2 = static_cast<float>(P->cfg.min_steal_log2 > 0 ? P->cfg.min_steal_log2 : std::log2(40320.0));
  S.lgfact = P->d_lgfact;
  S.trigger = static_cast<float>(P->cfg.steal_trigger > 0 ? P->cfg.steal_trigger : 1.0);
  S.lens = P->d_lens;
  S.max_split = P->cfg.max_split > 0 ? std::min(P->cfg.max_split, 63) : 4;
  const int blocks = (P->K + 7) / 8;
  for (int r = 0; r < P->rounds_per_sync; ++r) {
    ck(cudaEventRecord(P->evs[3 * r], P->stream), "event");
    for (int st = 0; st < P->big_steps; ++st) {
      // the pruning bound of this step: the host's best (device improvements of this round
      // reach it at the next synchronization; a higher bound only prunes less)
      int64_t inc = P->cfg.disable_pruning ? INT_MAX : (P->cfg.pinned ? P->pinned_ub : P->best_value);
      G.incumbent = static_cast<int>(std::min<int64_t>(inc, INT_MAX));
      ck(cudaMemsetAsync(P->d_bfstat, 0, 4 * sizeof(int), P->stream), "memset");
      big_select_kernel<8><<<blocks, 256, 0, P->stream>>>(BS);
      ck(cudaGetLastError(), "big_select_kernel");
      ck(cudaMemcpyAsync(P->h_bfstat, P->d_bfstat, 4 * sizeof(int), cudaMemcpyDeviceToHost, P->stream), "fstat");
      ck(cudaStreamSynchronize(P->stream), "sync");
      P->d2h_bytes += 4 * sizeof(int);
      P->launches += 1;
      if (P->h_bfstat[1] == 0) break;
      launch_big_bounding(P, G, P->K, P->h_bfstat[0], P->h_bfstat[2], P->h_bfstat[1]);
      big_branch_kernel<8><<<blocks, 256, 0, P->stream>>>(BS);
      ck(cudaGetLastError(), "big_branch_kernel");
      P->launches += 2;
    }
    ck(cudaEventRecord(P->evs[3 * r + 1], P->stream), "event");
    big_lens_kernel<<<(P->K + 127) / 128, 128, 0, P->stream>>>(P->BL, P->d_state, P->K, P->d_lgfact, P->d_lens);
    steal_kernel<<<1, kStealThreads, 0, P->stream>>>(S);
    big_split_thieves_kernel<<<(P->K + 127) / 128, 128, 0, P->stream>>>(P->BL, P->d_state, S.thief, S.victim, S.plan,
                                                                         P->d_ctr);
    big_split_victims_kernel<<<(P->K + 127) / 128, 128, 0, P->stream>>>(P->BL, P->d_state, S.victim, S.plan);
    ck(cudaGetLastError(), "big steal pipeline");
    ck(cudaEventRecord(P->evs[3 * r + 2], P->stream), "event");
    P->launches += 4;
  }
  read_counters(P);
  for (int r = 0; r < P->rounds_per_sync; ++r) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, P->evs[3 * r], P->evs[3 * r + 1]), "elapsed");
    P->kernel_ms += ms;
    ck(cudaEventElapsedTime(&ms, P->evs[3 * r + 1], P->evs[3 * r + 2]), "elapsed");
    P->steal_ms += ms;
  }
  P->rounds += static_cast<uint64_t>(P->rounds_per_sync);
  harvest_big(P);
  P->last_active = P->h_ctr->active;
  if (P->timeline) sample_timeline(P, P->h_ctr->active == 0);
  return P->h_ctr->active;
}

int run_round(pbbgpu_pool* P) {
  if (P->big_explore) return big_run_round(P);
  if (P->batch_only)
    throw StateError("pbbgpu: this n > 64 pool is bounding-only (decompose_batch); create it with explorers > 0 to explore");
  const int64_t offer = P->pending_offer.exchange(INT64_MAX);
  if (offer < P->best_value) {
    {
      std::scoped_lock lk(P->best_mu);
      P->best_value = offer;
    }
    if (!P->cfg.pinned) set_device_best(P, offer);
  }
  ExploreParams E = explore_params(P);
  if (P->cfg.pinned) E.pinned_ub = static_cast<int>(std::min<int64_t>(P->pinned_ub, INT_MAX));
  // adaptive round length: while many explorers are idle (ramp-up, tail) the steal phase is
  // what matters, so rounds are 4x shorter; when (almost) all are busy, full-length rounds
  if (E.budget_ns && P->rounds > 0 && P->last_active * 4 < P->K * 3)
    E.budget_ns = std::max<unsigned long long>(E.budget_ns / 4, 250000ull);
  StealParams S{};
  S.L = P->L;
  S.state = P->d_state;
  S.K = P->K;
  S.ptot = P->d_ptot;
  S.ctr = P->d_ctr;
  S.thief = P->d_wrk;
  S.victim = P->d_wrk + P->K;
  S.plan = P->d_wrk + 2 * P->K + 2;
  S.min_log2 = static_cast<float>(P->cfg.min_steal_log2 > 0 ? P->cfg.min_steal_log2 : std::log2(40320.0));
  S.lgfact = P->d_lgfact;
  S.trigger = static_cast<float>(P->cfg.steal_trigger > 0 ? P->cfg.steal_trigger : 1.0);
  S.lens = P->d_lens;
  S.max_split = P->cfg.max_split > 0 ? std::min(P->cfg.max_split, 63) : 4;
  S.split_mode = split_kind(P->cfg.split_mode);
  if (P->cfg.steal_policy != 1 && P->bound == kLB2 && P->G == 32 && P->n <= 32) {  // kLensInKernel
    E.lens = P->d_lens;
    E.lgfact = P->d_lgfact;
    E.lens_mode = S.split_mode;
  }
  // several (explore, steal) rounds back to back per host synchronization: the rounds are
  // device-timed, and a round after exhaustion costs only the state copy of an empty launch
  const int R = P->rounds_per_sync;
  StealRefParams SR{};
  if (P->cfg.steal_policy == 1) {
    SR.L = P->L;
    SR.state = P->d_state;
    SR.K = P->K;
    SR.ptot = P->d_ptot;
    SR.ctr = P->d_ctr;
    SR.len = P->d_ref_len;
    SR.flags = P->d_ref_flags;
    SR.pairs = P->d_ref_pairs;
    SR.order = P->d_ref_pairs + 2 * P->K;
    SR.min_steal = P->ref_min_steal;
  }
  for (int r = 0; r < R; ++r) {
    ck(cudaEventRecord(P->evs[3 * r], P->stream), "event");
    P->efn<<<P->grid, P->block, P->smem, P->stream>>>(E);
    ck(cudaGetLastError(), "explore_kernel launch");
    ck(cudaEventRecord(P->evs[3 * r + 1], P->stream), "event");
    if (P->cfg.steal_policy == 1) {  // the reference's steal_phase (explorer.cpp:251-340)
      steal_ref_kernel<<<1, kRefThreads, 0, P->stream>>>(SR);
      ck(cudaGetLastError(), "steal_ref_kernel launch");
      ck(cudaEventRecord(P->evs[3 * r + 2], P->stream), "event");
      P->launches += 2;
      continue;
    }
    if (!E.lens) launch_lens(P, S.split_mode);  // else written by the explore kernel (kLensInKernel)
    steal_kernel<<<1, kStealThreads, 0, P->stream>>>(S);
    ck(cudaGetLastError(), "steal_kernel launch");
    split_kernel<<<P->split_grid, kSplitWarps * 32, kSplitWarps * P->L.gstride, P->stream>>>(
        P->L, P->d_state, P->d_ptot, S.thief, S.victim, S.plan, P->d_ctr, S.split_mode);
    ck(cudaGetLastError(), "split_kernel launch");
    if (P->g_open) {  // inter-GPU exchange over peer memory (no host involvement)
      ck(cudaEventRecord(P->gev[r], P->stream), "event");
      const GroupParams G = group_params(P);
      group_exchange_kernel<<<1, kStealThreads, 0, P->stream>>>(P->L, P->d_state, P->d_ptot, P->d_ctr, G);
      ck(cudaGetLastError(), "group_exchange_kernel launch");
      launch_lens(P, S.split_mode);
      ck(cudaGetLastError(), "lens_kernel launch");
      group_export_kernel<<<1, kStealThreads, 0, P->stream>>>(S, G);
      ck(cudaGetLastError(), "group_export_kernel launch");
      P->launches += 3;
    }
    ck(cudaEventRecord(P->evs[3 * r + 2], P->stream), "event");
    P->launches += E.lens ? 3 : 4;
  }
  read_counters(P);
  for (int r = 0; r < R; ++r) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, P->evs[3 * r], P->evs[3 * r + 1]), "elapsed");
    P->kernel_ms += ms;
    ck(cudaEventElapsedTime(&ms, P->evs[3 * r + 1], P->evs[3 * r + 2]), "elapsed");
    P->steal_ms += ms;
    if (P->g_open) {
      ck(cudaEventElapsedTime(&ms, P->gev[r], P->evs[3 * r + 2]), "elapsed");
      P->group_ms += ms;
      P->group_rounds += 1;
    }
  }
  P->rounds += static_cast<uint64_t>(R);
  harvest(P);
  P->last_active = P->h_ctr->active;
  if (P->timeline) sample_timeline(P, P->h_ctr->active == 0);
  return P->h_ctr->active;
}

int set_err(const std::exception& e) {
  g_last_error = e.what();
  if (dynamic_cast<const CudaError*>(&e)) return PBBGPU_ERR_CUDA;
  if (dynamic_cast<const CapacityError*>(&e)) return PBBGPU_ERR_CAPACITY;
  if (dynamic_cast<const StateError*>(&e)) return PBBGPU_ERR_STATE;
  if (dynamic_cast<const std::logic_error*>(&e)) return PBBGPU_ERR_ARG;
  return PBBGPU_ERR_CUDA;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PBBGPU_OK;
  } catch (const std::exception& e) {
    return set_err(e);
  }
}

void check_digits(int n, const uint16_t* d) {
  for (int l = 0; l < n; ++l)
    if (d[l] > n - 1 - l) throw std::invalid_argument("factoradic digit out of radix at level " + std::to_string(l));
}

}  // namespace

// ------------------------------------------------------------------ C-ABI

void pbbgpu_internal_set_error(const char* msg) { g_last_error = msg ? msg : ""; }

extern "C" {

const char* pbbgpu_last_error(void) { return g_last_error.c_str(); }

int pbbgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int pbbgpu_int32_peak(int device, double* ops_per_s) {
  return guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw CudaError("pbbgpu: no CUDA device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "props");
    int* d_in = nullptr;
    int* d_out = nullptr;
    int h_in[24];
    for (int i = 0; i < 24; ++i) h_in[i] = (i * 7919) % 97 - 40;
    ck(cudaMalloc(&d_in, sizeof(h_in)), "malloc");
    ck(cudaMalloc(&d_out, 1 << 20), "malloc");
    ck(cudaMemcpy(d_in, h_in, sizeof(h_in), cudaMemcpyHostToDevice), "copy");
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    int32_peak_kernel<<<blocks, threads>>>(d_in, d_out, 256);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      ck(cudaEventRecord(a), "event");
      int32_peak_kernel<<<blocks, threads>>>(d_in, d_out, iters);
      ck(cudaEventRecord(b), "event");
      ck(cudaEventSynchronize(b), "sync");
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
      best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d_in);
    cudaFree(d_out);
    const double ops = static_cast<double>(blocks) * threads * iters * 8 * 4;  // 2 x (add, max)
    *ops_per_s = ops / (best * 1e-3);
  });
}

int pbbgpu_taillard(int n, int m, int32_t seed, int32_t* p_out) {
  return guarded([&] { taillard(n, m, seed, p_out); });
}

int pbbgpu_taillard_named(const char* name, int* n, int* m, int32_t* p_out) {
  return guarded([&] {
    const std::string s = name ? name : "";
    if (s.size() != 5 || (s.rfind("ta", 0) != 0 && s.rfind("Ta", 0) != 0)) throw std::invalid_argument("expected instance name of the form ta001..ta120");
    const int idx = std::atoi(s.c_str() + 2);
    if (idx < 1 || idx > 120) throw std::invalid_argument("instance number out of range 1..120");
    const TaClass& c = kTa[(idx - 1) / 10];
    *n = c.n;
    *m = c.m;
    if (p_out) taillard(c.n, c.m, c.seeds[(idx - 1) % 10], p_out);
  });
}

int64_t pbbgpu_makespan(int n, int m, const int32_t* p, const int32_t* perm) {
  try {
    return makespan_host(n, m, p, perm);
  } catch (const std::exception& e) {
    set_err(e);
    return -1;
  }
}

int64_t pbbgpu_neh(int n, int m, const int32_t* p, int32_t* perm_out) {
  try {
    return neh_host(n, m, p, perm_out);
  } catch (const std::exception& e) {
    set_err(e);
    return -1;
  }
}

int pbbgpu_create(int n, int m, const int32_t* p, int bound_kind, const pbbgpu_config_t* cfg, pbbgpu_pool** out) {
  *out = nullptr;
  pbbgpu_pool* P = new pbbgpu_pool();
  TraceScope ts("create");
  const int rc = guarded([&] { pool_init(P, n, m, p, bound_kind, cfg); });
  if (rc != PBBGPU_OK) {
    P->release();
    delete P;
    return rc;
  }
  *out = P;
  return PBBGPU_OK;
}

void pbbgpu_destroy(pbbgpu_pool* P) {
  if (!P) return;
  P->release();
  delete P;
}

int pbbgpu_load_instance(pbbgpu_pool* P, const int32_t* p) {
  return guarded([&] {
    if (!P || !p) throw std::invalid_argument("pbbgpu_load_instance: null argument");
    std::vector<int32_t> padded = pad_machines(P->n, P->m_real, P->m, p);
    if (validate_times(P->n, P->m, padded.data(), P->bound) && !P->wide && !P->batch_only)
      throw CapacityError("pbbgpu_load_instance: this instance needs 32-bit explorer tables ((n+m)*max p >= 2^16); create a new pool");
    const HostTables T = build_tables(P->n, P->m_real, P->m, P->bound, p, P->batch_only);
    if (P->bound == kLB2 && !P->batch_only && P->G == 32 && !T.packable)
      throw CapacityError("pbbgpu_load_instance: this instance's LB2 tables do not pack into 31 bits; create a new pool");
    ck(cudaStreamSynchronize(P->stream), "sync");
    P->p = std::move(padded);
    upload_tables(P, T);
    reset_search(P);
  });
}

int pbbgpu_K(const pbbgpu_pool* P) { return P ? P->K : 0; }

int pbbgpu_pool_shape(const pbbgpu_pool* P, int* n, int* m) {
  return guarded([&] {
    if (!P) throw std::invalid_argument("null pool");
    *n = P->n;
    *m = P->m_real;
  });
}

int pbbgpu_pool_times(const pbbgpu_pool* P, int32_t* p) {
  return guarded([&] {
    if (!P) throw std::invalid_argument("null pool");
    for (int j = 0; j < P->n; ++j)
      for (int k = 0; k < P->m_real; ++k) p[static_cast<size_t>(j) * P->m_real + k] = P->p[static_cast<size_t>(j) * P->m + k];
  });
}

int pbbgpu_set_initial_bound(pbbgpu_pool* P, int64_t ub, const int32_t* sched, int len) {
  return guarded([&] {
    if (ub <= 0) throw std::invalid_argument("incumbent must be positive");
    {
      std::scoped_lock lk(P->best_mu);
      P->best_value = ub;
      if (sched && len == P->n) {
        P->best_sched.assign(sched, sched + len);
        P->best_sched_value = ub;
      } else {
        P->best_sched.clear();
        P->best_sched_value = INT64_MAX;
      }
      P->pinned_ub = ub;
      P->improvement_mark = ub;  // explorer.cpp:112-120
      // a stale offer (e.g. a MIN exchanged at the end of the previous solve) must not lower
      // the new bound below a value that has no schedule behind it
      P->pending_offer.store(INT64_MAX);
    }
    set_device_best(P, ub);
  });
}

int pbbgpu_assign(pbbgpu_pool* P, const uint16_t* a, const uint16_t* b, const uint8_t* nf, int count) {
  return guarded([&] {
    if (count < 0 || count > P->K) throw std::invalid_argument("more intervals than explorers");
    if (count == 0) return;
    const int n = P->n;
    const std::vector<int> idle = idle_slots(P);
    if (static_cast<int>(idle.size()) < count) throw CapacityError("not enough idle explorers for the assignment");
    std::vector<int> da(static_cast<size_t>(count) * n), db(static_cast<size_t>(count) * n, 0), slots(static_cast<size_t>(count));
    std::vector<uint8_t> dn(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
      check_digits(n, a + static_cast<size_t>(i) * n);
      const bool inf = nf && nf[i];
      if (!inf) check_digits(n, b + static_cast<size_t>(i) * n);
      for (int l = 0; l < n; ++l) {
        da[static_cast<size_t>(i) * n + l] = a[static_cast<size_t>(i) * n + l];
        if (!inf) db[static_cast<size_t>(i) * n + l] = b[static_cast<size_t>(i) * n + l];
      }
      dn[static_cast<size_t>(i)] = inf ? 1 : 0;
      slots[static_cast<size_t>(i)] = idle[static_cast<size_t>(i)];
    }
    assign_digits(P, da, db, dn, slots);
  });
}

// ---- breadth-first seeding (planning only)
// The top of the tree is expanded level by level with the batch bounding kernel (the same
// decompose as the explorers: rows in ascending job order, MinMin direction, prune at the
// seeding bound) until the live frontier holds at least `target` nodes. [0, n!) is then cut
// at frontier nodes into <= target intervals, each starting at a live subtree, instead of
// n!/target-equal ranges that mostly start inside pruned subtrees and leave the explorers
// to find the work by stealing (the ramp-up of a short proof). Only the cut points come
// from the seeding: the explorers decompose everything in their intervals and the unique
// count rule holds for any partition, so counts are unchanged.
namespace {
void batch_bound(pbbgpu_pool* P, const std::vector<int>& perms, const std::vector<int>& d1, const std::vector<int>& d2,
                 int prune, std::vector<uint8_t>& pruned, std::vector<uint8_t>& dir) {
  const int n = P->n, count = static_cast<int>(d1.size());
  const size_t cn = static_cast<size_t>(count) * n;
  int* dp = scratch<int>(P, 0, cn);
  int* dd1 = scratch<int>(P, 1, count);
  int* dd2 = scratch<int>(P, 2, count);
  int* dlb = scratch<int>(P, 3, cn);
  int* dlf = scratch<int>(P, 4, cn);
  int* dlbw = scratch<int>(P, 5, cn);
  uint8_t* ddir = scratch<uint8_t>(P, 6, count);
  uint8_t* dpr = scratch<uint8_t>(P, 7, cn);
  xfer(P, dp, perms.data(), cn * sizeof(int), cudaMemcpyHostToDevice, "copy");
  xfer(P, dd1, d1.data(), count * sizeof(int), cudaMemcpyHostToDevice, "copy");
  xfer(P, dd2, d2.data(), count * sizeof(int), cudaMemcpyHostToDevice, "copy");
  BatchParams B{};
  B.L = P->L;
  B.perms = dp;
  B.d1 = dd1;
  B.d2 = dd2;
  B.count = count;
  B.incumbent = prune;
  B.p32 = P->d_p32;
  B.npairs = P->npairs;
  B.pk = P->d_pk;
  B.pl = P->d_pl;
  B.order = P->d_ord;
  B.lag = P->d_lag;
  B.packed = P->d_packed;
  B.invord = P->d_invord;
  B.child_lb = dlb;
  B.lb_fwd = dlf;
  B.lb_bwd = dlbw;
  B.dir = ddir;
  B.pruned = dpr;
  const int NG = P->block / P->G;
  const int grid = std::min((count + NG - 1) / NG, P->num_sms * 8);
  P->bfn<<<grid, P->block, P->smem, P->stream>>>(B);
  ck(cudaGetLastError(), "decompose_batch launch");
  P->launches += 1;
  pruned.resize(cn);
  dir.resize(static_cast<size_t>(count));
  xfer(P, pruned.data(), dpr, cn, cudaMemcpyDeviceToHost, "copy");
  xfer(P, dir.data(), ddir, static_cast<size_t>(count), cudaMemcpyDeviceToHost, "copy");
}

// Sorted cut points (digit vectors, n each, the first cut > 0) of a <= target interval partition.
std::vector<std::vector<int>> bfs_cuts(pbbgpu_pool* P, int prune, int target) {
  TraceScope ts("seed: breadth-first cuts");
  const int n = P->n;
  target = std::max(target, 1);
  // frontier nodes: digits (n each, zero padded) and perm = sigma1 ++ free ascending ++ sigma2
  std::vector<int> dig(static_cast<size_t>(n) * n, 0), perm(static_cast<size_t>(n) * n), d1v(static_cast<size_t>(n), 1),
      d2v(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j) {  // the root's children: never bounded, all live, Forward
    dig[static_cast<size_t>(j) * n] = j;
    int* pp = &perm[static_cast<size_t>(j) * n];
    int t = 0;
    pp[t++] = j;
    for (int x = 0; x < n; ++x)
      if (x != j) pp[t++] = x;
  }
  auto cuts_of = [&](const std::vector<int>& dg, long long F) {
    const long long G = std::min<long long>(F, target);
    std::vector<std::vector<int>> cuts;
    for (long long g = 1; g < G; ++g) {
      const size_t idx = static_cast<size_t>(g * F / G);
      cuts.emplace_back(dg.begin() + static_cast<long>(idx * n), dg.begin() + static_cast<long>((idx + 1) * n));
    }
    return cuts;
  };
  int depth = 1;
  // host memory of the next frontier (digits + perm, 8 bytes per job) capped at 64 MB
  const size_t kMaxChildren = (size_t(64) << 20) / (static_cast<size_t>(n) * 8);
  while (static_cast<int>(d1v.size()) < target && n - depth >= 3 &&
         d1v.size() * static_cast<size_t>(n - depth) <= kMaxChildren) {
    std::vector<uint8_t> pruned, dir;
    batch_bound(P, perm, d1v, d2v, prune, pruned, dir);
    const int cnt = static_cast<int>(d1v.size());
    // live children per node (prefix offsets), then either the next frontier or, when it
    // reaches the target, only the digits of the cut nodes
    std::vector<long long> off(static_cast<size_t>(cnt) + 1, 0);
    for (int i = 0; i < cnt; ++i) {
      const int f = n - d1v[static_cast<size_t>(i)] - d2v[static_cast<size_t>(i)];
      int live = 0;
      for (int c = 0; c < f; ++c) live += !pruned[static_cast<size_t>(i) * n + c];
      off[static_cast<size_t>(i) + 1] = off[static_cast<size_t>(i)] + live;
    }
    const long long F = off[static_cast<size_t>(cnt)];
    if (F == 0) break;  // everything below this level is pruned: keep this frontier
    auto child_digits = [&](long long k, int* out) {  // digits of live child number k
      const int i = static_cast<int>(std::upper_bound(off.begin(), off.end(), k) - off.begin()) - 1;
      long long r = k - off[static_cast<size_t>(i)];
      int c = 0;
      for (;; ++c)
        if (!pruned[static_cast<size_t>(i) * n + c] && r-- == 0) break;
      for (int l = 0; l < n; ++l) out[l] = l == depth ? c : dig[static_cast<size_t>(i) * n + l];
    };
    if (F >= target) {
      const long long G = target;
      std::vector<std::vector<int>> cuts;
      for (long long g = 1; g < G; ++g) {
        std::vector<int> v(static_cast<size_t>(n));
        child_digits(g * F / G, v.data());
        cuts.push_back(std::move(v));
      }
      return cuts;
    }
    std::vector<int> ndig(static_cast<size_t>(F) * n), nperm(static_cast<size_t>(F) * n), nd1(static_cast<size_t>(F)),
        nd2(static_cast<size_t>(F));
    long long k = 0;
    for (int i = 0; i < cnt; ++i) {
      const int a = d1v[static_cast<size_t>(i)], b = d2v[static_cast<size_t>(i)], f = n - a - b;
      const int* pp = &perm[static_cast<size_t>(i) * n];
      const bool fwd = dir[static_cast<size_t>(i)] == kFwd;
      for (int c = 0; c < f; ++c) {
        if (pruned[static_cast<size_t>(i) * n + c]) continue;
        int* dg = &ndig[static_cast<size_t>(k) * n];
        for (int l = 0; l < n; ++l) dg[l] = l == depth ? c : dig[static_cast<size_t>(i) * n + l];
        int* np = &nperm[static_cast<size_t>(k) * n];
        const int j = pp[a + c];
        int t = 0;
        for (int x = 0; x < a; ++x) np[t++] = pp[x];
        if (fwd) np[t++] = j;
        for (int x = 0; x < f; ++x)
          if (x != c) np[t++] = pp[a + x];
        if (!fwd) np[t++] = j;
        for (int x = n - b; x < n; ++x) np[t++] = pp[x];
        nd1[static_cast<size_t>(k)] = a + fwd;
        nd2[static_cast<size_t>(k)] = b + !fwd;
        ++k;
      }
    }
    dig.swap(ndig);
    perm.swap(nperm);
    d1v.swap(nd1);
    d2v.swap(nd2);
    ++depth;
  }
  return cuts_of(dig, static_cast<long long>(d1v.size()));
}
}  // namespace

int pbbgpu_seed(pbbgpu_pool* P, int64_t bound, int first, int stride, int total) {
  return guarded([&] {
    if (P->batch_only) throw StateError("pbbgpu: bounding-only pool has no explorers");
    if (stride < 1 || first < 0 || first >= stride) throw std::invalid_argument("bad seed rank/stride");
    if (total <= 0) total = stride * P->K;
    const int n = P->n;
    int prune = static_cast<int>(std::min<int64_t>(std::max<int64_t>(bound, 1), INT_MAX));
    if (P->cfg.disable_pruning) prune = INT_MAX;
    const std::vector<std::vector<int>> cuts = bfs_cuts(P, prune, total);
    const int I = static_cast<int>(cuts.size()) + 1;  // intervals [0, c1), [c1, c2), ..., [c_last, n!)
    std::vector<int> a, b, slots;
    std::vector<uint8_t> nf;
    for (int i = first; i < I; i += stride) {
      if (static_cast<int>(slots.size()) >= P->K) throw CapacityError("pbbgpu_seed: more intervals than explorers");
      for (int l = 0; l < n; ++l) a.push_back(i == 0 ? 0 : cuts[static_cast<size_t>(i - 1)][static_cast<size_t>(l)]);
      const bool last = i == I - 1;
      for (int l = 0; l < n; ++l) b.push_back(last ? 0 : cuts[static_cast<size_t>(i)][static_cast<size_t>(l)]);
      nf.push_back(last ? 1 : 0);
      slots.push_back(static_cast<int>(slots.size()));
    }
    clear_explorers(P);
    P->launches += 1;
    assign_digits(P, a, b, nf, slots);
  });
}

int pbbgpu_assign_split_range(pbbgpu_pool* P, int first, int count, int total) {
  return pbbgpu_assign_split_strided(P, first, 1, count, total);
}

int pbbgpu_assign_split_strided(pbbgpu_pool* P, int first, int stride, int count, int total) {
  return guarded([&] {
    if (total <= 0) total = P->K;
    if (count < 0) count = total;
    if (stride < 1) throw std::invalid_argument("bad split stride");
    if (first < 0 || count > P->K || (count > 0 && first + static_cast<int64_t>(count - 1) * stride >= total))
      throw std::invalid_argument("bad split range");
    const int n = P->n;
    // floor(i * n! / total) in factoradic, digit by digit: d_l = floor(r (n-l) / C),
    // r <- r (n-l) mod C (exact rational expansion, no big integers needed)
    auto digits_of = [&](int64_t i, int* out) {
      int64_t r = i;
      for (int l = 0; l < n; ++l) {
        r *= (n - l);
        out[l] = static_cast<int>(r / total);
        r %= total;
      }
    };
    std::vector<int> a(static_cast<size_t>(count) * n), b(static_cast<size_t>(count) * n, 0), slots(static_cast<size_t>(count));
    std::vector<uint8_t> nf(static_cast<size_t>(count), 0);
    for (int c = 0; c < count; ++c) {
      const int i = first + c * stride;
      digits_of(i, &a[static_cast<size_t>(c) * n]);
      if (i + 1 < total) digits_of(i + 1, &b[static_cast<size_t>(c) * n]);
      else nf[static_cast<size_t>(c)] = 1;
      slots[static_cast<size_t>(c)] = c;
    }
    clear_explorers(P);
    P->launches += 1;
    assign_digits(P, a, b, nf, slots);
  });
}

int pbbgpu_assign_split(pbbgpu_pool* P, int pieces) {
  if (pieces <= 0) pieces = P ? P->K : 0;
  return pbbgpu_assign_split_range(P, 0, pieces, pieces);
}

int pbbgpu_export(pbbgpu_pool* P, int max_count, uint16_t* a_out, uint16_t* b_out, uint8_t* nf_out, int* count) {
  return guarded([&] {
    *count = 0;
    if (max_count <= 0) return;
    if (P->batch_only && !P->big_explore) throw StateError("pbbgpu: bounding-only pool has no explorers");
    const int n = P->n;
    const int want = std::min(max_count, P->K);
    if (P->big_explore) {
      // n > 64 explorers (int16 IVMs in HBM): on the host through BlockRef -- the longest
      // remaining intervals (exact log2 lengths) are halved at their factoradic midpoint, the
      // explorer keeps [pos, mid) (shrink_end) and [mid, end) is exported
      std::vector<unsigned char> st = download_state(P);
      struct Cand {
        long lg;
        int i;
      };
      std::vector<Cand> cands;
      std::vector<int> pos, end;
      bool nf = false;
      for (int i = 0; i < P->K; ++i) {
        const BlockRef h = block_ref(P, st, i);
        if (h.state() != kActive) continue;  // replaying explorers are not split
        if (!block_span(h, pos, end, nf)) continue;
        const long lg = exact_log2_len(pos, end, nf, n);
        if (lg >= 1) cands.push_back({lg, i});
      }
      std::stable_sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) { return x.lg > y.lg; });
      int c = 0;
      for (const Cand& cd : cands) {
        if (c >= want) break;
        const BlockRef h = block_ref(P, st, cd.i);
        block_span(h, pos, end, nf);
        const std::vector<int> mid = factoradic_mid(pos, end, nf, n);
        if (mid == pos) continue;  // a single leaf left: nothing to give
        for (int l = 0; l < n; ++l) {
          a_out[static_cast<size_t>(c) * n + l] = static_cast<uint16_t>(mid[static_cast<size_t>(l)]);
          b_out[static_cast<size_t>(c) * n + l] = static_cast<uint16_t>(nf ? 0 : end[static_cast<size_t>(l)]);
        }
        nf_out[c] = nf ? 1 : 0;
        h.set_end(mid);
        ++c;
      }
      if (c) xfer(P, P->d_state, st.data(), st.size(), cudaMemcpyHostToDevice, "state copy");
      *count = c;
      return;
    }
    int* d_dig = scratch<int>(P, 0, static_cast<size_t>(want + 64) * 2 * n);
    uint8_t* d_nf = scratch<uint8_t>(P, 1, static_cast<size_t>(want + 64));
    int* d_cnt = scratch<int>(P, 2, 1);
    StealParams S{};
    S.L = P->L;
    S.state = P->d_state;
    S.K = P->K;
    S.ptot = P->d_ptot;
    S.ctr = P->d_ctr;
    S.thief = P->d_wrk;
    S.victim = P->d_wrk + P->K;
    S.min_log2 = static_cast<float>(P->cfg.min_steal_log2 > 0 ? P->cfg.min_steal_log2 : std::log2(40320.0));
    S.lgfact = P->d_lgfact;
    S.lens = P->d_lens;
    S.split_mode = split_kind(P->cfg.split_mode);
    launch_lens(P, S.split_mode);
    ck(cudaGetLastError(), "lens_kernel");
    P->launches += 1;
    export_kernel<<<1, kStealThreads, 0, P->stream>>>(S, want, d_dig, d_nf, d_cnt);
    ck(cudaGetLastError(), "export_kernel");
    P->launches += 1;
    int cnt = 0;
    xfer(P, &cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, "copy");
    ck(cudaStreamSynchronize(P->stream), "sync");
    std::vector<int> dig(static_cast<size_t>(cnt) * 2 * n);
    std::vector<uint8_t> nf(static_cast<size_t>(cnt));
    if (cnt > 0) {
      xfer(P, dig.data(), d_dig, dig.size() * sizeof(int), cudaMemcpyDeviceToHost, "copy");
      xfer(P, nf.data(), d_nf, nf.size(), cudaMemcpyDeviceToHost, "copy");
    }
    for (int i = 0; i < cnt; ++i) {
      for (int l = 0; l < n; ++l) {
        a_out[static_cast<size_t>(i) * n + l] = static_cast<uint16_t>(dig[static_cast<size_t>(i) * 2 * n + l]);
        b_out[static_cast<size_t>(i) * n + l] = static_cast<uint16_t>(dig[static_cast<size_t>(i) * 2 * n + n + l]);
      }
      nf_out[i] = nf[static_cast<size_t>(i)];
    }
    *count = cnt;
  });
}

int pbbgpu_run_round(pbbgpu_pool* P, int* active_out) {
  return guarded([&] {
    const int a = run_round(P);
    if (active_out) *active_out = a;
  });
}

int pbbgpu_active_count(pbbgpu_pool* P, int* active_out) {
  return guarded([&] { *active_out = count_active_host(P); });
}

int pbbgpu_snapshot(pbbgpu_pool* P, uint16_t* pos, uint16_t* end, uint8_t* end_nf, int cap, int* count) {
  uint64_t recount = 0;
  return pbbgpu_snapshot_ex(P, pos, end, end_nf, cap, count, &recount);
}

// Exact restart accounting. A resumed interval [pos, end) is re-seated by an init_at replay
// whose duplicates are discounted as min(L, lnz(pos)) (the steal rule). The path nodes at
// levels lnz(pos) .. level-1 of an explorer that is about to select pos's node were already
// decomposed (and counted) by this pool, and the replay counts them again; an explorer still
// replaying (kInit) has counted nrep replay decompositions that its re-seat redoes from
// scratch. Their sum is returned so that snapshot_count - resume_recount + the resumed
// pool's unique count equals a single run's count (fixed tree: same incumbent on both sides).
int pbbgpu_snapshot_ex(pbbgpu_pool* P, uint16_t* pos, uint16_t* end, uint8_t* end_nf, int cap, int* count,
                       uint64_t* resume_recount) {
  return guarded([&] {
    if (P->batch_only && !P->big_explore) throw StateError("pbbgpu: bounding-only pool has no explorers");
    const int n = P->n;
    uint64_t recount = 0;
    std::vector<unsigned char> st = download_state(P);  // either layout (BlockRef)
    std::vector<int> pv, ev;
    int c = 0;
    for (int i = 0; i < P->K; ++i) {
      const BlockRef h = block_ref(P, st, i);
      if (h.state() == kEmpty) continue;
      bool nf = false;
      // an explorer parked on a pruned/consumed cell (evaluated leaf, replay into a pruned
      // subtree) has covered that cell's whole subtree: its remaining work starts after it
      // (block_span's effective position, effective_pos in explore.cuh)
      if (!block_span(h, pv, ev, nf)) continue;
      if (c >= cap) throw CapacityError("snapshot buffer too small");
      const bool parked = h.state() == kActive && h.level() >= 0 && h.cell(h.level(), h.V(h.level())) <= 0;
      if (h.state() == kInit) {
        recount += static_cast<uint64_t>(h.nrep());
      } else if (!parked) {
        int lnz = 0;
        for (int l = 0; l < n; ++l)
          if (pv[static_cast<size_t>(l)] != 0) lnz = l;
        recount += static_cast<uint64_t>(std::max(0, h.level() - lnz));
      }
      for (int l = 0; l < n; ++l) {
        pos[static_cast<size_t>(c) * n + l] = static_cast<uint16_t>(pv[static_cast<size_t>(l)]);
        end[static_cast<size_t>(c) * n + l] = static_cast<uint16_t>(ev[static_cast<size_t>(l)]);
      }
      end_nf[c] = nf ? 1 : 0;
      ++c;
    }
    *count = c;
    if (resume_recount) *resume_recount = recount;
  });
}

int pbbgpu_debug_state(pbbgpu_pool* P, uint8_t* out, int64_t cap, int* gstride, int* offsets) {
  return guarded([&] {
    if (P->batch_only) throw StateError("pbbgpu_debug_state: the n <= 64 block layout only");
    const size_t bytes = static_cast<size_t>(P->K) * P->L.gstride;
    if (static_cast<int64_t>(bytes) > cap) throw std::invalid_argument("debug_state buffer too small");
    xfer(P, out, P->d_state, bytes, cudaMemcpyDeviceToHost, "state copy");
    *gstride = P->L.gstride;
    offsets[0] = P->L.o_cells;
    offsets[1] = P->L.o_v;
    offsets[2] = P->L.o_dir;
    offsets[3] = P->L.o_end;
    offsets[4] = P->L.o_tgt;
    offsets[5] = P->L.o_ft;
    offsets[6] = P->L.o_r;
  });
}

int pbbgpu_best(pbbgpu_pool* P, int64_t* value, int32_t* perm, int* has_perm) {
  return guarded([&] {
    std::scoped_lock lk(P->best_mu);
    *value = P->best_value;
    if (has_perm) *has_perm = P->best_sched.empty() ? 0 : 1;
    if (perm && !P->best_sched.empty()) std::copy(P->best_sched.begin(), P->best_sched.end(), perm);
  });
}

int pbbgpu_best_schedule(pbbgpu_pool* P, int64_t* cmax, int32_t* perm, int* has_perm) {
  return guarded([&] {
    std::scoped_lock lk(P->best_mu);
    *cmax = P->best_sched.empty() ? INT64_MAX : P->best_sched_value;
    if (has_perm) *has_perm = P->best_sched.empty() ? 0 : 1;
    if (perm && !P->best_sched.empty()) std::copy(P->best_sched.begin(), P->best_sched.end(), perm);
  });
}

int pbbgpu_offer_bound(pbbgpu_pool* P, int64_t v) {
  return guarded([&] {
    int64_t cur = P->pending_offer.load();
    while (v < cur && !P->pending_offer.compare_exchange_weak(cur, v)) {
    }
  });
}

int64_t pbbgpu_insertion_ls(int n, int m, const int32_t* p, const int32_t* seed, uint64_t max_iter, double max_seconds,
                            uint64_t rng_seed, int32_t* perm_out) {
  try {
    return insertion_ls_host(n, m, p, seed, max_iter, max_seconds, rng_seed, perm_out);
  } catch (const std::exception& e) {
    set_err(e);
    return -1;
  }
}

// offer_schedule (src/explorer.cpp:379-395): a schedule found elsewhere (heuristic agent);
// taken when it beats the bound or the pool's best schedule; the bound reaches the device
// at the next round (mailbox, like offer_bound).
int pbbgpu_offer_schedule(pbbgpu_pool* P, const int32_t* perm, int64_t cmax, int* taken) {
  return guarded([&] {
    if (taken) *taken = 0;
    if (!perm || cmax < 0) return;
    if (makespan_host(P->n, P->m, P->p.data(), perm) != cmax) throw std::invalid_argument("offer_schedule: cmax does not match the schedule");
    bool took = false;
    {
      std::scoped_lock lk(P->best_mu);
      if (cmax < P->best_sched_value) {
        P->best_sched.assign(perm, perm + P->n);
        P->best_sched_value = cmax;
        took = true;
      }
    }
    int64_t cur = P->pending_offer.load();
    while (cmax < cur && !P->pending_offer.compare_exchange_weak(cur, cmax)) {
    }
    {
      std::scoped_lock lk(P->best_mu);  // run_round updates best_value under the same lock
      if (cmax < P->best_value) {
        took = true;
        ++P->host_improvements;  // explorer.cpp:383-386
      }
    }
    if (taken) *taken = took ? 1 : 0;
  });
}

// promote_solutions (src/explorer.cpp:397-424): every active explorer's current node,
// completed by ordering its free jobs as in the best schedule, evaluated, best first.
int pbbgpu_promote(pbbgpu_pool* P, int capacity, int32_t* perms_out, int64_t* cmax_out, int* count) {
  return guarded([&] {
    *count = 0;
    std::vector<int32_t> inc;
    {
      std::scoped_lock lk(P->best_mu);
      inc = P->best_sched;
    }
    if (inc.empty() || capacity <= 0 || (P->batch_only && !P->big_explore)) return;
    const int n = P->n;
    std::vector<int> rank(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) rank[static_cast<size_t>(inc[static_cast<size_t>(i)])] = i;
    std::vector<unsigned char> st = download_state(P);  // either layout (BlockRef)
    std::vector<std::pair<int64_t, std::vector<int32_t>>> cands;
    std::vector<int32_t> perm(static_cast<size_t>(n));
    for (int i = 0; i < P->K; ++i) {
      const BlockRef h = block_ref(P, st, i);
      if (h.state() != kActive || h.level() < 0) continue;
      const int level = h.level();
      if (h.V(level) >= n - level) continue;
      int d1 = 0, d2 = 0;  // decode (src/ivm.cpp:152-172)
      for (int l = 0; l <= level; ++l) {
        const int x = h.cell(l, h.V(l));
        const int job = (x < 0 ? -x : x) - 1;
        if (h.dir(l) == kFwd) perm[static_cast<size_t>(d1++)] = job;
        else perm[static_cast<size_t>(n - 1 - d2++)] = job;
      }
      int pos = d1;
      for (int c = 0; c < n - level; ++c) {
        if (c == h.V(level)) continue;
        const int x = h.cell(level, c);
        perm[static_cast<size_t>(pos++)] = (x < 0 ? -x : x) - 1;
      }
      std::sort(perm.begin() + d1, perm.end() - d2, [&](int a, int b) { return rank[static_cast<size_t>(a)] < rank[static_cast<size_t>(b)]; });
      cands.emplace_back(makespan_host(n, P->m, P->p.data(), perm.data()), perm);
    }
    std::stable_sort(cands.begin(), cands.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const int c = std::min(capacity, static_cast<int>(cands.size()));
    for (int i = 0; i < c; ++i) {
      cmax_out[i] = cands[static_cast<size_t>(i)].first;
      std::copy(cands[static_cast<size_t>(i)].second.begin(), cands[static_cast<size_t>(i)].second.end(), perms_out + static_cast<size_t>(i) * n);
    }
    *count = c;
  });
}

// Per-explorer activity after the last round (timeline rows, src/explorer.cpp:448-464):
// log2 of the remaining leaves from the effective position; -2 = busy replaying (active, length
// not tracked), -3 = idle.
int pbbgpu_explorer_lengths(pbbgpu_pool* P, float* out, int cap) {
  return guarded([&] {
    if (P->batch_only && !P->big_explore) throw StateError("pbbgpu: bounding-only pool has no explorers");
    if (cap < P->K) throw std::invalid_argument("explorer_lengths buffer smaller than K");
    if (P->big_explore) big_lens_kernel<<<(P->K + 127) / 128, 128, 0, P->stream>>>(P->BL, P->d_state, P->K, P->d_lgfact, P->d_lens);
    else launch_lens(P, 1);
    ck(cudaGetLastError(), "lens_kernel");
    P->launches += 1;
    xfer(P, out, P->d_lens, static_cast<size_t>(P->K) * sizeof(float), cudaMemcpyDeviceToHost, "lens copy");
  });
}

int pbbgpu_stats(pbbgpu_pool* P, pbbgpu_stats_t* out) {
  return guarded([&] {
    if (P->batch_only && !P->big_explore) {
      std::memset(out, 0, sizeof(*out));
      out->kernel_launches = P->launches;
      out->batch_kernel_ms = P->batch_ms;
      out->h2d_bytes = P->h2d_bytes;
      out->d2h_bytes = P->d2h_bytes;
      return;
    }
    read_counters(P);
    const DevCounters& c = *P->h_ctr;
    std::memset(out, 0, sizeof(*out));
    out->decomposed = c.decomposed;
    out->replay_dups = c.dups;
    out->unique = c.decomposed - c.dups;
    out->leaves = c.leaves;
    out->improvements = c.improvements + P->host_improvements;
    out->local_steals = c.steals;
    out->steal_phases = c.steal_phases;
    out->intervals_initialized = c.inits;
    out->rounds = P->rounds;
    out->steps = c.steps;
    out->kernel_ms = P->kernel_ms;
    out->completed = P->last_active == 0;
    out->K = P->K;
    out->group = P->G;
    out->block = P->block;
    out->steps_per_round = P->steps;
    out->kernel_launches = P->launches;
    out->batch_kernel_ms = P->batch_ms;
    out->h2d_bytes = P->h2d_bytes;
    out->d2h_bytes = P->d2h_bytes;
    out->steal_kernel_ms = P->steal_ms;
  });
}

int pbbgpu_histogram(pbbgpu_pool* P, uint64_t* hist, int len) {
  return guarded([&] {
    const int n = P->n;
    std::vector<unsigned long long> h(static_cast<size_t>(n) + 1), d(static_cast<size_t>(n) + 1);
    xfer(P, h.data(), P->d_hist, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, "hist copy");
    xfer(P, d.data(), P->d_dhist, d.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, "hist copy");
    for (int f = 0; f < len; ++f) hist[f] = f <= n ? h[static_cast<size_t>(f)] - d[static_cast<size_t>(f)] : 0;
  });
}

int pbbgpu_decompose_batch(pbbgpu_pool* P, const int32_t* perms, const int32_t* d1, const int32_t* d2, int count,
                           int64_t incumbent, int64_t* child_lb, uint8_t* direction, uint8_t* pruned,
                           int64_t* lb_fwd, int64_t* lb_bwd) {
  return guarded([&] {
    if (count <= 0) return;
    if (incumbent <= 0) throw std::invalid_argument("decompose: incumbent must be positive");
    const int n = P->n;
    for (int i = 0; i < count; ++i) {
      const int a = d1[i], b = d2[i];
      if (a < 0 || b < 0 || a + b > n - 1) throw std::invalid_argument("decompose: no free jobs / bad depths");
      std::vector<char> seen(static_cast<size_t>(n), 0);
      for (int t = 0; t < n; ++t) {
        const int j = perms[static_cast<size_t>(i) * n + t];
        if (j < 0 || j >= n || seen[static_cast<size_t>(j)]) throw std::invalid_argument("subproblem perm is not a permutation");
        seen[static_cast<size_t>(j)] = 1;
      }
    }
    const size_t cn = static_cast<size_t>(count) * n;
    int* dp = scratch<int>(P, 0, cn);
    int* dd1 = scratch<int>(P, 1, count);
    int* dd2 = scratch<int>(P, 2, count);
    int* dlb = scratch<int>(P, 3, cn);
    int* dlf = scratch<int>(P, 4, cn);
    int* dlbw = scratch<int>(P, 5, cn);
    uint8_t* ddir = scratch<uint8_t>(P, 6, count);
    uint8_t* dpr = scratch<uint8_t>(P, 7, cn);
    xfer(P, dp, perms, cn * sizeof(int), cudaMemcpyHostToDevice, "copy");
    xfer(P, dd1, d1, count * sizeof(int), cudaMemcpyHostToDevice, "copy");
    xfer(P, dd2, d2, count * sizeof(int), cudaMemcpyHostToDevice, "copy");
    if (P->batch_only) {
      BigBatchParams G{};
      G.n = n;
      G.m = P->m;
      G.mp = P->mp;
      G.npairs = P->npairs;
      G.perms = dp;
      G.d1 = dd1;
      G.d2 = dd2;
      G.count = count;
      G.incumbent = static_cast<int>(std::min<int64_t>(incumbent, INT_MAX));
      G.p32 = P->d_p32;
      G.pk = P->d_pk;
      G.pl = P->d_pl;
      G.packed = P->d_packed64;
      G.inv16 = P->d_inv16;
      G.scratch = P->d_big_scratch;
      G.child_lb = dlb;
      G.lb_fwd = dlf;
      G.lb_bwd = dlbw;
      G.dir = ddir;
      G.pruned = dpr;
      ck(cudaEventRecord(P->ev0, P->stream), "event");
      int fmax = 0;
      long long fsum = 0;
      for (int i = 0; i < count; ++i) {
        fmax = std::max(fmax, n - d1[i] - d2[i]);
        fsum += n - d1[i] - d2[i];
      }
      launch_big_bounding(P, G, count, fmax, fsum, count);
      ck(cudaEventRecord(P->ev1, P->stream), "event");
    }
    BatchParams B{};
    B.L = P->L;
    B.perms = dp;
    B.d1 = dd1;
    B.d2 = dd2;
    B.count = count;
    B.incumbent = static_cast<int>(std::min<int64_t>(incumbent, INT_MAX));
    B.p32 = P->d_p32;
    B.npairs = P->npairs;
    B.pk = P->d_pk;
    B.pl = P->d_pl;
    B.order = P->d_ord;
    B.lag = P->d_lag;
    B.packed = P->d_packed;
    B.invord = P->d_invord;
    B.child_lb = dlb;
    B.lb_fwd = dlf;
    B.lb_bwd = dlbw;
    B.dir = ddir;
    B.pruned = dpr;
    if (!P->batch_only) {
      const int NG = P->block / P->G;
      const int grid = std::min((count + NG - 1) / NG, P->num_sms * 8);
      ck(cudaEventRecord(P->ev0, P->stream), "event");
      P->bfn<<<grid, P->block, P->smem, P->stream>>>(B);
      ck(cudaGetLastError(), "decompose_batch launch");
      ck(cudaEventRecord(P->ev1, P->stream), "event");
    }
    P->launches += 1;
    ck(cudaStreamSynchronize(P->stream), "sync");
    float bms = 0;
    ck(cudaEventElapsedTime(&bms, P->ev0, P->ev1), "elapsed");
    P->batch_ms += bms;
    std::vector<int> lb(cn), lf(cn), lbw(cn);
    std::vector<uint8_t> pr(cn);
    xfer(P, lb.data(), dlb, cn * sizeof(int), cudaMemcpyDeviceToHost, "copy");
    xfer(P, lf.data(), dlf, cn * sizeof(int), cudaMemcpyDeviceToHost, "copy");
    xfer(P, lbw.data(), dlbw, cn * sizeof(int), cudaMemcpyDeviceToHost, "copy");
    xfer(P, pr.data(), dpr, cn, cudaMemcpyDeviceToHost, "copy");
    xfer(P, direction, ddir, count, cudaMemcpyDeviceToHost, "copy");
    for (int i = 0; i < count; ++i) {
      const int f = n - d1[i] - d2[i];
      for (int c = 0; c < f; ++c) {
        const size_t s = static_cast<size_t>(i) * n + c;
        child_lb[s] = lb[s];
        pruned[s] = pr[s];
        if (lb_fwd) lb_fwd[s] = lf[s];
        if (lb_bwd) lb_bwd[s] = lbw[s];
      }
    }
  });
}

// ---- apply_work_update (src/explorer.cpp:162-199) on factoradic digit intervals: BigCount
// comparisons are lexicographic digit comparisons; an end of n! is a flag (greater than any
// digit vector). normalize / intersect_units / subtract_units follow src/workunit.cpp:8-51 and
// src/explorer.cpp:143-160.
namespace {
struct DInterval {
  std::vector<int> a, b;
  bool b_nf;
};
int dcmp(const std::vector<int>& x, const std::vector<int>& y) {
  for (size_t l = 0; l < x.size(); ++l)
    if (x[l] != y[l]) return x[l] < y[l] ? -1 : 1;
  return 0;
}
// point comparison with the n! flag
int pcmp(const std::vector<int>& x, bool xnf, const std::vector<int>& y, bool ynf) {
  if (xnf || ynf) return xnf == ynf ? 0 : (xnf ? 1 : -1);
  return dcmp(x, y);
}
bool dempty(const DInterval& iv) { return pcmp(iv.a, false, iv.b, iv.b_nf) >= 0; }

std::vector<DInterval> dnormalize(std::vector<DInterval> ivs) {
  ivs.erase(std::remove_if(ivs.begin(), ivs.end(), dempty), ivs.end());
  std::sort(ivs.begin(), ivs.end(), [](const DInterval& x, const DInterval& y) {
    const int c = dcmp(x.a, y.a);
    if (c) return c < 0;
    return pcmp(x.b, x.b_nf, y.b, y.b_nf) < 0;
  });
  std::vector<DInterval> out;
  for (DInterval& iv : ivs) {
    if (!out.empty() && pcmp(iv.a, false, out.back().b, out.back().b_nf) < 0) {
      if (pcmp(iv.b, iv.b_nf, out.back().b, out.back().b_nf) > 0) {
        out.back().b = iv.b;
        out.back().b_nf = iv.b_nf;
      }
    } else {
      out.push_back(std::move(iv));
    }
  }
  return out;
}

std::vector<DInterval> dintersect(const std::vector<DInterval>& A, const std::vector<DInterval>& B) {
  std::vector<DInterval> out;
  size_t i = 0, j = 0;
  while (i < A.size() && j < B.size()) {
    const std::vector<int>& lo = dcmp(A[i].a, B[j].a) > 0 ? A[i].a : B[j].a;
    const bool a_hi = pcmp(A[i].b, A[i].b_nf, B[j].b, B[j].b_nf) < 0;
    const DInterval& h = a_hi ? A[i] : B[j];
    if (pcmp(lo, false, h.b, h.b_nf) < 0) out.push_back({lo, h.b, h.b_nf});
    if (pcmp(A[i].b, A[i].b_nf, B[j].b, B[j].b_nf) <= 0) ++i;
    else ++j;
  }
  return out;
}

std::vector<DInterval> dsubtract(const std::vector<DInterval>& A, const std::vector<DInterval>& B) {
  std::vector<DInterval> out;
  for (const DInterval& iv : A) {
    std::vector<int> cur = iv.a;
    bool cur_nf = false;
    for (const DInterval& c : B) {
      if (pcmp(c.b, c.b_nf, cur, cur_nf) <= 0) continue;
      if (pcmp(c.a, false, iv.b, iv.b_nf) >= 0) break;
      if (pcmp(c.a, false, cur, cur_nf) > 0) out.push_back({cur, c.a, false});
      cur = c.b;
      cur_nf = c.b_nf;
      if (pcmp(cur, cur_nf, iv.b, iv.b_nf) >= 0) break;
    }
    if (pcmp(cur, cur_nf, iv.b, iv.b_nf) < 0) out.push_back({cur, iv.b, iv.b_nf});
  }
  return out;
}
}  // namespace

int pbbgpu_apply_work_update(pbbgpu_pool* P, const uint16_t* a, const uint16_t* b, const uint8_t* nf, int count) {
  return guarded([&] {
    if (P->batch_only && !P->big_explore) throw StateError("pbbgpu: bounding-only pool has no explorers");
    if (count < 0) throw std::invalid_argument("negative interval count");
    if (count > P->K) throw std::invalid_argument("work update holds more intervals than explorers");
    const int n = P->n;
    std::vector<DInterval> incoming;
    for (int i = 0; i < count; ++i) {
      check_digits(n, a + static_cast<size_t>(i) * n);
      const bool inf = nf && nf[i];
      if (!inf) check_digits(n, b + static_cast<size_t>(i) * n);
      DInterval iv{std::vector<int>(a + static_cast<size_t>(i) * n, a + static_cast<size_t>(i + 1) * n),
                   std::vector<int>(static_cast<size_t>(n), 0), inf};
      if (!inf) iv.b.assign(b + static_cast<size_t>(i) * n, b + static_cast<size_t>(i + 1) * n);
      if (pcmp(iv.a, false, iv.b, iv.b_nf) > 0) throw std::invalid_argument("interval with a > b");
      incoming.push_back(std::move(iv));
    }
    incoming = dnormalize(std::move(incoming));
    std::vector<unsigned char> st = download_state(P);
    std::vector<DInterval> kept;
    std::vector<int> idle;
    std::vector<unsigned long long> extra(static_cast<size_t>(n) + 1, 0);  // replay dups by f
    unsigned long long extra_dups = 0;
    // explorers re-seated from scratch: their start and the levels [lo, hi) whose path nodes
    // they have already counted (pbbgpu_snapshot_ex's recount), plus the dups a partial replay
    // would have been discounted had it finished (levels [0, min(nrep, lz)))
    struct Reset {
      std::vector<int> start;
      int lo, hi, lzcut;
    };
    std::vector<Reset> resets;
    std::vector<int> pos, end;
    for (int i = 0; i < P->K; ++i) {
      const BlockRef h = block_ref(P, st, i);
      if (h.state() == kEmpty) {
        idle.push_back(i);
        continue;
      }
      bool end_nf = false;
      std::vector<DInterval> mine;
      const bool has_span = block_span(h, pos, end, end_nf);
      if (has_span) mine = dintersect(incoming, {{pos, end, end_nf}});
      if (mine.size() == 1 && dcmp(mine[0].a, pos) == 0) {
        if (pcmp(mine[0].b, mine[0].b_nf, end, end_nf) < 0) h.set_end(mine[0].b);  // shrink_end (ivm.cpp:186-189)
        kept.push_back(std::move(mine[0]));
      } else {
        if (has_span) {
          int lnz = 0;
          for (int l = 0; l < n; ++l)
            if (pos[static_cast<size_t>(l)] != 0) lnz = l;
          if (h.state() == kInit) {
            resets.push_back({pos, 0, h.nrep(), std::min<int>(h.nrep(), lnz)});
          } else if (h.cell(h.level(), h.V(h.level())) > 0) {  // not parked
            resets.push_back({pos, lnz, std::max<int>(lnz, h.level()), 0});
          }
        }
        h.set_empty();
        idle.push_back(i);
      }
    }
    kept = dnormalize(std::move(kept));
    const std::vector<DInterval> to_place = dsubtract(incoming, kept);
    if (to_place.size() > idle.size()) throw CapacityError("work update fragments exceed explorer capacity");
    // a fragment re-seated exactly at a reset explorer's start replays the path nodes that
    // explorer already counted: discount them (the same recount as pbbgpu_snapshot_ex); a
    // partial replay not re-seated there keeps only its first-leaf-owned nodes
    for (const Reset& r : resets) {
      bool reseated = false;
      for (const DInterval& f : to_place)
        if (dcmp(f.a, r.start) == 0) reseated = true;
      const int lo = reseated ? r.lo : 0, hi = reseated ? r.hi : r.lzcut;
      for (int l = lo; l < hi; ++l) {
        ++extra_dups;
        ++extra[static_cast<size_t>(n - 1 - l)];
      }
    }
    xfer(P, P->d_state, st.data(), st.size(), cudaMemcpyHostToDevice, "state copy");
    if (extra_dups) {
      read_counters(P);
      const unsigned long long d = P->h_ctr->dups + extra_dups;
      xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, dups), &d, sizeof(d), cudaMemcpyHostToDevice, "copy");
      std::vector<unsigned long long> dh(static_cast<size_t>(n) + 1);
      xfer(P, dh.data(), P->d_dhist, dh.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, "copy");
      for (int f = 0; f <= n; ++f) dh[static_cast<size_t>(f)] += extra[static_cast<size_t>(f)];
      xfer(P, P->d_dhist, dh.data(), dh.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, "copy");
    }
    std::sort(idle.begin(), idle.end());
    std::vector<int> da, db, slots;
    std::vector<uint8_t> dn;
    for (size_t i = 0; i < to_place.size(); ++i) {
      da.insert(da.end(), to_place[i].a.begin(), to_place[i].a.end());
      if (to_place[i].b_nf) db.insert(db.end(), static_cast<size_t>(n), 0);
      else db.insert(db.end(), to_place[i].b.begin(), to_place[i].b.end());
      dn.push_back(to_place[i].b_nf ? 1 : 0);
      slots.push_back(idle[i]);
    }
    assign_digits(P, da, db, dn, slots);
    read_counters(P);
    P->last_active = static_cast<int>(P->K - idle.size() + to_place.size());
  });
}

int pbbgpu_improved_since_mark(pbbgpu_pool* P, int* improved) {
  return guarded([&] {
    std::scoped_lock lk(P->best_mu);
    *improved = 0;
    if (P->best_sched_value < P->improvement_mark) {
      P->improvement_mark = P->best_sched_value;
      *improved = 1;
    }
  });
}

int pbbgpu_steals_since_mark(pbbgpu_pool* P, uint64_t* steals) {
  return guarded([&] {
    if (P->batch_only) {
      *steals = 0;
      return;
    }
    read_counters(P);
    *steals = P->h_ctr->steals - P->steal_mark;
  });
}

int pbbgpu_reset_steal_mark(pbbgpu_pool* P) {
  return guarded([&] {
    if (P->batch_only) return;
    read_counters(P);
    P->steal_mark = P->h_ctr->steals;
  });
}

int pbbgpu_take_census(pbbgpu_pool* P, uint64_t* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    *count = 0;
    if (!P->d_census) throw StateError("take_census: the pool was created without record_census");
    read_counters(P);
    const int64_t c = P->h_ctr->census_count;
    if (c > P->census_cap) throw CapacityError("census buffer overflow: raise census_cap or take the census more often");
    if (c > cap) throw CapacityError("take_census: output buffer too small");
    if (c > 0) xfer(P, out, P->d_census, static_cast<size_t>(c) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, "census copy");
    const unsigned zero = 0;
    xfer(P, reinterpret_cast<char*>(P->d_ctr) + offsetof(DevCounters, census_count), &zero, sizeof(zero), cudaMemcpyHostToDevice, "copy");
    *count = c;
  });
}

int pbbgpu_flush_timeline(pbbgpu_pool* P) {
  return guarded([&] {
    if (!P->timeline) return;
    sample_timeline(P, true);
    std::fflush(P->timeline);
  });
}

// ---- multi-GPU group (one process per GPU; peer windows over CUDA IPC / NVLink)
int pbbgpu_group_handle_size(void) { return static_cast<int>(sizeof(cudaIpcMemHandle_t)); }

int pbbgpu_group_create(pbbgpu_pool* P, int world, int rank, void* handle_out) {
  return guarded([&] {
    if (P->batch_only) throw StateError("pbbgpu: bounding-only pool has no explorers");
    if (P->cfg.steal_policy == 1) throw std::invalid_argument("the reference steal policy is single-pool only");
    if (world < 2 || world > kMaxGroup || rank < 0 || rank >= world) throw std::invalid_argument("bad group world / rank");
    if (P->d_window) throw StateError("pbbgpu_group_create: the pool already has a group");
    ck(cudaSetDevice(P->cfg.device), "cudaSetDevice");
    P->g_cap = P->K;
    const size_t bytes = kWindowHeader + static_cast<size_t>(P->g_cap) * (2 * P->n * sizeof(int) + 1);
    ck(cudaMalloc(&P->d_window, bytes), "malloc window");
    ck(cudaMemset(P->d_window, 0, bytes), "memset window");
    ck(cudaMalloc(&P->d_gs, sizeof(GroupState)), "malloc");
    ck(cudaMallocHost(&P->h_gs, sizeof(GroupState)), "malloc host");
    P->g_world = world;
    P->g_rank = rank;
    P->g_peer[rank] = P->d_window;
    for (cudaEvent_t& e : P->gev)
      if (!e) ck(cudaEventCreate(&e), "event");
    ck(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out), P->d_window), "cudaIpcGetMemHandle");
  });
}

int pbbgpu_group_open(pbbgpu_pool* P, const void* handles) {
  return guarded([&] {
    if (!P->d_window) throw StateError("pbbgpu_group_open before pbbgpu_group_create");
    if (P->g_open) return;
    ck(cudaSetDevice(P->cfg.device), "cudaSetDevice");
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int q = 0; q < P->g_world; ++q) {
      if (q == P->g_rank) continue;
      void* ptr = nullptr;
      ck(cudaIpcOpenMemHandle(&ptr, h[q], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      P->g_peer[q] = static_cast<unsigned char*>(ptr);
    }
    P->g_open = true;
  });
}

// Own window back to its initial state (call on every rank, then a group barrier, before a solve).
int pbbgpu_group_reset(pbbgpu_pool* P) {
  return guarded([&] {
    if (!P->d_window) throw StateError("pbbgpu_group_reset: no group");
    PeerWindow w{};
    w.best = INT_MAX;
    w.active = 1 << 20;  // "not started": never terminal, never served, until the first publish
    xfer(P, P->d_window, &w, sizeof(w), cudaMemcpyHostToDevice, "window reset");
    GroupState z{};
    z.serve = -1;
    xfer(P, P->d_gs, &z, sizeof(z), cudaMemcpyHostToDevice, "group state reset");
  });
}

int pbbgpu_group_solve(pbbgpu_pool* P, int64_t initial_ub, int seed_div, double time_limit_s,
                       pbbgpu_group_stats_t* out) {
  return guarded([&] {
    if (!P->g_open) throw StateError("pbbgpu_group_solve: open the group first");
    std::memset(out, 0, sizeof(*out));
    int rc = pbbgpu_set_initial_bound(P, initial_ub, nullptr, 0);
    if (rc) throw std::runtime_error(g_last_error);
    const int W = P->g_world, r = P->g_rank;
    rc = seed_div > 0 ? pbbgpu_seed(P, initial_ub, r, W, std::max(W, W * P->K / seed_div))
                      : pbbgpu_assign_split_strided(P, r, W, P->K, W * P->K);
    if (rc) throw std::runtime_error(g_last_error);
    const auto t0 = std::chrono::steady_clock::now();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, P->stream), "event");
    bool completed = true, have_prev = false;
    GroupState prev{};
    uint64_t syncs = 0;
    const double g0 = P->group_ms;
    const uint64_t gr0 = P->group_rounds;
    for (;;) {
      run_round(P);
      ++syncs;
      xfer(P, P->h_gs, P->d_gs, sizeof(GroupState), cudaMemcpyDeviceToHost, "group state");
      const GroupState& g = *P->h_gs;
      bool terminal = true;
      unsigned long long ss = 0, rr = 0;
      for (int q = 0; q < W; ++q) {
        terminal = terminal && g.act[q] == 0;
        ss += g.sent[q];
        rr += g.recv[q];
      }
      terminal = terminal && ss == rr;
      if (terminal && have_prev) {
        bool same = true;
        for (int q = 0; q < W; ++q) same = same && prev.sent[q] == g.sent[q] && prev.recv[q] == g.recv[q];
        if (same) break;
      }
      have_prev = terminal;
      prev = g;
      if (time_limit_s > 0) {
        const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
        if (el.count() >= time_limit_s) {
          completed = false;
          break;
        }
      }
    }
    ck(cudaEventRecord(e1, P->stream), "event");
    ck(cudaEventSynchronize(e1), "event sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    xfer(P, P->h_gs, P->d_gs, sizeof(GroupState), cudaMemcpyDeviceToHost, "group state");
    out->syncs = syncs;
    out->exchanges = P->h_gs->exchanges;
    out->imported = P->h_gs->imported;
    out->exported = P->h_gs->exported;
    out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out->device_ms = ms;
    out->completed = completed ? 1 : 0;
    out->exchange_us_per_round = P->group_rounds > gr0 ? 1000.0 * (P->group_ms - g0) / static_cast<double>(P->group_rounds - gr0) : 0.0;
  });
}

int pbbgpu_group_close(pbbgpu_pool* P) {
  return guarded([&] {
    if (!P->d_window) return;
    ck(cudaStreamSynchronize(P->stream), "sync");
    for (int q = 0; q < P->g_world; ++q) {
      if (q != P->g_rank && P->g_peer[q]) cudaIpcCloseMemHandle(P->g_peer[q]);
      P->g_peer[q] = nullptr;
    }
    cudaFree(P->d_window);
    cudaFree(P->d_gs);
    cudaFreeHost(P->h_gs);
    P->d_window = nullptr;
    P->d_gs = nullptr;
    P->h_gs = nullptr;
    P->g_open = false;
    P->g_world = 0;
  });
}

int pbbgpu_solve(pbbgpu_pool* P, int64_t initial_ub, const uint16_t* a, const uint16_t* b, const uint8_t* nf,
                 int count, int64_t* best_value, int32_t* best_perm, int* has_perm, pbbgpu_stats_t* stats) {
  int rc = pbbgpu_set_initial_bound(P, initial_ub, nullptr, 0);
  if (rc) return rc;
  rc = count > 0 ? pbbgpu_assign(P, a, b, nf, count) : pbbgpu_assign_split(P, 0);
  if (rc) return rc;
  const auto t0 = std::chrono::steady_clock::now();
  bool completed = true;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  float dev_ms = 0.f;
  rc = guarded([&] {
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, P->stream), "event");
    for (;;) {
      const int act = run_round(P);
      if (act == 0) break;
      if (P->cfg.time_limit_s > 0) {
        const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
        if (el.count() >= P->cfg.time_limit_s) {
          completed = false;
          break;
        }
      }
    }
    ck(cudaEventRecord(e1, P->stream), "event");
    ck(cudaEventSynchronize(e1), "event sync");
    ck(cudaEventElapsedTime(&dev_ms, e0, e1), "elapsed");
  });
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (rc) return rc;
  const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
  rc = pbbgpu_best(P, best_value, best_perm, has_perm);
  if (rc) return rc;
  if (stats) {
    rc = pbbgpu_stats(P, stats);
    stats->wall_s = el.count();
    stats->completed = completed ? 1 : 0;
    stats->device_ms = dev_ms;
  }
  return rc;
}

}  // extern "C"
