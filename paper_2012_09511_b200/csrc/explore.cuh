// B200-native PFSP Branch-and-Bound device code (sm_100a).
//
// One explorer (IVM: Integer-Vector-Matrix, §2.5 / src/ivm.cpp) per group of G
// lanes; a 128-thread CTA holds 128/G explorers whose whole state lives in shared memory
// for the duration of a persistent launch ("round"). Each group loops
//     select (or replay) -> [leaf: makespan | internal: bound children -> MinMin -> prune
//     -> branch]
// entirely out of shared memory; the only global traffic per step is the incumbent read.
//
// Semantics follow the reference bit-for-bit (paths under /root/reference/proj):
//   select_next + end test      src/ivm.cpp:90-122
//   decode (free jobs in row order minus the selected cell)  src/ivm.cpp:152-172
//   LB1 children, fwd/bwd       src/bound.cpp:61-88
//   MinMin + prune (>=)         src/bound.cpp:109-138
//   branch                      src/ivm.cpp:124-145
//   leaf = one free job, improve iff mk < improve bound   src/explorer.cpp:42-57
//   init_at replay              src/ivm.cpp:48-88
// LB2 follows SURVEY.md §8 row a22 (no reference implementation exists).
//
// Incremental node tables (B200 design, not in the reference): instead of re-scanning the
// prefix/suffix of every node (bound_tables, src/bound.cpp:20-46), the explorer keeps
//   FS[d] = front of the first d forward jobs, TS[d] = tail of the first d backward jobs
// in one (n+1)*m uint16 stack (FS grows from slot 0, TS from slot n; d1+d2 <= n-1 keeps
// them disjoint) and R = per-machine sum over the jobs of the current row, updated by
// +-p on descend/backtrack. A node's tables then cost one O(m) extension.
#pragma once

#include <climits>
#include <cstdint>
#include <type_traits>

#include "pbb_layout.h"

namespace pbbgpu {

__host__ __device__ inline int tri_off(int l, int n) { return l * n - (l * (l - 1)) / 2; }
__host__ __device__ inline int round_up(int x, int a) { return (x + a - 1) / a * a; }

// Per-CTA shared instance region (identical computation on host and device).
struct InstLayout {
  int o_p32, o_psf, o_psb, o_pk, o_pl, o_ord, o_lag, o_pk32, o_inv, o_cnt, o_cta, o_hist, o_dhist, o_roff, bytes;
};

// packed = warp-per-explorer LB2 (children_lb2_w): one uint32 per (position, pair),
// transposed [t][q]; otherwise the group LB2 tables (order [q][t], lag [q][j]).
// wide = 32-bit times: the exclusive and inclusive sums are two int32 [n][mp] arrays.
__host__ __device__ inline InstLayout inst_layout(int n, int mp, int npairs, bool packed = false, bool wide = false) {
  InstLayout s;
  int o = 0;
  s.o_p32 = o;
  o += n * mp * 4;
  s.o_psf = o;  // [n][mp] prefix sums of p: exclusive | inclusive << 16
  o += n * mp * (wide ? 8 : 4);
  s.o_psb = o;  // [n][mp] suffix sums of p: exclusive | inclusive << 16
  o += n * mp * (wide ? 8 : 4);
  s.o_lag = o;
  o += packed ? 0 : round_up(npairs * n * 2, 16);
  s.o_pk32 = o;
  o += packed ? round_up(round_up(npairs, 32) * n * 4, 16) : 0;
  s.o_inv = o;  // [job][pair] position of the job in the pair's order (packed mode)
  o += packed ? round_up(npairs * n, 16) : 0;
  s.o_pk = o;
  o += round_up(npairs, 16);
  s.o_pl = o;
  o += round_up(npairs, 16);
  s.o_ord = o;
  o += packed ? 0 : round_up(npairs * n, 16);
  s.o_cnt = o;
  o += 64;
  s.o_cta = o;
  s.o_hist = o;
  o += round_up((n + 1) * 4, 16);
  s.o_dhist = o;
  o += round_up((n + 1) * 4, 16);
  s.o_roff = o;  // [n + 1] uint16: tri_off(l, n), the IVM row offsets
  o += round_up((n + 1) * 2, 16);
  s.bytes = round_up(o, 128);
  return s;
}

__host__ __device__ inline IvmLayout ivm_layout(int n, int m, int bound, int lanes, bool wide = false) {
  IvmLayout L;
  L.n = n;
  L.m = m;
  L.mp = round_up(m, 4);
  L.ftb = wide ? 4 : 2;
  int o = 8;  // IvmHdr
  L.o_cells = o;
  o += n * (n + 1) / 2;
  L.o_v = o;
  o += n;
  L.o_dir = o;
  o += n;
  L.o_end = o;
  o += n;
  L.o_tgt = o;
  o += n;
  o = round_up(o, 4);
  L.o_ft = o;
  o += (n + 1) * m * L.ftb;
  L.o_r = o;
  o += m * L.ftb;
  L.gstride = round_up(o, 16);
  o = L.gstride;
  L.o_fr = o;
  o += L.mp * 4;
  L.o_tl = o;
  o += L.mp * 4;
  L.o_rm = o;
  o += L.mp * 4;
  if (bound == kLB1) {  // remain + tail, front + remain: LB1's children only
    L.o_rt = o;
    o += L.mp * 4;
    L.o_frm = o;
    o += L.mp * 4;
  } else {
    L.o_rt = L.o_frm = -1;
  }
  if (bound == kLB2 && lanes == 32 && n <= 32) {
    L.o_lbf = -1;  // children bounds stay in registers (decompose_branch)
  } else {
    L.o_lbf = o;  // lbf / lbb: two int32 [n] arrays
    o += round_up(2 * n * 4, 16);
  }
  L.o_free = o;
  o += round_up(n, 16);
  if (bound == kLB2) {
    L.o_heads = o;
    o += round_up(n * m * 2, 16);
    L.o_tails = o;
    o += round_up(n * m * 2, 16);
    L.o_lst = o;
    if (lanes == 32) {
      // per-lane [job][32] table: int32 PM' then S_j (n <= 32), int16 PM' only (n > 32: S_j is
      // folded into the child bounds in the backward pass)
      o += round_up(n * 32 * (n <= 32 ? 4 : 2), 16);
      L.o_pos = 0;
    } else {
      o += n * 16;
      L.o_pos = o;
      o += round_up(n, 16);
    }
    L.o_msk = 0;
    if (lanes == 32 && n <= 32) {  // RowMask: [round][32] uint32 per explorer
      o = round_up(o, 16);
      L.o_msk = o;
      o += ((m * (m - 1) / 2 + 31) / 32) * 32 * 4;
    }
  } else {
    L.o_heads = L.o_tails = L.o_lst = L.o_pos = L.o_msk = 0;
  }
  o = round_up(o, 16);
  // stride == 16 (mod 128): the groups of one warp hit distinct bank quads on LDS.128
  L.sstride = o + ((16 - (o % 128)) + 128) % 128;
  return L;
}

#ifdef __CUDACC__

template <int G>
struct Group {
  unsigned mask;
  int g;
  int base;
  __device__ __forceinline__ Group() {
    const int lane = threadIdx.x & 31;
    g = lane & (G - 1);
    base = lane & ~(G - 1);
    mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << base);
  }
  __device__ __forceinline__ unsigned ballot(bool p) const {
    const unsigned b = __ballot_sync(mask, p);
    return G == 32 ? b : ((b >> base) & ((1u << G) - 1u));
  }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ int bcast(int v, int src) const { return __shfl_sync(mask, v, src, G); }
  // REDUX (sm_80+): one instruction per reduction over the group's lanes
  __device__ __forceinline__ int rmin(int v) const { return __reduce_min_sync(mask, v); }
  __device__ __forceinline__ int rmax(int v) const { return __reduce_max_sync(mask, v); }
  __device__ __forceinline__ int rsum(int v) const { return __reduce_add_sync(mask, v); }
  __device__ __forceinline__ unsigned long long ror64(unsigned long long v) const {
#pragma unroll
    for (int o = G / 2; o; o >>= 1) v |= __shfl_xor_sync(mask, v, o, G);
    return v;
  }
};

// FT / R entry type: uint16 unless the instance needs wide times (IvmLayout::ftb == 4)
template <bool W>
using FtT = typename std::conditional<W, uint32_t, uint16_t>::type;

// Shared-memory view of one explorer.
struct IvmView {
  IvmHdr* hdr;
  int8_t* cells;
  int8_t* V;
  uint8_t* dir;
  int8_t* endd;
  int8_t* tgt;
  uint16_t* ft;
  uint16_t* R;
  int* fr;
  int* tl;
  int* rm;
  int* rt;
  int* frm;
  int* lbf;
  int* lbb;
  uint8_t* freej;
  uint16_t* heads;
  uint16_t* tails;
  int4* lst;
  uint8_t* pos;
  int16_t* pm;
  int16_t* sm;
  __device__ __forceinline__ IvmView(unsigned char* b, const IvmLayout& L) {
    hdr = reinterpret_cast<IvmHdr*>(b);
    cells = reinterpret_cast<int8_t*>(b + L.o_cells);
    V = reinterpret_cast<int8_t*>(b + L.o_v);
    dir = b + L.o_dir;
    endd = reinterpret_cast<int8_t*>(b + L.o_end);
    tgt = reinterpret_cast<int8_t*>(b + L.o_tgt);
    ft = reinterpret_cast<uint16_t*>(b + L.o_ft);
    R = reinterpret_cast<uint16_t*>(b + L.o_r);
    fr = reinterpret_cast<int*>(b + L.o_fr);
    tl = reinterpret_cast<int*>(b + L.o_tl);
    rm = reinterpret_cast<int*>(b + L.o_rm);
    rt = reinterpret_cast<int*>(b + L.o_rt);    // LB1 only
    frm = reinterpret_cast<int*>(b + L.o_frm);
    lbf = reinterpret_cast<int*>(b + L.o_lbf);
    lbb = lbf + L.n;
    freej = b + L.o_free;
    heads = reinterpret_cast<uint16_t*>(b + L.o_heads);
    tails = reinterpret_cast<uint16_t*>(b + L.o_tails);
    lst = reinterpret_cast<int4*>(b + L.o_lst);
    pos = b + L.o_pos;
    pm = reinterpret_cast<int16_t*>(b + L.o_lst);
    sm = pm + L.n * 32;
  }
  template <bool W>
  __device__ __forceinline__ FtT<W>* ftw() const { return reinterpret_cast<FtT<W>*>(ft); }
  template <bool W>
  __device__ __forceinline__ FtT<W>* Rw() const { return reinterpret_cast<FtT<W>*>(R); }
};

struct InstView {
  const int* p32;  // [n][mp]
  const uint32_t* psf;  // [n][mp] sum_{i<k} p | sum_{i<=k} p << 16
  const uint32_t* psb;  // [n][mp] sum_{i>k} p | sum_{i>=k} p << 16
  const uint8_t* pk;
  const uint8_t* pl;
  const uint8_t* ord;
  const uint16_t* lag;
  const uint32_t* packed;  // [n][npairs]: a | job << 7 | b << 13 | lag << 20
  const uint8_t* invord;   // [n][npairs]: position of job j in pair q's order
  const uint16_t* roff;    // [n + 1]: IVM row offsets tri_off(l, n)
  int npairs;
};

// Row offset of IVM level l: a shared-memory table for the lane-group kernels (LB1: their steps
// are issue-bound and select / branch / backtrack each need one), the arithmetic for the
// warp-per-explorer LB2 kernels (left as compiled: their register allocation is tight).
template <int G>
__device__ __forceinline__ int row_off(const InstView& in, int l, int n) {
  if constexpr (G < 32) return in.roff[l];
  else return tri_off(l, n);
}

// ------------------------------------------------------------------ bounding
//
// Input (shared, per explorer): fr/tl/rm/rt/frm tables of the node, freej[0..f-1].
// Output: lbf[c], lbb[c] = bound of the forward child sigma1.j and of the backward child
// j.sigma2 for free job j = freej[c].

// LB1 (src/bound.cpp:61-88), rewritten so each machine costs 4 integer ops per direction:
//   fwd: t = max(prev, front[k]); best = max(best, t + remain[k] + tail[k]); prev = t + p
//   bwd: t = max(prev, tail[k]);  best = max(best, t + front[k] + remain[k]); prev = t + p
// (prev + remain - p + tail with prev = t + p is exactly t + remain + tail).
template <int M, int G>
__device__ __forceinline__ void children_lb1(const Group<G>& grp, const IvmView& iv,
                                             const InstView& in, int mp, int f) {
  // node tables and p rows are padded to mp (a multiple of 4) and 16-byte aligned: LDS.128
  constexpr int Q = (M + 3) / 4;
  const int4* fr4 = reinterpret_cast<const int4*>(iv.fr);
  const int4* rt4 = reinterpret_cast<const int4*>(iv.rt);
  const int4* tl4 = reinterpret_cast<const int4*>(iv.tl);
  const int4* frm4 = reinterpret_cast<const int4*>(iv.frm);
  for (int c = grp.g; c < f; c += G) {
    const int j = iv.freej[c];
    const int4* pr4 = reinterpret_cast<const int4*>(in.p32 + j * mp);
    int prev = 0, best = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int4 a = fr4[q], r = rt4[q], w = pr4[q];
      const int av[4] = {a.x, a.y, a.z, a.w}, rv[4] = {r.x, r.y, r.z, r.w}, pv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (4 * q + e < M) {
          const int t = max(prev, av[e]);
          best = max(best, t + rv[e]);
          prev = t + pv[e];
        }
      }
    }
    iv.lbf[c] = best;
    prev = 0;
    best = 0;
#pragma unroll
    for (int q = Q - 1; q >= 0; --q) {
      const int4 a = tl4[q], r = frm4[q], w = pr4[q];
      const int av[4] = {a.x, a.y, a.z, a.w}, rv[4] = {r.x, r.y, r.z, r.w}, pv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 3; e >= 0; --e) {
        if (4 * q + e < M) {
          const int t = max(prev, av[e]);
          best = max(best, t + rv[e]);
          prev = t + pv[e];
        }
      }
    }
    iv.lbb[c] = best;
  }
}

// LB2: for every machine pair (k<l) the free jobs are taken in that pair's Johnson/Mitten
// order (precomputed per instance); each child c evaluates
//   t0 = r[k], t1 = r[l]; for j in order, j free, j != job(c):
//       t0 += p[j][k]; t1 = max(t1, t0 + lag_j) + p[j][l]
//   lb_kl = max(t0 + q[k], t1 + q[l])
// with (r, q) = (extended head, node tail) for forward children and (node head, extended
// tail) for backward children; LB2 = max over pairs.
// Per pair the group first compacts the node's free jobs in pair order (ballot), then the
// lanes run the 2f child chains over the compacted sequence (broadcast LDS.128 reads).
template <int M, int G>
__device__ __forceinline__ void children_lb2(const Group<G>& grp, const IvmView& iv,
                                             const InstView& in, int n, int mp, int f,
                                             unsigned long long fmask) {
  // child heads / tails
  for (int c = grp.g; c < f; c += G) {
    const int j = iv.freej[c];
    const int* pr = in.p32 + j * mp;
    int prev = 0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      prev = max(prev, iv.fr[k]) + pr[k];
      iv.heads[c * M + k] = static_cast<uint16_t>(prev);
    }
    prev = 0;
#pragma unroll
    for (int k = M - 1; k >= 0; --k) {
      prev = max(prev, iv.tl[k]) + pr[k];
      iv.tails[c * M + k] = static_cast<uint16_t>(prev);
    }
    iv.lbf[c] = 0;
    iv.lbb[c] = 0;
  }
  grp.sync();
  for (int q = 0; q < in.npairs; ++q) {
    const int k = in.pk[q], l = in.pl[q];
    const uint8_t* ord = in.ord + q * n;
    const uint16_t* lag = in.lag + q * n;
    int cnt = 0;
    for (int b0 = 0; b0 < n; b0 += G) {
      const int t = b0 + grp.g;
      const int j = t < n ? ord[t] : 0;
      const bool isf = t < n && ((fmask >> j) & 1ull);
      const unsigned bal = grp.ballot(isf);
      if (isf) {
        const int idx = cnt + __popc(bal & ((1u << grp.g) - 1u));
        iv.lst[idx] = make_int4(in.p32[j * mp + k], in.p32[j * mp + l], lag[j], 0);
        iv.pos[j] = static_cast<uint8_t>(idx);
      }
      cnt += __popc(bal);
    }
    grp.sync();
    const int qk = iv.tl[k], ql = iv.tl[l], rk = iv.fr[k], rl = iv.fr[l];
    for (int cc = grp.g; cc < 2 * f; cc += G) {
      const bool fwd = cc < f;
      const int c = fwd ? cc : cc - f;
      const int s = iv.pos[iv.freej[c]];
      int t0, t1, q0, q1;
      if (fwd) {
        t0 = iv.heads[c * M + k];
        t1 = iv.heads[c * M + l];
        q0 = qk;
        q1 = ql;
      } else {
        t0 = rk;
        t1 = rl;
        q0 = iv.tails[c * M + k];
        q1 = iv.tails[c * M + l];
      }
      for (int i = 0; i < f; ++i) {
        const int4 e = iv.lst[i];
        if (i != s) {
          t0 += e.x;
          t1 = max(t1, t0 + e.z) + e.y;
        }
      }
      const int v = max(t0 + q0, t1 + q1);
      int* dst = fwd ? &iv.lbf[c] : &iv.lbb[c];
      *dst = max(*dst, v);
    }
    grp.sync();
  }
}

// 16x2 unsigned SIMD (sm_90+: VIADD.16x2 / VIADDMNMX.U16x2, one instruction each)
__device__ __forceinline__ uint32_t add_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ int bfind_u32(uint32_t x) {  // index of the highest set bit (FLO)
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t max_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// LB2, warp per explorer, lanes over machine pairs, exact max-plus prefix/suffix form.
// For one pair (k,l) and the node's free jobs s_1..s_f in that pair's Johnson order the
// chain of row a22 unrolls to
//   t1 = max(r_l + B, r_k + max_i X_i),  X_i = A_{<=i} + lag_i + B_{>=i}
// (A, B: sums of p[.][k], p[.][l]); a child that removes s_i = j keeps the X terms before
// i reduced by b_j and those after i reduced by a_j, so with PM_j = max_{i'<i} X_i',
// SM_j = max_{i'>i} X_i' (one forward and one backward pass per pair):
//   t0 = r_k + A - a_j,  t1 = max(r_l + B - b_j, r_k + max(PM_j - b_j, SM_j - a_j))
//   lb_kl(child) = max(t0 + q_k, t1 + q_l)
// Integer-exact, identical values to the per-child chains, O(P (n + f)) per node.
//
// Evaluation form. The child's head on machine m is h_m = h'_m + p_jm with
// h'_m = max(h_{m-1}, front_m) (tails alike: t_m = t'_m + p_jm), so the p_j terms cancel:
//   fwd child (r = child heads, q = node tails):
//     lb = max(h'_k + max(A + q_k, I' + q_l), h'_l + (B + q_l))
//   bwd child (r = node fronts, q = child tails):
//     lb = max(t'_l + max(r_l + B, r_k + I''), t'_k + (r_k + A))
//   I' = max(PM_j + a_j - b_j, SM_j) + B,  I'' = I' + b_j - a_j
// The backward pass stores S_j = max(A + q_k, I' + q_l) | max(r_l + B, r_k + I'') << 16 per
// (job, lane); the child tables hold H'[c][m] = h'_m | t'_m << 16. Every term is a partial
// sum of a bound below 2^16 (the (n+m) max p < 2^16 invariant), so one child costs two
// byte permutes, one VIADD.16x2 and one VIADDMNMX.U16x2 for both directions. Each lane owns
// a pair (32 pairs per round, the last round's spare lanes repeat pair P-1); per child the
// 32 pair bounds are combined with REDUX.MAX.
// Per-lane free-position masks of the current IVM row, one 32-bit word per pair round
// (n <= 32, warp-per-explorer LB2), kept in the explorer's shared scratch ([round][lane],
// IvmLayout::o_msk): bit t of word r is set when the job at position t of pair (32 r + lane)'s
// Johnson order is in the row. A node's free set is its row minus the selected job, so the
// masks follow the explorer incrementally -- branch: the node's masks become the next row's;
// backtrack: the job selected one level up is added back -- instead of being rebuilt from the
// free jobs at every node (f inverse-order lookups per pair round). Rebuilt from the row at
// every launch (the steal / split / exchange kernels only touch the persistent block).
template <int M, bool ON>
struct RowMask {
  uint32_t* w = nullptr;  // this lane's words, stride 32
  int R = 0, P = 0;
  __device__ __forceinline__ void bind(const IvmView& iv, const IvmLayout& L, int npairs) {
    if constexpr (ON) {
      w = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(iv.hdr) + L.o_msk) + (threadIdx.x & 31);
      P = npairs;
      R = (npairs + 31) >> 5;
    }
  }
  __device__ __forceinline__ uint32_t bit(const InstView& in, int job, int r) const {
    const int q = min(32 * r + static_cast<int>(threadIdx.x & 31), P - 1);
    return 1u << in.invord[job * P + q];
  }
  __device__ __forceinline__ void build(const IvmView& iv, const InstView& in, int n, int level) {
    if constexpr (ON) {
      if (level < 0) return;
      const int8_t* row = iv.cells + tri_off(level, n);
      for (int r = 0; r < R; ++r) {
        uint32_t acc = 0;
        for (int c = 0; c < n - level; ++c) {
          const int x = row[c];
          acc |= bit(in, (x < 0 ? -x : x) - 1, r);
        }
        w[r * 32] = acc;
      }
    }
  }
  __device__ __forceinline__ void add(const InstView& in, int job) {
    if constexpr (ON) {
      for (int r = 0; r < R; ++r) w[r * 32] |= bit(in, job, r);
    }
  }
};

// Fold each S_j into child j's bounds inside the backward pass (shared atomicMax, no S table
// pass and no per-child REDUX pair) instead of a separate child loop: measured faster for n > 32
// (ta056 LB2 18.8 -> 22.0 M nodes/s, f ~ 30) and slower for n <= 32 (ta021 LB2 225 -> 275 ms,
// f ~ 10: the lanes' Johnson orders collide on the same jobs and the atomics serialize).
template <bool SMALLN>
constexpr bool kFusedCombine = !SMALLN;

// One pair round of children_lb2_w: lane q's pair, the forward / backward passes over the set
// bits of Fr (the node's free positions in the pair's order), then every child's bound for
// the round's 32 pairs folded into acc (lane c holds child c).
template <int M, bool SMALLN>
__device__ __forceinline__ void lb2_round(const IvmView& iv, const InstView& in, int f, int q0, uint32_t Fr32,
                                          unsigned long long Fq, uint32_t& acc0, uint32_t& acc1) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NEG = -30000;
  const int lane = threadIdx.x & 31;
  const uint32_t* H = reinterpret_cast<const uint32_t*>(iv.heads);  // [c][M] h' | t' << 16
  const int P = in.npairs;
  // packed rows are padded to a multiple of 32 pairs: lane q always reads bank q mod 32,
  // whatever position t each lane is at (the set-bit passes diverge in t)
  const int PS = round_up(P, 32);
  int* Sl = reinterpret_cast<int*>(iv.pm) + lane;  // [j][32]: PM'_j (forward pass), then S_j
  const int q = min(q0 + lane, P - 1);
  const int k = in.pk[q], l = in.pl[q];
  const int Atot = iv.rm[k], Btot = iv.rm[l];
  const int qk = iv.tl[k], ql = iv.tl[l], rk = iv.fr[k], rl = iv.fr[l];
  const int cAq = Atot + qk, cRB = rl + Btot;
  // packed entries e = job << 7 | u << 13 | v << 24 (u = a + lag, v = a - b signed): e & 0x1f80 is
  // the byte offset of row `job` of the per-lane [job][32] int32 table. With E = Btot + sum of
  // v over the earlier free positions, X'_i = X_i + Btot = E + u_i (forward); going backward
  // from G = Atot, G -= v_i gives X'_i = G + u_i. PM' and SM' carry the + Btot, so
  //   I1 = max(PM'_i + v_i, SM'_i),  lo = max(A + q_k, I1 + q_l),  hi = max(r_l + B, I1 + r_k - v_i)
  const unsigned char* pq = reinterpret_cast<const unsigned char*>(in.packed + q);
  const int strideB = PS * 4;
  unsigned char* Sb = reinterpret_cast<unsigned char*>(Sl);
  const uint32_t C = static_cast<uint32_t>(Btot + ql) | static_cast<uint32_t>(rk + Atot) << 16;
  // S_j of the backward pass: kept for the child loop below, or (kFusedCombine<SMALLN>) folded at once
  // into child j's bounds: V = max(H'_k|H'_l + S_j, H'_l|H'_k + C) with job-indexed H' rows and
  // shared-memory atomicMax into the job-indexed lbf / lbb
  const uint32_t* Hk = H + k;
  const int dkl = l - k;
  auto fold = [&](unsigned e, uint32_t S, int* slot) {
    if constexpr (kFusedCombine<SMALLN>) {
      const int job = static_cast<int>((e >> 7) & 63u);
      const uint32_t* hp = Hk + job * M;
      const uint32_t hk = hp[0], hl = hp[dkl];
      const uint32_t V = max_u16x2(add_u16x2(__byte_perm(hk, hl, 0x7610), S), add_u16x2(__byte_perm(hl, hk, 0x7610), C));
      atomicMax(reinterpret_cast<unsigned*>(iv.lbf) + job, V & 0xffffu);
      atomicMax(reinterpret_cast<unsigned*>(iv.lbb) + job, V >> 16);
    } else {
      *slot = static_cast<int>(S);
    }
  };
  if constexpr (SMALLN) {
    // both passes walk exactly the f set bits with bfind: the backward pass on the mask, the
    // forward pass on its bit reversal (position t = 31 - u, address pq31 - u * stride)
    const unsigned char* pq31 = pq + 31 * strideB;
    const int nstride = -strideB;
    int E = Btot, pm = NEG;
    for (uint32_t w = __brev(Fr32); w;) {
      const int u = bfind_u32(w);
      w ^= 1u << u;
      const unsigned e = *reinterpret_cast<const unsigned*>(pq31 + u * nstride);
      *reinterpret_cast<int*>(Sb + (e & 0x1f80u)) = pm;
      pm = max(pm, E + static_cast<int>((e >> 13) & 0x7ffu));
      E += static_cast<int>(e) >> 24;
    }
    int G = Atot, sm = NEG;
    for (uint32_t w = Fr32; w;) {  // descending positions
      const int t = bfind_u32(w);
      w ^= 1u << t;
      const unsigned e = *reinterpret_cast<const unsigned*>(pq + t * strideB);
      int* slot = reinterpret_cast<int*>(Sb + (e & 0x1f80u));
      const int v = static_cast<int>(e) >> 24;
      const int I1 = max(*slot + v, sm);
      const int lo = max(cAq, I1 + ql), hi = max(cRB, I1 + (rk - v));
      fold(e, __byte_perm(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi), 0x5410), slot);
      G -= v;
      sm = max(sm, G + static_cast<int>((e >> 13) & 0x7ffu));
    }
  } else {
    // n <= 64: same set-bit iteration over a 64-bit free-position mask; S_j is folded at once
    // (kFusedCombine), so the per-lane table only carries PM' and is int16 ([job][32] x 2 B)
    static_assert(kFusedCombine<SMALLN>, "the n > 32 path keeps only PM' in its lane table");
    unsigned char* Pb = reinterpret_cast<unsigned char*>(reinterpret_cast<int16_t*>(iv.pm) + lane);
    // the 64-bit mask walked as two 32-bit words (one FLO per set bit instead of the 64-bit
    // find-first / count-leading sequences)
    int E = Btot, pm = NEG;
    auto fwd = [&](int t) {
      const unsigned e = *reinterpret_cast<const unsigned*>(pq + t * strideB);
      *reinterpret_cast<int16_t*>(Pb + ((e & 0x1f80u) >> 1)) = static_cast<int16_t>(pm);
      pm = max(pm, E + static_cast<int>((e >> 13) & 0x7ffu));
      E += static_cast<int>(e) >> 24;
    };
    // every lane's mask has exactly f set bits, but split differently over the two words: one
    // loop of f iterations that switches words when the first runs dry keeps the warp converged
    // (two loops per word would run max(lo bits) + max(hi bits) divergent iterations)
    const uint32_t lo32 = static_cast<uint32_t>(Fq), hi32 = static_cast<uint32_t>(Fq >> 32);
    {
      uint32_t w = __brev(lo32), w2 = __brev(hi32);  // ascending: positions 31 - u, then 63 - u
      int top = 31;
      for (int i = 0; i < f; ++i) {
        if (w == 0) {
          w = w2;
          top = 63;
        }
        const int u = bfind_u32(w);
        w ^= 1u << u;
        fwd(top - u);
      }
    }
    __syncwarp();
    int G = Atot, sm = NEG;
    auto bwd = [&](int t) {
      const unsigned e = *reinterpret_cast<const unsigned*>(pq + t * strideB);
      int* slot = nullptr;
      const int v = static_cast<int>(e) >> 24;
      const int I1 = max(static_cast<int>(*reinterpret_cast<const int16_t*>(Pb + ((e & 0x1f80u) >> 1))) + v, sm);
      const int lo = max(cAq, I1 + ql), hi = max(cRB, I1 + (rk - v));
      fold(e, __byte_perm(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi), 0x5410), slot);
      G -= v;
      sm = max(sm, G + static_cast<int>((e >> 13) & 0x7ffu));
    };
    {
      uint32_t w = hi32;  // descending: positions 32 + t, then t
      int base = 32;
      for (int i = 0; i < f; ++i) {
        if (w == 0) {
          w = lo32;
          base = 0;
        }
        const int t = bfind_u32(w);
        w ^= 1u << t;
        bwd(base + t);
      }
    }
    __syncwarp();
  }
  if constexpr (kFusedCombine<SMALLN>) return;
  const uint32_t* Hl = H + l;
  for (int c = 0; c < f; ++c) {
    const int j = iv.freej[c];
    const uint32_t hk = Hk[c * M], hl = Hl[c * M];
    const uint32_t S = static_cast<uint32_t>(Sl[j * 32]);
    const uint32_t V = max_u16x2(add_u16x2(__byte_perm(hk, hl, 0x7610), S), add_u16x2(__byte_perm(hl, hk, 0x7610), C));
    const uint32_t vF = __reduce_max_sync(FULL, V & 0xffffu);
    const uint32_t vB = __reduce_max_sync(FULL, V) & 0xffff0000u;
    if (SMALLN) {
      if (lane == c) acc0 = max_u16x2(acc0, vF | vB);
    } else if (lane == (c & 31)) {
      if (c < 32) acc0 = max_u16x2(acc0, vF | vB);
      else acc1 = max_u16x2(acc1, vF | vB);
    }
  }
}

// LB2, warp per explorer, lanes over machine pairs, exact max-plus prefix/suffix form.
// (derivation above children_lb2_w's H tables; rounds in lb2_round). With RM (n <= 32 explorer
// path) the node's free-position masks come from the explorer's row masks (RowMask) minus the
// selected job, and become the next row's masks (the caller branches); otherwise they are built
// from the free jobs through the static inverse order.
// n <= 32: returns lane c's child bounds (lbf | lbb << 16; lbf / lbb are not written),
// otherwise writes lbf / lbb.
template <int M, bool SMALLN, bool RM = false>
__device__ __forceinline__ uint32_t children_lb2_w(const IvmView& iv, const InstView& in, int n, int mp, int f,
                                               unsigned long long fmask, RowMask<M, RM>* rowmask = nullptr,
                                               int seljob = 0) {
  const int lane = threadIdx.x & 31;
  uint32_t* H = reinterpret_cast<uint32_t*>(iv.heads);  // [c][M] (kFusedCombine: [job][M]) h' | t' << 16
  for (int c = lane; c < f; c += 32) {
    const int j = iv.freej[c];
    const int* pr = in.p32 + j * mp;
    const int row = kFusedCombine<SMALLN> ? j : c;
    if (kFusedCombine<SMALLN>) iv.lbf[j] = iv.lbb[j] = 0;
    int hp[M];
    int prev = 0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      hp[k] = max(prev, iv.fr[k]);
      prev = hp[k] + pr[k];
    }
    prev = 0;
#pragma unroll
    for (int k = M - 1; k >= 0; --k) {
      const int tp = max(prev, iv.tl[k]);
      prev = tp + pr[k];
      H[row * M + k] = static_cast<uint32_t>(hp[k]) | static_cast<uint32_t>(tp) << 16;
    }
  }
  __syncwarp();
  uint32_t acc0 = 0, acc1 = 0;
  const int P = in.npairs;
  if constexpr (RM) {
    for (int r = 0; r < rowmask->R; ++r) {
      const uint32_t Fr = rowmask->w[r * 32] & ~rowmask->bit(in, seljob, r);
      rowmask->w[r * 32] = Fr;  // the caller branches: the node's free set is the next row
      lb2_round<M, SMALLN>(iv, in, f, 32 * r, Fr, 0, acc0, acc1);
    }
  } else {
    for (int q0 = 0; q0 < P; q0 += 32) {
      const int q = min(q0 + lane, P - 1);
      uint32_t Fr = 0;
      unsigned long long Fq = 0;
      if constexpr (SMALLN) {
        for (int c = 0; c < f; ++c) Fr |= 1u << in.invord[iv.freej[c] * P + q];
      } else {
        for (int c = 0; c < f; ++c) Fq |= 1ull << in.invord[iv.freej[c] * P + q];
      }
      lb2_round<M, SMALLN>(iv, in, f, q0, Fr, Fq, acc0, acc1);
    }
  }
  if constexpr (kFusedCombine<SMALLN>) {  // job-indexed -> child-indexed (lane c holds children c, c + 32)
    __syncwarp();
    int a0 = 0, b0 = 0, a1 = 0, b1 = 0;
    if (lane < f) {
      a0 = iv.lbf[iv.freej[lane]];
      b0 = iv.lbb[iv.freej[lane]];
    }
    if (lane + 32 < f) {
      a1 = iv.lbf[iv.freej[lane + 32]];
      b1 = iv.lbb[iv.freej[lane + 32]];
    }
    acc0 = static_cast<uint32_t>(a0) | static_cast<uint32_t>(b0) << 16;
    acc1 = static_cast<uint32_t>(a1) | static_cast<uint32_t>(b1) << 16;
    __syncwarp();
  }
  if constexpr (!SMALLN) {
    if (lane < f) {
      iv.lbf[lane] = static_cast<int>(acc0 & 0xffffu);
      iv.lbb[lane] = static_cast<int>(acc0 >> 16);
    }
    if (lane + 32 < f) {
      iv.lbf[lane + 32] = static_cast<int>(acc1 & 0xffffu);
      iv.lbb[lane + 32] = static_cast<int>(acc1 >> 16);
    }
  }
  return acc0;
}

// MinMin (src/bound.cpp:109-131): lo over the union, fewer occurrences of lo wins, then the
// larger sum, then Forward.
// Wide times (W): the count and sum differences are reduced separately (the sum of n bounds
// stays below 2^31, validate_times).
template <int G, bool W = false>
__device__ __forceinline__ int minmin(const Group<G>& grp, const IvmView& iv, int f) {
  // one pass: per-lane minimum with its fwd/bwd occurrence counts and the running
  // sum difference; lanes whose minimum is the group's contribute their count difference.
  // One REDUX sums (cf - cb) << 24 + (sf - sb): |sf - sb| < 64 * 2^16 = 2^22 and
  // |cf - cb| <= 64, so both fields survive in 32 bits.
  int lo = INT_MAX, cf = 0, cb = 0, sd = 0;
  for (int c = grp.g; c < f; c += G) {
    const int a = iv.lbf[c], b = iv.lbb[c];
    const int mn = min(a, b);
    if (mn < lo) {
      lo = mn;
      cf = 0;
      cb = 0;
    }
    cf += a == lo;
    cb += b == lo;
    sd += a - b;
  }
  const int glo = grp.rmin(lo);
  if constexpr (W) {
    const int cd = grp.rsum(lo == glo ? cf - cb : 0);
    if (cd) return cd < 0 ? kFwd : kBwd;
    const int v = grp.rsum(sd);
    if (v) return v > 0 ? kFwd : kBwd;
    return kFwd;
  }
  const int v = grp.rsum(((lo == glo ? cf - cb : 0) << 24) + sd);
  const int cd = (v + (1 << 23)) >> 24;
  if (cd) return cd < 0 ? kFwd : kBwd;  // fewer occurrences of lo wins
  if (v) return v > 0 ? kFwd : kBwd;    // then the larger sum
  return kFwd;
}

// MinMin over a warp whose lane c holds child c's bounds (a = forward, b = backward).
__device__ __forceinline__ int minmin_lane(bool valid, int a, int b) {
  constexpr unsigned FULL = 0xffffffffu;
  const int glo = __reduce_min_sync(FULL, valid ? min(a, b) : INT_MAX);
  const int cd = valid ? static_cast<int>(a == glo) - static_cast<int>(b == glo) : 0;
  const int v = __reduce_add_sync(FULL, (cd << 24) + (valid ? a - b : 0));
  const int c = (v + (1 << 23)) >> 24;
  if (c) return c < 0 ? kFwd : kBwd;
  if (v) return v > 0 ? kFwd : kBwd;
  return kFwd;
}

// R (per-machine sum of the jobs of the current row) in registers, machine-chunked like
// node_tables (lane g holds machines g*C .. g*C+C-1): set from the node's remain on branch,
// + p of the job one level up on backtrack; the block's R is only read at entry and written
// at the write-back.
template <int M, int G>
struct RowSum {
  static constexpr int C = (M + G - 1) / G;
  int v[C];
  template <bool W>
  __device__ __forceinline__ void load(const Group<G>& grp, const IvmView& iv) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int k = grp.g * C + c;
      v[c] = k < M ? static_cast<int>(iv.Rw<W>()[k]) : 0;
    }
  }
  template <bool W>
  __device__ __forceinline__ void store(const Group<G>& grp, const IvmView& iv) const {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int k = grp.g * C + c;
      if (k < M) iv.Rw<W>()[k] = static_cast<FtT<W>>(v[c]);
    }
  }
  __device__ __forceinline__ void add(const Group<G>& grp, const int* pr) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int k = grp.g * C + c;
      if (k < M) v[c] += pr[k];
    }
  }
};

// Node tables from the incremental stacks: node at `level` with selected job `job` placed
// by dir[level]; d1/d2 include it. SET: the node's remain becomes the row sum (branch).
// RTF: also write remain + tail / front + remain (LB1's children; not LB2, not leaves)
template <int M, int G, bool W = false, bool RTF = true, bool SET = false>
__device__ __forceinline__ void node_tables(const Group<G>& grp, const IvmView& iv,
                                            const InstView& in, int n, int mp, int job, int dI,
                                            int d1, int d2, RowSum<M, G>& rs) {
  // The extended table (front of sigma1.job, or tail of job.sigma2) is the max-plus
  // recurrence e[k] = max(e[k-1], src[k]) + p[k] (e[M] = 0 backward). Unrolled with the
  // prefix sums of p it is a prefix max: e[k] = Sin[k] + max_{i<=k} (src[i] - Sex[i])
  // (suffix max backward), so each lane scans a chunk of C machines and the group joins the
  // chunks with log2(G) shuffles instead of one lane walking all M machines.
  constexpr int C = (M + G - 1) / G;
  constexpr int NEG = -(1 << 30);
  const FtT<W>* fsrc = iv.ftw<W>() + (dI == kFwd ? d1 - 1 : d1) * M;
  const FtT<W>* tsrc = iv.ftw<W>() + (n - (dI == kBwd ? d2 - 1 : d2)) * M;
  const int* pr = in.p32 + job * mp;
  const int k0 = grp.g * C;
  int loc[C], inc[C];
  int run = NEG;
  if (dI == kFwd) {
    const uint32_t* ps = in.psf + job * mp;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int k = k0 + c;
      if (k < M) {
        const uint32_t u = ps[k];
        run = max(run, static_cast<int>(fsrc[k]) - static_cast<int>(W ? u : u & 0xffffu));
        inc[c] = static_cast<int>(W ? ps[n * mp + k] : u >> 16);
      }
      loc[c] = run;
    }
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int t = __shfl_up_sync(grp.mask, run, o, G);
      if (grp.g >= o) run = max(run, t);
    }
    int ex = __shfl_up_sync(grp.mask, run, 1, G);
    if (grp.g == 0) ex = NEG;
#pragma unroll
    for (int c = 0; c < C; ++c) loc[c] = max(loc[c], ex);
  } else {
    const uint32_t* ps = in.psb + job * mp;
#pragma unroll
    for (int c = C - 1; c >= 0; --c) {
      const int k = k0 + c;
      if (k < M) {
        const uint32_t u = ps[k];
        run = max(run, static_cast<int>(tsrc[k]) - static_cast<int>(W ? u : u & 0xffffu));
        inc[c] = static_cast<int>(W ? ps[n * mp + k] : u >> 16);
      }
      loc[c] = run;
    }
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      const int t = __shfl_down_sync(grp.mask, run, o, G);
      if (grp.g + o < G) run = max(run, t);
    }
    int ex = __shfl_down_sync(grp.mask, run, 1, G);
    if (grp.g == G - 1) ex = NEG;
#pragma unroll
    for (int c = 0; c < C; ++c) loc[c] = max(loc[c], ex);
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int k = k0 + c;
    if (k < M) {
      const int e = inc[c] + loc[c];
      const int rmk = rs.v[c] - pr[k];
      if (SET) rs.v[c] = rmk;
      const int frk = dI == kFwd ? e : static_cast<int>(fsrc[k]);
      const int tlk = dI == kFwd ? static_cast<int>(tsrc[k]) : e;
      iv.rm[k] = rmk;
      iv.fr[k] = frk;
      iv.tl[k] = tlk;
      if (RTF) {
        iv.rt[k] = rmk + tlk;
        iv.frm[k] = frk + rmk;
      }
    }
  }
}

// Free jobs of the node (row minus the selected cell, row order, src/ivm.cpp:164-169).
template <int G>
__device__ __forceinline__ unsigned long long gather_free(const Group<G>& grp, const IvmView& iv,
                                                          const int8_t* row, int sel, int f) {
  unsigned long long m = 0;
  for (int c = grp.g; c < f; c += G) {
    const int x = row[c < sel ? c : c + 1];
    const int j = (x < 0 ? -x : x) - 1;
    iv.freej[c] = static_cast<uint8_t>(j);
    m |= 1ull << j;
  }
  return m;
}

// ------------------------------------------------------------------ explorer steps


// position_reached_end (src/ivm.cpp:90-97): padded V >= end, digit by digit.
template <int G>
__device__ __forceinline__ bool reached_end(const Group<G>& grp, const IvmView& iv, int n, int level) {
  for (int b0 = 0; b0 < n; b0 += G) {
    const int l = b0 + grp.g;
    int pv = 0, ev = 0;
    if (l < n) {
      pv = l <= level ? iv.V[l] : 0;
      ev = iv.endd[l];
    }
    const unsigned b = grp.ballot(pv != ev);
    if (b) {
      const int src = __ffs(b) - 1;
      return grp.bcast(pv, src) > grp.bcast(ev, src);
    }
  }
  return true;
}


// The end test kept incrementally (register state, uniform over the group) instead of a
// digit-by-digit comparison of padded V and end at every select: eq = length of the common
// prefix of V[0..level-1] and end (levels above the current row), lt = V[eq] < end[eq] when
// eq < level, enz = the last non-zero end digit. V only changes at the current row, so a
// descent extends or fixes the prefix and a backtrack truncates it.
struct EndTrack {
  int eq = 0, enz = -1;
  bool lt = false;
  template <int G>
  __device__ __forceinline__ void init(const Group<G>& grp, const IvmView& iv, int n, int level) {
    int d = level, z = -1;
    for (int b0 = 0; b0 < n; b0 += G) {
      const int l = b0 + grp.g;
      const bool in = l < n;
      const int e = in ? iv.endd[l] : 0;
      if (in && l < level && iv.V[l] != e) d = min(d, l);
      if (in && e != 0) z = l;
    }
    eq = grp.rmin(d);
    enz = grp.rmax(z);
    lt = eq < level ? iv.V[eq] < iv.endd[eq] : false;
  }
  // position_reached_end (src/ivm.cpp:90-97) for V[level] = found: padded V >= end
  __device__ __forceinline__ bool reached(const IvmView& iv, int level, int found) const {
    if (eq < level) return !lt;
    const int e = iv.endd[level];
    if (found != e) return found > e;
    return level >= enz;
  }
  __device__ __forceinline__ void descend(const IvmView& iv, int level, int sel) {
    if (eq == level) {
      const int e = iv.endd[level];
      if (sel == e) eq = level + 1;
      else lt = sel < e;
    }
  }
  __device__ __forceinline__ void up(int level) { eq = min(eq, level); }
};

constexpr int kNoHint = -2;

// select_next (src/ivm.cpp:99-122) with the incremental R / d1 / d2 bookkeeping.
// Returns the selected cell, or -1 when the explorer is exhausted. hint: the first unpruned
// cell of the current row when decompose_branch has just written it (-1: every child pruned,
// backtrack at once), so the row is not scanned again; the IVM state stays the reference's.
template <int M, int G, bool RM, bool W = false, bool INC = true>
__device__ __forceinline__ int select_next(const Group<G>& grp, const IvmView& iv,
                                           const InstView& in, int n, int mp, bool has_end,
                                           int& level, int& d1, int& d2, RowMask<M, RM>& rowmask,
                                           RowSum<M, G>& rs, EndTrack& et, int hint = kNoHint) {
  // INC (LB1): the scan start of the row one level up comes back from a backtrack in a register
  // (lane 0's V read broadcast by a shuffle), so V is only ever written by lane 0 and read by
  // the group before a ballot or shuffle that orders it: no group barriers on this path.
  int cnext = -1;
  for (;;) {
    if (level < 0) return -1;
    const int len = n - level;
    const int8_t* row = iv.cells + row_off<G>(in, level, n);
    int found = -1;
    if (hint != kNoHint) {
      // the row was just written by decompose_branch (V = 0): its first unpruned cell is known
      found = hint;
      hint = kNoHint;
    } else {
      const int c0 = (INC && cnext >= 0) ? cnext : iv.V[level];
      for (int b0 = c0; b0 < len; b0 += G) {
        const int c = b0 + grp.g;
        const unsigned b = grp.ballot(c < len && row[c] > 0);
        if (b) {
          found = b0 + __ffs(b) - 1;
          break;
        }
      }
    }
    cnext = -1;
    if (found < 0) {  // row exhausted: backtrack
      const int dl = iv.dir[level];
      d1 -= dl == kFwd;
      d2 -= dl == kBwd;
      if (!INC) grp.sync();
      if (grp.g == 0) iv.V[level] = 0;
      --level;
      if (INC) et.up(level);
      if (level >= 0) {
        const int psel = INC ? grp.bcast(grp.g == 0 ? iv.V[level] : 0, 0) : iv.V[level];
        const int x = iv.cells[row_off<G>(in, level, n) + psel];
        const int job = (x < 0 ? -x : x) - 1;
        rs.add(grp, in.p32 + job * mp);
        rowmask.add(in, job);  // the row one level up holds the job selected there
        if (!INC) grp.sync();
        if (grp.g == 0) iv.V[level] = static_cast<int8_t>(psel + 1);
        cnext = psel + 1;
      }
      if (!INC) grp.sync();
      continue;
    }
    if (!INC) grp.sync();
    if (grp.g == 0) iv.V[level] = static_cast<int8_t>(found);
    if (!INC) grp.sync();
    if (has_end && (INC ? et.reached(iv, level, found) : reached_end(grp, iv, n, level))) return -1;
    return found;
  }
}

struct StepCounters {
  unsigned int decomposed, leaves, dups, improvements, steps, steals;
};

// Decompose the node at (level, sel) and branch (bound.cpp:98-139 + ivm.cpp:124-145).
template <int M, int G, int BOUND, bool SMALLN, bool RM, bool W = false>
__device__ __forceinline__ int decompose_branch(const Group<G>& grp, const IvmView& iv,
                                                 const InstView& in, int n, int mp, int sel,
                                                 int prune, int& level, int& d1, int& d2,
                                                 unsigned* shist, RowMask<M, RM>& rowmask, RowSum<M, G>& rs) {
  const int I = level;
  const int f = n - 1 - I;
  int8_t* row = iv.cells + row_off<G>(in, I, n);
  const int x = row[sel];
  const int job = (x < 0 ? -x : x) - 1;
  const int dI = iv.dir[I];
  node_tables<M, G, W, BOUND == kLB1, true>(grp, iv, in, n, mp, job, dI, d1, d2, rs);
  const unsigned long long fm0 = gather_free<G>(grp, iv, row, sel, f);
  unsigned long long fm = 0;
  if constexpr (BOUND == kLB2) fm = grp.ror64(fm0);  // LB1 does not use the free set mask
  grp.sync();
  int8_t* nrow = iv.cells + row_off<G>(in, I + 1, n);
  int dir, first;
  if constexpr (BOUND == kLB2 && G == 32 && SMALLN) {
    // lane c holds child c's two bounds in registers (no lbf / lbb round trip)
    const uint32_t acc = children_lb2_w<M, SMALLN, RM>(iv, in, n, mp, f, fm, &rowmask, job);
    const int a = static_cast<int>(acc & 0xffffu), b = static_cast<int>(acc >> 16);
    dir = minmin_lane(grp.g < f, a, b);
    const int lb = dir == kFwd ? a : b;
    if (grp.g < f) {
      const int j1 = iv.freej[grp.g] + 1;
      nrow[grp.g] = static_cast<int8_t>(lb >= prune ? -j1 : j1);
    }
    first = __ffs(__ballot_sync(0xffffffffu, grp.g < f && lb < prune)) - 1;
  } else {
    if constexpr (BOUND == kLB1) {
      children_lb1<M, G>(grp, iv, in, mp, f);
    } else if constexpr (G == 32) {
      children_lb2_w<M, SMALLN, RM>(iv, in, n, mp, f, fm, &rowmask, job);
    } else {
      children_lb2<M, G>(grp, iv, in, n, mp, f, fm);
    }
    grp.sync();
    dir = minmin<G, W>(grp, iv, f);
    first = f;
    for (int c = grp.g; c < f; c += G) {
      const int lb = dir == kFwd ? iv.lbf[c] : iv.lbb[c];
      const int j1 = iv.freej[c] + 1;
      nrow[c] = static_cast<int8_t>(lb >= prune ? -j1 : j1);
      if (lb < prune) first = min(first, c);
    }
    first = grp.rmin(first);
    if (first == f) first = -1;
  }
  FtT<W>* ft = iv.ftw<W>();
  for (int k = grp.g; k < M; k += G) {
    if (dI == kFwd) ft[d1 * M + k] = static_cast<FtT<W>>(iv.fr[k]);
    else ft[(n - d2) * M + k] = static_cast<FtT<W>>(iv.tl[k]);
  }
  if (grp.g == 0) {
    iv.dir[I + 1] = static_cast<uint8_t>(dir);
    iv.V[I + 1] = 0;
    atomicAdd(&shist[f], 1u);
  }
  grp.sync();
  level = I + 1;
  d1 += dir == kFwd;
  d2 += dir == kBwd;
  return first;
}

// Leaf: one free job (explorer.cpp:42-57). Makespan of sigma1.j.sigma2 from the node
// tables: C = max_k (front_{sigma1.j}[k] + tail_{sigma2}[k]).
template <int M, int G, bool W = false>
__device__ __forceinline__ void leaf(const Group<G>& grp, const IvmView& iv, const InstView& in, RowSum<M, G>& rs,
                                     int n, int mp, int sel, int level, int d1, int d2,
                                     int improve, DevCounters* ctr, ImpRecord* imp,
                                     StepCounters& sc, unsigned long long* census = nullptr,
                                     int census_cap = 0) {
  int8_t* row = iv.cells + row_off<G>(in, level, n);
  const int x = row[sel];
  const int job = (x < 0 ? -x : x) - 1;
  const int dI = iv.dir[level];
  node_tables<M, G, W, false>(grp, iv, in, n, mp, job, dI, d1, d2, rs);
  grp.sync();
  if (grp.g == 0) {
    const int len = n - level;
    int jf = -1;
    for (int c = 0; c < len; ++c) {
      if (c == sel) continue;
      const int y = row[c];
      jf = (y < 0 ? -y : y) - 1;
    }
    int mk = 0;
    if (jf >= 0) {
      const int* pr = in.p32 + jf * mp;
      int prev = 0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        prev = max(prev, iv.fr[k]) + pr[k];
        mk = max(mk, prev + iv.tl[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < M; ++k) mk = max(mk, iv.fr[k] + iv.tl[k]);
    }
    row[sel] = static_cast<int8_t>(x < 0 ? x : -x);  // prune_current
    ++sc.leaves;
    if (census) {  // census->push_back(ivm.position_u64()) (src/explorer.cpp:47)
      unsigned long long pos = 0;
      for (int l = 0; l < n; ++l) pos = pos * static_cast<unsigned long long>(n - l) + (l <= level ? iv.V[l] : 0);
      const unsigned slot = atomicAdd(&ctr->census_count, 1u);
      if (static_cast<int>(slot) < census_cap) census[slot] = pos;
    }
    if (mk < improve) {
      const int old = atomicMin(&ctr->best, mk);
      if (mk < old) {
        ++sc.improvements;
        // ring of records: the newest (best) improvements survive an overflow; the host
        // re-evaluates every record's schedule and keeps the best valid one
        const int slot = atomicAdd(&ctr->imp_count, 1) % kImpCap;
        {
          ImpRecord* r = imp + slot;
          int a = 0, b = 0;
          for (int l = 0; l <= level; ++l) {
            const int y = iv.cells[tri_off(l, n) + iv.V[l]];
            const int jj = (y < 0 ? -y : y) - 1;
            if (iv.dir[l] == kFwd) r->perm[a++] = static_cast<int8_t>(jj);
            else r->perm[n - 1 - b++] = static_cast<int8_t>(jj);
          }
          if (jf >= 0) r->perm[a] = static_cast<int8_t>(jf);
          r->mk = mk;
        }
      }
    }
  }
  grp.sync();
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Effective start of an explorer's remaining work: the padded V, moved past the current
// cell's subtree when that cell is pruned/consumed (an explorer parked on a pruned cell
// after a replay, or on an evaluated leaf, has already covered the whole subtree; its
// padded V lies *before* its actual progress). Returns false when nothing remains (>= n!).
template <typename T>
__device__ __forceinline__ bool effective_pos(const T* V, int level, const T* cells, int n, int* pos) {
  for (int l = 0; l < n; ++l) pos[l] = l <= level ? V[l] : 0;
  if (cells[tri_off(level, n) + V[level]] > 0) return true;
  for (int l = level; l >= 0; --l) {  // + (n-1-level)!: increment digit `level` with carry
    if (++pos[l] <= n - 1 - l) return true;
    pos[l] = 0;
  }
  return false;
}

// log2 of end - pos: exact factoradic subtraction (borrows from the least significant digit;
// end = n! when !has_end), then the leading non-zero digit (+ the next one) gives the
// magnitude. -1 when nothing remains.
template <typename T>
__device__ __forceinline__ float remaining_log2_pos(const int* pos, const T* E, bool has_end, int n,
                                                    const float* lgfact) {
  int lead = -1, d0 = 0, d1 = 0;
  if (has_end) {
    int borrow = 0;
    int D1 = 0;
    for (int l = n - 1; l >= 0; --l) {
      int d = E[l] - pos[l] - borrow;
      borrow = d < 0;
      if (borrow) d += n - l;
      if (d) {
        lead = l;
        d0 = d;
        d1 = D1;
      }
      D1 = d;
    }
    if (borrow) return -1.f;
  } else {  // n! - pos = ((n! - 1) - pos) + 1
    int carry = 1, D1 = 0;
    for (int l = n - 1; l >= 0; --l) {
      int d = n - 1 - l - pos[l] + carry;
      carry = d > n - 1 - l;
      if (carry) d = 0;
      if (d) {
        lead = l;
        d0 = d;
        d1 = D1;
      }
      D1 = d;
    }
    if (carry) return lgfact[n];
  }
  if (lead < 0) return -1.f;
  float d = static_cast<float>(d0);
  if (lead + 1 < n) d += static_cast<float>(d1) / static_cast<float>(n - 1 - lead);
  return lgfact[n - 1 - lead] + __log2f(d);
}

// ---- remaining work of one explorer for the steal phase: log2 of its leaves, -2 busy /
// unsplittable, -3 idle (lens_kernel, on a shared-memory copy of the block). mode 0: the live
// siblings of the shallowest level holding any (pool.cu live_siblings), (cnt + 1) (n-1-l*)!;
// mode 1: the exact factoradic length of [effective position, end).
__device__ __forceinline__ int live_count(const unsigned char* vb, const IvmLayout& L, int& lstar) {
  const int n = L.n;
  const IvmHdr* h = reinterpret_cast<const IvmHdr*>(vb);
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
    for (int c = V[l] + 1; c < lim; ++c) cnt += row[c] > 0;
    if (cnt) {
      lstar = l;
      return cnt;
    }
  }
  return 0;
}

__device__ __forceinline__ float explorer_lens(const unsigned char* blk, const IvmLayout& L, const float* lgfact, int mode) {
  const IvmHdr* h = reinterpret_cast<const IvmHdr*>(blk);
  if (h->state == kInit) return -2.f;
  if (h->state != kActive) return -3.f;
  float lg = -2.f;
  int cnt = 0;
  if (mode != 1) {
    int lstar = 0;
    cnt = live_count(blk, L, lstar);
    if (cnt > 0) lg = log2f(static_cast<float>(cnt + 1)) + lgfact[L.n - 1 - lstar];
  }
  if (mode == 1 || (mode == 0 && cnt == 0)) {
    int pos[kMaxN];
    if (effective_pos(reinterpret_cast<const int8_t*>(blk + L.o_v), h->level,
                      reinterpret_cast<const int8_t*>(blk + L.o_cells), L.n, pos)) {
      const float r = remaining_log2_pos(pos, reinterpret_cast<const int8_t*>(blk + L.o_end), h->has_end != 0, L.n, lgfact);
      if (r >= 0.f) lg = r;
    }
  }
  return lg;
}

// Prefix / suffix sums of every job's row (node_tables' max-plus scans), built from the
// global p32 table while the CTA stages the instance.
__device__ __forceinline__ void stage_prefix_sums(unsigned char* smem, const InstLayout& IL, const int* p32, int n,
                                                  int mp, bool wide) {
  uint32_t* pf = reinterpret_cast<uint32_t*>(smem + IL.o_psf);
  uint32_t* pb = reinterpret_cast<uint32_t*>(smem + IL.o_psb);
  const int nm = n * mp;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int* pr = p32 + j * mp;
    uint32_t acc = 0;
    for (int k = 0; k < mp; ++k) {
      const uint32_t v = static_cast<uint32_t>(pr[k]);
      if (wide) {
        pf[j * mp + k] = acc;
        pf[nm + j * mp + k] = acc + v;
      } else {
        pf[j * mp + k] = acc | ((acc + v) << 16);
      }
      acc += v;
    }
    acc = 0;
    for (int k = mp - 1; k >= 0; --k) {
      const uint32_t v = static_cast<uint32_t>(pr[k]);
      if (wide) {
        pb[j * mp + k] = acc;
        pb[nm + j * mp + k] = acc + v;
      } else {
        pb[j * mp + k] = acc | ((acc + v) << 16);
      }
      acc += v;
    }
  }
}

// incremental row masks (RowMask, shared memory) for the warp-per-explorer LB2 path with
// n <= 32. (Held in registers instead -- 6 more per lane -- they cost warps and spilled: 249 ms
// vs 227 ms on the ta021 LB2 proof.)
template <int BOUND, int G, bool SMALLN>
constexpr bool kRowMask = BOUND == kLB2 && G == 32 && SMALLN;
template <int BOUND, int G, bool SMALLN>
constexpr int kExploreThreads = 1024;
// Steal lengths evaluated at the explore kernel's write-back (a noinline call, once per explorer
// and launch) instead of by lens_kernel after it: measured per variant -- the call site changes
// ptxas' allocation of the register-capped explorer loop, which the n <= 32 LB2 warp kernel
// likes (ta021 LB2 proof 196 -> 192 ms) and LB1 / n > 32 LB2 do not (ta021 LB1 176 -> 182 ms,
// ta056 LB2 30 -> 24 M nodes/s at 5 s).
template <int BOUND, int G, bool SMALLN>
constexpr bool kLensInKernel = BOUND == kLB2 && G == 32 && SMALLN;
__device__ __noinline__ float explorer_lens_call(const unsigned char* blk, const IvmLayout& L, const float* lgfact,
                                                 int mode) {
  return explorer_lens(blk, L, lgfact, mode);
}

// W: wide (32-bit) FT / R / prefix sums, LB1 only (pool_init)
template <int M, int G, int BOUND, bool SMALLN = false, bool W = false>
__global__ void __launch_bounds__(kExploreThreads<BOUND, G, SMALLN>) explore_kernel(const ExploreParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const IvmLayout& L = P.L;
  const int n = L.n, mp = L.mp;
  const int NG = blockDim.x / G;  // explorers per CTA
  constexpr bool PACKED = BOUND == kLB2 && G == 32;
  constexpr bool RM = kRowMask<BOUND, G, SMALLN>;
  const InstLayout IL = inst_layout(n, mp, BOUND == kLB2 ? P.npairs : 0, PACKED, W);

  // ---- stage the instance (and LB2 pair tables) into shared memory
  {
    int* sp = reinterpret_cast<int*>(smem + IL.o_p32);
    for (int i = threadIdx.x; i < n * mp; i += blockDim.x) sp[i] = P.p32[i];
    stage_prefix_sums(smem, IL, P.p32, n, mp, W);
    for (int i = threadIdx.x; i <= n; i += blockDim.x) reinterpret_cast<uint16_t*>(smem + IL.o_roff)[i] = static_cast<uint16_t>(tri_off(i, n));
    if (PACKED) {
      uint32_t* sk = reinterpret_cast<uint32_t*>(smem + IL.o_pk32);
      for (int i = threadIdx.x; i < round_up(P.npairs, 32) * n; i += blockDim.x) sk[i] = P.packed[i];
      for (int i = threadIdx.x; i < P.npairs * n; i += blockDim.x) smem[IL.o_inv + i] = P.invord[i];
      for (int i = threadIdx.x; i < P.npairs; i += blockDim.x) {
        smem[IL.o_pk + i] = P.pk[i];
        smem[IL.o_pl + i] = P.pl[i];
      }
    } else if (BOUND == kLB2) {
      uint16_t* sl = reinterpret_cast<uint16_t*>(smem + IL.o_lag);
      for (int i = threadIdx.x; i < P.npairs * n; i += blockDim.x) {
        sl[i] = P.lag[i];
        smem[IL.o_ord + i] = P.order[i];
      }
      for (int i = threadIdx.x; i < P.npairs; i += blockDim.x) {
        smem[IL.o_pk + i] = P.pk[i];
        smem[IL.o_pl + i] = P.pl[i];
      }
    }
    unsigned* h = reinterpret_cast<unsigned*>(smem + IL.o_hist);
    unsigned* dh = reinterpret_cast<unsigned*>(smem + IL.o_dhist);
    for (int i = threadIdx.x; i <= n; i += blockDim.x) h[i] = dh[i] = 0;
    unsigned* cnt = reinterpret_cast<unsigned*>(smem + IL.o_cnt);
    if (threadIdx.x < 16) cnt[threadIdx.x] = 0;
  }
  // ---- stage this CTA's explorers (a warp per explorer block, 16-byte words over the lanes)
  const int first = blockIdx.x * NG;
  unsigned char* ivbase = smem + IL.bytes;
  {
    const int words = L.gstride / 16, nw = blockDim.x >> 5;
    for (int i = threadIdx.x >> 5; i < NG && first + i < P.K; i += nw) {
      const uint4* src = reinterpret_cast<const uint4*>(P.state + static_cast<size_t>(first + i) * L.gstride);
      uint4* dst = reinterpret_cast<uint4*>(ivbase + i * L.sstride);
      for (int w = threadIdx.x & 31; w < words; w += 32) dst[w] = src[w];
    }
  }
  __syncthreads();

  InstView in;
  in.p32 = reinterpret_cast<const int*>(smem + IL.o_p32);
  in.psf = reinterpret_cast<const uint32_t*>(smem + IL.o_psf);
  in.psb = reinterpret_cast<const uint32_t*>(smem + IL.o_psb);
  in.pk = smem + IL.o_pk;
  in.pl = smem + IL.o_pl;
  in.ord = smem + IL.o_ord;
  in.lag = reinterpret_cast<const uint16_t*>(smem + IL.o_lag);
  in.packed = reinterpret_cast<const uint32_t*>(smem + IL.o_pk32);
  in.invord = smem + IL.o_inv;
  in.roff = reinterpret_cast<const uint16_t*>(smem + IL.o_roff);
  in.npairs = P.npairs;
  unsigned* shist = reinterpret_cast<unsigned*>(smem + IL.o_hist);
  unsigned* sdhist = reinterpret_cast<unsigned*>(smem + IL.o_dhist);

  Group<G> grp;
  const int gi = threadIdx.x / G;
  StepCounters sc = {0, 0, 0, 0, 0, 0};
  if (first + gi < P.K) {
    IvmView iv(ivbase + gi * L.sstride, L);
    int level = iv.hdr->level, state = iv.hdr->state, d1 = iv.hdr->d1, d2 = iv.hdr->d2;
    int rlev = iv.hdr->rlev, nrep = iv.hdr->nrep;
    const bool has_end = iv.hdr->has_end != 0;
    RowMask<M, RM> rowmask;
    rowmask.bind(iv, L, in.npairs);
    if (state != kEmpty) rowmask.build(iv, in, n, level);
    RowSum<M, G> rs;
    rs.template load<W>(grp, iv);
    if (grp.g == 0 && state != kEmpty) atomicAdd(reinterpret_cast<unsigned*>(smem + IL.o_cnt) + 6, 1u);
    int best = grp.bcast(grp.g == 0 ? *reinterpret_cast<volatile int*>(&P.ctr->best) : 0, 0);
    int step = 0, hint = kNoHint;
    // the survivor hint and the incremental end test pay for LB1 (select / backtrack dominate
    // its steps: ta021 proof 192 -> 176 ms); the LB2 warp kernels are register-capped and lose
    // more to the extra live state than the selects cost them (ta021 LB2 192 -> 199 ms)
    constexpr bool INC = BOUND == kLB1;
    EndTrack et;
    if (INC && has_end && state == kActive) et.init(grp, iv, n, level);
    unsigned long long t_end = ~0ull;
    if (P.budget_ns) t_end = globaltimer_ns() + P.budget_ns;
    while (step < P.steps) {
      // budget check every 4th step; every step for LB2 warps (a step costs tens of us there,
      // and the whole CTA waits for its slowest explorer at the round's end)
      constexpr int kCheck = (BOUND == kLB2 && G == 32) ? 0 : 3;
      if (P.budget_ns && (step & kCheck) == 0 && grp.bcast(grp.g == 0 ? (globaltimer_ns() >= t_end) : 0, 0)) break;
      if (state == kEmpty) break;
      if ((step & 15) == 15) best = grp.bcast(grp.g == 0 ? *reinterpret_cast<volatile int*>(&P.ctr->best) : 0, 0);
      ++step;
      const int prune = P.prune_mode == 0 ? best : (P.prune_mode == 1 ? P.pinned_ub : INT_MAX);
      const int improve = P.prune_mode == 1 ? 0 : best;
      ++sc.steps;
      if (state == kInit) {
        // one replay level of init_at (src/ivm.cpp:70-86); under the reference steal policy the
        // replay is part of the steal phase (synchronous there), not of the round's batch steps
        step -= P.free_replay;
        const int l = rlev;
        const int digit = iv.tgt[l];
        int8_t* row = iv.cells + tri_off(l, n);
        level = l;
        for (int c = grp.g; c < digit; c += G) {
          const int x = row[c];
          if (x > 0) row[c] = static_cast<int8_t>(-x);
        }
        grp.sync();
        if (grp.g == 0) iv.V[l] = static_cast<int8_t>(digit);
        grp.sync();
        if (row[digit] < 0 || l >= n - 2) {
          // positioned: duplicates = min(L, lnz(a)) (SURVEY.md §7 hard part 1)
          int lz = 0;
          for (int t = grp.g; t < n; t += G)
            if (iv.tgt[t] != 0) lz = max(lz, t);
          lz = grp.rmax(lz);
          const int dup = min(nrep, lz);
          if (grp.g == 0) {
            sc.dups += dup;
            for (int t = 0; t < dup; ++t) atomicAdd(&sdhist[n - 1 - t], 1u);
          }
          state = kActive;
          if (INC && has_end) et.init(grp, iv, n, level);
          continue;
        }
        decompose_branch<M, G, BOUND, SMALLN, RM, W>(grp, iv, in, n, mp, digit, prune, level, d1, d2, shist, rowmask, rs);
        ++sc.decomposed;
        ++nrep;
        rlev = level;
        continue;
      }
      const int sel = select_next<M, G, RM, W, INC>(grp, iv, in, n, mp, has_end, level, d1, d2, rowmask, rs, et, hint);
      hint = kNoHint;
      if (sel < 0) {
        state = kEmpty;
        break;
      }
      if (n - 1 - level <= 1) {
        leaf<M, G, W>(grp, iv, in, rs, n, mp, sel, level, d1, d2, improve, P.ctr, P.imp, sc, P.census, P.census_cap);
        continue;
      }
      if (INC && has_end) et.descend(iv, level, sel);
      hint = decompose_branch<M, G, BOUND, SMALLN, RM, W>(grp, iv, in, n, mp, sel, prune, level, d1, d2, shist, rowmask, rs);
      if (!INC) hint = kNoHint;
      ++sc.decomposed;
    }
    rs.template store<W>(grp, iv);
    if (grp.g == 0) {
      iv.hdr->level = static_cast<int16_t>(level);
      iv.hdr->state = static_cast<uint8_t>(state);
      iv.hdr->d1 = static_cast<uint8_t>(d1);
      iv.hdr->d2 = static_cast<uint8_t>(d2);
      iv.hdr->rlev = static_cast<uint8_t>(rlev);
      iv.hdr->nrep = static_cast<uint8_t>(nrep);
      if constexpr (kLensInKernel<BOUND, G, SMALLN>)
        if (P.lens) P.lens[first + gi] = explorer_lens_call(reinterpret_cast<const unsigned char*>(iv.hdr), L, P.lgfact, P.lens_mode);
      unsigned* cnt = reinterpret_cast<unsigned*>(smem + IL.o_cnt);
      atomicAdd(&cnt[0], sc.decomposed);
      atomicAdd(&cnt[1], sc.leaves);
      atomicAdd(&cnt[2], sc.dups);
      atomicAdd(&cnt[3], sc.improvements);
      atomicAdd(&cnt[4], sc.steps);
      atomicAdd(&cnt[5], sc.steals);
    }
  }
  __syncthreads();
  // ---- write back explorers and counters
  {
    const int words = L.gstride / 16, nw = blockDim.x >> 5;
    for (int i = threadIdx.x >> 5; i < NG && first + i < P.K; i += nw) {
      uint4* dst = reinterpret_cast<uint4*>(P.state + static_cast<size_t>(first + i) * L.gstride);
      const uint4* src = reinterpret_cast<const uint4*>(ivbase + i * L.sstride);
      for (int w = threadIdx.x & 31; w < words; w += 32) dst[w] = src[w];
    }
    const unsigned* cnt = reinterpret_cast<const unsigned*>(smem + IL.o_cnt);
    if (threadIdx.x == 0) {
      if (cnt[0]) atomicAdd(&P.ctr->decomposed, static_cast<unsigned long long>(cnt[0]));
      if (cnt[1]) atomicAdd(&P.ctr->leaves, static_cast<unsigned long long>(cnt[1]));
      if (cnt[2]) atomicAdd(&P.ctr->dups, static_cast<unsigned long long>(cnt[2]));
      if (cnt[3]) atomicAdd(&P.ctr->improvements, static_cast<unsigned long long>(cnt[3]));
      if (cnt[4]) atomicAdd(&P.ctr->steps, static_cast<unsigned long long>(cnt[4]));
      if (cnt[5]) {
        atomicAdd(&P.ctr->steals, static_cast<unsigned long long>(cnt[5]));
        atomicAdd(&P.ctr->inits, static_cast<unsigned long long>(cnt[5]));
      }
      if (cnt[6]) atomicAdd(&P.ctr->round_live, static_cast<int>(cnt[6]));
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x) {
      if (shist[i]) atomicAdd(&P.hist[i], static_cast<unsigned long long>(shist[i]));
      if (sdhist[i]) atomicAdd(&P.dhist[i], static_cast<unsigned long long>(sdhist[i]));
    }
  }
}

// Batched decompose of explicit nodes (the per-node parity hook, bound.hpp:78-79):
// node i = perm[i*n .. i*n+n-1], d1[i], d2[i]. Tables are rebuilt from scratch
// (bound_tables, src/bound.cpp:20-46); outputs are the chosen-direction bounds.
struct BatchParams {
  IvmLayout L;
  const int* perms;
  const int* d1;
  const int* d2;
  int count;
  int incumbent;
  const int* p32;
  int npairs;
  const uint8_t* pk;
  const uint8_t* pl;
  const uint8_t* order;
  const uint16_t* lag;
  const uint32_t* packed;
  const uint8_t* invord;
  int* child_lb;   // [count*n]
  int* lb_fwd;     // [count*n] both sets (before MinMin), for the parity tests
  int* lb_bwd;
  uint8_t* dir;    // [count]
  uint8_t* pruned; // [count*n]
};

template <int M, int G, int BOUND, bool SMALLN = false, bool W = false>
__global__ void __launch_bounds__(1024) decompose_batch_kernel(const BatchParams B) {
  extern __shared__ __align__(128) unsigned char smem[];
  const IvmLayout& L = B.L;
  const int n = L.n, mp = L.mp;
  const int NG = blockDim.x / G;
  constexpr bool PACKED = BOUND == kLB2 && G == 32;
  const InstLayout IL = inst_layout(n, mp, BOUND == kLB2 ? B.npairs : 0, PACKED, W);
  {
    int* sp = reinterpret_cast<int*>(smem + IL.o_p32);
    for (int i = threadIdx.x; i < n * mp; i += blockDim.x) sp[i] = B.p32[i];
    stage_prefix_sums(smem, IL, B.p32, n, mp, W);
    for (int i = threadIdx.x; i <= n; i += blockDim.x) reinterpret_cast<uint16_t*>(smem + IL.o_roff)[i] = static_cast<uint16_t>(tri_off(i, n));
    if (PACKED) {
      uint32_t* sk = reinterpret_cast<uint32_t*>(smem + IL.o_pk32);
      for (int i = threadIdx.x; i < round_up(B.npairs, 32) * n; i += blockDim.x) sk[i] = B.packed[i];
      for (int i = threadIdx.x; i < B.npairs * n; i += blockDim.x) smem[IL.o_inv + i] = B.invord[i];
      for (int i = threadIdx.x; i < B.npairs; i += blockDim.x) {
        smem[IL.o_pk + i] = B.pk[i];
        smem[IL.o_pl + i] = B.pl[i];
      }
    } else if (BOUND == kLB2) {
      uint16_t* sl = reinterpret_cast<uint16_t*>(smem + IL.o_lag);
      for (int i = threadIdx.x; i < B.npairs * n; i += blockDim.x) {
        sl[i] = B.lag[i];
        smem[IL.o_ord + i] = B.order[i];
      }
      for (int i = threadIdx.x; i < B.npairs; i += blockDim.x) {
        smem[IL.o_pk + i] = B.pk[i];
        smem[IL.o_pl + i] = B.pl[i];
      }
    }
  }
  __syncthreads();
  InstView in;
  in.p32 = reinterpret_cast<const int*>(smem + IL.o_p32);
  in.psf = reinterpret_cast<const uint32_t*>(smem + IL.o_psf);
  in.psb = reinterpret_cast<const uint32_t*>(smem + IL.o_psb);
  in.pk = smem + IL.o_pk;
  in.pl = smem + IL.o_pl;
  in.ord = smem + IL.o_ord;
  in.lag = reinterpret_cast<const uint16_t*>(smem + IL.o_lag);
  in.packed = reinterpret_cast<const uint32_t*>(smem + IL.o_pk32);
  in.invord = smem + IL.o_inv;
  in.roff = reinterpret_cast<const uint16_t*>(smem + IL.o_roff);
  in.npairs = B.npairs;
  Group<G> grp;
  const int gi = threadIdx.x / G;
  IvmView iv(smem + IL.bytes + gi * L.sstride, L);
  for (int node = blockIdx.x * NG + gi; node < B.count; node += gridDim.x * NG) {
    const int* perm = B.perms + static_cast<size_t>(node) * n;
    const int d1 = B.d1[node], d2 = B.d2[node];
    const int f = n - d1 - d2;
    if (grp.g == 0) {
      for (int k = 0; k < M; ++k) iv.fr[k] = iv.tl[k] = iv.rm[k] = 0;
      for (int i = 0; i < d1; ++i) {  // front (bound.cpp:25-30)
        const int* pr = in.p32 + perm[i] * mp;
        int prev = 0;
        for (int k = 0; k < M; ++k) {
          prev = max(prev, iv.fr[k]) + pr[k];
          iv.fr[k] = prev;
        }
      }
      for (int i = n - 1; i >= n - d2; --i) {  // tail (bound.cpp:35-39)
        const int* pr = in.p32 + perm[i] * mp;
        int prev = 0;
        for (int k = M - 1; k >= 0; --k) {
          prev = max(prev, iv.tl[k]) + pr[k];
          iv.tl[k] = prev;
        }
      }
      for (int i = d1; i < n - d2; ++i) {
        const int* pr = in.p32 + perm[i] * mp;
        for (int k = 0; k < M; ++k) iv.rm[k] += pr[k];
      }
      if constexpr (BOUND == kLB1) {
        for (int k = 0; k < M; ++k) {
          iv.rt[k] = iv.rm[k] + iv.tl[k];
          iv.frm[k] = iv.fr[k] + iv.rm[k];
        }
      }
    }
    unsigned long long fm = 0;
    for (int c = grp.g; c < f; c += G) {
      const int j = perm[d1 + c];
      iv.freej[c] = static_cast<uint8_t>(j);
      fm |= 1ull << j;
    }
    fm = grp.ror64(fm);
    grp.sync();
    if constexpr (BOUND == kLB2 && G == 32 && SMALLN) {  // lane c: child c's bounds in registers
      const uint32_t acc = children_lb2_w<M, SMALLN>(iv, in, n, mp, f, fm);
      const int a = static_cast<int>(acc & 0xffffu), b = static_cast<int>(acc >> 16);
      const int dir = minmin_lane(grp.g < f, a, b);
      if (grp.g < f) {
        const size_t o = static_cast<size_t>(node) * n + grp.g;
        const int lb = dir == kFwd ? a : b;
        B.child_lb[o] = lb;
        B.lb_fwd[o] = a;
        B.lb_bwd[o] = b;
        B.pruned[o] = lb >= B.incumbent;
      }
      if (grp.g == 0) B.dir[node] = static_cast<uint8_t>(dir);
      grp.sync();
      continue;
    }
    if constexpr (BOUND == kLB1) children_lb1<M, G>(grp, iv, in, mp, f);
    else if constexpr (G == 32) children_lb2_w<M, SMALLN>(iv, in, n, mp, f, fm);
    else children_lb2<M, G>(grp, iv, in, n, mp, f, fm);
    grp.sync();
    const int dir = minmin<G, W>(grp, iv, f);
    for (int c = grp.g; c < f; c += G) {
      const int lb = dir == kFwd ? iv.lbf[c] : iv.lbb[c];
      B.child_lb[static_cast<size_t>(node) * n + c] = lb;
      B.lb_fwd[static_cast<size_t>(node) * n + c] = iv.lbf[c];
      B.lb_bwd[static_cast<size_t>(node) * n + c] = iv.lbb[c];
      B.pruned[static_cast<size_t>(node) * n + c] = lb >= B.incumbent;
    }
    if (grp.g == 0) B.dir[node] = static_cast<uint8_t>(dir);
    grp.sync();
  }
}

#endif  // __CUDACC__

}  // namespace pbbgpu
