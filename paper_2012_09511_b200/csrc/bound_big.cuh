// Batched decompose for large instances (64 < n <= 512, e.g. ta111 500x20): the
// bounding-throughput path of BASELINE config 5.
//
//   LB1  two kernels, chosen per batch by the host (mean f vs n/2):
//        decompose_big_lb1g_kernel  lane-per-node node tables (one register recurrence over
//                                   sigma1 then reversed sigma2), lane-per-child children
//        decompose_big_lb1_kernel   warp per node: lane-per-machine wavefront tables,
//                                   lane-per-child children
//        (bound_tables / children_bounds / decompose, src/bound.cpp:20-139)
//   LB2  decompose_big_kernel, one 256-thread CTA per node: wavefront node tables, child
//        heads/tails, then a thread per machine pair (P = 190 for m = 20) walks only the
//        free positions of its Johnson order (per-pair bitmask built from the inverse-order
//        table, f set bits): the forward pass stores PM_j, the backward pass carries SM and
//        evaluates every child in O(1) (max-plus prefix/suffix form, explore.cuh); the
//        order entries stream from L2 16 per thread in flight; per-child maxima over pairs
//        by shared-memory atomicMax; block MinMin (src/bound.cpp:109-138)
#pragma once

#include "explore.cuh"

namespace pbbgpu {

constexpr int kBigMaxN = 512;
constexpr int kBigThreads = 256;
constexpr int kPf = 16;  // LB2 pair passes: order entries prefetched per thread

struct BigBatchParams {
  int n, m, mp, npairs;
  const int* perms;
  const int* d1;
  const int* d2;
  int count;
  int incumbent;
  const int* p32;        // [n][mp]
  const uint8_t* pk;
  const uint8_t* pl;
  const uint2* packed;   // [n][npairs]: x = job | a << 16, y = b | lag << 16
  const uint16_t* inv16; // [n][npairs]: position of job j in pair q's Johnson order
  int* scratch;          // [gridDim.x][n][kBigThreads]: PM_j of the thread's pair
  int* child_lb;         // [count*n]
  int* lb_fwd;
  int* lb_bwd;
  uint8_t* dir;
  uint8_t* pruned;
};

__host__ __device__ inline int big_smem_bytes(int n, int mp, int m) {
  return n * mp * 4 + 2 * n * m * 2 + round_up(n, 16) + 2 * n * 4 + 3 * round_up(m, 4) * 4 + 64 * 4 + round_up(n, 8) * 2 +
         m * (m - 1) / 2 * ((n + 31) / 32) * 4;
}

#ifdef __CUDACC__

// One lane of a max-plus wavefront over `len` jobs of the warp's staged perm (forward from
// position 0, or backward from n-1 when rev): at step s the lane at wave position wp handles
// job s - wp on machine k. The loads are independent of the chain, so they run two steps
// ahead (indices clamped into range; out-of-range steps leave C unchanged and add 0).
// MP = 0: row stride passed at run time.
template <int MP, typename PT = int>
__device__ __forceinline__ void big_wave(const PT* sp, const uint16_t* spm, int n, int len, bool rev, int k,
                                         int wp, bool act, int steps, int& C, int& sum, int mp = MP) {
  const int hi = max(len - 1, 0);
  auto at = [&](int s) {
    const int i = min(max(s - wp, 0), hi);
    return static_cast<int>(spm[rev ? n - 1 - i : i]);
  };
  int jn = at(1);
  int pn = static_cast<int>(sp[at(0) * mp + k]);
  for (int s = 0; s < steps; ++s) {
    const int pv = pn;
    pn = static_cast<int>(sp[jn * mp + k]);
    jn = at(s + 2);
    int left = __shfl_up_sync(0xffffffffu, C, 1);
    if (wp == 0) left = 0;
    const int i = s - wp;
    if (act && i >= 0 && i < len) {
      C = max(C, left) + pv;
      sum += pv;
    }
  }
}

template <int M, int BOUND>
__global__ void __launch_bounds__(kBigThreads) decompose_big_kernel(const BigBatchParams B) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = B.n, mp = B.mp, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* sp = reinterpret_cast<int*>(smem);                         // [n][mp]
  uint16_t* heads = reinterpret_cast<uint16_t*>(sp + n * mp);     // [job][M]
  uint16_t* tails = heads + n * M;
  int* accf = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(tails + n * M) + round_up(n, 16));  // [job]
  int* accb = accf + n;
  int* fr = accb + n;  // [mp] each
  int* tl = fr + round_up(M, 4);
  int* rm = tl + round_up(M, 4);
  int* red = rm + round_up(M, 4);  // 8 x 4 reduction scratch
  uint16_t* spm = reinterpret_cast<uint16_t*>(red + 64);  // the node's perm
  const int MW = (n + 31) >> 5;
  uint32_t* fmask = reinterpret_cast<uint32_t*>(spm + round_up(n, 8));  // LB2: [MW][pair] free positions
  for (int i = tid; i < n * mp; i += blockDim.x) sp[i] = B.p32[i];
  __syncthreads();
  for (int node = blockIdx.x; node < B.count; node += gridDim.x) {
    const int* perm = B.perms + static_cast<size_t>(node) * n;
    const int d1 = B.d1[node], d2 = B.d2[node], f = n - d1 - d2;
    if (d1 < 0) continue;  // no node in this slot (big explorer pool steps)
    for (int j = tid; j < n; j += blockDim.x) {
      accf[j] = 0;
      accb[j] = 0;
    }
    if (tid < M) rm[tid] = 0;
    if (BOUND == kLB2)
      for (int i = tid; i < B.npairs * MW; i += blockDim.x) fmask[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) spm[i] = static_cast<uint16_t>(perm[i]);
    __syncthreads();
    if (BOUND == kLB2 && warp >= 2) {
      // per pair, the free jobs' positions in its Johnson order as a bitmask, word-major
      // ([MW][pair]: the pairs of a warp hit distinct banks), built by warps 2.. while warps 0/1
      // run the node-table wavefronts
      static_assert(kBigThreads - 64 >= 20 * 19 / 2, "a mask thread per pair (m <= 20)");
      const int P = B.npairs, t0 = tid - 64, cs = (kBigThreads - 64) / P;  // thread -> (pair, first child)
      if (t0 < cs * P) {
        const int q = t0 % P;
        int c = t0 / P;
        for (; c + 15 * cs < f; c += 16 * cs) {  // 16 inverse-order loads in flight
          int pos[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) pos[u] = B.inv16[static_cast<size_t>(spm[d1 + c + u * cs]) * P + q];
#pragma unroll
          for (int u = 0; u < 16; ++u) atomicOr(&fmask[(pos[u] >> 5) * P + q], 1u << (pos[u] & 31));
        }
        for (; c < f; c += cs) {
          const int pos = B.inv16[static_cast<size_t>(spm[d1 + c]) * P + q];
          atomicOr(&fmask[(pos >> 5) * P + q], 1u << (pos & 31));
        }
      }
    }
    if (warp < 2) {  // front (warp 0) / tail (warp 1): wavefronts over (job, machine)
      int C = 0, unused = 0;
      const int k = warp ? M - 1 - lane : lane;
      if (warp == 0) big_wave<0>(sp, spm, n, d1, false, lane < M ? k : 0, lane, lane < M, d1 + M - 1, C, unused, mp);
      else big_wave<0>(sp, spm, n, d2, true, lane < M ? k : 0, lane, lane < M, d2 + M - 1, C, unused, mp);
      if (lane < M) (warp ? tl : fr)[k] = C;
    }
    {  // remain: per-warp partial sums over the free jobs, lane = machine
      int acc = 0;
      if (lane < M)
        for (int c = warp; c < f; c += blockDim.x / 32) acc += sp[spm[d1 + c] * mp + lane];
      __syncthreads();
      if (lane < M) atomicAdd(&rm[lane], acc);
    }
    __syncthreads();
    if (BOUND == kLB1) {
      for (int c = tid; c < f; c += blockDim.x) {
        const int j = spm[d1 + c];
        const int* pr = sp + j * mp;
        int prev = 0, best = 0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const int t = max(prev, fr[k]);
          best = max(best, t + rm[k] + tl[k]);
          prev = t + pr[k];
        }
        accf[j] = best;
        prev = 0;
        best = 0;
#pragma unroll
        for (int k = M - 1; k >= 0; --k) {
          const int t = max(prev, tl[k]);
          best = max(best, t + fr[k] + rm[k]);
          prev = t + pr[k];
        }
        accb[j] = best;
      }
    } else {
      for (int c = tid; c < f; c += blockDim.x) {  // child heads / tails, by job
        const int j = spm[d1 + c];
        const int* pr = sp + j * mp;
        int prev = 0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          prev = max(prev, fr[k]) + pr[k];
          heads[j * M + k] = static_cast<uint16_t>(prev);
        }
        prev = 0;
#pragma unroll
        for (int k = M - 1; k >= 0; --k) {
          prev = max(prev, tl[k]) + pr[k];
          tails[j * M + k] = static_cast<uint16_t>(prev);
        }
      }
      __syncthreads();
      int* PM = B.scratch + static_cast<size_t>(blockIdx.x) * n * kBigThreads + tid;
      constexpr int NEG = -(1 << 29);
      for (int q = tid; q < B.npairs; q += blockDim.x) {
        const int k = B.pk[q], l = B.pl[q];
        const int Atot = rm[k], Btot = rm[l];
        const int qk = tl[k], ql = tl[l], rk = fr[k], rl = fr[l];
        int A = 0, Bp = 0, pm = NEG;
        const uint2* col = B.packed + q;
        {
        // the pair's Johnson order streams from L2, only at the free positions (set bits of
        // the pair's mask, f of them): kPf entries in flight per thread
        // PM_i is kept by rank (the i-th free position of the walk): every thread of a warp is
        // at the same rank at every step, so the scratch accesses are coalesced
        const uint32_t* mk = fmask + q;
        const int P = B.npairs;
        int w = 0, rank = 0;
        uint32_t bits = mk[0];
        for (int left = f; left > 0; left -= kPf) {
          const int cnt = min(left, kPf);
          uint2 ev[kPf];
#pragma unroll
          for (int u = 0; u < kPf; ++u) {
            if (u < cnt) {
              while (bits == 0) bits = mk[++w * P];
              const int t = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              ev[u] = col[static_cast<size_t>(t) * B.npairs];
            }
          }
#pragma unroll
          for (int u = 0; u < kPf; ++u) {
            if (u < cnt) {
              const uint2 e = ev[u];
              A += e.x >> 16;
              const int X = A + static_cast<int>(e.y >> 16) - Bp;
              PM[(rank++) * kBigThreads] = pm;
              pm = max(pm, X);
              Bp += e.y & 0xffff;
            }
          }
        }
        int As = 0, Bs = Atot - Btot, sm = NEG;
        w = MW - 1;
        bits = mk[w * P];
        for (int left = f; left > 0; left -= kPf) {
          const int cnt = min(left, kPf);
          uint2 ev[kPf];
#pragma unroll
          for (int u = 0; u < kPf; ++u) {
            if (u < cnt) {
              while (bits == 0) bits = mk[--w * P];
              const int b = 31 - __clz(bits);
              bits &= ~(1u << b);
              ev[u] = col[static_cast<size_t>(w * 32 + b) * B.npairs];
            }
          }
          int pmv[kPf];  // the forward pass's PM of this batch (ranks left-1 .. left-cnt), all loads in flight
#pragma unroll
          for (int u = 0; u < kPf; ++u) pmv[u] = u < cnt ? PM[(left - 1 - u) * kBigThreads] : 0;
#pragma unroll
          for (int u = 0; u < kPf; ++u) {
            if (u < cnt) {
              const uint2 e = ev[u];
              const int j = e.x & 0xffff;
              const int a = e.x >> 16, b = e.y & 0xffff;
              Bs += b;
              const int X = static_cast<int>(e.y >> 16) + Bs - As;
              const int inner = max(pmv[u] - b, sm - a) + Btot;
              const int hk = heads[j * M + k], hl = heads[j * M + l];
              const int vF = max(hk + Atot - a + qk, max(hl + Btot - b, hk + inner) + ql);
              const int vB = max(rk + Atot - a + tails[j * M + k], max(rl + Btot - b, rk + inner) + tails[j * M + l]);
              atomicMax(&accf[j], vF);
              atomicMax(&accb[j], vB);
              sm = max(sm, X);
              As += a;
            }
          }
        }
        }
      }
    }
    __syncthreads();
    // MinMin over children in decode order (src/bound.cpp:109-131)
    int lo = INT_MAX;
    for (int c = tid; c < f; c += blockDim.x) {
      const int j = spm[d1 + c];
      lo = min(lo, min(accf[j], accb[j]));
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    if (lane == 0) red[warp] = lo;
    __syncthreads();
    lo = INT_MAX;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) lo = min(lo, red[w]);
    __syncthreads();
    int cf = 0, cb = 0, sf = 0, sb = 0;
    for (int c = tid; c < f; c += blockDim.x) {
      const int j = spm[d1 + c];
      cf += accf[j] == lo;
      cb += accb[j] == lo;
      sf += accf[j];
      sb += accb[j];
    }
    cf = __reduce_add_sync(0xffffffffu, cf);
    cb = __reduce_add_sync(0xffffffffu, cb);
    sf = __reduce_add_sync(0xffffffffu, sf);
    sb = __reduce_add_sync(0xffffffffu, sb);
    if (lane == 0) {
      red[8 + warp] = cf;
      red[16 + warp] = cb;
      red[24 + warp] = sf;
      red[32 + warp] = sb;
    }
    __syncthreads();
    cf = cb = sf = sb = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
      cf += red[8 + w];
      cb += red[16 + w];
      sf += red[24 + w];
      sb += red[32 + w];
    }
    int d = kFwd;
    if (cf != cb) d = cf < cb ? kFwd : kBwd;
    else if (sf != sb) d = sf > sb ? kFwd : kBwd;
    for (int c = tid; c < f; c += blockDim.x) {
      const int j = spm[d1 + c];
      const int lb = d == kFwd ? accf[j] : accb[j];
      const size_t o = static_cast<size_t>(node) * n + c;
      B.child_lb[o] = lb;
      B.lb_fwd[o] = accf[j];
      B.lb_bwd[o] = accb[j];
      B.pruned[o] = lb >= B.incumbent;
    }
    if (tid == 0) B.dir[node] = static_cast<uint8_t>(d);
    __syncthreads();
  }
}

#endif  // __CUDACC__

// LB1 for large n: one WARP per node, kBig1Warps nodes in flight per CTA, the instance
// table staged once per CTA.
//   tables     front over sigma1 / tail over sigma2 as lane-per-machine wavefronts
//              (bound_tables, src/bound.cpp:20-46); for M <= 16 the front runs in lanes 0-15
//              and the tail in lanes 16-31 of the same loop. The same loads accumulate the
//              fixed jobs' machine sums, so remain = ptot - sum(sigma1) - sum(sigma2) costs no
//              pass over the free jobs.
//   children   lane per child (children_bounds, src/bound.cpp:61-88), rows as LDS.128,
//              results stored coalesced; MinMin (src/bound.cpp:109-131) from per-lane
//              (min, count-at-min, sum) triples reduced with REDUX, so one pass suffices;
//              the second pass writes child_lb / pruned from the chosen direction.
constexpr int kBig1Warps = 16;

__host__ __device__ inline int big1_smem_bytes(int n, int mp, int m) {
  return n * mp * 4 + kBig1Warps * (round_up(n, 8) * 2 + 4 * round_up(m, 4) * 4);
}

#ifdef __CUDACC__

// Children of one node, lane per child (children_bounds, src/bound.cpp:61-88), and MinMin
// (src/bound.cpp:109-131) from per-lane (min, count-at-min, sum) triples; fr/tl/rt/frm are the
// node's warp-uniform tables in shared memory, jobs[d1 + c] its free jobs in decode order.
template <int M, int MP, typename JobT>
__device__ __forceinline__ void big1_children(const BigBatchParams& B, const int* sp, const JobT* jobs, int d1, int f,
                                              int node, const int* fr, const int* tl, const int* rt, const int* frm,
                                              int lane) {
    const int n = B.n;
    // children: lane per child; per-lane MinMin triples
    int lo = INT_MAX, cf = 0, cb = 0, sf = 0, sb = 0;
    const size_t ob = static_cast<size_t>(node) * n;
    for (int c = lane; c < f; c += 32) {
      const int4* pr4 = reinterpret_cast<const int4*>(sp + jobs[d1 + c] * MP);
      const int4* fr4 = reinterpret_cast<const int4*>(fr);
      const int4* rt4 = reinterpret_cast<const int4*>(rt);
      const int4* tl4 = reinterpret_cast<const int4*>(tl);
      const int4* fm4 = reinterpret_cast<const int4*>(frm);
      int prev = 0, vf = 0;
#pragma unroll
      for (int k4 = 0; k4 < MP / 4; ++k4) {
        const int4 a = fr4[k4], r = rt4[k4], w = pr4[k4];
        const int av[4] = {a.x, a.y, a.z, a.w}, rv[4] = {r.x, r.y, r.z, r.w}, pv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k4 * 4 + u < M) {
            const int t = max(prev, av[u]);
            vf = max(vf, t + rv[u]);
            prev = t + pv[u];
          }
        }
      }
      prev = 0;
      int vb = 0;
#pragma unroll
      for (int k4 = MP / 4 - 1; k4 >= 0; --k4) {
        const int4 a = tl4[k4], r = fm4[k4], w = pr4[k4];
        const int av[4] = {a.x, a.y, a.z, a.w}, rv[4] = {r.x, r.y, r.z, r.w}, pv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 3; u >= 0; --u) {
          if (k4 * 4 + u < M) {
            const int t = max(prev, av[u]);
            vb = max(vb, t + rv[u]);
            prev = t + pv[u];
          }
        }
      }
      B.lb_fwd[ob + c] = vf;
      B.lb_bwd[ob + c] = vb;
      const int v = min(vf, vb);
      if (v < lo) {
        lo = v;
        cf = cb = 0;
      }
      cf += vf == lo;
      cb += vb == lo;
      sf += vf;
      sb += vb;
    }
    const int glo = __reduce_min_sync(0xffffffffu, lo);
    cf = __reduce_add_sync(0xffffffffu, lo == glo ? cf : 0);
    cb = __reduce_add_sync(0xffffffffu, lo == glo ? cb : 0);
    sf = __reduce_add_sync(0xffffffffu, sf);
    sb = __reduce_add_sync(0xffffffffu, sb);
    int d = kFwd;
    if (cf != cb) d = cf < cb ? kFwd : kBwd;
    else if (sf != sb) d = sf > sb ? kFwd : kBwd;
    for (int c = lane; c < f; c += 32) {
      const int lb = d == kFwd ? B.lb_fwd[ob + c] : B.lb_bwd[ob + c];
      B.child_lb[ob + c] = lb;
      B.pruned[ob + c] = lb >= B.incumbent;
    }
    if (lane == 0) B.dir[node] = static_cast<uint8_t>(d);
}

template <int M>
__global__ void __launch_bounds__(kBig1Warps * 32, M > 16 ? 1 : 2) decompose_big_lb1_kernel(const BigBatchParams B, const int* ptot) {
  constexpr int MP = (M + 3) / 4 * 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = B.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* sp = reinterpret_cast<int*>(smem);  // [n][MP]
  uint16_t* spm = reinterpret_cast<uint16_t*>(sp + n * MP) + warp * round_up(n, 8);  // this warp's perm
  int* wt = reinterpret_cast<int*>(reinterpret_cast<uint16_t*>(sp + n * MP) + kBig1Warps * round_up(n, 8)) +
            warp * 4 * MP;
  int* fr = wt;            // front
  int* tl = wt + MP;       // tail
  int* rt = wt + 2 * MP;   // remain + tail
  int* frm = wt + 3 * MP;  // front + remain
  for (int i = tid; i < n * MP; i += blockDim.x) sp[i] = B.p32[i];
  __syncthreads();
  constexpr bool kDual = M <= 16;
  const int half = lane >> 4, hk = lane & 15;
  for (int node = blockIdx.x * kBig1Warps + warp; node < B.count; node += gridDim.x * kBig1Warps) {
    const int* perm = B.perms + static_cast<size_t>(node) * n;
    const int d1 = B.d1[node], d2 = B.d2[node], f = n - d1 - d2;
    if (d1 < 0) continue;  // no node in this slot
    for (int i = lane; i < n; i += 32) spm[i] = static_cast<uint16_t>(perm[i]);
    __syncwarp();
    int sum = 0;  // fixed jobs' processing times on this lane's machine
    if (kDual) {
      // lanes 0..15: front, machine hk over sigma1; lanes 16..31: tail, machine M-1-hk over sigma2
      const int len = half ? d2 : d1;
      const int k = half ? M - 1 - hk : hk;
      const int steps = max(d1, d2) + M - 1;
      int C = 0;
      big_wave<MP>(sp, spm, n, len, half, k, hk, hk < M, steps, C, sum);
      if (hk < M) (half ? tl : fr)[k] = C;
      // machine k's fixed sum = front lane k + tail lane 16 + (M-1-k)
      const int tsum = __shfl_sync(0xffffffffu, sum, half ? lane : 16 + ((M - 1 - hk) & 15));
      if (!half && hk < M) frm[hk] = ptot[hk] - sum - tsum;  // remain, folded below
    } else {
      int C = 0;
      big_wave<MP>(sp, spm, n, d1, false, lane < M ? lane : 0, lane, lane < M, d1 + M - 1, C, sum);
      if (lane < M) fr[lane] = C;
      C = 0;
      const int k = M - 1 - lane;
      int tsum = 0;
      big_wave<MP>(sp, spm, n, d2, true, lane < M ? k : 0, lane, lane < M, d2 + M - 1, C, tsum);
      if (lane < M) tl[k] = C;
      __syncwarp();
      const int ts = __shfl_sync(0xffffffffu, tsum, (M - 1 - lane) & 31);
      if (lane < M) frm[lane] = ptot[lane] - sum - ts;  // remain, fixed below
    }
    __syncwarp();
    if (lane < M) {
      const int r = frm[lane];
      rt[lane] = r + tl[lane];
      frm[lane] = fr[lane] + r;
    }
    __syncwarp();
    big1_children<M, MP>(B, sp, spm, d1, f, node, fr, tl, rt, frm, lane);
    __syncwarp();
  }
}


// LB2 for large n, one WARP per node (batches whose nodes have f <= kBig2wFmax free jobs; the
// CTA-per-node decompose_big_kernel keeps the rest). A CTA stages the instance once and runs
// up to 20 nodes at a time (one per warp), so the serial parts of a node (its wavefront
// tables) overlap other warps' pair passes instead of idling a whole CTA at a barrier:
//   tables     front / tail as lane-per-machine wavefronts (as decompose_big_lb1_kernel),
//              remain = ptot - fixed sums (no pass over the free jobs)
//   heads      lane per child: H'[c][k] = h'_k | t'_k << 16 (explore.cuh children_lb2_w)
//   pairs      lane per machine pair, 32 pairs per round: the free positions of the pair's
//              Johnson order as a lane-private bitmask in shared memory (from the inverse
//              order, coalesced over the lanes), then the forward / backward passes of the
//              O(P (n + f)) max-plus form over exactly the f set bits, order entries
//              (job | u << 9 | v << 24, u = a + lag, v = a - b) streamed from L2 kPf per lane
//              in flight, PM'_i kept per rank in a per-warp global scratch (all lanes are at
//              the same rank at every step: coalesced), every S_j folded into child j's bounds
//              at once with shared-memory atomicMax (as explore.cuh lb2_round, n > 32)
//   MinMin     lanes over children, REDUX (src/bound.cpp:109-131)
constexpr int kBig2wFmax = 128;
constexpr int kBig2wMaxWarps = 20;

__host__ __device__ inline int big2w_warp_bytes(int n, int m, int fmax) {
  const int mw = (n + 31) / 32;
  return round_up(round_up(n, 8) * 2 * 2 + 3 * round_up(m, 4) * 4 + mw * 32 * 4 + 2 * round_up(fmax, 4) * 4 +
                      fmax * m * 4 + fmax * 32 * (4 + 2),
                  16);
}

__host__ __device__ inline int big2w_smem_bytes(int n, int mp, int m, int fmax, int warps) {
  return round_up(n * mp * 2, 16) + warps * big2w_warp_bytes(n, m, fmax);  // p as uint16
}

#ifdef __CUDACC__

template <int M>
__global__ void __launch_bounds__(kBig2wMaxWarps * 32) decompose_big_lb2w_kernel(const BigBatchParams B, const int* ptot,
                                                                              const uint32_t* packed32, int fmax,
                                                                              int* pm_scratch) {
  constexpr int MP = (M + 3) / 4 * 4;
  constexpr int NEG = -30000;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = B.n, P = B.npairs, PS = round_up(P, 32), MW = (n + 31) >> 5;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  uint16_t* sp = reinterpret_cast<uint16_t*>(smem);  // [n][MP] (p < 2^16: validate_times)
  unsigned char* wb = smem + round_up(n * MP * 2, 16) + warp * big2w_warp_bytes(n, M, fmax);
  uint16_t* spm = reinterpret_cast<uint16_t*>(wb);                  // the node's perm
  uint16_t* cidx = spm + round_up(n, 8);                             // job -> child (0xffff: fixed)
  int* fr = reinterpret_cast<int*>(cidx + round_up(n, 8));
  int* tl = fr + MP;
  int* rm = tl + MP;
  uint32_t* mask = reinterpret_cast<uint32_t*>(rm + MP);             // [MW][32] lane-private words
  int* accf = reinterpret_cast<int*>(mask + MW * 32);                // [fmax] child-indexed
  int* accb = accf + round_up(fmax, 4);
  uint32_t* H = reinterpret_cast<uint32_t*>(accb + round_up(fmax, 4));  // [fmax][M] h' | t' << 16
  uint32_t* ent = H + fmax * M + lane;                                 // [rank][32]: the walk's order entries
  int16_t* pml = reinterpret_cast<int16_t*>(H + fmax * M + fmax * 32) + lane;  // [rank][32]: PM'
  (void)pm_scratch;
  for (int i = tid; i < n * MP; i += blockDim.x) sp[i] = static_cast<uint16_t>(B.p32[i]);
  __syncthreads();
  for (int node = blockIdx.x * nwarps + warp; node < B.count; node += gridDim.x * nwarps) {
    const int* perm = B.perms + static_cast<size_t>(node) * n;
    const int d1 = B.d1[node], d2 = B.d2[node], f = n - d1 - d2;
    if (d1 < 0) continue;  // no node in this slot
    for (int i = lane; i < n; i += 32) {
      spm[i] = static_cast<uint16_t>(perm[i]);
      cidx[i] = 0xffff;
    }
    __syncwarp();
    for (int c = lane; c < f; c += 32) cidx[spm[d1 + c]] = static_cast<uint16_t>(c);
    {  // node tables (bound_tables, src/bound.cpp:20-46)
      int C = 0, sum = 0, tsum = 0;
      big_wave<MP, uint16_t>(sp, spm, n, d1, false, lane < M ? lane : 0, lane, lane < M, d1 + M - 1, C, sum);
      if (lane < M) fr[lane] = C;
      C = 0;
      const int k = M - 1 - lane;
      big_wave<MP, uint16_t>(sp, spm, n, d2, true, lane < M ? k : 0, lane, lane < M, d2 + M - 1, C, tsum);
      if (lane < M) tl[k] = C;
      const int ts = __shfl_sync(0xffffffffu, tsum, (M - 1 - lane) & 31);
      if (lane < M) rm[lane] = ptot[lane] - sum - ts;
    }
    __syncwarp();
    for (int c = lane; c < f; c += 32) {  // child heads / tails without the job's own time
      const uint16_t* pr = sp + spm[d1 + c] * MP;
      int hp[M];
      int prev = 0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        hp[k] = max(prev, fr[k]);
        prev = hp[k] + pr[k];
      }
      prev = 0;
#pragma unroll
      for (int k = M - 1; k >= 0; --k) {
        const int tp = max(prev, tl[k]);
        prev = tp + pr[k];
        H[c * M + k] = static_cast<uint32_t>(hp[k]) | static_cast<uint32_t>(tp) << 16;
      }
      accf[c] = 0;
      accb[c] = 0;
    }
    __syncwarp();
    for (int q0 = 0; q0 < P; q0 += 32) {
      const int q = min(q0 + lane, P - 1);
      const int k = B.pk[q], l = B.pl[q];
      const int Atot = rm[k], Btot = rm[l];
      const int qk = tl[k], ql = tl[l], rk = fr[k], rl = fr[l];
      const int cAq = Atot + qk, cRB = rl + Btot;
      const uint32_t Cc = static_cast<uint32_t>(Btot + ql) | static_cast<uint32_t>(rk + Atot) << 16;
      // free positions of the pair's order: lane-private mask words (inverse order, coalesced
      // loads; shared-memory atomicOr so the updates pipeline instead of chaining through
      // load-modify-store) and a summary of the non-empty words (n <= 512: 16 words)
      for (int w = 0; w < MW; ++w) mask[w * 32 + lane] = 0;
      uint32_t nonempty = 0;
      __syncwarp();
      {
        const uint16_t* iq = B.inv16 + q;
        int c = 0;
        for (; c + 16 <= f; c += 16) {  // 16 inverse-order loads in flight per lane
          int pos[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) pos[u] = iq[static_cast<size_t>(spm[d1 + c + u]) * P];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            atomicOr(&mask[(pos[u] >> 5) * 32 + lane], 1u << (pos[u] & 31));
            nonempty |= 1u << (pos[u] >> 5);
          }
        }
        for (; c < f; ++c) {
          const int pos = iq[static_cast<size_t>(spm[d1 + c]) * P];
          atomicOr(&mask[(pos >> 5) * 32 + lane], 1u << (pos & 31));
          nonempty |= 1u << (pos >> 5);
        }
      }
      __syncwarp();
      const uint32_t* col = packed32 + q;
      // every lane walks exactly f positions (its pair's free jobs): the forward pass gathers the
      // order entries from L2 in position order (4 in flight) and keeps them with PM'_i in the
      // warp's shared lists by rank; the backward pass reads both back in reverse
      uint32_t words = nonempty, bits = 0;
      int w = 0;
      auto next_up = [&]() {  // ascending set bits over the non-empty words
        if (bits == 0) {
          w = __ffs(words) - 1;
          words &= words - 1;
          bits = mask[w * 32 + lane];
        }
        const int t = w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        return t;
      };
      int E = Btot, pm = NEG, rank = 0;
      auto fwd = [&](uint32_t e) {  // PM'_i = prefix max of X' over the earlier free positions
        ent[rank * 32] = e;
        pml[rank * 32] = static_cast<int16_t>(pm);
        ++rank;
        pm = max(pm, E + static_cast<int>((e >> 9) & 0x7ffu));
        E += static_cast<int>(e) >> 24;
      };
      int i = 0;
      for (; i + 16 <= f; i += 16) {  // 16 order entries in flight per lane
        uint32_t e[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) e[u] = col[static_cast<size_t>(next_up()) * PS];
#pragma unroll
        for (int u = 0; u < 16; ++u) fwd(e[u]);
      }
      for (; i + 4 <= f; i += 4) {
        uint32_t e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = col[static_cast<size_t>(next_up()) * PS];
#pragma unroll
        for (int u = 0; u < 4; ++u) fwd(e[u]);
      }
      for (; i < f; ++i) fwd(col[static_cast<size_t>(next_up()) * PS]);
      int G = Atot, sm = NEG;
      for (int r = f - 1; r >= 0; --r) {  // S_j folded into child j's bounds
        const uint32_t e = ent[r * 32];
        const int v = static_cast<int>(e) >> 24;
        const int c = cidx[e & 0x1ffu];
        const int I1 = max(static_cast<int>(pml[r * 32]) + v, sm);
        const int lo = max(cAq, I1 + ql), hi = max(cRB, I1 + (rk - v));
        const uint32_t S = __byte_perm(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi), 0x5410);
        const uint32_t hk = H[c * M + k], hl = H[c * M + l];
        const uint32_t V = max_u16x2(add_u16x2(__byte_perm(hk, hl, 0x7610), S), add_u16x2(__byte_perm(hl, hk, 0x7610), Cc));
        atomicMax(reinterpret_cast<unsigned*>(accf) + c, V & 0xffffu);
        atomicMax(reinterpret_cast<unsigned*>(accb) + c, V >> 16);
        G -= v;
        sm = max(sm, G + static_cast<int>((e >> 9) & 0x7ffu));
      }
    }
    __syncwarp();
    // MinMin over children in decode order (src/bound.cpp:109-131) and the outputs
    int lo = INT_MAX, cf = 0, cb = 0, sf = 0, sb = 0;
    for (int c = lane; c < f; c += 32) {
      const int vf = accf[c], vb = accb[c];
      const int v = min(vf, vb);
      if (v < lo) {
        lo = v;
        cf = cb = 0;
      }
      cf += vf == lo;
      cb += vb == lo;
      sf += vf;
      sb += vb;
    }
    const int glo = __reduce_min_sync(0xffffffffu, lo);
    cf = __reduce_add_sync(0xffffffffu, lo == glo ? cf : 0);
    cb = __reduce_add_sync(0xffffffffu, lo == glo ? cb : 0);
    sf = __reduce_add_sync(0xffffffffu, sf);
    sb = __reduce_add_sync(0xffffffffu, sb);
    int d = kFwd;
    if (cf != cb) d = cf < cb ? kFwd : kBwd;
    else if (sf != sb) d = sf > sb ? kFwd : kBwd;
    const size_t ob = static_cast<size_t>(node) * n;
    for (int c = lane; c < f; c += 32) {
      const int vf = accf[c], vb = accb[c];
      const int lb = d == kFwd ? vf : vb;
      B.lb_fwd[ob + c] = vf;
      B.lb_bwd[ob + c] = vb;
      B.child_lb[ob + c] = lb;
      B.pruned[ob + c] = lb >= B.incumbent;
    }
    if (lane == 0) B.dir[node] = static_cast<uint8_t>(d);
    __syncwarp();
  }
}

#endif  // __CUDACC__

// LB1 for large n, node tables lane-per-node: a warp takes 32 nodes at a time; each lane runs
// its node's front over sigma1 and then its tail over reversed sigma2 as one sequence of
// d1 + d2 fixed jobs (bound_tables, src/bound.cpp:20-46) -- the tail reads machine-reversed
// rows, so both halves are the same register recurrence C[k] = max(C[k], C[k-1]) + p[k]
// (20 VIADDMNMX-class ops per job and lane, rows as LDS.128, no shuffles). The 32 nodes'
// tables go through shared memory to the lane-per-child children pass (big1_children).
constexpr int kBig1gWarps = 8;

__host__ __device__ inline int big1g_smem_bytes(int n, int mp) {
  return 2 * n * mp * 4 + kBig1gWarps * 32 * 4 * mp * 4;
}

template <int M>
__global__ void __launch_bounds__(kBig1gWarps * 32, 1) decompose_big_lb1g_kernel(const BigBatchParams B, const int* ptot) {
  constexpr int MP = (M + 3) / 4 * 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = B.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* sp = reinterpret_cast<int*>(smem);  // [n][MP] rows
  int* sr = sp + n * MP;                   // [n][MP] machine-reversed rows
  int* stage = sr + n * MP + warp * 32 * 4 * MP;  // [32 nodes][fr | tl | rt | frm][MP]
  for (int i = tid; i < n * MP; i += blockDim.x) {
    const int j = i / MP, k = i - j * MP;
    sp[i] = B.p32[i];
    sr[i] = k < M ? B.p32[j * MP + M - 1 - k] : 0;
  }
  __syncthreads();
  const int groups = (B.count + 31) / 32;
  // groups interleaved over the CTAs (warp-major), so a batch smaller than one full wave
  // still spreads over every SM
  for (int g = warp * gridDim.x + blockIdx.x; g < groups; g += gridDim.x * kBig1gWarps) {
    const int node = g * 32 + lane;
    const int rd1 = node < B.count ? B.d1[node] : -1;  // -1: no node in this slot
    const bool live = rd1 >= 0;
    const int d1 = live ? rd1 : 0, d2 = live ? B.d2[node] : 0;
    const int len = d1 + d2;
    const int steps = __reduce_max_sync(0xffffffffu, len);
    const int* perm = B.perms + static_cast<size_t>(live ? node : 0) * n;
    int C[M], S[M];
#pragma unroll
    for (int k = 0; k < M; ++k) C[k] = S[k] = 0;
    int* st = stage + lane * 4 * MP;
    auto flip = [&]() {  // end of sigma1: save the front, restart for the tail, reverse the sums
#pragma unroll
      for (int k = 0; k < M; ++k) {
        st[k] = C[k];
        C[k] = 0;
      }
#pragma unroll
      for (int k = 0; k < M / 2; ++k) {
        const int t = S[k];
        S[k] = S[M - 1 - k];
        S[M - 1 - k] = t;
      }
    };
    // the lane's job sequence (sigma1, then sigma2 from the end) is read kJq steps ahead
    constexpr int kJq = 8;
    auto job_at = [&](int t) { return t < len ? perm[t < d1 ? t : n - 1 - (t - d1)] : 0; };
    int jq[kJq];
#pragma unroll
    for (int u = 0; u < kJq; ++u) jq[u] = job_at(u);
    for (int t = 0; t < steps; ++t) {
      const int j = jq[0];
#pragma unroll
      for (int u = 0; u + 1 < kJq; ++u) jq[u] = jq[u + 1];
      jq[kJq - 1] = job_at(t + kJq);
      if (t == d1 && t < len) flip();
      if (t < len) {
        const bool tail = t >= d1;
        const int4* r4 = reinterpret_cast<const int4*>((tail ? sr : sp) + j * MP);
        int prev = 0;
#pragma unroll
        for (int k4 = 0; k4 < MP / 4; ++k4) {
          const int4 w = r4[k4];
          const int pv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (k4 * 4 + u < M) {
              prev = max(C[k4 * 4 + u], prev) + pv[u];
              C[k4 * 4 + u] = prev;
              S[k4 * 4 + u] += pv[u];
            }
          }
        }
      }
    }
    if (len == d1) flip();  // no tail jobs (also covers len == 0)
    // C = tail in reversed machine order, S = fixed sums in reversed order
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const int tlk = C[M - 1 - k];
      const int rem = ptot[k] - S[M - 1 - k];
      const int frk = st[k];
      st[MP + k] = tlk;
      st[2 * MP + k] = rem + tlk;
      st[3 * MP + k] = frk + rem;
    }
    __syncwarp();
    const int last = min(32, B.count - g * 32);
    for (int q = 0; q < last; ++q) {
      const int nd = g * 32 + q;
      const int* sq = stage + q * 4 * MP;
      const int qd1 = __shfl_sync(0xffffffffu, d1, q), qd2 = __shfl_sync(0xffffffffu, d2, q);
      if (!__shfl_sync(0xffffffffu, static_cast<int>(live), q)) continue;
      big1_children<M, MP>(B, sp, B.perms + static_cast<size_t>(nd) * n, qd1, n - qd1 - qd2, nd, sq, sq + MP,
                           sq + 2 * MP, sq + 3 * MP, lane);
    }
    __syncwarp();
  }
}

#endif  // __CUDACC__

}  // namespace pbbgpu
