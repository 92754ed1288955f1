// Explorer pool for 64 < n <= 512 (ta061-ta120): IVM explorers in global memory, stepped in
// lock step with the large-n bounding kernels (bound_big.cuh) as their decompose operator.
//
// An explorer's IVM (ivm.hpp:21-94) has int16 cells (job + 1, negative = pruned / consumed)
// in a triangular matrix, int16 V / end / replay-target digits and a header; at n = 500 that
// is 254 KB, so the explorers live in HBM (K x 254 KB) rather than shared memory. One step:
//   big_select_kernel   warp per explorer: one init_at replay level (ivm.cpp:70-86), or
//                       select_next (ivm.cpp:99-122, end test ivm.cpp:90-97); the selected node
//                       is decoded (ivm.cpp:152-172) into the explorer's batch slot (perm, d1,
//                       d2), leaves (one free job, explorer.cpp:42) included: their only child
//                       bound IS the schedule's makespan (front_{sigma1 j} + tail_{sigma2} over
//                       the machines, for LB1 and LB2 alike)
//   bounding            decompose_big_* over the K slots (inactive slots have d1 < 0)
//   big_branch_kernel   warp per explorer: branch (ivm.cpp:124-145) with the slot's MinMin
//                       direction and prune flags, or the leaf's evaluation and prune_current
//                       (explorer.cpp:42-57); replay bookkeeping
// Work is split between explorers by the same log2-bucket steal plan as the small-n pool
// (steal_kernel reads only the lens array) with int16-digit lens / split kernels here.
// Included by pool.cu inside its kernel section (seat / split helpers are templated there).
#pragma once

struct BigHdr {
  int16_t level, d1, d2, rlev, nrep;
  uint8_t state, has_end;
  int16_t pad;
};

struct BigIvmLayout {
  int n, o_cells, o_v, o_end, o_tgt, o_dir, stride;
};

inline BigIvmLayout big_ivm_layout(int n) {
  BigIvmLayout L{};
  L.n = n;
  int o = 16;  // BigHdr
  L.o_cells = o;
  o += n * (n + 1) / 2 * 2;
  L.o_v = o;
  o += n * 2;
  L.o_end = o;
  o += n * 2;
  L.o_tgt = o;
  o += n * 2;
  L.o_dir = o;
  o += n;
  L.stride = round_up(o, 16);
  return L;
}

struct BigImp {
  int mk;
  int16_t perm[kBigMaxN];
};
constexpr int kBigImpCap = 256;

struct BigStepParams {
  BigIvmLayout L;
  unsigned char* state;
  int K;
  int* perms;        // [K][n] batch slot perms
  int* d1;           // [K] (-1: no node this step)
  int* d2;
  uint8_t* kind;     // [K]: 0 none, 1 node, 2 replay node, 3 leaf
  int* fstat;        // [0] max f, [1] slots with a node, [2] sum f (low 31 bits), [3] explorers not Empty
  DevCounters* ctr;
  unsigned long long* hist;
  unsigned long long* dhist;
  const uint8_t* dir;     // bounding outputs
  const uint8_t* pruned;  // [K][n]
  const int* lb_fwd;      // [K][n]
  int prune_mode, pinned_ub;
  BigImp* imp;
};

__device__ __forceinline__ BigHdr* bhdr(unsigned char* b) { return reinterpret_cast<BigHdr*>(b); }
__device__ __forceinline__ int16_t* bcells(unsigned char* b, const BigIvmLayout& L) { return reinterpret_cast<int16_t*>(b + L.o_cells); }
__device__ __forceinline__ int16_t* bV(unsigned char* b, const BigIvmLayout& L) { return reinterpret_cast<int16_t*>(b + L.o_v); }
__device__ __forceinline__ int16_t* bE(unsigned char* b, const BigIvmLayout& L) { return reinterpret_cast<int16_t*>(b + L.o_end); }
__device__ __forceinline__ int16_t* bT(unsigned char* b, const BigIvmLayout& L) { return reinterpret_cast<int16_t*>(b + L.o_tgt); }
__device__ __forceinline__ uint8_t* bD(unsigned char* b, const BigIvmLayout& L) { return b + L.o_dir; }

// init_root + targets (ivm.cpp:38-64) for an interval [a, b) (has_end: b < n!)
__device__ void big_seat(unsigned char* blk, const BigIvmLayout& L, const int* a, const int* b, bool has_end, int lane,
                         int width) {
  const int n = L.n;
  int16_t* C = bcells(blk, L);
  int16_t *V = bV(blk, L), *E = bE(blk, L), *T = bT(blk, L);
  uint8_t* D = bD(blk, L);
  for (int c = lane; c < n; c += width) C[c] = static_cast<int16_t>(c + 1);
  for (int l = lane; l < n; l += width) {
    V[l] = 0;
    D[l] = kFwd;
    T[l] = static_cast<int16_t>(a[l]);
    E[l] = static_cast<int16_t>(has_end ? b[l] : 0);
  }
  if (lane == 0) {
    bool empty = false;
    if (has_end) {
      int cmp = 0;
      for (int l = 0; l < n && !cmp; ++l) cmp = a[l] < b[l] ? -1 : (a[l] > b[l] ? 1 : 0);
      empty = cmp >= 0;
    }
    BigHdr* h = bhdr(blk);
    h->level = 0;
    h->d1 = 1;
    h->d2 = 0;
    h->rlev = 0;
    h->nrep = 0;
    h->state = static_cast<uint8_t>(empty ? kEmpty : kInit);
    h->has_end = has_end ? 1 : 0;
  }
}

__global__ void big_init_kernel(BigIvmLayout L, unsigned char* state, const int* a, const int* b, const uint8_t* b_nfact,
                                const int* slots, int count) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= count) return;
  big_seat(state + static_cast<size_t>(slots[i]) * L.stride, L, a + static_cast<size_t>(i) * L.n,
           b + static_cast<size_t>(i) * L.n, !b_nfact[i], threadIdx.x & 31, 32);
}

__global__ void big_clear_kernel(BigIvmLayout L, unsigned char* state, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  BigHdr* h = bhdr(state + static_cast<size_t>(i) * L.stride);
  h->state = kEmpty;
  h->level = -1;
}

// Decode the node (level, V[level]) into the slot: sigma1 from the Forward levels, sigma2 from
// the Backward levels (filled from the end), the row's other cells in row order between them.
__device__ void big_decode(unsigned char* blk, const BigIvmLayout& L, int level, int* perm, int& d1, int& d2, int lane) {
  const int n = L.n;
  const int16_t* C = bcells(blk, L);
  const int16_t* V = bV(blk, L);
  const uint8_t* D = bD(blk, L);
  // path: prefix counts of Forward levels by ballot
  int a = 0, b = 0;
  for (int l0 = 0; l0 <= level; l0 += 32) {
    const int l = l0 + lane;
    const bool on = l <= level;
    const bool fw = on && D[l] == kFwd;
    const unsigned mf = __ballot_sync(0xffffffffu, fw), mb = __ballot_sync(0xffffffffu, on && !fw);
    if (on) {
      const int x = C[tri_off(l, n) + V[l]];
      const int job = (x < 0 ? -x : x) - 1;
      const unsigned below = (1u << lane) - 1u;
      if (fw) perm[a + __popc(mf & below)] = job;
      else perm[n - 1 - (b + __popc(mb & below))] = job;
    }
    a += __popc(mf);
    b += __popc(mb);
  }
  const int len = n - level, sel = V[level];
  const int16_t* row = C + tri_off(level, n);
  for (int c = lane; c < len - 1; c += 32) {
    const int x = row[c < sel ? c : c + 1];
    perm[a + c] = (x < 0 ? -x : x) - 1;
  }
  d1 = a;
  d2 = b;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) big_select_kernel(BigStepParams S) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (i >= S.K) return;
  const BigIvmLayout& L = S.L;
  const int n = L.n;
  unsigned char* blk = S.state + static_cast<size_t>(i) * L.stride;
  BigHdr* h = bhdr(blk);
  int16_t* C = bcells(blk, L);
  int16_t* V = bV(blk, L);
  int* perm = S.perms + static_cast<size_t>(i) * n;
  int state = h->state, level = h->level;
  uint8_t kind = 0;
  for (;;) {
    if (state == kEmpty) break;
    if (state == kInit) {  // one replay level of init_at (ivm.cpp:70-86)
      const int l = h->rlev, digit = bT(blk, L)[l];
      int16_t* row = C + tri_off(l, n);
      for (int c = lane; c < digit; c += 32)
        if (row[c] > 0) row[c] = static_cast<int16_t>(-row[c]);
      __syncwarp();
      if (lane == 0) V[l] = static_cast<int16_t>(digit);
      __syncwarp();
      level = l;
      if (row[digit] < 0 || l >= n - 2) {  // positioned: duplicates = min(L, lnz(a))
        int lz = 0;
        for (int t = lane; t < n; t += 32)
          if (bT(blk, L)[t] != 0) lz = max(lz, t);
        lz = __reduce_max_sync(0xffffffffu, lz);
        const int dup = min(static_cast<int>(h->nrep), lz);
        if (lane == 0) {
          if (dup) atomicAdd(&S.ctr->dups, static_cast<unsigned long long>(dup));
          for (int t = 0; t < dup; ++t) atomicAdd(&S.dhist[n - 1 - t], 1ull);
          h->state = kActive;
          h->level = static_cast<int16_t>(level);
        }
        state = kActive;
        __syncwarp();
        continue;
      }
      kind = 2;  // the replay node is decomposed by this step's bounding
      break;
    }
    // select_next (ivm.cpp:99-122)
    bool exhausted = false;
    for (;;) {
      if (level < 0) {
        exhausted = true;
        break;
      }
      const int len = n - level;
      const int16_t* row = C + tri_off(level, n);
      int found = -1;
      for (int b0 = V[level]; b0 < len; b0 += 32) {
        const int c = b0 + lane;
        const unsigned bal = __ballot_sync(0xffffffffu, c < len && row[c] > 0);
        if (bal) {
          found = b0 + __ffs(bal) - 1;
          break;
        }
      }
      if (found < 0) {  // backtrack
        __syncwarp();
        if (lane == 0) {
          V[level] = 0;
          if (level > 0) V[level - 1] = static_cast<int16_t>(V[level - 1] + 1);
        }
        --level;
        __syncwarp();
        continue;
      }
      __syncwarp();
      if (lane == 0) V[level] = static_cast<int16_t>(found);
      __syncwarp();
      if (h->has_end) {  // position_reached_end (ivm.cpp:90-97): padded V >= end
        const int16_t* E = bE(blk, L);
        int res = 0;  // 1 reached, -1 below
        for (int b0 = 0; b0 < n && !res; b0 += 32) {
          const int l = b0 + lane;
          int pv = 0, ev = 0;
          if (l < n) {
            pv = l <= level ? V[l] : 0;
            ev = E[l];
          }
          const unsigned bal = __ballot_sync(0xffffffffu, l < n && pv != ev);
          if (bal) {
            const int src = __ffs(bal) - 1;
            res = __shfl_sync(0xffffffffu, pv, src) > __shfl_sync(0xffffffffu, ev, src) ? 1 : -1;
          }
        }
        if (res >= 0) exhausted = true;
      }
      break;
    }
    if (exhausted) {
      state = kEmpty;
      break;
    }
    kind = n - 1 - level <= 1 ? 3 : 1;
    break;
  }
  int d1 = -1, d2 = 0;
  if (kind) big_decode(blk, L, level, perm, d1, d2, lane);
  if (lane == 0) {
    h->state = static_cast<uint8_t>(state);
    h->level = static_cast<int16_t>(state == kEmpty ? -1 : level);
    S.d1[i] = kind ? d1 : -1;
    S.d2[i] = d2;
    S.kind[i] = kind;
    if (kind) {
      const int f = n - d1 - d2;
      atomicMax(&S.fstat[0], f);
      atomicAdd(&S.fstat[1], 1);
      atomicAdd(&S.fstat[2], f);
    }
    if (state != kEmpty) atomicAdd(&S.fstat[3], 1);
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) big_branch_kernel(BigStepParams S) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (i >= S.K) return;
  const int kind = S.kind[i];
  if (!kind) return;
  const BigIvmLayout& L = S.L;
  const int n = L.n;
  unsigned char* blk = S.state + static_cast<size_t>(i) * L.stride;
  BigHdr* h = bhdr(blk);
  int16_t* C = bcells(blk, L);
  int16_t* V = bV(blk, L);
  const int level = h->level;
  const int* perm = S.perms + static_cast<size_t>(i) * n;
  const int d1 = S.d1[i], d2 = S.d2[i], f = n - d1 - d2;
  if (kind == 3) {  // leaf (explorer.cpp:42-57): its only child bound is the makespan
    const int mk = S.lb_fwd[static_cast<size_t>(i) * n];
    int slot = -1;
    if (lane == 0) {
      int16_t& x = C[tri_off(level, n) + V[level]];
      if (x > 0) x = static_cast<int16_t>(-x);  // prune_current
      atomicAdd(&S.ctr->leaves, 1ull);
      const int improve = S.prune_mode == 1 ? 0 : *reinterpret_cast<volatile int*>(&S.ctr->best);
      if (mk < improve) {
        const int old = atomicMin(&S.ctr->best, mk);
        if (mk < old) {
          atomicAdd(&S.ctr->improvements, 1ull);
          slot = atomicAdd(&S.ctr->imp_count, 1) % kBigImpCap;
          S.imp[slot].mk = mk;
        }
      }
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    // the record's schedule: the slot's perm is the complete schedule (a ring overwrite can
    // tear a record; the host re-evaluates every record's makespan)
    if (slot >= 0)
      for (int t = lane; t < n; t += 32) S.imp[slot].perm[t] = static_cast<int16_t>(perm[t]);
    return;
  }
  // branch (ivm.cpp:124-145): row level+1 = the free jobs in row order, pruned negated
  const int dir = S.dir[i];
  int16_t* nrow = C + tri_off(level + 1, n);
  const uint8_t* pr = S.pruned + static_cast<size_t>(i) * n;
  for (int c = lane; c < f; c += 32) {
    const int j1 = perm[d1 + c] + 1;
    nrow[c] = static_cast<int16_t>(pr[c] ? -j1 : j1);
  }
  __syncwarp();
  if (lane == 0) {
    bD(blk, L)[level + 1] = static_cast<uint8_t>(dir);
    V[level + 1] = 0;
    h->level = static_cast<int16_t>(level + 1);
    h->d1 = static_cast<int16_t>(d1 + (dir == kFwd));
    h->d2 = static_cast<int16_t>(d2 + (dir == kBwd));
    atomicAdd(&S.ctr->decomposed, 1ull);
    atomicAdd(&S.hist[f], 1ull);
    if (kind == 2) {
      h->nrep = static_cast<int16_t>(h->nrep + 1);
      h->rlev = static_cast<int16_t>(level + 1);
    }
  }
}

// ---- steal helpers on int16 digits
__global__ void big_lens_kernel(BigIvmLayout L, unsigned char* state, int K, const float* lgfact, float* lens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  unsigned char* blk = state + static_cast<size_t>(i) * L.stride;
  const BigHdr* h = bhdr(blk);
  float lg = -3.f;
  if (h->state == kInit) {
    lg = -2.f;
  } else if (h->state == kActive) {
    lg = -2.f;
    int pos[kBigMaxN];
    if (effective_pos(bV(blk, L), h->level, bcells(blk, L), L.n, pos)) {
      const float r = remaining_log2_pos(pos, bE(blk, L), h->has_end != 0, L.n, lgfact);
      if (r >= 0.f) lg = r;
    }
  }
  lens[i] = lg;
}

__device__ int big_split_setup(unsigned char* vb, const BigIvmLayout& L, int r, int* pos, int* D, int& top) {
  const BigHdr* vh = bhdr(vb);
  if (vh->state != kActive) return 0;
  if (!effective_pos(bV(vb, L), vh->level, bcells(vb, L), L.n, pos)) return 0;
  if (!diff_digits(pos, bE(vb, L), vh->has_end != 0, L.n, D, top)) return 0;
  if (!top) {
    long long small = 0;
    bool big = false;
    for (int l = 0; l < L.n && !big; ++l) {
      small = small * (L.n - l) + D[l];
      if (small > (1ll << 40)) big = true;
    }
    if (!big) {
      if (small < 2) return 0;
      r = static_cast<int>(min(static_cast<long long>(r), max(small / 2 - 1, 1ll)));
    }
  }
  return r;
}

// one thread per (victim, part): thief seated on part i of the victim's [pos, end)
__global__ void big_split_thieves_kernel(BigIvmLayout L, unsigned char* state, const int* thief, const int* victim,
                                         const int* plan, DevCounters* ctr) {
  const int nv = plan[0], rs = plan[1];
  const int g0 = blockIdx.x * blockDim.x + threadIdx.x;
  int ok = 0;
  if (g0 < nv * rs) {
    const int v = g0 / rs, i = g0 % rs + 1;
    unsigned char* vb = state + static_cast<size_t>(victim[v]) * L.stride;
    int pos[kBigMaxN], D[kBigMaxN], b0[kBigMaxN], b1[kBigMaxN];
    int top = 0;
    const int r = big_split_setup(vb, L, rs, pos, D, top);
    if (i <= r) {
      const bool last = i == r;
      split_point(pos, D, top, i, r + 1, L.n, b0);
      if (last) {
        const int16_t* E = bE(vb, L);
        for (int l = 0; l < L.n; ++l) b1[l] = E[l];
      } else {
        split_point(pos, D, top, i + 1, r + 1, L.n, b1);
      }
      big_seat(state + static_cast<size_t>(thief[v * rs + i - 1]) * L.stride, L, b0, b1,
               last ? bhdr(vb)->has_end != 0 : true, 0, 1);
      ok = 1;
    }
  }
  const unsigned cnt = __popc(__ballot_sync(0xffffffffu, ok));
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(&ctr->active, static_cast<int>(cnt));
    atomicAdd(&ctr->steals, static_cast<unsigned long long>(cnt));
    atomicAdd(&ctr->inits, static_cast<unsigned long long>(cnt));
  }
}

__global__ void big_split_victims_kernel(BigIvmLayout L, unsigned char* state, const int* victim, const int* plan) {
  const int nv = plan[0], rs = plan[1];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  unsigned char* vb = state + static_cast<size_t>(victim[v]) * L.stride;
  int pos[kBigMaxN], D[kBigMaxN], b[kBigMaxN];
  int top = 0;
  const int r = big_split_setup(vb, L, rs, pos, D, top);
  if (r < 1) return;
  split_point(pos, D, top, 1, r + 1, L.n, b);
  int16_t* E = bE(vb, L);
  for (int l = 0; l < L.n; ++l) E[l] = static_cast<int16_t>(b[l]);
  bhdr(vb)->has_end = 1;
}
