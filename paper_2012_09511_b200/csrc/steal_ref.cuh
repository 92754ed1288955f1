// The reference pool's own steal policy on the device (pbbgpu_config_t.steal_policy = 1):
// ExplorerPool::steal_phase / do_steal, src/explorer.cpp:251-340, reproduced exactly so that
// a GPU pool with batch_steps-long rounds reports the reference's PoolStats (raw decomposed,
// local_steals, steal_phases, intervals_initialized) and not only its partition-invariant
// unique count:
//   trigger      active * 5 < 4K after the round (explorer.cpp:251)
//   lengths      remaining_length = end - position (raw, zero-padded V; ivm.cpp:195-200),
//                exact in 128-bit integers (n <= 30)
//   eligible(v)  Active, unclaimed, len > floor(sum len / K), len > min_steal_len
//   matching     K = 4^c: for digit 1..c, j 1..3, every idle unsatisfied thief tries the
//                victim whose base-4 digit is (d - j) mod 4 (one pass is a bijection thief ->
//                victim, so the thieves of a pass run in parallel); otherwise every idle thief,
//                in index order, takes the largest eligible victim (ties: lowest index)
//   do_steal     refused when len < 2; mid = floor((pos + end) / 2); the victim keeps
//                [pos, mid), the thief is seated on [mid, end) (init_at replay in the next
//                launch, whose replay steps do not consume the round's batch steps)
// One CTA; arrays in global scratch. Fixed-tree runs (no incumbent change) are deterministic in
// the reference for any thread count, so the counters are comparable exactly.
// Included by pool.cu inside its kernel section (uses seat_explorer / diff_digits / split_point).
#pragma once

using u128 = unsigned __int128;

struct StealRefParams {
  IvmLayout L;
  unsigned char* state;
  int K;
  const int* ptot;
  DevCounters* ctr;
  u128* len;         // [K]
  uint8_t* flags;    // [K]: bit0 active, bit1 eligible, bit2 claimed, bit3 satisfied
  int* pairs;        // [2K]: victim, thief
  int* order;        // [K] scratch: idle thieves in index order / victims by rank
  u128 min_steal;    // min(8!, ceil(n!/4K)) or the configured length
};

constexpr int kRefThreads = 1024;

__device__ __forceinline__ u128 fact128(int k) {
  u128 f = 1;
  for (int i = 2; i <= k; ++i) f *= static_cast<u128>(i);
  return f;
}

// to_decimal of a digit vector (MSD first, digit l has radix n - l): Horner form
__device__ __forceinline__ u128 dec128(const int* d, int n) {
  u128 v = 0;
  for (int l = 0; l < n; ++l) v = v * static_cast<u128>(n - l) + static_cast<u128>(d[l]);
  return v;
}

__device__ __forceinline__ void raw_position(const unsigned char* blk, const IvmLayout& L, int* pos) {
  const IvmHdr* h = reinterpret_cast<const IvmHdr*>(blk);
  const int8_t* V = reinterpret_cast<const int8_t*>(blk + L.o_v);
  for (int l = 0; l < L.n; ++l) pos[l] = l <= h->level ? V[l] : 0;
}

__device__ __forceinline__ u128 end_dec128(const unsigned char* blk, const IvmLayout& L, u128 nfact) {
  const IvmHdr* h = reinterpret_cast<const IvmHdr*>(blk);
  if (!h->has_end) return nfact;
  const int8_t* E = reinterpret_cast<const int8_t*>(blk + L.o_end);
  int e[kMaxN];
  for (int l = 0; l < L.n; ++l) e[l] = E[l];
  return dec128(e, L.n);
}

__global__ void __launch_bounds__(kRefThreads) steal_ref_kernel(StealRefParams S) {
  __shared__ u128 s_sum[kRefThreads];
  __shared__ int s_cnt[kRefThreads];
  __shared__ int s_npairs, s_ok;
  const int t = threadIdx.x, K = S.K, n = S.L.n;
  const int live = S.ctr->round_live;
  __syncthreads();
  if (live == 0) {  // a round that started with no explorer: pool_run had already stopped
    if (t == 0) S.ctr->active = 0;
    return;
  }
  const u128 nfact = fact128(n);
  u128 sum = 0;
  int act = 0;
  for (int i = t; i < K; i += kRefThreads) {
    const unsigned char* blk = S.state + static_cast<size_t>(i) * S.L.gstride;
    const IvmHdr* h = reinterpret_cast<const IvmHdr*>(blk);
    u128 len = 0;
    uint8_t fl = 0;
    if (h->state != kEmpty) {
      fl = 1;
      ++act;
      int pos[kMaxN];
      raw_position(blk, S.L, pos);
      const u128 p = dec128(pos, n), e = end_dec128(blk, S.L, nfact);
      len = p < e ? e - p : 0;
    }
    S.len[i] = len;
    S.flags[i] = fl;
    sum += len;
  }
  s_sum[t] = sum;
  s_cnt[t] = act;
  __syncthreads();
  for (int off = kRefThreads / 2; off; off >>= 1) {
    if (t < off) {
      s_sum[t] += s_sum[t + off];
      s_cnt[t] += s_cnt[t + off];
    }
    __syncthreads();
  }
  const int total_active = s_cnt[0];
  const u128 avg = s_sum[0] / static_cast<u128>(K);
  if (t == 0) S.ctr->round_live = 0;
  if (total_active * 5 >= 4 * K) {
    if (t == 0) S.ctr->active = total_active;
    return;
  }
  for (int i = t; i < K; i += kRefThreads) {
    const u128 len = S.len[i];
    if ((S.flags[i] & 1) && len > avg && len > S.min_steal) S.flags[i] |= 2;
  }
  if (t == 0) {
    s_npairs = 0;
    s_ok = 0;
  }
  __syncthreads();
  bool pow4 = K >= 4;
  for (int k = K; k > 1 && pow4; k /= 4) pow4 = k % 4 == 0;
  if (pow4) {
    int c = 0;
    for (int k = K; k > 1; k /= 4) ++c;
    int stride = 1;
    for (int digit = 1; digit <= c; ++digit, stride *= 4) {
      for (int j = 1; j <= 3; ++j) {
        for (int th = t; th < K; th += kRefThreads) {
          if (S.flags[th] & (1 | 8)) continue;  // active, or already satisfied
          const int d = (th / stride) % 4;
          const int nd = ((d - j) % 4 + 4) % 4;
          const int v = th + (nd - d) * stride;
          const uint8_t fv = S.flags[v];
          if ((fv & 2) && !(fv & 4)) {  // eligible and unclaimed (v is this pass's only claimant)
            S.flags[v] = fv | 4;
            S.flags[th] |= 8;
            const int p = atomicAdd(&s_npairs, 1);
            S.pairs[2 * p] = v;
            S.pairs[2 * p + 1] = th;
          }
        }
        __syncthreads();
      }
    }
  } else {
    // idle thieves in index order, eligible victims ranked by (len desc, index asc)
    __shared__ int s_idle[kRefThreads];
    const int CH = (K + kRefThreads - 1) / kRefThreads;
    const int lo = t * CH, hi = min(K, lo + CH);
    int idle = 0;
    for (int i = lo; i < hi; ++i) idle += !(S.flags[i] & 1);
    s_idle[t] = idle;
    __syncthreads();
    for (int off = 1; off < kRefThreads; off <<= 1) {
      const int v = t >= off ? s_idle[t - off] : 0;
      __syncthreads();
      s_idle[t] += v;
      __syncthreads();
    }
    int r = s_idle[t] - idle;
    const int nidle = s_idle[kRefThreads - 1];
    for (int i = lo; i < hi; ++i)
      if (!(S.flags[i] & 1)) S.order[r++] = i;  // order[0..nidle): thieves
    __syncthreads();
    for (int v = t; v < K; v += kRefThreads) {
      if (!(S.flags[v] & 2)) continue;
      const u128 lv = S.len[v];
      int rank = 0;
      for (int u = 0; u < K; ++u)
        if ((S.flags[u] & 2) && (S.len[u] > lv || (S.len[u] == lv && u < v))) ++rank;
      if (rank < nidle) {
        const int p = atomicAdd(&s_npairs, 1);
        S.pairs[2 * p] = v;
        S.pairs[2 * p + 1] = S.order[rank];
      }
    }
    __syncthreads();
  }
  const int np = s_npairs;
  for (int p = t; p < np; p += kRefThreads) {
    const int v = S.pairs[2 * p], th = S.pairs[2 * p + 1];
    if (S.len[v] < 2) continue;  // do_steal refuses: end < pos + 2
    unsigned char* vb = S.state + static_cast<size_t>(v) * S.L.gstride;
    IvmHdr* vh = reinterpret_cast<IvmHdr*>(vb);
    int8_t* E = reinterpret_cast<int8_t*>(vb + S.L.o_end);
    int pos[kMaxN], D[kMaxN], mid[kMaxN], oe[kMaxN];
    raw_position(vb, S.L, pos);
    const bool had_end = vh->has_end != 0;
    int top = 0;
    diff_digits(pos, E, had_end, n, D, top);
    split_point(pos, D, top, 1, 2, n, mid);  // pos + floor((end - pos) / 2)
    for (int l = 0; l < n; ++l) oe[l] = E[l];
    for (int l = 0; l < n; ++l) E[l] = static_cast<int8_t>(mid[l]);
    vh->has_end = 1;
    seat_explorer(S.state + static_cast<size_t>(th) * S.L.gstride, S.L, S.ptot, mid, oe, had_end);
    atomicAdd(&s_ok, 1);
  }
  __syncthreads();
  if (t == 0) {
    S.ctr->steal_phases += 1ull;
    S.ctr->steals += static_cast<unsigned long long>(s_ok);
    S.ctr->inits += static_cast<unsigned long long>(s_ok);
    S.ctr->active = total_active + s_ok;
  }
}
