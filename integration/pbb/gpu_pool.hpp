// pbb/gpu_pool.hpp — reference-side binding of the B200 explorer pool (what a maintainer of
// /root/reference/proj adds next to include/pbb/explorer.hpp).
//
// GpuExplorerPool has ExplorerPool's method set (include/pbb/explorer.hpp:66-103) so that
// worker_run (src/worker.cpp:138-296) and pool_run-style drivers can swap it in. It wraps the
// C-ABI of libpbbgpu.so (include/pbbgpu.h): BigCount interval endpoints become factoradic
// digit vectors at this boundary (from_decimal / to_decimal, src/factoradic.cpp:18-49), the
// C-ABI's status codes become the reference's exception types.
//
// Compiled against the reference headers by integration/Makefile (integration/gpu_worker.cpp).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbb/explorer.hpp"
#include "pbb/factoradic.hpp"
#include "pbb/instance.hpp"
#include "pbb/workunit.hpp"
#include "pbbgpu.h"

namespace pbb {

inline void pbbgpu_check(int rc) {
  if (rc == PBBGPU_OK) return;
  const std::string msg = pbbgpu_last_error();
  if (rc == PBBGPU_ERR_ARG) throw std::invalid_argument(msg);
  if (rc == PBBGPU_ERR_STATE) throw std::logic_error(msg);
  throw std::runtime_error(msg);  // capacity, device
}

class GpuExplorerPool {
 public:
  // bound: PBBGPU_LB1 (the reference's decompose) or PBBGPU_LB2. steal_policy 1 reproduces the
  // reference's steal_phase and round length exactly (raw PoolStats equal on fixed trees).
  GpuExplorerPool(const Instance& inst, const PoolConfig& cfg, int bound = PBBGPU_LB1, int steal_policy = 0)
      : inst_(inst) {
    pbbgpu_config_t c{};
    c.explorers = cfg.explorers > 0 ? cfg.explorers : 0;  // 0 = fill the GPU
    c.disable_pruning = cfg.disable_pruning ? 1 : 0;
    c.time_limit_s = cfg.time_limit_s;
    c.record_census = cfg.record_census ? 1 : 0;
    c.timeline_path = cfg.timeline_path.empty() ? nullptr : cfg.timeline_path.c_str();
    c.steal_policy = steal_policy;
    if (steal_policy == 1) c.steps_per_round = cfg.batch_steps;
    pbbgpu_check(pbbgpu_create(inst.n, inst.m, inst.p.data(), bound, &c, &h_));
  }
  ~GpuExplorerPool() { pbbgpu_destroy(h_); }
  GpuExplorerPool(const GpuExplorerPool&) = delete;
  GpuExplorerPool& operator=(const GpuExplorerPool&) = delete;

  int K() const { return pbbgpu_K(h_); }
  const Instance& instance() const { return inst_; }

  void set_initial_bound(std::int64_t ub, std::span<const int> sched) {
    pbbgpu_check(pbbgpu_set_initial_bound(h_, ub, sched.data(), static_cast<int>(sched.size())));
  }
  void assign_fresh(std::span<const Interval> intervals) {
    Digits d = digits(intervals);
    pbbgpu_check(pbbgpu_assign(h_, d.a.data(), d.b.data(), d.nf.data(), d.count));
  }
  void apply_work_update(std::span<const Interval> intervals) {
    Digits d = digits(intervals);
    pbbgpu_check(pbbgpu_apply_work_update(h_, d.a.data(), d.b.data(), d.nf.data(), d.count));
  }
  int run_round() {
    int a = 0;
    pbbgpu_check(pbbgpu_run_round(h_, &a));
    return a;
  }
  int active_count() const {
    int a = 0;
    pbbgpu_check(pbbgpu_active_count(h_, &a));
    return a;
  }
  std::vector<Interval> snapshot_intervals() const {
    const int n = inst_.n, k = K();
    std::vector<std::uint16_t> pos(static_cast<std::size_t>(k) * n), end(static_cast<std::size_t>(k) * n);
    std::vector<std::uint8_t> nf(static_cast<std::size_t>(k));
    int cnt = 0;
    std::uint64_t recount = 0;
    pbbgpu_check(pbbgpu_snapshot_ex(h_, pos.data(), end.data(), nf.data(), k, &cnt, &recount));
    const BigCount nfact = BigCount::factorial(n);
    std::vector<Interval> out;
    for (int i = 0; i < cnt; ++i) {
      const BigCount a = to_decimal(fact(pos.data() + static_cast<std::size_t>(i) * n));
      const BigCount b = nf[static_cast<std::size_t>(i)] ? nfact : to_decimal(fact(end.data() + static_cast<std::size_t>(i) * n));
      if (a < b) out.emplace_back(a, b);
    }
    return normalize(std::move(out));
  }
  std::int64_t best_value() const {
    std::int64_t v = 0;
    pbbgpu_check(pbbgpu_best(h_, &v, nullptr, nullptr));
    return v;
  }
  Schedule best_schedule() const {
    std::int64_t v = 0;
    int has = 0;
    Schedule s;
    s.perm.assign(static_cast<std::size_t>(inst_.n), 0);
    pbbgpu_check(pbbgpu_best_schedule(h_, &v, s.perm.data(), &has));
    if (!has) return Schedule{};
    s.cmax = v;
    return s;
  }
  void offer_bound(std::int64_t v) { pbbgpu_check(pbbgpu_offer_bound(h_, v)); }
  bool offer_schedule(const Schedule& cand) {
    if (cand.perm.empty() || cand.cmax < 0) return false;
    int taken = 0;
    pbbgpu_check(pbbgpu_offer_schedule(h_, cand.perm.data(), cand.cmax, &taken));
    return taken != 0;
  }
  bool improved_since_mark() {
    int v = 0;
    pbbgpu_check(pbbgpu_improved_since_mark(h_, &v));
    return v != 0;
  }
  std::uint64_t steals_since_mark() const {
    std::uint64_t v = 0;
    pbbgpu_check(pbbgpu_steals_since_mark(h_, &v));
    return v;
  }
  void reset_steal_mark() { pbbgpu_check(pbbgpu_reset_steal_mark(h_)); }
  std::vector<Schedule> promote_solutions(int capacity) {
    std::vector<Schedule> out;
    if (capacity <= 0) return out;
    std::vector<std::int32_t> perms(static_cast<std::size_t>(capacity) * inst_.n);
    std::vector<std::int64_t> cm(static_cast<std::size_t>(capacity));
    int cnt = 0;
    pbbgpu_check(pbbgpu_promote(h_, capacity, perms.data(), cm.data(), &cnt));
    for (int i = 0; i < cnt; ++i) {
      Schedule s;
      s.perm.assign(perms.begin() + static_cast<std::ptrdiff_t>(i) * inst_.n,
                    perms.begin() + static_cast<std::ptrdiff_t>(i + 1) * inst_.n);
      s.cmax = cm[static_cast<std::size_t>(i)];
      out.push_back(std::move(s));
    }
    return out;
  }
  PoolStats stats() const {
    pbbgpu_stats_t s{};
    pbbgpu_check(pbbgpu_stats(h_, &s));
    PoolStats st;
    st.decomposed = s.decomposed;  // raw (replays included), PoolStats semantics
    st.leaves = s.leaves;
    st.improvements = s.improvements;
    st.local_steals = s.local_steals;
    st.steal_phases = s.steal_phases;
    st.intervals_initialized = s.intervals_initialized;
    st.completed = s.completed != 0;
    return st;
  }
  // the partition-invariant count (raw minus replay duplicates), not in PoolStats
  std::uint64_t unique_decomposed() const {
    pbbgpu_stats_t s{};
    pbbgpu_check(pbbgpu_stats(h_, &s));
    return s.unique;
  }
  std::vector<std::uint64_t> take_census() {
    std::vector<std::uint64_t> out(1u << 20);
    std::int64_t cnt = 0;
    pbbgpu_check(pbbgpu_take_census(h_, out.data(), static_cast<std::int64_t>(out.size()), &cnt));
    out.resize(static_cast<std::size_t>(cnt));
    return out;
  }
  void flush_timeline() { pbbgpu_check(pbbgpu_flush_timeline(h_)); }

 private:
  struct Digits {
    std::vector<std::uint16_t> a, b;
    std::vector<std::uint8_t> nf;
    int count = 0;
  };
  Digits digits(std::span<const Interval> intervals) const {
    Digits d;
    const int n = inst_.n;
    const BigCount nfact = BigCount::factorial(n);
    for (const Interval& iv : intervals) {
      if (iv.a > iv.b) throw std::invalid_argument("interval with a > b");
      if (iv.b > nfact) throw std::invalid_argument("interval beyond n!");
      if (iv.empty()) continue;
      for (int x : from_decimal(iv.a, n).digits) d.a.push_back(static_cast<std::uint16_t>(x));
      const bool inf = !(iv.b < nfact);
      d.nf.push_back(inf ? 1 : 0);
      const Factoradic fb = inf ? Factoradic::zero(n) : from_decimal(iv.b, n);
      for (int x : fb.digits) d.b.push_back(static_cast<std::uint16_t>(x));
      ++d.count;
    }
    return d;
  }
  Factoradic fact(const std::uint16_t* p) const {
    return Factoradic(std::vector<int>(p, p + inst_.n));
  }

  Instance inst_;
  pbbgpu_pool* h_ = nullptr;
};

}  // namespace pbb
