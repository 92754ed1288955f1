// ref_driver — command-line probe over the REFERENCE solver's public API.
//
// TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never the product).
// Built by oracle/Makefile against the unmodified reference sources under
// /root/reference/proj/src into oracle/_ref/ref_driver.  It drives:
//   * pool_run              (include/pbb/explorer.hpp:145, src/explorer.cpp:473-507)
//   * Ivm::init_at / explore_step (src/ivm.cpp:48-88, src/explorer.cpp:37-63)
//   * decompose             (src/bound.cpp:98-139)
//   * neh                   (src/heuristic.cpp:73-103)
// and prints one JSON object per run (or a text fixture for `nodes`).
//
// Modes
//   solve  <ta> <ub|neh> <K> <threads> [time_limit_s]      pool_run
//   hist   <ta|gen:n:m:seed> <ub>                         K=1 fixed tree + per-f histogram
//   nodes  <ta> <ub> <seed> <starts> <per_start>          per-node decompose dump
//   pinned <ta> <ub> <threads> <seconds> <prefix_depth>   prune>=ub, never improve
//   neh    <ta>                                           NEH makespan + perm
//   inst   <ta>                                           processing-time matrix
//   ils    <ta> <iterations> <rng_seed>                   NEH + insertion_local_search
//   ckpt   <ta> <path>  /  ckptload <ta> <path>           checkpoint_save / checkpoint_load
//   stats  <ta|gen:n:m:seed> <ub> <K> <threads> <batch_steps> <disable_pruning> <census>
//                                                         pool_run with every PoolStats field
//                                                         (+ the sorted census when asked)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pbb/bound.hpp"
#include "pbb/coordinator.hpp"
#include "pbb/explorer.hpp"
#include "pbb/factoradic.hpp"
#include "pbb/heuristic.hpp"
#include "pbb/instance.hpp"
#include "pbb/ivm.hpp"
#include "pbb/protocol.hpp"

using namespace pbb;

namespace {

std::int64_t parse_ub(const Instance& inst, const char* s) {
  if (std::strcmp(s, "neh") == 0) return neh(inst).cmax;
  return std::strtoll(s, nullptr, 10);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int lnz(const Factoradic& a) {
  int r = 0;
  for (int l = 0; l < a.size(); ++l)
    if (a.digits[l] != 0) r = l;
  return r;
}

Instance named_or_generated(const char* s) {
  if (std::strncmp(s, "gen:", 4) == 0) {
    int n = 0, m = 0;
    long seed = 0;
    if (std::sscanf(s + 4, "%d:%d:%ld", &n, &m, &seed) != 3) throw std::invalid_argument("gen:n:m:seed");
    return generate_taillard(n, m, static_cast<std::int32_t>(seed));
  }
  return taillard_named(s);
}

int cmd_solve(int argc, char** argv) {
  if (argc < 6) return 2;
  Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  PoolConfig cfg;
  cfg.explorers = std::atoi(argv[4]);
  cfg.threads = std::atoi(argv[5]);
  if (argc > 6) cfg.time_limit_s = std::atof(argv[6]);
  PoolResult r = pool_run(inst, ub, {}, cfg);
  std::printf(
      "{\"mode\":\"solve\",\"instance\":\"%s\",\"initial_ub\":%lld,\"best_value\":%lld,"
      "\"improved\":%s,\"decomposed\":%llu,\"leaves\":%llu,\"improvements\":%llu,"
      "\"local_steals\":%llu,\"intervals_initialized\":%llu,\"wall_s\":%.6f,\"completed\":%s,"
      "\"threads\":%d,\"explorers\":%d,\"best\":[",
      argv[2], (long long)ub, (long long)r.best_value, r.best.perm.empty() ? "false" : "true",
      (unsigned long long)r.stats.decomposed, (unsigned long long)r.stats.leaves,
      (unsigned long long)r.stats.improvements, (unsigned long long)r.stats.local_steals,
      (unsigned long long)r.stats.intervals_initialized, r.stats.wall_s,
      r.stats.completed ? "true" : "false", cfg.threads, cfg.explorers);
  for (std::size_t i = 0; i < r.best.perm.size(); ++i)
    std::printf("%s%d", i ? "," : "", r.best.perm[i]);
  std::printf("]}\n");
  return 0;
}

// K=1 fixed tree exactly as pool_run does it (init_at(0) replay, then the
// explore loop), with a histogram of decomposed nodes by free-job count f.
int cmd_hist(int argc, char** argv) {
  if (argc < 4) return 2;
  Instance inst = named_or_generated(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  const int n = inst.n;
  Ivm ivm(n);
  BoundScratch scratch;
  Decomposition dec;
  std::uint64_t decomposed = 0, leaves = 0, improvements = 0;
  std::int64_t best = ub;
  std::vector<std::uint64_t> hist(static_cast<std::size_t>(n) + 1, 0);
  const double t0 = now_s();
  ivm.init_at(Factoradic::zero(n), std::nullopt, BigCount::factorial(n), inst, best, scratch,
              &decomposed);
  for (std::uint64_t l = 0; l < decomposed; ++l) ++hist[static_cast<std::size_t>(n - 1 - l)];
  Schedule improved;
  for (;;) {
    const std::uint64_t before = decomposed;
    StepOutcome o = explore_step(ivm, inst, best, best, scratch, dec, decomposed, leaves, &improved,
                                 nullptr);
    if (o == StepOutcome::Exhausted) break;
    if (o == StepOutcome::ImprovedBest) {
      best = improved.cmax;
      ++improvements;
    }
    if (decomposed != before) ++hist[static_cast<std::size_t>(scratch.sub.free_count())];
  }
  const double wall = now_s() - t0;
  std::printf(
      "{\"mode\":\"hist\",\"instance\":\"%s\",\"initial_ub\":%lld,\"best_value\":%lld,"
      "\"decomposed\":%llu,\"leaves\":%llu,\"improvements\":%llu,\"wall_s\":%.6f,\"hist\":{",
      argv[2], (long long)ub, (long long)best, (unsigned long long)decomposed,
      (unsigned long long)leaves, (unsigned long long)improvements, wall);
  bool first = true;
  for (int f = 0; f <= n; ++f) {
    if (!hist[static_cast<std::size_t>(f)]) continue;
    std::printf("%s\"%d\":%llu", first ? "" : ",", f, (unsigned long long)hist[static_cast<std::size_t>(f)]);
    first = false;
  }
  std::printf("}}\n");
  return 0;
}

// Per-node decompose dump (SURVEY §8(d) sampler): uniform random factoradic
// starts, init_at with an infinite incumbent, then explore_step(prune=ub,
// improve=0); every decomposition prints one line
//   perm... | d1 d2 | dir | child_lb... | pruned...
int cmd_nodes(int argc, char** argv) {
  if (argc < 7) return 2;
  Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  std::mt19937_64 rng(std::strtoull(argv[4], nullptr, 10));
  const int starts = std::atoi(argv[5]);
  const int per_start = std::atoi(argv[6]);
  const int n = inst.n;
  BoundScratch scratch;
  Decomposition dec;
  std::printf("# instance %s n %d m %d ub %lld\n", argv[2], n, inst.m, (long long)ub);
  for (int s = 0; s < starts; ++s) {
    Factoradic a = Factoradic::zero(n);
    for (int l = 0; l < n; ++l) a.digits[l] = static_cast<int>(rng() % static_cast<std::uint64_t>(n - l));
    Ivm ivm(n);
    std::uint64_t decomposed = 0, leaves = 0;
    ivm.init_at(a, std::nullopt, BigCount::factorial(n), inst, kNoIncumbent, scratch, &decomposed);
    int emitted = 0;
    for (int guard = 0; emitted < per_start && guard < 50 * per_start; ++guard) {
      const std::uint64_t before = decomposed;
      StepOutcome o =
          explore_step(ivm, inst, ub, 0, scratch, dec, decomposed, leaves, nullptr, nullptr);
      if (o == StepOutcome::Exhausted) break;
      if (decomposed == before) continue;
      const Subproblem& sub = scratch.sub;
      for (int i = 0; i < n; ++i) std::printf("%s%d", i ? " " : "", sub.perm[i]);
      std::printf(" | %d %d | %d |", sub.d1, sub.d2, static_cast<int>(dec.direction));
      for (auto v : dec.child_lb) std::printf(" %lld", (long long)v);
      std::printf(" |");
      for (auto v : dec.pruned) std::printf(" %d", static_cast<int>(v));
      std::printf("\n");
      ++emitted;
    }
  }
  return 0;
}

// Pinned-UB throughput: prune >= ub, never improve; threads pull
// prefix-depth subtrees [a, a + (n-depth)!) from a shared counter.
int cmd_pinned(int argc, char** argv) {
  if (argc < 7) return 2;
  Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  const int threads = std::atoi(argv[4]);
  const double seconds = std::atof(argv[5]);
  const int depth = std::atoi(argv[6]);
  const int n = inst.n;
  std::uint64_t pieces = 1;
  for (int l = 0; l < depth; ++l) pieces *= static_cast<std::uint64_t>(n - l);
  std::atomic<std::uint64_t> next{0};
  std::atomic<bool> stop{false};
  std::atomic<std::uint64_t> tot_raw{0}, tot_unique{0}, tot_leaves{0};
  const double t0 = now_s();
  auto work = [&] {
    BoundScratch scratch;
    Decomposition dec;
    std::uint64_t raw = 0, dups = 0, leaves = 0;
    for (;;) {
      const std::uint64_t id = next.fetch_add(1);
      if (id >= pieces || stop.load(std::memory_order_relaxed)) break;
      Factoradic a = Factoradic::zero(n);
      std::uint64_t rest = id;
      for (int l = depth - 1; l >= 0; --l) {
        a.digits[l] = static_cast<int>(rest % static_cast<std::uint64_t>(n - l));
        rest /= static_cast<std::uint64_t>(n - l);
      }
      std::optional<Factoradic> b;
      BigCount bdec = BigCount::factorial(n);
      if (id + 1 < pieces) {
        Factoradic bb = Factoradic::zero(n);
        rest = id + 1;
        for (int l = depth - 1; l >= 0; --l) {
          bb.digits[l] = static_cast<int>(rest % static_cast<std::uint64_t>(n - l));
          rest /= static_cast<std::uint64_t>(n - l);
        }
        bdec = to_decimal(bb);
        b = bb;
      }
      Ivm ivm(n);
      std::uint64_t replay = 0;
      ivm.init_at(a, b, bdec, inst, ub, scratch, &replay);
      raw += replay;
      dups += std::min<std::uint64_t>(replay, static_cast<std::uint64_t>(lnz(a)));
      for (std::uint64_t it = 0;; ++it) {
        if ((it & 1023) == 0 && now_s() - t0 >= seconds) {
          stop.store(true);
          break;
        }
        if (explore_step(ivm, inst, ub, 0, scratch, dec, raw, leaves, nullptr, nullptr) ==
            StepOutcome::Exhausted)
          break;
      }
      if (stop.load(std::memory_order_relaxed)) break;
    }
    tot_raw += raw;
    tot_unique += raw - dups;
    tot_leaves += leaves;
  };
  std::vector<std::thread> team;
  for (int t = 1; t < threads; ++t) team.emplace_back(work);
  work();
  for (auto& th : team) th.join();
  const double wall = now_s() - t0;
  std::printf(
      "{\"mode\":\"pinned\",\"instance\":\"%s\",\"ub\":%lld,\"threads\":%d,\"decomposed\":%llu,"
      "\"unique\":%llu,\"leaves\":%llu,\"wall_s\":%.6f,\"nodes_per_s\":%.1f,\"exhausted\":%s}\n",
      argv[2], (long long)ub, threads, (unsigned long long)tot_raw.load(),
      (unsigned long long)tot_unique.load(), (unsigned long long)tot_leaves.load(), wall,
      static_cast<double>(tot_unique.load()) / wall, stop.load() ? "false" : "true");
  return 0;
}

int cmd_neh(int argc, char** argv) {
  if (argc < 3) return 2;
  Instance inst = taillard_named(argv[2]);
  Schedule s = neh(inst);
  std::printf("{\"mode\":\"neh\",\"instance\":\"%s\",\"cmax\":%lld,\"perm\":[", argv[2], (long long)s.cmax);
  for (std::size_t i = 0; i < s.perm.size(); ++i) std::printf("%s%d", i ? "," : "", s.perm[i]);
  std::printf("]}\n");
  return 0;
}

// NEH then insertion_local_search (src/heuristic.cpp:105-155) with an iteration budget.
int cmd_ils(int argc, char** argv) {
  if (argc < 5) return 2;
  Instance inst = taillard_named(argv[2]);
  SearchBudget budget;
  budget.max_iterations = std::strtoull(argv[3], nullptr, 10);
  Schedule s = insertion_local_search(inst, neh(inst), budget, std::strtoull(argv[4], nullptr, 10));
  std::printf("{\"mode\":\"ils\",\"instance\":\"%s\",\"iterations\":%s,\"rng_seed\":%s,\"cmax\":%lld,\"perm\":[",
              argv[2], argv[3], argv[4], (long long)s.cmax);
  for (std::size_t i = 0; i < s.perm.size(); ++i) std::printf("%s%d", i ? "," : "", s.perm[i]);
  std::printf("]}\n");
  return 0;
}

// checkpoint_save / checkpoint_load (src/coordinator.cpp:22-102) on fixed sample data
int cmd_ckpt(int argc, char** argv) {
  if (argc < 4) return 2;
  Instance inst = taillard_named(argv[2]);
  CheckpointData d;
  Schedule s = neh(inst);
  d.best_value = s.cmax;
  d.best_schedule = s.perm;
  d.total_nodes = 123456789;
  const BigCount nf = BigCount::factorial(inst.n);
  WorkUnit u1;
  u1.kmax = 4;
  u1.intervals = {Interval(BigCount(0), BigCount(1000)), Interval(BigCount(5000), nf)};
  WorkUnit u2;
  u2.kmax = 2;
  u2.intervals = {Interval(nf / 2, nf / 2 + BigCount(7))};
  d.units = {u1, u2};
  checkpoint_save(argv[3], inst, d);
  return 0;
}

int cmd_ckptload(int argc, char** argv) {
  if (argc < 4) return 2;
  Instance inst = taillard_named(argv[2]);
  CheckpointData d = checkpoint_load(argv[3], inst);
  std::printf("{\"best\":%lld,\"nodes\":%llu,\"units\":[", (long long)d.best_value, (unsigned long long)d.total_nodes);
  for (std::size_t u = 0; u < d.units.size(); ++u) {
    std::printf("%s{\"kmax\":%u,\"intervals\":[", u ? "," : "", d.units[u].kmax);
    for (std::size_t i = 0; i < d.units[u].intervals.size(); ++i)
      std::printf("%s[\"%s\",\"%s\"]", i ? "," : "", d.units[u].intervals[i].a.str().c_str(), d.units[u].intervals[i].b.str().c_str());
    std::printf("]}");
  }
  std::printf("]}\n");
  return 0;
}

int cmd_stats(int argc, char** argv) {
  if (argc < 9) return 2;
  Instance inst = named_or_generated(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  PoolConfig cfg;
  cfg.explorers = std::atoi(argv[4]);
  cfg.threads = std::atoi(argv[5]);
  cfg.batch_steps = std::atoi(argv[6]);
  cfg.disable_pruning = std::atoi(argv[7]) != 0;
  cfg.record_census = std::atoi(argv[8]) != 0;
  PoolResult r = pool_run(inst, ub, {}, cfg);
  std::sort(r.census.begin(), r.census.end());
  std::printf(
      "{\"mode\":\"stats\",\"instance\":\"%s\",\"initial_ub\":%lld,\"best_value\":%lld,\"explorers\":%d,"
      "\"threads\":%d,\"batch_steps\":%d,\"disable_pruning\":%d,\"decomposed\":%llu,\"leaves\":%llu,"
      "\"improvements\":%llu,\"local_steals\":%llu,\"steal_phases\":%llu,\"intervals_initialized\":%llu,"
      "\"completed\":%s,\"census_size\":%zu,\"census_distinct\":%zu}\n",
      argv[2], (long long)ub, (long long)r.best_value, cfg.explorers, cfg.threads, cfg.batch_steps,
      cfg.disable_pruning ? 1 : 0, (unsigned long long)r.stats.decomposed, (unsigned long long)r.stats.leaves,
      (unsigned long long)r.stats.improvements, (unsigned long long)r.stats.local_steals,
      (unsigned long long)r.stats.steal_phases, (unsigned long long)r.stats.intervals_initialized,
      r.stats.completed ? "true" : "false", r.census.size(),
      static_cast<size_t>(std::unique(r.census.begin(), r.census.end()) - r.census.begin()));
  return 0;
}

// Wire frames encoded by the reference (src/protocol.cpp) for the codec golden file: one line
// per frame, "<sender> <n> <hex>" (sender W = worker, C = coordinator; n = the instance size the
// intervals belong to).
int cmd_frames(int, char**) {
  std::mt19937_64 rng(2012);
  auto emit = [](const char* who, int n, const Message& m) {
    const std::vector<std::uint8_t> fr = encode(m);
    std::printf("%s %d ", who, n);
    for (std::uint8_t b : fr) std::printf("%02x", b);
    std::printf("\n");
  };
  for (int n : {5, 20, 50, 500}) {
    const BigCount nf = BigCount::factorial(n);
    std::vector<BigCount> pts;  // random points from random digit vectors, cut into pieces
    for (int t = 0; t < 12; ++t) {
      Factoradic x = Factoradic::zero(n);
      for (int l = 0; l < n; ++l) x.digits[l] = static_cast<int>(rng() % static_cast<std::uint64_t>(n - l));
      pts.push_back(to_decimal(x));
    }
    std::sort(pts.begin(), pts.end());
    std::vector<Interval> ivs;
    for (std::size_t t = 0; t + 1 < pts.size(); t += 2)
      if (pts[t] < pts[t + 1]) ivs.emplace_back(pts[t], pts[t + 1]);
    ivs.emplace_back(pts.back(), nf);
    std::vector<Interval> norm = normalize(ivs);
    WorkRequest req;
    req.worker_id = static_cast<std::uint32_t>(n);
    req.nodes_since_checkpoint = 1234567890123ull + static_cast<std::uint64_t>(n);
    req.kmax = 4736;
    req.intervals = norm;
    emit("W", n, req);
    emit("W", n, WorkRequest{7, 0, 16, {}});
    emit("C", n, WorkReply{norm});
    emit("C", n, WorkReply{{Interval(BigCount(1), BigCount(2))}});
  }
  std::vector<std::uint32_t> sched;
  for (std::uint32_t j = 0; j < 20; ++j) sched.push_back((j * 7) % 20);
  emit("W", 20, BestMsg{2297, sched});
  emit("C", 20, BestMsg{2297, {}});
  emit("C", 20, BestMsg{kNoMakespan, {}});
  emit("W", 20, EndMsg{1278, sched});
  emit("C", 20, EndMsg{kNoMakespan, {}});
  return 0;
}

int cmd_inst(int argc, char** argv) {
  if (argc < 3) return 2;
  Instance inst = taillard_named(argv[2]);
  std::printf("%d %d\n", inst.n, inst.m);
  for (int j = 0; j < inst.n; ++j) {
    for (int k = 0; k < inst.m; ++k) std::printf("%s%d", k ? " " : "", inst.pt(j, k));
    std::printf("\n");
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver solve|hist|nodes|pinned|neh|inst ...\n");
    return 2;
  }
  const std::string mode = argv[1];
  int rc = 2;
  try {
    if (mode == "solve") rc = cmd_solve(argc, argv);
    else if (mode == "hist") rc = cmd_hist(argc, argv);
    else if (mode == "nodes") rc = cmd_nodes(argc, argv);
    else if (mode == "pinned") rc = cmd_pinned(argc, argv);
    else if (mode == "neh") rc = cmd_neh(argc, argv);
    else if (mode == "inst") rc = cmd_inst(argc, argv);
    else if (mode == "ils") rc = cmd_ils(argc, argv);
    else if (mode == "ckpt") rc = cmd_ckpt(argc, argv);
    else if (mode == "ckptload") rc = cmd_ckptload(argc, argv);
    else if (mode == "stats") rc = cmd_stats(argc, argv);
    else if (mode == "frames") rc = cmd_frames(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver: %s\n", e.what());
    return 1;
  }
  if (rc == 2) std::fprintf(stderr, "ref_driver: bad arguments for %s\n", mode.c_str());
  return rc;
}
