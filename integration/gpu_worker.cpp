// gpu_worker — the reference's own distributed runtime driving B200 explorer pools.
//
// Integration harness (not the product): compiled against the UNMODIFIED reference headers
// and objects (oracle/_ref/*.o, built from /root/reference/proj/src by oracle/Makefile) plus
// libpbbgpu.so, through the reference-side binding integration/pbb/gpu_pool.hpp.
//
//   gpu_worker pool <ta> <ub> <K> <lb1|lb2> <steal_policy> <batch_steps>
//       pool_run's loop (src/explorer.cpp:473-507) over GpuExplorerPool
//   gpu_worker tcp <ta> <ub> <workers> <lb1|lb2>
//       Coordinator::run over the reference's TcpListener (src/transport.cpp) on 127.0.0.1,
//       workers = libpbbgpu's own worker role and wire codec (pbbgpu_worker_run,
//       csrc/wire.cpp), one GPU pool each: the product speaking the reference's protocol
//   gpu_worker cluster <ta> <ub> <workers> <lb1|lb2>
//       Coordinator::run (src/coordinator.cpp:241-306) over make_inproc_cluster (every message
//       encoded / decoded by src/protocol.cpp), one GPU worker thread per transport endpoint,
//       each running worker_run's pool-role loop (src/worker.cpp:138-296) on a GpuExplorerPool:
//       apply_work_update -> run_round -> improved_since_mark -> BEST, snapshot triggers
//       (steals_since_mark >= K/5, checkpoint timer, exhaustion) -> WORK checkpoints.
//       The comm agent's request/reply exchange runs inline (one outstanding message, as the
//       reference's single-slot outbox enforces); no heuristic agents.
// Prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "pbb/coordinator.hpp"
#include "pbb/gpu_pool.hpp"
#include "pbb/heuristic.hpp"
#include "pbb/protocol.hpp"
#include "pbb/transport.hpp"
#include "pbb/worker.hpp"  // WorkerConfig / the worker_run contract (worker.cpp itself is not linked)

using namespace pbb;

namespace {

int bound_of(const char* s) { return std::strcmp(s, "lb2") == 0 ? PBBGPU_LB2 : PBBGPU_LB1; }

std::int64_t parse_ub(const Instance& inst, const char* s) {
  if (std::strcmp(s, "neh") == 0) return neh(inst).cmax;
  return std::strtoll(s, nullptr, 10);
}

int cmd_pool(int argc, char** argv) {
  if (argc < 8) return 2;
  const Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  PoolConfig cfg;
  cfg.explorers = std::atoi(argv[4]);
  cfg.batch_steps = std::atoi(argv[7]);
  GpuExplorerPool pool(inst, cfg, bound_of(argv[5]), std::atoi(argv[6]));
  pool.set_initial_bound(ub, {});
  const Interval all(BigCount(0), BigCount::factorial(inst.n));
  pool.assign_fresh(std::span<const Interval>(&all, 1));
  while (pool.run_round() > 0) {
  }
  const PoolStats st = pool.stats();
  const Schedule best = pool.best_schedule();
  std::printf(
      "{\"mode\":\"pool\",\"instance\":\"%s\",\"initial_ub\":%lld,\"best_value\":%lld,\"has_schedule\":%s,"
      "\"decomposed\":%llu,\"unique\":%llu,\"leaves\":%llu,\"local_steals\":%llu,\"steal_phases\":%llu,"
      "\"intervals_initialized\":%llu,\"K\":%d}\n",
      argv[2], (long long)ub, (long long)pool.best_value(), best.evaluated() ? "true" : "false",
      (unsigned long long)st.decomposed, (unsigned long long)pool.unique_decomposed(),
      (unsigned long long)st.leaves, (unsigned long long)st.local_steals, (unsigned long long)st.steal_phases,
      (unsigned long long)st.intervals_initialized, pool.K());
  return 0;
}

struct GpuWorkerResult {
  Schedule local_best;
  PoolStats stats;
  std::uint64_t unique = 0;
  std::uint64_t checkpoints_sent = 0;
  std::uint64_t bests_sent = 0;
  std::uint64_t updates_applied = 0;
};

std::vector<std::uint32_t> to_wire(const std::vector<int>& perm) { return {perm.begin(), perm.end()}; }

// worker_run's pool role (src/worker.cpp:138-296) with a GpuExplorerPool.
GpuWorkerResult gpu_worker_run(WorkerTransport& transport, const Instance& inst, const WorkerConfig& cfg,
                               int bound) {
  using clock = std::chrono::steady_clock;
  GpuExplorerPool pool(inst, cfg.pool, bound);
  Schedule seed = neh(inst);
  if (inst.n > 1) {
    SearchBudget bud;
    bud.max_iterations = 2000;
    seed = insertion_local_search(inst, seed, bud, cfg.rng_seed);
  }
  pool.set_initial_bound(seed.cmax, seed.perm);
  if (cfg.initial_ub != kNoIncumbent) pool.offer_bound(cfg.initial_ub);
  pool.improved_since_mark();

  GpuWorkerResult res;
  std::optional<std::vector<Interval>> work;
  bool done = false;
  // one request / reply exchange (the comm agent's loop body, src/worker.cpp:158-202)
  auto exchange = [&](const Message& msg) {
    transport.send(msg);
    Message reply = transport.receive();
    if (const auto* best = std::get_if<BestMsg>(&reply)) {
      if (best->makespan != kNoMakespan) pool.offer_bound(static_cast<std::int64_t>(best->makespan));
    } else if (auto* w = std::get_if<WorkReply>(&reply)) {
      work = std::move(w->intervals);
    } else if (const auto* end = std::get_if<EndMsg>(&reply)) {
      if (end->makespan != kNoMakespan) pool.offer_bound(static_cast<std::int64_t>(end->makespan));
      const Schedule local = pool.best_schedule();
      EndMsg bye;
      if (local.evaluated()) {
        bye.makespan = static_cast<std::uint64_t>(local.cmax);
        bye.schedule = to_wire(local.perm);
      }
      transport.send(bye);
      done = true;
    } else {
      throw std::runtime_error("unexpected message from coordinator");
    }
  };

  const std::uint64_t steal_threshold = std::max<std::uint64_t>(1, (static_cast<std::uint64_t>(pool.K()) + 4) / 5);
  auto last_checkpoint = clock::time_point{};
  std::uint64_t nodes_at_last_snapshot = 0;
  bool pending_best = cfg.send_initial_best;
  while (!done) {
    if (work) {
      pool.apply_work_update(*work);
      work.reset();
      ++res.updates_applied;
    }
    const int active = pool.run_round();
    if (pool.improved_since_mark()) pending_best = true;
    if (pending_best) {
      const Schedule b = pool.best_schedule();
      if (b.evaluated()) {
        exchange(BestMsg{static_cast<std::uint64_t>(b.cmax), to_wire(b.perm)});
        ++res.bests_sent;
      }
      pending_best = false;
      if (done) break;
    }
    const double since_cp = std::chrono::duration<double>(clock::now() - last_checkpoint).count();
    if (pool.steals_since_mark() >= steal_threshold || since_cp >= cfg.checkpoint_period_s || active == 0) {
      WorkRequest req;
      req.worker_id = cfg.worker_id;
      const std::uint64_t nodes = pool.stats().decomposed;
      req.nodes_since_checkpoint = nodes - nodes_at_last_snapshot;
      req.kmax = static_cast<std::uint32_t>(pool.K());
      req.intervals = pool.snapshot_intervals();
      exchange(req);
      nodes_at_last_snapshot = nodes;
      pool.reset_steal_mark();
      last_checkpoint = clock::now();
      ++res.checkpoints_sent;
      if (active == 0 && !work && !done) std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  res.local_best = pool.best_schedule();
  res.stats = pool.stats();
  res.unique = pool.unique_decomposed();
  return res;
}

int cmd_cluster(int argc, char** argv) {
  if (argc < 6) return 2;
  const Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  const int W = std::atoi(argv[4]);
  const int bound = bound_of(argv[5]);
  InProcCluster cl = make_inproc_cluster(W);
  CoordinatorConfig ccfg;
  Coordinator coord(inst, ccfg);
  coord.add_initial_interval();
  std::vector<GpuWorkerResult> results(static_cast<std::size_t>(W));
  std::vector<std::string> errors(static_cast<std::size_t>(W));
  std::vector<std::thread> workers;
  for (int w = 0; w < W; ++w) {
    workers.emplace_back([&, w] {
      try {
        WorkerConfig wc;
        wc.worker_id = static_cast<std::uint32_t>(w);
        wc.initial_ub = ub;
        wc.checkpoint_period_s = 0.05;
        wc.rng_seed = 1 + static_cast<std::uint64_t>(w);
        results[static_cast<std::size_t>(w)] = gpu_worker_run(*cl.workers[static_cast<std::size_t>(w)], inst, wc, bound);
      } catch (const std::exception& e) {
        errors[static_cast<std::size_t>(w)] = e.what();
      }
    });
  }
  const CoordinatorResult cr = coord.run(*cl.coordinator);
  for (auto& t : workers) t.join();
  for (const std::string& e : errors)
    if (!e.empty()) throw std::runtime_error("worker failed: " + e);
  std::uint64_t unique = 0, raw = 0, leaves = 0, updates = 0, cps = 0;
  for (const GpuWorkerResult& r : results) {
    unique += r.unique;
    raw += r.stats.decomposed;
    leaves += r.stats.leaves;
    updates += r.updates_applied;
    cps += r.checkpoints_sent;
  }
  std::printf(
      "{\"mode\":\"cluster\",\"instance\":\"%s\",\"initial_ub\":%lld,\"workers\":%d,\"best_value\":%lld,"
      "\"coordinator_total_nodes\":%llu,\"splits\":%llu,\"messages\":%llu,\"decomposed\":%llu,\"unique\":%llu,"
      "\"leaves\":%llu,\"updates_applied\":%llu,\"checkpoints\":%llu,\"wall_s\":%.3f}\n",
      argv[2], (long long)ub, W, (long long)cr.best_value, (unsigned long long)cr.total_nodes,
      (unsigned long long)cr.splits, (unsigned long long)cr.messages, (unsigned long long)raw,
      (unsigned long long)unique, (unsigned long long)leaves, (unsigned long long)updates, (unsigned long long)cps,
      cr.wall_s);
  return 0;
}

int cmd_tcp(int argc, char** argv) {
  if (argc < 6) return 2;
  const Instance inst = taillard_named(argv[2]);
  const std::int64_t ub = parse_ub(inst, argv[3]);
  const int W = std::atoi(argv[4]);
  const int bound = bound_of(argv[5]);
  TcpListener listener("127.0.0.1", 0);
  const int port = listener.port();
  std::vector<pbbgpu_worker_result_t> res(static_cast<std::size_t>(W));
  std::vector<pbbgpu_stats_t> st(static_cast<std::size_t>(W));
  std::vector<std::string> errors(static_cast<std::size_t>(W));
  std::vector<std::thread> workers;
  for (int w = 0; w < W; ++w) {
    workers.emplace_back([&, w] {
      pbbgpu_pool* pool = nullptr;
      pbbgpu_config_t c{};
      int rc = pbbgpu_create(inst.n, inst.m, inst.p.data(), bound, &c, &pool);
      if (rc == PBBGPU_OK) {
        pbbgpu_worker_config_t wc{};
        wc.worker_id = static_cast<std::uint32_t>(w);
        wc.initial_ub = ub;
        wc.checkpoint_period_s = 0.05;
        wc.rng_seed = 1 + static_cast<std::uint64_t>(w);
        rc = pbbgpu_worker_run(pool, "127.0.0.1", port, &wc, &res[static_cast<std::size_t>(w)]);
        if (rc == PBBGPU_OK) rc = pbbgpu_stats(pool, &st[static_cast<std::size_t>(w)]);
      }
      if (rc != PBBGPU_OK) errors[static_cast<std::size_t>(w)] = pbbgpu_last_error();
      pbbgpu_destroy(pool);
    });
  }
  CoordinatorConfig ccfg;
  Coordinator coord(inst, ccfg);
  coord.add_initial_interval();
  const std::shared_ptr<CoordinatorTransport> transport = listener.accept_workers(W);
  const CoordinatorResult cr = coord.run(*transport);
  for (auto& t : workers) t.join();
  for (const std::string& e : errors)
    if (!e.empty()) throw std::runtime_error("worker failed: " + e);
  std::uint64_t unique = 0, raw = 0, leaves = 0, updates = 0, msgs = 0;
  for (int w = 0; w < W; ++w) {
    unique += st[static_cast<std::size_t>(w)].unique;
    raw += st[static_cast<std::size_t>(w)].decomposed;
    leaves += st[static_cast<std::size_t>(w)].leaves;
    updates += res[static_cast<std::size_t>(w)].updates_applied;
    msgs += res[static_cast<std::size_t>(w)].messages;
  }
  std::printf(
      "{\"mode\":\"tcp\",\"instance\":\"%s\",\"initial_ub\":%lld,\"workers\":%d,\"best_value\":%lld,"
      "\"coordinator_total_nodes\":%llu,\"splits\":%llu,\"messages\":%llu,\"worker_messages\":%llu,"
      "\"decomposed\":%llu,\"unique\":%llu,\"leaves\":%llu,\"updates_applied\":%llu,\"wall_s\":%.3f}\n",
      argv[2], (long long)ub, W, (long long)cr.best_value, (unsigned long long)cr.total_nodes,
      (unsigned long long)cr.splits, (unsigned long long)cr.messages, (unsigned long long)msgs,
      (unsigned long long)raw, (unsigned long long)unique, (unsigned long long)leaves, (unsigned long long)updates,
      cr.wall_s);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: gpu_worker pool|cluster ...\n");
    return 2;
  }
  int rc = 2;
  try {
    if (std::strcmp(argv[1], "pool") == 0) rc = cmd_pool(argc, argv);
    else if (std::strcmp(argv[1], "cluster") == 0) rc = cmd_cluster(argc, argv);
    else if (std::strcmp(argv[1], "tcp") == 0) rc = cmd_tcp(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "gpu_worker: %s\n", e.what());
    return 1;
  }
  if (rc == 2) std::fprintf(stderr, "gpu_worker: bad arguments\n");
  return rc;
}
