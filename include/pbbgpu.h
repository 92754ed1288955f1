/* pbbgpu.h — C-ABI of the B200-native PFSP Branch-and-Bound explorer pool.
 *
 * Drop-in boundary for the reference solver's solve/explore path. Each entry point names
 * the reference interface it replaces (paths under /root/reference/proj):
 *
 *   pbbgpu_create / pbbgpu_destroy  <- ExplorerPool::ExplorerPool(const Instance&, PoolConfig)
 *                                      (include/pbb/explorer.hpp:68, src/explorer.cpp:87-106)
 *   pbbgpu_K                        <- ExplorerPool::K()                (explorer.hpp:70)
 *   pbbgpu_set_initial_bound        <- ExplorerPool::set_initial_bound  (explorer.hpp:73)
 *   pbbgpu_assign                   <- ExplorerPool::assign_fresh       (explorer.hpp:76)
 *   pbbgpu_assign_split             <- assign_fresh of [0,n!) cut into K equal ranges
 *                                      (pool_run's default interval, explorer.cpp:479)
 *   pbbgpu_assign_split_range       <- initial partition of [0,n!) over GPUs
 *   pbbgpu_export                   <- split_unit right halves for another worker
 *                                      (src/workunit.cpp:59-74, src/coordinator.cpp:170-187)
 *   pbbgpu_run_round                <- ExplorerPool::run_round          (explorer.hpp:85)
 *   pbbgpu_apply_work_update        <- ExplorerPool::apply_work_update  (explorer.hpp:78-81)
 *   pbbgpu_improved_since_mark      <- ExplorerPool::improved_since_mark (explorer.hpp:94)
 *   pbbgpu_steals_since_mark / pbbgpu_reset_steal_mark
 *                                   <- steals_since_mark / reset_steal_mark (explorer.hpp:95-96)
 *   pbbgpu_take_census              <- ExplorerPool::take_census        (explorer.hpp:102)
 *   pbbgpu_flush_timeline           <- ExplorerPool::flush_timeline     (explorer.hpp:103)
 *   pbbgpu_active_count             <- ExplorerPool::active_count       (explorer.hpp:87)
 *   pbbgpu_snapshot                 <- ExplorerPool::snapshot_intervals (explorer.hpp:88)
 *   pbbgpu_best                     <- best_value / best_schedule       (explorer.hpp:90-91)
 *   pbbgpu_best_schedule            <- best_schedule with its own makespan (explorer.cpp:352-377)
 *   pbbgpu_offer_bound              <- ExplorerPool::offer_bound        (explorer.hpp:92)
 *   pbbgpu_stats                    <- ExplorerPool::stats              (explorer.hpp:101)
 *   pbbgpu_histogram                <- (new) decomposed nodes by free-job count (roofline)
 *   pbbgpu_decompose_batch          <- decompose(inst, sub, incumbent, ...) (bound.hpp:78-79)
 *   pbbgpu_solve                    <- pool_run(inst, ub, intervals, cfg) (explorer.hpp:145-146)
 *   pbbgpu_insertion_ls             <- insertion_local_search           (heuristic.hpp:27, heuristic.cpp:105-155)
 *   pbbgpu_offer_schedule           <- ExplorerPool::offer_schedule     (explorer.hpp:93)
 *   pbbgpu_promote                  <- ExplorerPool::promote_solutions  (explorer.hpp:99, explorer.cpp:397-424)
 *   pbbgpu_explorer_lengths         <- timeline sampling                (explorer.cpp:71-85, 448-464)
 *   pbbgpu_int32_peak               <- (new) integer-ALU roofline denominator
 *   pbbgpu_worker_run               <- worker_run's pool role over the reference's TCP protocol
 *                                      (src/worker.cpp:138-296, src/protocol.cpp, src/transport.cpp)
 *   pbbgpu_wire_reencode            <- encode / decode (src/protocol.cpp:104-177)
 *   pbbgpu_group_*                  <- Coordinator/worker WORK+BEST exchange inside one box
 *                                      (src/coordinator.cpp:170-306, src/workunit.cpp:59-74) over
 *                                      NVLink peer memory
 *   pbbgpu_taillard / pbbgpu_makespan / pbbgpu_neh
 *                                   <- generate_taillard / taillard_named / makespan / neh
 *                                      (instance.hpp:42-48, heuristic.hpp:21)
 *
 * Conventions: int status, 0 = OK, negative = error class (no exceptions cross the ABI);
 * pbbgpu_last_error() returns the message of the last failure on the calling thread.
 * Factoradic vectors are MSD first, digit l in [0, n-1-l] (factoradic.hpp:12-26); an
 * interval end equal to n! is passed with b_is_nfact = 1. Bounds are int64 makespans;
 * kNoIncumbent = INT64_MAX. The product path has no CPU fallback: every compute entry
 * fails with PBBGPU_ERR_CUDA when no sm_100 device is present.
 */
#ifndef PBBGPU_H
#define PBBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBBGPU_OK 0
#define PBBGPU_ERR_ARG -1      /* std::invalid_argument in the reference */
#define PBBGPU_ERR_STATE -2    /* std::logic_error */
#define PBBGPU_ERR_CUDA -3     /* device / driver failure, no GPU */
#define PBBGPU_ERR_CAPACITY -4 /* std::runtime_error (capacity) */
#define PBBGPU_ERR_TRANSPORT -5 /* TransportError (transport.hpp:15-17): peer loss, malformed frames */

#define PBBGPU_LB1 1
#define PBBGPU_LB2 2

typedef struct pbbgpu_pool pbbgpu_pool;

typedef struct {
  int explorers;         /* K; 0 = fill the GPU (occupancy) */
  int group;             /* lanes per explorer (4, 8, 16, 32); 0 = auto */
  int steps_per_round;   /* explore steps per explorer per round; 0 = auto */
  int disable_pruning;   /* PoolConfig.disable_pruning (explorer.hpp:37) */
  int pinned;            /* prune >= initial ub, never improve (explore_step(ub, 0)) */
  double time_limit_s;   /* pbbgpu_solve only; 0 = none */
  double min_steal_log2; /* log2 of the minimal stolen interval length; 0 = log2(8!) */
  int device;            /* CUDA device ordinal */
  int block;             /* threads per CTA (128, 256, 512); 0 = auto */
  double round_us;       /* device time per round; 0 = auto (2000 us, 2500 us for warp explorers, or steps_per_round if set) */
  double steal_trigger;  /* steal phase when active < trigger*K; 0 = 1.0 (reference pool: 0.8) */
  int rounds_per_sync;   /* (explore, steal) rounds per pbbgpu_run_round host sync; 0 = 3, max 8 */
  int max_split;         /* thieves one victim may feed per steal phase (multi-way split); 0 = 4 */
  int split_mode;        /* 0 = factoradic interval split (the reference's steal_right_half,
                            explorer.cpp:265-280, generalised to r-way); 1 = live-sibling split
                            (thieves take unexplored, unpruned subtrees of the shallowest level
                            holding any; best on irregular pinned trees); 2 = live-sibling where
                            the victim has decomposed siblings left, factoradic otherwise */
  int steal_policy;      /* 0 = B200 policy (every idle explorer is a thief each round, longest
                            remaining intervals split r ways); 1 = the reference's steal_phase
                            exactly (explorer.cpp:251-340: trigger active*5 < 4K, eligible
                            len > avg and > min_steal_len, 4-ary hypercube matching when K = 4^c,
                            else largest eligible; midpoint of the raw position; rounds of
                            steps_per_round steps (default 1024 = batch_steps) whose replays are
                            free): raw PoolStats then equal the reference's on fixed trees. n <= 30 */
  int record_census;     /* PoolConfig.record_census (explorer.hpp:39): leaf positions, n <= 20 */
  int census_cap;        /* census capacity (leaf positions held between take_census calls); 0 = 2^20 */
  const char* timeline_path; /* PoolConfig.timeline_path (explorer.hpp:40): activity CSV, NULL = none */
} pbbgpu_config_t;

typedef struct {
  uint64_t decomposed;          /* raw, PoolStats.decomposed semantics */
  uint64_t unique;              /* decomposed - replay duplicates (partition invariant) */
  uint64_t replay_dups;
  uint64_t leaves;
  uint64_t improvements;
  uint64_t local_steals;
  uint64_t steal_phases;
  uint64_t intervals_initialized;
  uint64_t rounds;
  uint64_t steps;
  double wall_s;                /* pbbgpu_solve only */
  double kernel_ms;             /* device time of explore kernels (CUDA events) */
  int completed;                /* pbbgpu_solve only */
  int K;
  int group;
  int steps_per_round;
  double device_ms;             /* pbbgpu_solve only: CUDA-event time from the first round to the last */
  uint64_t kernel_launches;     /* kernels launched by the pool so far (explore + steal + init) */
  uint64_t h2d_bytes;           /* host->device bytes copied by the pool so far */
  uint64_t d2h_bytes;           /* device->host bytes copied by the pool so far */
  int block;                    /* threads per CTA of the explore kernel */
  double batch_kernel_ms;       /* device time of decompose_batch kernels (CUDA events) */
  double steal_kernel_ms;       /* device time of the between-round lens + steal kernels (CUDA events) */
} pbbgpu_stats_t;

const char* pbbgpu_last_error(void);
int pbbgpu_device_count(void);

/* instance helpers (host) */
int pbbgpu_taillard(int n, int m, int32_t seed, int32_t* p_out);
int pbbgpu_taillard_named(const char* name, int* n, int* m, int32_t* p_out /* n*m */);
int64_t pbbgpu_makespan(int n, int m, const int32_t* p, const int32_t* perm);
int64_t pbbgpu_neh(int n, int m, const int32_t* p, int32_t* perm_out);

/* pool */
int pbbgpu_create(int n, int m, const int32_t* p_jobmajor, int bound_kind,
                  const pbbgpu_config_t* cfg, pbbgpu_pool** out);
void pbbgpu_destroy(pbbgpu_pool* pool);
/* Reuse a pool for another instance of the same shape (n, m, bound): the instance tables are
 * rebuilt and re-uploaded in place, counters / incumbent / explorers reset as after create
 * (no device allocation; a serving loop keeps one pool per shape). Replaces constructing a
 * new ExplorerPool per instance (include/pbb/explorer.hpp ExplorerPool(const Instance&, ...)). */
int pbbgpu_load_instance(pbbgpu_pool* pool, const int32_t* p_jobmajor);
int pbbgpu_K(const pbbgpu_pool* pool);
int pbbgpu_set_initial_bound(pbbgpu_pool* pool, int64_t ub, const int32_t* sched, int len);
int pbbgpu_assign(pbbgpu_pool* pool, const uint16_t* a_digits, const uint16_t* b_digits,
                  const uint8_t* b_is_nfact, int count);
int pbbgpu_assign_split(pbbgpu_pool* pool, int pieces);
/* pieces [first, first+count) of [0,n!) cut into `total` equal ranges (multi-GPU partition) */
int pbbgpu_assign_split_range(pbbgpu_pool* pool, int first, int count, int total);
/* pieces first, first+stride, ... (count of them) of [0,n!) cut into `total` ranges: the
 * interleaved multi-GPU partition (rank r of W: first = r, stride = W) */
int pbbgpu_assign_split_strided(pbbgpu_pool* pool, int first, int stride, int count, int total);
/* Breadth-first seeding: expand the top of the tree with the batch bounding kernel (prune at
 * `bound`, the pool's pinned / disable_pruning flags respected) until the live frontier holds
 * >= total nodes, cut [0,n!) at frontier nodes into <= total intervals (each starting at a
 * live subtree) and seat intervals first, first+stride, ... (rank r of W: first = r,
 * stride = W). total <= 0: stride*K. Replaces the equal-range split of pool_run's
 * assign_fresh (explorer.cpp:473-507); counts are unchanged (any partition is exact). */
int pbbgpu_seed(pbbgpu_pool* pool, int64_t bound, int first, int stride, int total);
/* hand the right halves [mid, end) of the `max_count` longest remaining intervals to another
 * pool (inter-GPU stealing); the explorers keep [pos, mid) */
int pbbgpu_export(pbbgpu_pool* pool, int max_count, uint16_t* a_out, uint16_t* b_out,
                  uint8_t* b_is_nfact_out, int* count);
int pbbgpu_run_round(pbbgpu_pool* pool, int* active_out);
/* apply_work_update (explorer.hpp:78-81, src/explorer.cpp:162-199): the new interval set
 * (normalized here) intersected with every explorer's remaining [position, end): an explorer
 * whose intersection is one interval starting at its position keeps its search state (its
 * end shrinks to the interval's end); any other explorer goes idle; the update minus what was
 * kept is seated on idle explorers. More intervals than K: PBBGPU_ERR_ARG; more fragments
 * than idle explorers: PBBGPU_ERR_CAPACITY (std::runtime_error in the reference). */
int pbbgpu_apply_work_update(pbbgpu_pool* pool, const uint16_t* a_digits, const uint16_t* b_digits,
                             const uint8_t* b_is_nfact, int count);
/* improved_since_mark (explorer.hpp:94, explorer.cpp:379-386): 1 when the best schedule improved
 * on the mark (the mark moves to it), else 0. */
int pbbgpu_improved_since_mark(pbbgpu_pool* pool, int* improved);
/* steals_since_mark / reset_steal_mark (explorer.hpp:95-96) */
int pbbgpu_steals_since_mark(pbbgpu_pool* pool, uint64_t* steals);
int pbbgpu_reset_steal_mark(pbbgpu_pool* pool);
/* take_census (explorer.hpp:102, explorer.cpp:438-445): leaf positions (decimal, position_u64)
 * recorded since the last call (record_census), then cleared. PBBGPU_ERR_CAPACITY when more
 * than census_cap leaves were recorded (or more than cap requested). */
int pbbgpu_take_census(pbbgpu_pool* pool, uint64_t* out, int64_t cap, int64_t* count);
/* flush_timeline (explorer.hpp:103, explorer.cpp:466-471): forced timeline sample + flush */
int pbbgpu_flush_timeline(pbbgpu_pool* pool);
int pbbgpu_active_count(pbbgpu_pool* pool, int* active_out);
int pbbgpu_snapshot(pbbgpu_pool* pool, uint16_t* pos_digits, uint16_t* end_digits,
                    uint8_t* end_is_nfact, int cap, int* count);
/* snapshot + exact restart accounting: *resume_recount = nodes this pool already counted that
 * a pool resumed on the snapshot intervals counts again (path nodes of the explorers between
 * lnz(pos) and their level; partial replays). A checkpoint stores unique - resume_recount, so
 * checkpointed + resumed counts add up to one run's count exactly (fixed tree). */
int pbbgpu_snapshot_ex(pbbgpu_pool* pool, uint16_t* pos_digits, uint16_t* end_digits,
                       uint8_t* end_is_nfact, int cap, int* count, uint64_t* resume_recount);
int pbbgpu_best(pbbgpu_pool* pool, int64_t* value, int32_t* perm_or_null, int* has_perm);
/* the pool's best schedule and ITS makespan (best_sched_value_, src/explorer.cpp:352-377);
 * *cmax = INT64_MAX and *has_perm = 0 when the pool holds no schedule. May exceed the
 * pool's bound (an offered bound has no schedule behind it). */
int pbbgpu_best_schedule(pbbgpu_pool* pool, int64_t* cmax, int32_t* perm_or_null, int* has_perm);
int pbbgpu_offer_bound(pbbgpu_pool* pool, int64_t value);
int pbbgpu_stats(pbbgpu_pool* pool, pbbgpu_stats_t* out);
int pbbgpu_histogram(pbbgpu_pool* pool, uint64_t* hist_out, int len);
/* n > 64 (up to 512, e.g. ta111): created with explorers == 0 the pool is bounding-only
 * (decompose_batch; exploration entry points return PBBGPU_ERR_STATE); with explorers > 0 it
 * explores with int16 IVMs in HBM (assign / run_round / solve / stats / best / offer /
 * snapshot_ex / apply_work_update / promote / explorer_lengths / timeline), while census and
 * the peer-memory group stay n <= 64 (PBBGPU_ERR_STATE). */
int pbbgpu_decompose_batch(pbbgpu_pool* pool, const int32_t* perms, const int32_t* d1,
                           const int32_t* d2, int count, int64_t incumbent, int64_t* child_lb,
                           uint8_t* direction, uint8_t* pruned, int64_t* lb_fwd_or_null,
                           int64_t* lb_bwd_or_null);

/* raw explorer blocks (debugging): K * gstride bytes; offsets = cells, V, dir, end, tgt, ft, R */
int pbbgpu_debug_state(pbbgpu_pool* pool, uint8_t* out, int64_t cap, int* gstride, int* offsets);

/* heuristic cooperation (the worker's heuristic agents) */
int64_t pbbgpu_insertion_ls(int n, int m, const int32_t* p, const int32_t* seed_perm, uint64_t max_iter,
                            double max_seconds, uint64_t rng_seed, int32_t* perm_out);
int pbbgpu_offer_schedule(pbbgpu_pool* pool, const int32_t* perm, int64_t cmax, int* taken);
int pbbgpu_promote(pbbgpu_pool* pool, int capacity, int32_t* perms_out, int64_t* cmax_out, int* count);

/* activity timeline (explorer.cpp:448-464): per explorer log2 remaining leaves, -2 busy, -3 idle */
int pbbgpu_explorer_lengths(pbbgpu_pool* pool, float* out, int cap);

/* INT32 ALU microbenchmark (add + max streams, the bounding kernels' instruction mix):
 * measured integer-op throughput of the device, the roofline denominator of the bounding
 * kernels (MEASURED_PEAKS.json has no integer peak). */
int pbbgpu_int32_peak(int device, double* ops_per_s);

/* ---- multi-GPU group: one process per GPU, peer memory over NVLink.
 * Replaces the coordinator / worker exchange inside one box (src/coordinator.cpp:170-306,
 * src/workunit.cpp:59-74): each rank's pool owns a peer window (CUDA IPC); every round the
 * device itself shares the incumbent (system-scope atomicMin), publishes its activity, requests
 * work when below K/2 active explorers, and serves a less busy peer's request by splitting its
 * longest intervals straight into that peer's inbox. The host only detects termination.
 *   create -> exchange handles (any side channel, e.g. torch.distributed) -> open
 *   per solve: reset -> barrier -> solve -> barrier ; close after a final barrier */
typedef struct {
  uint64_t syncs;       /* host synchronizations (run_round calls) */
  uint64_t exchanges;   /* device exchange rounds */
  uint64_t imported;    /* intervals seated from peers */
  uint64_t exported;    /* intervals deposited into peers */
  double wall_s;
  double device_ms;     /* CUDA-event time of the solve loop */
  int completed;        /* 0 when the time limit stopped it */
  double exchange_us_per_round; /* device time of the exchange kernels (incumbent MIN, import,
                                   request / claim, export into the peer) per round */
} pbbgpu_group_stats_t;
int pbbgpu_group_handle_size(void);
int pbbgpu_group_create(pbbgpu_pool* pool, int world, int rank, void* handle_out);
int pbbgpu_group_open(pbbgpu_pool* pool, const void* handles /* world * handle_size bytes, rank order */);
int pbbgpu_group_reset(pbbgpu_pool* pool);
/* this rank's share of [0,n!) (interleaved equal ranges, or breadth-first seeding when
 * seed_div > 0), rounds until the group terminates (or the time limit); counters are local */
int pbbgpu_group_solve(pbbgpu_pool* pool, int64_t initial_ub, int seed_div, double time_limit_s,
                       pbbgpu_group_stats_t* out);
int pbbgpu_group_close(pbbgpu_pool* pool);

/* the pool's instance as given to pbbgpu_create: n, m and the job-major n*m matrix */
int pbbgpu_pool_shape(const pbbgpu_pool* pool, int* n, int* m);
int pbbgpu_pool_times(const pbbgpu_pool* pool, int32_t* p_out);

/* ---- the reference's wire protocol and a GPU worker speaking it
 * Frames of src/protocol.cpp:104-177 over blocking TCP (src/transport.cpp:108-341), so a pool
 * joins the reference's own Coordinator (src/coordinator.cpp) as a worker process. */
typedef struct {
  uint32_t worker_id;          /* WorkerConfig.worker_id (worker.hpp:15) */
  double checkpoint_period_s;  /* WORK checkpoint timer; 0 = 30 s */
  int64_t initial_ub;          /* offered after the seed; <= 0 = none */
  uint64_t rng_seed;           /* insertion_local_search seed; 0 = 1 */
  int ils_iterations;          /* seed descent budget; 0 = 2000 (worker.cpp:146-149) */
  int send_initial_best;       /* WorkerConfig.send_initial_best; set -1 for false (0 = default true) */
} pbbgpu_worker_config_t;
typedef struct {
  int64_t local_best;          /* makespan of the pool's best schedule (INT64_MAX = none) */
  int has_schedule;
  uint64_t checkpoints_sent, bests_sent, updates_applied, messages;
} pbbgpu_worker_result_t;
/* worker_run's pool role (src/worker.cpp:138-296) on `pool`, connected to a coordinator at
 * host:port; returns after END. PBBGPU_ERR_TRANSPORT on peer loss / protocol violations. */
int pbbgpu_worker_run(pbbgpu_pool* pool, const char* host, int port, const pbbgpu_worker_config_t* cfg,
                      pbbgpu_worker_result_t* out);
/* decode one frame (sender_is_worker selects the WORK layout) and encode it again, intervals
 * passed through factoradic digits when n > 0: byte-identical to the input for every frame the
 * reference's encode() produces (the codec's parity hook; no GPU needed) */
int pbbgpu_wire_reencode(const uint8_t* frame, int64_t len, int sender_is_worker, int n, uint8_t* out,
                         int64_t cap, int64_t* out_len);

/* pool_run: assign [0,n!) (or the given intervals), run rounds to exhaustion or time limit */
int pbbgpu_solve(pbbgpu_pool* pool, int64_t initial_ub, const uint16_t* a_digits,
                 const uint16_t* b_digits, const uint8_t* b_is_nfact, int count,
                 int64_t* best_value, int32_t* best_perm, int* has_perm, pbbgpu_stats_t* stats);

#ifdef __cplusplus
}
#endif

#endif
