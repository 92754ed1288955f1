"""Heuristic cooperation around the GPU pool.

Mirrors the reference worker's heuristic agents (src/worker.cpp:144-152, 204-219):
  initial UB   NEH then insertion local search (src/heuristic.cpp:73-155)
  promotion    at round boundaries the driving thread asks the pool for its current nodes
               completed in incumbent order (promote_solutions, src/explorer.cpp:397-424)
  agents       a host thread improves promoted schedules with insertion local search and
               offers better ones back (offer_schedule, src/explorer.cpp:379-395)
The GPU explores; the host cores (otherwise idle) search for better upper bounds.
"""
from __future__ import annotations

import queue
import threading
import time
from dataclasses import dataclass
from typing import Optional

from .instance import Instance, Schedule, insertion_local_search, neh
from .pool import GpuPool, PoolConfig


@dataclass
class CoopResult:
    best: Schedule
    best_value: int
    initial_ub: int
    unique: int
    leaves: int
    offered: int
    accepted: int
    wall_s: float
    completed: bool


def solve_cooperative(inst: Instance, bound="lb2", cfg: Optional[PoolConfig] = None, ls_iterations: int = 2000,
                      promote_every: int = 4, promote_capacity: int = 4, rng_seed: int = 0,
                      time_limit_s: float = 0.0) -> CoopResult:
    seed = neh(inst)
    start = insertion_local_search(inst, seed, max_iterations=ls_iterations, rng_seed=rng_seed)
    t0 = time.time()
    work: "queue.Queue[Optional[Schedule]]" = queue.Queue(maxsize=64)
    stats = {"offered": 0, "accepted": 0}
    with GpuPool(inst, cfg or PoolConfig(), bound=bound) as pool:
        pool.set_initial_bound(start.cmax, start.perm)
        pool.assign_split()

        def agent():
            k = 0
            while True:
                s = work.get()
                if s is None:
                    return
                k += 1
                better = insertion_local_search(inst, s, max_iterations=ls_iterations, rng_seed=rng_seed + k)
                if better.cmax < pool.best_value():
                    stats["offered"] += 1
                    stats["accepted"] += int(pool.offer_schedule(better))

        th = threading.Thread(target=agent, daemon=True)
        th.start()
        rounds = 0
        completed = True
        while pool.run_round() > 0:
            rounds += 1
            if rounds % promote_every == 0:
                for s in pool.promote_solutions(promote_capacity):
                    try:
                        work.put_nowait(s)
                    except queue.Full:
                        break
            if time_limit_s and time.time() - t0 >= time_limit_s:
                completed = False
                break
        work.put(None)
        th.join()
        st = pool.stats()
        best = pool.best_schedule()
        return CoopResult(best, pool.best_value(), start.cmax, st.unique, st.leaves, stats["offered"],
                          stats["accepted"], time.time() - t0, completed)
