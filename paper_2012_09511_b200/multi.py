"""Multi-GPU solve: one process per GPU, torch.distributed for the plumbing.

  partition   [0, n!) cut into world*K equal ranges; rank r seats pieces r, r+W, r+2W, ...
              (pbbgpu_assign_split_strided): interleaved so that every rank samples the
              whole, highly irregular tree -- the intra-box analogue of the coordinator's
              initial work units (src/coordinator.cpp)
  per round   every rank runs one pool round (explore + intra-GPU steal kernels), then one
              all_gather of (active explorers, incumbent, exported intervals)
  incumbent   MIN over ranks (the BEST message of src/protocol.cpp), fed back through
              offer_bound
  stealing    a rank whose active explorers drop below `low` receives the right halves of a
              busy rank's longest intervals (pbbgpu_export -> all_gather -> pbbgpu_assign);
              the donor keeps [pos, mid) -- the coordinator's split_unit
              (src/workunit.cpp:59-74) between GPUs
  termination all ranks report 0 active explorers in the same gathered snapshot
Node counts stay exact: replays on the receiving GPU are discounted by the same
unique = raw - min(L, lnz(a)) rule, which is partition invariant.
Two data planes:
  native      (GpuPool on CUDA, the default for world > 1) the pools exchange over NVLink peer
              memory by themselves (pbbgpu_group_*, csrc/pool.cu): every round the device
              shares the incumbent with system-scope atomicMin, requests work below K/2 active
              explorers and serves a less busy peer by writing split intervals straight into its
              inbox; torch.distributed only exchanges the CUDA IPC handles once, brackets each
              solve with barriers and reduces the counters at the end
  host-staged (any object with the GpuPool surface, e.g. the simulated pool of the CPU tests)
              per sync one all_gather of (active, incumbent, stop) and of exported intervals
The orchestration logic of the host-staged plane is tested on CPU with a simulated pool and
the gloo backend (tests/test_multi.py); the native plane on GPUs (tests/test_gpu_multi.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np


@dataclass
class DistResult:
    best_value: int
    best_perm: list
    unique: int
    decomposed: int
    leaves: int
    improvements: int
    local_steals: int
    remote_intervals: int
    rounds: int
    exchanges: int
    hist: Dict[int, int]
    completed: bool
    exchange_us_per_round: float = 0.0  # native plane: device time of the exchange kernels per round


_DELTA = ("unique", "decomposed", "leaves", "improvements", "local_steals")


def _solve_native(pool, ub, group, device, time_limit_s, seed_div, world, rank) -> DistResult:
    import torch.distributed as dist

    st0 = pool.stats()
    h0 = pool.histogram()
    if not getattr(pool, "_group_ready", False):
        handle = pool.group_create(world, rank)
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        pool.group_open(handles)
        pool._group_ready = True
    pool.group_reset()
    dist.barrier(group=group)        # every window reset before any rank pushes into it
    gst = pool.group_solve(ub, seed_div, time_limit_s)
    dist.barrier(group=group)        # nobody reads or writes a peer window after this
    res = _finish(pool, st0, h0, group, device, world, rank, int(gst["imported"]), int(gst["syncs"]),
                  int(gst["exchanges"]), bool(gst["completed"]))
    res.exchange_us_per_round = float(gst["exchange_us_per_round"])
    return res


def solve_distributed(pool, ub: int, group=None, device=None, export_max: Optional[int] = None,
                      low_fraction: float = 0.5, time_limit_s: float = 0.0, seed_div: int = 0,
                      native: Optional[bool] = None) -> DistResult:
    """Run `pool` (a GpuPool, or any object with its surface) to exhaustion cooperatively with
    the other ranks of `group` (torch.distributed). world_size == 1 degenerates to pool_run.

    The initial partition is [0, n!) cut into world*K equal ranges, interleaved over the ranks
    (seed_div = 0), or breadth-first seeding (pbbgpu_seed) into world*K/seed_div intervals
    that each start at a live subtree (better on irregular trees such as pinned ta041)."""
    import time

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 1 and native is not False and hasattr(pool, "group_solve"):
        return _solve_native(pool, ub, group, device, time_limit_s, seed_div, world, rank)
    n = pool.inst.n
    K = pool.K()
    st0 = pool.stats()
    h0 = pool.histogram()
    pool.set_initial_bound(ub)
    # interleaved partition: rank r seats pieces r, r + W, r + 2W, ... of [0,n!) cut into W*K
    # ranges, so every rank samples the whole (highly irregular) tree from the start
    if seed_div > 0 and hasattr(pool, "seed"):  # breadth-first seeding, interleaved over the ranks
        pool.seed(ub, rank, world, max(world, world * K // seed_div))
    elif world > 1 and hasattr(pool, "assign_split_strided"):
        pool.assign_split_strided(rank, world, K, world * K)
    else:
        pool.assign_split_range(rank * K, K, world * K)
    X = export_max if export_max else max(1, K // 2)
    low = int(K * low_fraction)
    remote = 0
    rounds = 0
    exchanges = 0
    completed = True
    t0 = time.time()
    width = 2 * n + 1
    # phase-1 buffers, allocated once: pinned host row -> device -> all_gather -> pinned host
    dev = torch.device(device) if device is not None else torch.device("cpu")
    pin = dev.type == "cuda"
    info_h = torch.zeros(3, dtype=torch.int64, pin_memory=pin)
    info_d = info_h.to(dev)
    gath_d = torch.zeros(world * 3, dtype=torch.int64, device=dev)
    gath_h = torch.zeros(world * 3, dtype=torch.int64, pin_memory=pin)
    while True:
        active = pool.run_round()
        rounds += 1
        if world == 1:
            if active == 0:
                break
            if time_limit_s and time.time() - t0 >= time_limit_s:
                completed = False
                break
            continue
        exchanges += 1
        best = pool.best_value()
        stop = int(bool(time_limit_s) and time.time() - t0 >= time_limit_s)
        # phase 1: who is idle, who is busy, incumbent, time limit
        info_h[0], info_h[1], info_h[2] = active, min(best, (1 << 62)), stop
        info_d.copy_(info_h, non_blocking=pin)
        dist.all_gather_into_tensor(gath_d, info_d, group=group)
        gath_h.copy_(gath_d, non_blocking=pin)
        if pin:
            torch.cuda.current_stream(dev).synchronize()
        g = gath_h.numpy().reshape(world, 3)
        actives, bests = g[:, 0], g[:, 1]
        gbest = int(bests.min())
        if gbest < best:
            pool.offer_bound(gbest)
        if int(actives.sum()) == 0:
            break
        if int(g[:, 2].max()):
            completed = False
            break
        # receivers run low and hold less than half of the busiest rank; donors hold at least
        # half of it (multi-way splits let even a handful of explorers feed a receiver)
        amax = int(actives.max())
        receivers = [r for r in range(world) if actives[r] < low and 2 * actives[r] < amax]
        donors = [int(r) for r in np.argsort(-actives, kind="stable") if actives[r] > 0 and 2 * actives[r] >= amax]
        if not receivers or not donors:
            continue
        # phase 2: donors export, everybody gathers, receivers seat their share. The phase-1
        # counts are exact (no round runs in between): a donor exports at most its receivers'
        # idle explorers, and each receiver takes a contiguous share no larger than its idle.
        pairs = {}
        for i, r in enumerate(receivers):
            pairs.setdefault(int(donors[i % len(donors)]), []).append(r)
        buf = np.zeros((X, width), dtype=np.int32)
        cnt = 0
        if rank in pairs:
            room = sum(K - int(actives[r]) for r in pairs[rank])
            a, b, nf = pool.export_work(min(X, room))
            cnt = len(nf)
            buf[:cnt, :n] = a
            buf[:cnt, n:2 * n] = b
            buf[:cnt, 2 * n] = nf
        sbuf = torch.from_numpy(np.concatenate([buf.reshape(-1), np.array([cnt], dtype=np.int32)])).to(device)
        allb = [torch.zeros_like(sbuf) for _ in range(world)]
        dist.all_gather(allb, sbuf, group=group)
        for donor, recvs in pairs.items():
            if rank not in recvs:
                continue
            arr = allb[donor].cpu().numpy()
            c = int(arr[-1])
            rows = arr[:-1].reshape(X, width)[:c]
            # shares in proportion to the receivers' idle explorers, in receiver order
            idle = [K - int(actives[r]) for r in recvs]
            tot = max(1, sum(idle))
            shares = [c * i // tot for i in idle]
            for i in range(c - sum(shares)):
                shares[i % len(shares)] += 1
            me = recvs.index(rank)
            off = sum(shares[:me])
            if shares[me] > idle[me]:
                raise RuntimeError("inter-GPU exchange: share exceeds the receiver's idle explorers")
            mine = rows[off:off + shares[me]]
            if len(mine):
                pool.import_work(mine[:, :n].astype(np.uint16), mine[:, n:2 * n].astype(np.uint16),
                                 mine[:, 2 * n].astype(np.uint8))
                remote += len(mine)
    return _finish(pool, st0, h0, group, device, world, rank, remote, rounds, exchanges, completed)


def _finish(pool, st0, h0, group, device, world, rank, remote, rounds, exchanges, completed) -> DistResult:
    """This solve's counters (the pool's are cumulative), summed over the ranks; the best
    schedule broadcast from the rank that holds it."""
    import torch
    import torch.distributed as dist

    n = pool.inst.n
    st1 = pool.stats()
    h1 = pool.histogram()
    # this solve only (the pool's counters are cumulative)
    st = type(st1)(**{k: (getattr(st1, k) - getattr(st0, k)) if k in _DELTA else getattr(st1, k)
                      for k in st1.__dataclass_fields__})
    hist = {f: v - h0.get(f, 0) for f, v in h1.items() if v - h0.get(f, 0)}
    bsched = pool.best_schedule()
    if world > 1:
        vec = torch.tensor([st.unique, st.decomposed, st.leaves, st.improvements, st.local_steals, remote],
                           dtype=torch.int64, device=device)
        dist.all_reduce(vec, group=group)
        hv = torch.zeros(n + 1, dtype=torch.int64, device=device)
        for f, v in hist.items():
            hv[f] = v
        dist.all_reduce(hv, group=group)
        # the schedule owner: the rank holding the best schedule by ITS makespan (every rank's
        # bound equals the global MIN after the exchanges, so bound values cannot tell)
        sv = bsched.cmax if bsched.perm else (1 << 62)
        bv = torch.tensor([pool.best_value(), sv, rank], dtype=torch.int64, device=device)
        allbv = [torch.zeros_like(bv) for _ in range(world)]
        dist.all_gather(allbv, bv, group=group)
        bvals = torch.stack(allbv).cpu().numpy()
        owner = int(bvals[np.argmin(bvals[:, 1]), 2])
        pv = torch.tensor(bsched.perm if bsched.perm else [-1] * n, dtype=torch.int64, device=device)
        src = dist.get_global_rank(group, owner) if group is not None else owner
        dist.broadcast(pv, src=src, group=group)
        perm = [int(x) for x in pv.cpu().numpy()]
        v = vec.cpu().numpy()
        return DistResult(int(bvals[:, 0].min()), perm if perm[0] >= 0 else [], int(v[0]), int(v[1]), int(v[2]),
                          int(v[3]), int(v[4]), int(v[5]), rounds, exchanges,
                          {f: int(x) for f, x in enumerate(hv.cpu().numpy()) if x}, completed)
    return DistResult(pool.best_value(), bsched.perm, st.unique, st.decomposed, st.leaves, st.improvements,
                      st.local_steals, 0, rounds, exchanges, hist, completed)
