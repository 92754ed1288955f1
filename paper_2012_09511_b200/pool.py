"""GPU explorer pool — host mirror of the reference's ExplorerPool / pool_run / decompose.

Reference interfaces mirrored (paths under /root/reference/proj):
  PoolConfig / PoolStats / PoolResult   include/pbb/explorer.hpp:34-61
  ExplorerPool                           include/pbb/explorer.hpp:66-103
  pool_run                               include/pbb/explorer.hpp:145-146, src/explorer.cpp:473-507
  Subproblem / Decomposition / decompose include/pbb/bound.hpp:19-79
Intervals are (a, b) pairs of Python integers over [0, n!) (BigCount); they cross the
C-ABI as factoradic digit vectors.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from math import factorial
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .factoradic import from_decimal, to_decimal
from .instance import Instance, Schedule

NO_INCUMBENT = (1 << 63) - 1
FORWARD, BACKWARD = 0, 1
Interval = Tuple[int, int]

_u16p = ctypes.POINTER(ctypes.c_uint16)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)


@dataclass
class PoolConfig:
    explorers: int = 0          # K; 0 = fill the GPU
    group: int = 0              # lanes per explorer; 0 = auto
    batch_steps: int = 0        # explore steps per explorer per round; 0 = auto
    disable_pruning: bool = False
    pinned: bool = False        # prune >= ub, never improve (explore_step(ub, 0))
    time_limit_s: float = 0.0
    min_steal_len: int = 0      # 0 = 8!
    device: int = 0
    block: int = 0              # threads per CTA; 0 = auto
    round_us: float = 0.0       # device time per round; 0 = auto
    steal_trigger: float = 0.0  # steal when active < trigger*K; 0 = 1.0 (reference: 0.8)
    rounds_per_sync: int = 0    # device rounds per run_round() call; 0 = 3
    max_split: int = 0          # thieves per victim per steal phase (multi-way split); 0 = 4
    split_mode: int = 0         # 0 = factoradic (reference), 1 = live siblings, 2 = live else factoradic
    steal_policy: int = 0       # 0 = B200 policy; 1 = the reference's steal_phase exactly (explorer.cpp:251-340)
    record_census: bool = False  # PoolConfig.record_census: leaf positions (n <= 20), take_census()
    census_cap: int = 0         # census entries held between take_census calls; 0 = 2^20
    timeline_path: str = ""     # PoolConfig.timeline_path: activity CSV written by the pool

    def to_c(self) -> _lib.Config:
        c = _lib.Config()
        c.explorers = self.explorers
        c.group = self.group
        c.steps_per_round = self.batch_steps
        c.disable_pruning = int(self.disable_pruning)
        c.pinned = int(self.pinned)
        c.time_limit_s = self.time_limit_s
        c.min_steal_log2 = float(np.log2(self.min_steal_len)) if self.min_steal_len > 1 else 0.0
        c.device = self.device
        c.block = self.block
        c.round_us = self.round_us
        c.steal_trigger = self.steal_trigger
        c.rounds_per_sync = self.rounds_per_sync
        c.max_split = self.max_split
        c.split_mode = self.split_mode
        c.steal_policy = self.steal_policy
        c.record_census = int(self.record_census)
        c.census_cap = self.census_cap
        c.timeline_path = self.timeline_path.encode() if self.timeline_path else None
        return c


@dataclass
class PoolStats:
    decomposed: int = 0
    unique: int = 0
    replay_dups: int = 0
    leaves: int = 0
    improvements: int = 0
    local_steals: int = 0
    steal_phases: int = 0
    intervals_initialized: int = 0
    rounds: int = 0
    steps: int = 0
    wall_s: float = 0.0
    kernel_ms: float = 0.0
    completed: bool = True
    K: int = 0
    group: int = 0
    steps_per_round: int = 0
    device_ms: float = 0.0
    kernel_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    block: int = 0
    batch_kernel_ms: float = 0.0
    steal_kernel_ms: float = 0.0


@dataclass
class PoolResult:
    best: Schedule
    best_value: int
    stats: PoolStats
    hist: Dict[int, int] = field(default_factory=dict)


@dataclass
class Subproblem:
    perm: List[int]
    d1: int = 0
    d2: int = 0

    def free_count(self) -> int:
        return len(self.perm) - self.d1 - self.d2


@dataclass
class Decomposition:
    direction: int
    child_lb: List[int]
    pruned: List[int]


def _bound_kind(bound) -> int:
    if bound in (1, "lb1", "LB1"):
        return _lib.LB1
    if bound in (2, "lb2", "LB2"):
        return _lib.LB2
    raise ValueError(f"unknown bound {bound!r}")


def _digits(intervals: Sequence[Interval], n: int):
    nf = factorial(n)
    a = np.zeros((len(intervals), n), dtype=np.uint16)
    b = np.zeros((len(intervals), n), dtype=np.uint16)
    inf = np.zeros(len(intervals), dtype=np.uint8)
    for i, (lo, hi) in enumerate(intervals):
        if lo < 0 or hi > nf or lo > hi:
            raise ValueError("interval outside [0, n!)")
        a[i] = from_decimal(min(lo, nf - 1), n) if lo < nf else from_decimal(nf - 1, n)
        if hi >= nf:
            inf[i] = 1
        else:
            b[i] = from_decimal(hi, n)
    return a, b, inf


def normalize(intervals: Sequence[Interval]) -> List[Interval]:
    """src/workunit.cpp:8-27: drop empties, sort, merge overlaps (adjacent kept apart)."""
    for a, b in intervals:
        if a > b:
            raise ValueError("interval with a > b")
    ivs = sorted((a, b) for a, b in intervals if a < b)
    out: List[Interval] = []
    for a, b in ivs:
        if out and a < out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


class GpuPool:
    """ExplorerPool on one B200: K IVM explorers resident in shared memory."""

    def __init__(self, inst: Instance, cfg: Optional[PoolConfig] = None, bound="lb1"):
        self.inst = inst
        self.cfg = cfg or PoolConfig()
        self.bound = _bound_kind(bound)
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        c = self.cfg.to_c()
        _lib.check(self._lib.pbbgpu_create(inst.n, inst.m, inst.ptr(), self.bound, ctypes.byref(c), ctypes.byref(h)))
        self._h = h
        self.resumed_nodes = 0  # node total carried over from a checkpoint (checkpoint.resume_pool)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pbbgpu_destroy(self._h)
            self._h = None

    def load_instance(self, inst: Instance) -> None:
        """Reuse this pool for another instance of the same shape (pbbgpu_load_instance): tables
        re-uploaded in place, search state reset as after construction."""
        if (inst.n, inst.m) != (self.inst.n, self.inst.m):
            raise ValueError("load_instance needs an instance of the pool's shape (n, m)")
        _lib.check(self._lib.pbbgpu_load_instance(self._h, inst.ptr()))
        self.inst = inst

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- ExplorerPool surface -------------------------------------------------------------
    def K(self) -> int:
        return self._lib.pbbgpu_K(self._h)

    def set_initial_bound(self, ub: int, sched: Sequence[int] = ()) -> None:
        arr = np.ascontiguousarray(np.asarray(list(sched), dtype=np.int32))
        ptr = arr.ctypes.data_as(_i32p) if arr.size else None
        _lib.check(self._lib.pbbgpu_set_initial_bound(self._h, int(min(ub, NO_INCUMBENT)), ptr, int(arr.size)))

    def assign_fresh(self, intervals: Sequence[Interval]) -> None:
        ivs = normalize(intervals)
        if len(ivs) > self.K():
            raise ValueError("more intervals than explorers")
        a, b, inf = _digits(ivs, self.inst.n)
        _lib.check(self._lib.pbbgpu_assign(self._h, a.ctypes.data_as(_u16p), b.ctypes.data_as(_u16p),
                                           inf.ctypes.data_as(_u8p), len(ivs)))

    def assign_split(self, pieces: int = 0) -> None:
        _lib.check(self._lib.pbbgpu_assign_split(self._h, pieces))

    def assign_split_range(self, first: int, count: int, total: int) -> None:
        _lib.check(self._lib.pbbgpu_assign_split_range(self._h, first, count, total))

    def assign_split_strided(self, first: int, stride: int, count: int, total: int) -> None:
        _lib.check(self._lib.pbbgpu_assign_split_strided(self._h, first, stride, count, total))

    def seed(self, bound: int, first: int = 0, stride: int = 1, total: int = 0) -> None:
        """Breadth-first seeding (pbbgpu_seed): [0, n!) cut at live frontier nodes, intervals
        first, first + stride, ... seated."""
        _lib.check(self._lib.pbbgpu_seed(self._h, int(min(bound, NO_INCUMBENT)), first, stride, total))

    def export_work(self, max_count: int):
        """Right halves of the longest remaining intervals, as digit arrays (a, b, b_is_nfact)."""
        n = self.inst.n
        a = np.zeros((max_count, n), dtype=np.uint16)
        b = np.zeros((max_count, n), dtype=np.uint16)
        nf = np.zeros(max_count, dtype=np.uint8)
        cnt = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_export(self._h, max_count, a.ctypes.data_as(_u16p), b.ctypes.data_as(_u16p),
                                           nf.ctypes.data_as(_u8p), ctypes.byref(cnt)))
        c = cnt.value
        return a[:c].copy(), b[:c].copy(), nf[:c].copy()

    def import_work(self, a, b, nf) -> None:
        """Seat digit intervals (e.g. from another GPU's export_work) on idle explorers."""
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        nf = np.ascontiguousarray(nf, dtype=np.uint8)
        if len(nf) == 0:
            return
        _lib.check(self._lib.pbbgpu_assign(self._h, a.ctypes.data_as(_u16p), b.ctypes.data_as(_u16p),
                                           nf.ctypes.data_as(_u8p), len(nf)))

    def apply_work_update(self, intervals: Sequence[Interval]) -> None:
        """apply_work_update (explorer.cpp:162-199): adopt a coordinator's interval set; explorers
        whose remaining work starts the same keep their state (end shrunk), the rest go idle,
        the new parts are seated on idle explorers."""
        if len(intervals) > self.K():
            raise ValueError("work update holds more intervals than explorers")
        for lo, hi in intervals:
            if lo > hi:
                raise ValueError("interval with a > b")
        ivs = [(a, b) for a, b in intervals if a < b]
        a, b, inf = _digits(ivs, self.inst.n) if ivs else (np.zeros((0, self.inst.n), np.uint16),) * 2 + (
            np.zeros(0, np.uint8),)
        _lib.check(self._lib.pbbgpu_apply_work_update(self._h, a.ctypes.data_as(_u16p), b.ctypes.data_as(_u16p),
                                                      inf.ctypes.data_as(_u8p), len(ivs)))

    def improved_since_mark(self) -> bool:
        """improved_since_mark (explorer.hpp:94): the best schedule improved; resets the mark."""
        v = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_improved_since_mark(self._h, ctypes.byref(v)))
        return bool(v.value)

    def steals_since_mark(self) -> int:
        v = ctypes.c_uint64()
        _lib.check(self._lib.pbbgpu_steals_since_mark(self._h, ctypes.byref(v)))
        return int(v.value)

    def reset_steal_mark(self) -> None:
        _lib.check(self._lib.pbbgpu_reset_steal_mark(self._h))

    def take_census(self) -> List[int]:
        """take_census (explorer.hpp:102): leaf positions recorded since the last call."""
        cap = self.cfg.census_cap or (1 << 20)
        buf = np.zeros(cap, dtype=np.uint64)
        cnt = ctypes.c_int64()
        _lib.check(self._lib.pbbgpu_take_census(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap,
                                                ctypes.byref(cnt)))
        return [int(x) for x in buf[:cnt.value]]

    def flush_timeline(self) -> None:
        """flush_timeline (explorer.hpp:103): forced sample + flush of the pool's timeline CSV."""
        _lib.check(self._lib.pbbgpu_flush_timeline(self._h))

    # -- multi-GPU group over peer memory (pbbgpu_group_*; multi.solve_distributed drives it) -------
    def group_create(self, world: int, rank: int) -> bytes:
        """Create this rank's peer window; returns its CUDA IPC handle (to all_gather)."""
        size = self._lib.pbbgpu_group_handle_size()
        buf = ctypes.create_string_buffer(size)
        _lib.check(self._lib.pbbgpu_group_create(self._h, world, rank, buf))
        return buf.raw

    def group_open(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        _lib.check(self._lib.pbbgpu_group_open(self._h, ctypes.c_char_p(blob)))

    def group_reset(self) -> None:
        _lib.check(self._lib.pbbgpu_group_reset(self._h))

    def group_solve(self, ub: int, seed_div: int = 0, time_limit_s: float = 0.0) -> dict:
        gs = _lib.GroupStats()
        _lib.check(self._lib.pbbgpu_group_solve(self._h, int(min(ub, NO_INCUMBENT)), seed_div, time_limit_s,
                                                ctypes.byref(gs)))
        return gs.as_dict()

    def group_close(self) -> None:
        _lib.check(self._lib.pbbgpu_group_close(self._h))

    def worker_run(self, host: str, port: int, worker_id: int = 0, initial_ub: int = 0,
                   checkpoint_period_s: float = 30.0, rng_seed: int = 1) -> dict:
        """worker_run's pool role (src/worker.cpp:138-296) against a coordinator speaking the
        reference's wire protocol over TCP (pbbgpu_worker_run); returns after END."""
        c = _lib.WorkerConfig()
        c.worker_id = worker_id
        c.checkpoint_period_s = checkpoint_period_s
        c.initial_ub = initial_ub
        c.rng_seed = rng_seed
        r = _lib.WorkerResult()
        _lib.check(self._lib.pbbgpu_worker_run(self._h, host.encode(), port, ctypes.byref(c), ctypes.byref(r)))
        return r.as_dict()

    def run_round(self) -> int:
        act = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_run_round(self._h, ctypes.byref(act)))
        return act.value

    def active_count(self) -> int:
        act = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_active_count(self._h, ctypes.byref(act)))
        return act.value

    def snapshot_intervals(self) -> List[Interval]:
        """snapshot_intervals (explorer.cpp:342-350): the remaining work [position, end)."""
        return self.snapshot()[0]

    def snapshot(self) -> Tuple[List[Interval], int]:
        """Remaining intervals plus the resume recount (pbbgpu_snapshot_ex): nodes this pool has
        counted that a pool resumed on these intervals will count again. A checkpoint records
        unique - recount, so checkpointed + resumed counts equal one run's count exactly."""
        K, n = self.K(), self.inst.n
        pos = np.zeros((K, n), dtype=np.uint16)
        end = np.zeros((K, n), dtype=np.uint16)
        inf = np.zeros(K, dtype=np.uint8)
        cnt = ctypes.c_int()
        rec = ctypes.c_uint64()
        _lib.check(self._lib.pbbgpu_snapshot_ex(self._h, pos.ctypes.data_as(_u16p), end.ctypes.data_as(_u16p),
                                                inf.ctypes.data_as(_u8p), K, ctypes.byref(cnt), ctypes.byref(rec)))
        nf = factorial(n)
        out = []
        for i in range(cnt.value):
            a = to_decimal([int(x) for x in pos[i]])
            b = nf if inf[i] else to_decimal([int(x) for x in end[i]])
            if a < b:
                out.append((a, b))
        return normalize(out), int(rec.value)

    def best_value(self) -> int:
        v = ctypes.c_int64()
        _lib.check(self._lib.pbbgpu_best(self._h, ctypes.byref(v), None, None))
        return v.value

    def best_schedule(self) -> Schedule:
        """best_schedule (explorer.cpp:356-362): the best schedule seen and ITS makespan
        (cmax = -1 and an empty perm when the pool holds none)."""
        v = ctypes.c_int64()
        has = ctypes.c_int()
        perm = np.zeros(self.inst.n, dtype=np.int32)
        _lib.check(self._lib.pbbgpu_best_schedule(self._h, ctypes.byref(v), perm.ctypes.data_as(_i32p),
                                                  ctypes.byref(has)))
        if not has.value:
            return Schedule([], -1)
        return Schedule([int(x) for x in perm], int(v.value))

    def offer_bound(self, value: int) -> None:
        _lib.check(self._lib.pbbgpu_offer_bound(self._h, int(value)))

    def offer_schedule(self, sched: Schedule) -> bool:
        """offer_schedule (explorer.cpp:379-395): True when it improved the bound or best schedule."""
        arr = np.ascontiguousarray(np.asarray(sched.perm, dtype=np.int32))
        taken = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_offer_schedule(self._h, arr.ctypes.data_as(_i32p), int(sched.cmax), ctypes.byref(taken)))
        return bool(taken.value)

    def promote_solutions(self, capacity: int) -> List[Schedule]:
        """promote_solutions (explorer.cpp:397-424): current nodes completed in incumbent order."""
        n = self.inst.n
        perms = np.zeros((max(capacity, 1), n), dtype=np.int32)
        cm = np.zeros(max(capacity, 1), dtype=np.int64)
        cnt = ctypes.c_int()
        _lib.check(self._lib.pbbgpu_promote(self._h, capacity, perms.ctypes.data_as(_i32p), cm.ctypes.data_as(_i64p),
                                            ctypes.byref(cnt)))
        return [Schedule([int(x) for x in perms[i]], int(cm[i])) for i in range(cnt.value)]

    def stats(self) -> PoolStats:
        s = _lib.Stats()
        _lib.check(self._lib.pbbgpu_stats(self._h, ctypes.byref(s)))
        d = s.as_dict()
        d["completed"] = bool(d["completed"])
        return PoolStats(**d)

    def explorer_lengths(self) -> np.ndarray:
        """log2 remaining leaves per explorer (-2 busy replaying, -3 idle)."""
        out = np.zeros(self.K(), dtype=np.float32)
        _lib.check(self._lib.pbbgpu_explorer_lengths(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.size))
        return out

    def histogram(self) -> Dict[int, int]:
        n = self.inst.n
        h = np.zeros(n + 1, dtype=np.uint64)
        _lib.check(self._lib.pbbgpu_histogram(self._h, h.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n + 1))
        return {f: int(v) for f, v in enumerate(h) if v}

    # -- per-node bounding operator (bound.hpp:78-79) -----------------------------------------
    def decompose_batch(self, perms, d1, d2, incumbent: int):
        perms = np.ascontiguousarray(np.asarray(perms, dtype=np.int32).reshape(-1, self.inst.n))
        d1 = np.ascontiguousarray(np.asarray(d1, dtype=np.int32).reshape(-1))
        d2 = np.ascontiguousarray(np.asarray(d2, dtype=np.int32).reshape(-1))
        cnt = perms.shape[0]
        lb = np.zeros((cnt, self.inst.n), dtype=np.int64)
        lf = np.zeros((cnt, self.inst.n), dtype=np.int64)
        lbw = np.zeros((cnt, self.inst.n), dtype=np.int64)
        dr = np.zeros(cnt, dtype=np.uint8)
        pr = np.zeros((cnt, self.inst.n), dtype=np.uint8)
        _lib.check(self._lib.pbbgpu_decompose_batch(
            self._h, perms.ctypes.data_as(_i32p), d1.ctypes.data_as(_i32p), d2.ctypes.data_as(_i32p), cnt,
            int(min(incumbent, NO_INCUMBENT)), lb.ctypes.data_as(_i64p), dr.ctypes.data_as(_u8p),
            pr.ctypes.data_as(_u8p), lf.ctypes.data_as(_i64p), lbw.ctypes.data_as(_i64p)))
        return lb, dr, pr, lf, lbw

    def decompose(self, sub: Subproblem, incumbent: int) -> Decomposition:
        lb, dr, pr, _, _ = self.decompose_batch([sub.perm], [sub.d1], [sub.d2], incumbent)
        f = sub.free_count()
        return Decomposition(int(dr[0]), [int(x) for x in lb[0, :f]], [int(x) for x in pr[0, :f]])


def pool_run(inst: Instance, initial_ub: int, intervals: Sequence[Interval] = (),
             cfg: Optional[PoolConfig] = None, bound="lb1") -> PoolResult:
    """pool_run (src/explorer.cpp:473-507) on one GPU: [0, n!) by default, cut evenly over K."""
    cfg = cfg or PoolConfig()
    with GpuPool(inst, cfg, bound) as pool:
        return solve_pool(pool, initial_ub, intervals)


def solve_pool(pool: GpuPool, initial_ub: int, intervals: Sequence[Interval] = ()) -> PoolResult:
    """One pbbgpu_solve on an existing pool (fresh, or re-loaded with GpuPool.load_instance)."""
    inst = pool.inst
    lib = pool._lib
    ivs = normalize(list(intervals))
    a = b = inf = None
    if ivs:
        a, b, inf = _digits(ivs, inst.n)
    best = ctypes.c_int64()
    has = ctypes.c_int()
    perm = np.zeros(inst.n, dtype=np.int32)
    st = _lib.Stats()
    _lib.check(lib.pbbgpu_solve(
        pool._h, int(min(initial_ub, NO_INCUMBENT)),
        a.ctypes.data_as(_u16p) if ivs else None, b.ctypes.data_as(_u16p) if ivs else None,
        inf.ctypes.data_as(_u8p) if ivs else None, len(ivs), ctypes.byref(best),
        perm.ctypes.data_as(_i32p), ctypes.byref(has), ctypes.byref(st)))
    d = st.as_dict()
    d["completed"] = bool(d["completed"])
    sched = Schedule([int(x) for x in perm], int(best.value)) if has.value else Schedule([], -1)
    return PoolResult(sched, int(best.value), PoolStats(**d), pool.histogram())


def int32_peak(device: int = 0) -> float:
    """Measured INT32 add/max throughput of the device (ops/s), the bounding roofline."""
    v = ctypes.c_double()
    _lib.check(_lib.load().pbbgpu_int32_peak(device, ctypes.byref(v)))
    return v.value


class Timeline:
    """Activity timeline CSV (src/explorer.cpp:71-85, 448-471): one row per explorer per sample,
    `timestamp_ms,explorer_id,active,interval_length_log2`, samples >= 50 ms apart, forced at
    exhaustion. The GPU's per-explorer lengths come from pbbgpu_explorer_lengths."""

    MIN_GAP_S = 0.05

    def __init__(self, path: str):
        import time
        self._time = time
        self.f = open(path, "w")
        self.f.write("timestamp_ms,explorer_id,active,interval_length_log2\n")
        self.t0 = time.monotonic()
        self.last = -1e9

    def sample(self, pool: "GpuPool", force: bool = False) -> bool:
        now = self._time.monotonic()
        if not force and now - self.last < self.MIN_GAP_S:
            return False
        self.last = now
        ts = int((now - self.t0) * 1000)
        lens = pool.explorer_lengths()
        rows = []
        for i, lg in enumerate(lens):
            active = lg != -3.0
            rows.append(f"{ts},{i},{1 if active else 0},{int(lg) if lg >= 0 else -1}")
        self.f.write("\n".join(rows) + "\n")
        return True

    def close(self):
        self.f.close()


def wire_reencode(frame: bytes, sender_is_worker: bool, n: int = 0) -> bytes:
    """Decode one frame of the reference's wire protocol (src/protocol.cpp) and encode it again,
    interval endpoints passed through factoradic digits when n > 0 (pbbgpu_wire_reencode)."""
    lib = _lib.load()
    cap = 2 * len(frame) + 64
    out = ctypes.create_string_buffer(cap)
    ln = ctypes.c_int64()
    _lib.check(lib.pbbgpu_wire_reencode(frame, len(frame), int(sender_is_worker), n, out, cap, ctypes.byref(ln)))
    return out.raw[:ln.value]
