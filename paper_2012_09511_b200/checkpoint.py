"""Checkpoint / restart of GPU pools in the reference's coordinator checkpoint format
(src/coordinator.cpp:22-102, instance fingerprint
src/instance.cpp:185-205).

    pbb-checkpoint 1
    instance <n> <m> <fnv1a-64 hex>
    best <value|-> <len> <schedule...>
    nodes <total>
    units <count>
    unit <kmax> <count>
    <a> <b>            (decimal interval endpoints, [a, b) over [0, n!))
    end

Files are written to <path>.tmp and renamed (atomic replace), and refuse to load against a
different instance. A pool checkpoint is one unit holding the pool's snapshot intervals.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

from .instance import Instance
from .pool import NO_INCUMBENT, GpuPool, PoolConfig, normalize

Interval = Tuple[int, int]


def instance_fingerprint(inst: Instance) -> int:
    """FNV-1a over (n, m, p) as 8 little-endian bytes each (src/instance.cpp:185-205)."""
    h = 1469598103934665603
    mask = (1 << 64) - 1

    def mix(v: int) -> None:
        nonlocal h
        for i in range(8):
            h ^= (v >> (8 * i)) & 0xFF
            h = (h * 1099511628211) & mask

    mix(inst.n)
    mix(inst.m)
    for v in inst.p.reshape(-1):
        mix(int(v) & 0xFFFFFFFF)
    return h


@dataclass
class WorkUnitData:
    kmax: int
    intervals: List[Interval] = field(default_factory=list)


@dataclass
class CheckpointData:
    units: List[WorkUnitData] = field(default_factory=list)
    best_value: int = NO_INCUMBENT
    best_schedule: List[int] = field(default_factory=list)
    total_nodes: int = 0


def checkpoint_save(path: str, inst: Instance, data: CheckpointData) -> None:
    lines = ["pbb-checkpoint 1", f"instance {inst.n} {inst.m} {instance_fingerprint(inst):016x}"]
    if data.best_value == NO_INCUMBENT:
        lines.append("best - 0")
    else:
        lines.append(" ".join(["best", str(data.best_value), str(len(data.best_schedule))] +
                              [str(j) for j in data.best_schedule]))
    lines.append(f"nodes {data.total_nodes}")
    lines.append(f"units {len(data.units)}")
    for u in data.units:
        lines.append(f"unit {u.kmax} {len(u.intervals)}")
        lines.extend(f"{a} {b}" for a, b in u.intervals)
    lines.append("end")
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(lines) + "\n")
        f.flush()
        os.fsync(f.fileno())
    os.replace(tmp, path)


def checkpoint_load(path: str, inst: Instance) -> CheckpointData:
    with open(path) as f:
        tok = f.read().split()
    it = iter(tok)

    def take(expect: Optional[str] = None) -> str:
        try:
            t = next(it)
        except StopIteration:
            raise ValueError("checkpoint truncated") from None
        if expect is not None and t != expect:
            raise ValueError(f"checkpoint: expected {expect!r}, got {t!r}")
        return t

    take("pbb-checkpoint")
    if take() != "1":
        raise ValueError("not a recognized checkpoint file")
    take("instance")
    n, m, fp = int(take()), int(take()), take()
    if n != inst.n or m != inst.m or fp != f"{instance_fingerprint(inst):016x}":
        raise ValueError("checkpoint belongs to a different instance")
    take("best")
    bt = take()
    d = CheckpointData()
    ln = int(take())
    if bt != "-":
        d.best_value = int(bt)
    d.best_schedule = [int(take()) for _ in range(ln)]
    take("nodes")
    d.total_nodes = int(take())
    take("units")
    for _ in range(int(take())):
        take("unit")
        kmax, cnt = int(take()), int(take())
        ivs = [(int(take()), int(take())) for _ in range(cnt)]
        d.units.append(WorkUnitData(kmax, normalize(ivs)))
    take("end")
    return d


def save_pool(pool: GpuPool, path: str, total_nodes: Optional[int] = None, base_nodes: int = 0) -> CheckpointData:
    """Snapshot a pool between rounds (snapshot_intervals, explorer.cpp:342-350) into a file.

    `nodes` = base_nodes (what earlier runs of this proof had already counted, e.g. the
    `total_nodes` a resumed pool carries) + this pool's unique count - the resume recount
    (nodes the resumed pool will decompose again), so node totals stay exact across any
    number of checkpoint/restart cycles. The schedule is written only when its own makespan
    is the recorded bound (an offered bound has no schedule behind it)."""
    st = pool.stats()
    best = pool.best_schedule()
    ivs, recount = pool.snapshot()
    bv = pool.best_value()
    base = getattr(pool, "resumed_nodes", 0) + base_nodes
    d = CheckpointData([WorkUnitData(pool.K(), ivs)], bv,
                       best.perm if best.perm and best.cmax == bv else [],
                       base + st.unique - recount if total_nodes is None else total_nodes)
    checkpoint_save(path, pool.inst, d)
    return d


def resume_pool(path: str, inst: Instance, cfg: Optional[PoolConfig] = None, bound="lb1") -> GpuPool:
    """A fresh pool seated on a checkpoint's remaining intervals (Coordinator::restore analogue,
    src/coordinator.cpp:129-140). The checkpoint's node total is kept on the pool
    (`resumed_nodes`) and added by the next save_pool, like the coordinator's running total."""
    d = checkpoint_load(path, inst)
    pool = GpuPool(inst, cfg, bound)
    pool.resumed_nodes = d.total_nodes
    pool.set_initial_bound(d.best_value, d.best_schedule)
    ivs = normalize([iv for u in d.units for iv in u.intervals])
    if ivs:
        pool.assign_fresh(ivs)
    return pool
