"""GPU parity tests: the sm_100a kernels (through the C-ABI) against the reference's golden
outputs and the C oracle. Bit-exact integer parity everywhere.
"""
import itertools
import json
import math
import os
import subprocess

import numpy as np
import pytest

import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200 import _lib
from oracle import oracle as orc
from tests import golden_io

pytestmark = pytest.mark.gpu


def _hist_str(h):
    return {str(k): int(v) for k, v in h.items() if v}


# ---------------------------------------------------------------- per-node bounding parity

@pytest.mark.parametrize("name", ["ta001", "ta021", "ta041", "ta056"])
def test_decompose_batch_matches_reference_nodes(name):
    nodes, ub = golden_io.ref_nodes(name)
    inst = pbb.taillard_named(name)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=512)) as pool:
        perms = np.array([x[0] for x in nodes])
        lb, dr, pr, _, _ = pool.decompose_batch(perms, [x[1] for x in nodes], [x[2] for x in nodes], ub)
    for i, (perm, d1, d2, direction, lbs, pruned) in enumerate(nodes):
        f = len(lbs)
        assert int(dr[i]) == direction
        assert [int(x) for x in lb[i, :f]] == lbs
        assert [int(x) for x in pr[i, :f]] == pruned


def _random_nodes(n, count, seed):
    rng = np.random.default_rng(seed)
    perms, d1s, d2s = [], [], []
    for _ in range(count):
        perms.append(rng.permutation(n))
        f = int(rng.integers(1, n + 1))
        d1 = int(rng.integers(0, n - f + 1))
        d1s.append(d1)
        d2s.append(n - f - d1)
    return np.array(perms), d1s, d2s


@pytest.mark.parametrize("bound", ["lb1", "lb2"])
@pytest.mark.parametrize("name", ["ta001", "ta011", "ta021", "ta031", "ta041", "ta056"])
@pytest.mark.parametrize("group", [4, 8, 32])
def test_decompose_batch_matches_oracle(bound, name, group):
    inst = pbb.taillard_named(name)
    count = 400 if bound == "lb2" else 1500
    perms, d1s, d2s = _random_nodes(inst.n, count, 17)
    prob = orc.Problem(inst.p, orc.LB1 if bound == "lb1" else orc.LB2)
    inc = int(pbb.neh(inst).cmax)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=256, group=group), bound=bound) as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, inc)
    for i in range(count):
        f = inst.n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        d, clb, cpr = prob.decompose(perms[i], d1s[i], d2s[i], inc)
        assert [int(x) for x in lf[i, :f]] == fw
        assert [int(x) for x in lbw[i, :f]] == bw
        assert int(dr[i]) == d
        assert [int(x) for x in lb[i, :f]] == clb
        assert [int(x) for x in pr[i, :f]] == cpr


def test_decompose_errors():
    inst = pbb.taillard_named("ta001")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=64)) as pool:
        with pytest.raises(ValueError):
            pool.decompose(pbb.Subproblem(list(range(20)), 10, 10), 1278)   # no free jobs
        with pytest.raises(ValueError):
            pool.decompose(pbb.Subproblem(list(range(20)), 1, 1), 0)        # incumbent <= 0
        with pytest.raises(ValueError):
            pool.decompose(pbb.Subproblem([0] * 20, 1, 1), 1278)            # not a permutation


# ---------------------------------------------------------------- fixed trees (UB = optimum)

@pytest.mark.parametrize("key", ["ta001@1278", "ta011@1582", "ta031@2724", "ta041@2991"])
@pytest.mark.parametrize("explorers", [0, 64, 1000])
def test_fixed_tree_lb1_matches_reference(key, explorers):
    ref = golden_io.ref_counts()[key]
    name, ub = key.split("@")
    res = pbb.pool_run(pbb.taillard_named(name), int(ub), cfg=pbb.PoolConfig(explorers=explorers))
    assert res.stats.completed
    assert res.stats.unique == ref["decomposed"]
    assert res.stats.leaves == ref["leaves"]
    assert res.best_value == ref["best_value"]
    assert not res.best.perm              # no improvement below the optimum
    assert _hist_str(res.hist) == ref["hist"]


def test_fixed_tree_ta021_lb1_full_proof():
    """462,443,491 decomposed nodes / 1,440 leaves: the reference's 534.8 s K=1 proof."""
    res = pbb.pool_run(pbb.taillard_named("ta021"), 2297)
    assert res.stats.completed
    assert res.stats.unique == golden_io.TA021_LB1["decomposed"]
    assert res.stats.leaves == golden_io.TA021_LB1["leaves"]
    assert res.hist == golden_io.TA021_LB1["hist"]


@pytest.mark.parametrize("key", ["ta001@1278", "ta011@1582", "ta031@2724", "ta041@2991", "ta021@2297"])
def test_fixed_tree_lb2_matches_oracle(key):
    gold = golden_io.lb2_counts()[key]
    name, ub = key.split("@")
    res = pbb.pool_run(pbb.taillard_named(name), int(ub), bound="lb2")
    assert res.stats.completed
    assert res.stats.unique == gold["unique"]
    assert res.stats.leaves == gold["leaves"]
    assert _hist_str(res.hist) == gold["hist"]


@pytest.mark.timeout(180)
@pytest.mark.parametrize("split_mode", [0, 1, 2])
@pytest.mark.parametrize("steps,explorers,min_steal", [(64, 200, 2), (31, 333, 24), (200, 4096, 40320)])
def test_unique_count_invariant_under_stealing(steps, explorers, min_steal, split_mode):
    """Tiny rounds + many thieves: the unique-count rule must hold under heavy stealing, for
    the factoradic, live-sibling and hybrid split policies."""
    ref = golden_io.ref_counts()["ta011@1582"]
    cfg = pbb.PoolConfig(explorers=explorers, batch_steps=steps, min_steal_len=min_steal, split_mode=split_mode)
    res = pbb.pool_run(pbb.taillard_named("ta011"), 1582, cfg=cfg)
    assert res.stats.unique == ref["decomposed"]
    assert res.stats.leaves == ref["leaves"]
    assert res.stats.local_steals > 0
    assert _hist_str(res.hist) == ref["hist"]


def test_user_intervals_partition_invariance():
    """Any partition of [0, n!) into intervals gives the K=1 unique count."""
    ref = golden_io.ref_counts()["ta041@2991"]
    inst = pbb.taillard_named("ta041")
    nf = math.factorial(inst.n)
    rng = np.random.default_rng(5)
    cuts = sorted({int(x) * (nf >> 62) for x in rng.integers(1, 2 ** 62, 40)} | {nf // 3, nf // 2})
    bounds = [0] + cuts + [nf]
    ivs = list(zip(bounds[:-1], bounds[1:]))
    res = pbb.pool_run(inst, 2991, intervals=ivs, cfg=pbb.PoolConfig(explorers=128))
    assert res.stats.unique == ref["decomposed"]
    assert res.stats.leaves == ref["leaves"]


# ---------------------------------------------------------------- improving search

@pytest.mark.parametrize("name,opt", [("ta001", 1278), ("ta011", 1582), ("ta031", 2724), ("ta041", 2991)])
@pytest.mark.parametrize("bound", ["lb1", "lb2"])
def test_optimum_from_neh(name, opt, bound):
    inst = pbb.taillard_named(name)
    ub = pbb.neh(inst).cmax
    res = pbb.pool_run(inst, ub, bound=bound)
    assert res.best_value == opt
    if ub > opt:
        assert res.best.cmax == opt
        assert pbb.makespan(inst, res.best.perm) == opt
        assert res.stats.improvements >= 1


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("bound", ["lb1", "lb2"])
def test_optimum_matches_brute_force(seed, bound):
    n, m = 8, 5
    inst = pbb.generate_taillard(n, m, 4242 + seed)
    best = min(pbb.makespan(inst, perm) for perm in itertools.permutations(range(n)))
    res = pbb.pool_run(inst, 10 ** 6, bound=bound, cfg=pbb.PoolConfig(explorers=128))
    assert res.best_value == best
    assert pbb.makespan(inst, res.best.perm) == best


def test_census_without_pruning_visits_every_leaf():
    """disable_pruning: exactly n! leaves are evaluated (SPEC.md acceptance 4)."""
    n, m = 8, 5
    inst = pbb.generate_taillard(n, m, 77)
    res = pbb.pool_run(inst, 10 ** 6, cfg=pbb.PoolConfig(explorers=100, disable_pruning=True, batch_steps=64))
    assert res.stats.leaves == math.factorial(n)


@pytest.mark.parametrize("name,ub", [("ta041", 2992), ("ta011", 1583)])
def test_pinned_mode_matches_oracle(name, ub):
    """Pinned UB (prune >= ub, never improve) just above the optimum is a fixed tree too."""
    inst = pbb.taillard_named(name)
    ref = orc.Problem(inst.p, orc.LB1).solve(ub, pinned=True, threads=4, prefix_depth=2)
    res = pbb.pool_run(inst, ub, cfg=pbb.PoolConfig(pinned=True, explorers=300))
    assert res.stats.unique == ref["unique"]
    assert res.stats.leaves == ref["leaves"]
    assert res.stats.improvements == 0
    # the bench's pinned configuration: live-sibling splitting + breadth-first seeding
    from paper_2012_09511_b200.multi import solve_distributed
    with pbb.GpuPool(inst, pbb.PoolConfig(pinned=True, split_mode=1), bound="lb1") as pool:
        r = solve_distributed(pool, ub, seed_div=16)
    assert r.completed and r.unique == ref["unique"] and r.leaves == ref["leaves"] and r.improvements == 0


# ---------------------------------------------------------------- pool surface

def test_pool_rounds_snapshot_and_offer_bound():
    inst = pbb.taillard_named("ta021")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=512, batch_steps=256, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(2297)
        pool.assign_fresh([(0, math.factorial(20))])
        assert pool.active_count() == 1
        for _ in range(3):
            pool.run_round()
        snap = pool.snapshot_intervals()
        assert snap and all(a < b for a, b in snap)
        assert all(snap[i][1] <= snap[i + 1][0] for i in range(len(snap) - 1))
        pool.offer_bound(2296)
        pool.run_round()
        assert pool.best_value() == 2296
        st = pool.stats()
        assert st.rounds == 4 and st.decomposed > 0


@pytest.mark.parametrize("name,ub,rounds", [("ta011", 1582, 3), ("ta011", 1582, 7), ("ta021", 2297, 5)])
def test_snapshot_resume_preserves_count(name, ub, rounds):
    """Snapshot the remaining work after a few rounds, restart it in a fresh pool:
    nodes before - resume recount + nodes after == the reference's count, exactly."""
    # ta021@2297: the reference's 534.8-s K=1 proof
    ref = golden_io.ref_counts().get(f"{name}@{ub}", {"decomposed": 462443491, "leaves": 1440})
    inst = pbb.taillard_named(name)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=256, batch_steps=64, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(ub)
        pool.assign_split(256)
        for _ in range(rounds):
            pool.run_round()
        snap, recount = pool.snapshot()
        done = pool.stats()
    assert snap and recount >= 0
    res = pbb.pool_run(inst, ub, intervals=snap, cfg=pbb.PoolConfig(explorers=max(512, len(snap))))
    # path nodes between lnz(pos) and each explorer's level are decomposed again by the resumed
    # pool's replays (partial replays: redone from scratch); the recount removes exactly those
    assert done.unique - recount + res.stats.unique == ref["decomposed"]
    assert done.leaves + res.stats.leaves == ref["leaves"]


# ---------------------------------------------------------------- large n (ta111, 500 x 20): bounding-only pools

def _nodes_with_f(n, fs, seed):
    rng = np.random.default_rng(seed)
    perms, d1s, d2s = [], [], []
    for f in fs:
        perms.append(rng.permutation(n))
        d1 = int(rng.integers(0, n - f + 1))
        d1s.append(d1)
        d2s.append(n - f - d1)
    return np.array(perms), d1s, d2s


@pytest.mark.parametrize("bound,fs", [("lb1", [1, 2, 7, 50, 137, 256, 499, 500, 333, 64, 65, 300] * 4),
                                      ("lb2", [1, 2, 5, 17, 40, 64, 65, 90])])
def test_large_n_decompose_matches_oracle(bound, fs):
    inst = pbb.taillard_named("ta111")
    perms, d1s, d2s = _nodes_with_f(inst.n, fs, 23)
    prob = orc.Problem(inst.p, orc.LB1 if bound == "lb1" else orc.LB2)
    inc = 26670
    with pbb.GpuPool(inst, bound=bound) as pool:
        assert pool.K() == 0
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, inc)
        with pytest.raises(_lib.PbbError):
            pool.assign_split()
    for i in range(len(fs)):
        f = inst.n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        d, clb, cpr = prob.decompose(perms[i], d1s[i], d2s[i], inc)
        assert [int(x) for x in lf[i, :f]] == fw
        assert [int(x) for x in lbw[i, :f]] == bw
        assert int(dr[i]) == d
        assert [int(x) for x in lb[i, :f]] == clb
        assert [int(x) for x in pr[i, :f]] == cpr


@pytest.mark.parametrize("name", ["ta111", "ta091", "ta081", "ta061"])
@pytest.mark.parametrize("fdist", ["deep", "shallow"])
def test_large_n_lb1_batch_kernels(name, fdist):
    """Both large-n LB1 kernels over batches that fill many CTAs (ragged f, partial last
    group): "deep" batches (mean f < n/2) run the lane-per-node table kernel, "shallow" ones
    the warp-per-node kernel; m = 20 (two wavefront passes) and m = 5 / 10 (front and tail in
    the two half-warps); d2 = 0 and d1 = 0 nodes included. Node by node against the oracle."""
    inst = pbb.taillard_named(name)
    n = inst.n
    rng = np.random.default_rng(7)
    cnt = 16 * 148 + 13
    fs = rng.integers(1, n // 3, cnt) if fdist == "deep" else rng.integers(2 * n // 3, n + 1, cnt)
    fs[:4] = [1, n, 2, n - 1]
    perms = rng.random((cnt, n)).argsort(axis=1).astype(np.int32)
    d1s = np.array([int(rng.integers(0, n - f + 1)) for f in fs])
    d1s[4:40:3] = 0
    d1s[5:40:3] = n - fs[5:40:3]  # d2 = 0
    d2s = n - fs - d1s
    prob = orc.Problem(inst.p, orc.LB1)
    inc = int(rng.integers(1000, 30000))
    with pbb.GpuPool(inst, bound="lb1") as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, inc)
    for i in list(range(64)) + list(rng.integers(0, cnt, 400)) + [cnt - 1]:
        f = int(fs[i])
        fw, bw = prob.children_bounds(perms[i], int(d1s[i]), int(d2s[i]))
        d, clb, cpr = prob.decompose(perms[i], int(d1s[i]), int(d2s[i]), inc)
        assert [int(x) for x in lf[i, :f]] == fw, i
        assert [int(x) for x in lbw[i, :f]] == bw, i
        assert int(dr[i]) == d, i
        assert [int(x) for x in lb[i, :f]] == clb, i
        assert [int(x) for x in pr[i, :f]] == cpr, i


@pytest.mark.parametrize("name", ["ta111", "ta081"])
def test_large_n_lb2_shallow_batch(name):
    """LB2 on shallow nodes (f up to n: every position of each pair's Johnson order is free,
    the free-position bitmask walk crosses all 16 mask words), against the oracle."""
    inst = pbb.taillard_named(name)
    n = inst.n
    fs = [n, n - 1, 2 * n // 3, 3 * n // 4, n - 7, 1, 3, n // 2 + 1] * 2
    perms, d1s, d2s = _nodes_with_f(n, fs, 29)
    prob = orc.Problem(inst.p, orc.LB2)
    inc = 26670 if name == "ta111" else 6000
    with pbb.GpuPool(inst, bound="lb2") as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, inc)
    for i in range(len(fs)):
        f = n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        d, clb, cpr = prob.decompose(perms[i], d1s[i], d2s[i], inc)
        assert [int(x) for x in lf[i, :f]] == fw, i
        assert [int(x) for x in lbw[i, :f]] == bw, i
        assert int(dr[i]) == d, i
        assert [int(x) for x in lb[i, :f]] == clb, i
        assert [int(x) for x in pr[i, :f]] == cpr, i


# ---------------------------------------------------------------- heuristic cooperation (§8(f) #1)

def test_promote_and_offer_schedule():
    inst = pbb.taillard_named("ta021")
    start = pbb.neh(inst)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=512), bound="lb1") as pool:
        pool.set_initial_bound(start.cmax, start.perm)
        pool.assign_split()
        pool.run_round()
        proms = pool.promote_solutions(5)
        assert 0 < len(proms) <= 5
        assert [p.cmax for p in proms] == sorted(p.cmax for p in proms)
        for p in proms:
            assert sorted(p.perm) == list(range(20)) and pbb.makespan(inst, p.perm) == p.cmax
        better = pbb.insertion_local_search(inst, start, max_iterations=500, rng_seed=1)
        assert better.cmax < start.cmax
        assert pool.offer_schedule(better)
        pool.run_round()
        assert pool.best_value() <= better.cmax
        assert pool.best_schedule().cmax <= better.cmax
        with pytest.raises(ValueError):
            pool.offer_schedule(pbb.Schedule(better.perm, better.cmax - 1))  # cmax must match


@pytest.mark.parametrize("name,opt,bound", [("ta041", 2991, "lb1"), ("ta011", 1582, "lb2"), ("ta031", 2724, "lb1")])
def test_cooperative_solve_finds_optimum(name, opt, bound):
    r = pbb.solve_cooperative(pbb.taillard_named(name), bound=bound, ls_iterations=500)
    assert r.completed and r.best_value == opt
    assert r.initial_ub >= opt
    if r.best.perm:
        assert pbb.makespan(pbb.taillard_named(name), r.best.perm) == r.best.cmax


# ---------------------------------------------------------------- checkpoint / restart (§8(f) #2)

def test_checkpoint_restart_completes_the_proof(tmp_path):
    """Stop a proof after a few rounds, checkpoint (reference format), resume in a new pool,
    checkpoint again, resume again, finish: node and leaf totals equal the reference's
    single-run counts exactly, the bound and schedule survive."""
    from paper_2012_09511_b200 import checkpoint as ck

    ref = golden_io.ref_counts()["ta011@1582"]
    inst = pbb.taillard_named("ta011")
    path = str(tmp_path / "ta011.ckpt")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=256, batch_steps=64, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(1582)
        pool.assign_split()
        for _ in range(3):
            pool.run_round()
        first = pool.stats()
        d = ck.save_pool(pool, path)
    assert d.units[0].intervals and d.total_nodes <= first.unique
    with ck.resume_pool(path, inst, pbb.PoolConfig(explorers=4096, batch_steps=64, rounds_per_sync=1)) as pool2:
        assert pool2.resumed_nodes == d.total_nodes
        for _ in range(2):
            pool2.run_round()
        second = pool2.stats()
        d2 = ck.save_pool(pool2, path)   # carries the first checkpoint's total
    with ck.resume_pool(path, inst, pbb.PoolConfig(explorers=4096)) as pool3:
        while pool3.run_round():
            pass
        rest = pool3.stats()
        assert pool3.best_value() == 1582
    assert first.leaves + second.leaves + rest.leaves == ref["leaves"]
    assert d2.total_nodes + rest.unique == ref["decomposed"]


def test_timeline_csv(tmp_path):
    """Activity timeline rows in the reference format; forced sample at exhaustion."""
    import csv

    inst = pbb.taillard_named("ta011")
    path = tmp_path / "tl.csv"
    tl = pbb.Timeline(str(path))
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=300, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(1582)
        pool.assign_split()
        tl.sample(pool, force=True)
        assert not tl.sample(pool)                 # < 50 ms after the previous sample
        while pool.run_round():
            tl.sample(pool, force=True)
        tl.sample(pool, force=True)
    tl.close()
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["timestamp_ms", "explorer_id", "active", "interval_length_log2"]
    body = rows[1:]
    assert len(body) >= 2 * 300 and len(body) % 300 == 0
    last = body[-300:]
    assert all(r[2] == "0" and r[3] == "-1" for r in last)         # exhausted: all idle
    assert any(r[2] == "1" and int(r[3]) > 0 for r in body[:-300])  # remaining work is tracked


# ---------------------------------------------------------------- pool reuse (serving loop)

@pytest.mark.parametrize("bound", ["lb1", "lb2"])
def test_load_instance_matches_fresh_pools(bound):
    """One pool fed several same-shape instances gives exactly the fresh pools' results."""
    ta001 = pbb.taillard_named("ta001")
    others = [pbb.taillard_named(f"ta00{i}") for i in (2, 3)]
    optimum = {"ta001": 1278, "ta002": 1359, "ta003": 1081}  # fixed trees: UB = optimum
    with pbb.GpuPool(ta001, bound=bound) as pool:
        for inst in others + [ta001]:
            ub = optimum[inst.label]
            pool.load_instance(inst)
            got = pbb.solve_pool(pool, ub)
            want = pbb.pool_run(inst, ub, bound=bound)
            assert got.stats.completed and want.stats.completed
            assert got.stats.unique == want.stats.unique
            assert got.stats.leaves == want.stats.leaves
            assert got.best_value == want.best_value
            assert got.hist == want.hist
            if got.best.perm:
                assert pbb.makespan(inst, got.best.perm) == got.best_value
    if bound == "lb1":
        ref = golden_io.ref_counts()["ta001@1278"]
        with pbb.GpuPool(others[0], bound=bound) as pool:
            pool.load_instance(ta001)
            res = pbb.solve_pool(pool, 1278)
            assert res.stats.unique == ref["decomposed"]
            assert _hist_str(res.hist) == ref["hist"]


def test_load_instance_rejects_other_shapes():
    with pbb.GpuPool(pbb.taillard_named("ta001"), bound="lb1") as pool:
        with pytest.raises(ValueError):
            pool.load_instance(pbb.taillard_named("ta011"))


def test_load_instance_batch_only_pool():
    a, b = pbb.taillard_named("ta111"), pbb.taillard_named("ta112")
    perms, d1s, d2s = _nodes_with_f(a.n, [1, 50, 300, 499], 5)
    with pbb.GpuPool(a, bound="lb2") as pool:
        pool.load_instance(b)
        got = pool.decompose_batch(perms, d1s, d2s, 1 << 30)
    with pbb.GpuPool(b, bound="lb2") as fresh:
        want = fresh.decompose_batch(perms, d1s, d2s, 1 << 30)
    for x, y in zip(got, want):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("key", ["ta011@1582", "ta041@2991"])
@pytest.mark.parametrize("div", [1, 16])
def test_breadth_first_seeding_keeps_counts(key, div):
    """pbbgpu_seed cuts [0, n!) at live frontier nodes: any partition keeps the exact count."""
    from paper_2012_09511_b200.multi import solve_distributed
    ref = golden_io.ref_counts()[key]
    name, ub = key.split("@")
    with pbb.GpuPool(pbb.taillard_named(name), bound="lb1") as pool:
        r = solve_distributed(pool, int(ub), seed_div=div)
    assert r.completed
    assert r.unique == ref["decomposed"]
    assert r.leaves == ref["leaves"]
    assert _hist_str(r.hist) == ref["hist"]


# ---------------------------------------------------------------- LB2 pinned to its definition

def _nodes_small_f(n, count, fmax, seed):
    rng = np.random.default_rng(seed)
    perms, d1s, d2s = [], [], []
    for _ in range(count):
        perms.append(rng.permutation(n))
        f = int(rng.integers(1, min(fmax, n) + 1))
        d1 = int(rng.integers(0, n - f + 1))
        d1s.append(d1)
        d2s.append(n - f - d1)
    return np.array(perms), d1s, d2s


@pytest.mark.parametrize("name,fmax,count", [("ta001", 12, 300), ("ta021", 10, 100), ("ta056", 10, 60),
                                             ("ta041", 11, 120), ("ta111", 8, 12)])
def test_gpu_lb2_equals_relaxation_optimum(name, fmax, count):
    """Every GPU LB2 child bound (small-n warp kernel, and the large-n kernel for ta111) equals
    the maximum over machine pairs of the two-machine time-lag relaxation's optimum over ALL job
    orders (oracle subset DP, no Johnson order involved)."""
    inst = pbb.taillard_named(name)
    perms, d1s, d2s = _nodes_small_f(inst.n, count, fmax, 31)
    prob = orc.Problem(inst.p, orc.LB2)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=256), bound="lb2") as pool:
        _, _, _, lf, lbw = pool.decompose_batch(perms, d1s, d2s, 10 ** 6)
    for i in range(count):
        f = inst.n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds_lb2_exact(perms[i], d1s[i], d2s[i])
        assert [int(x) for x in lf[i, :f]] == fw
        assert [int(x) for x in lbw[i, :f]] == bw


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("m", [5, 10, 20])
def test_gpu_lb2_optimal_under_ties(seed, m):
    """Tie-heavy instances (times in {1, 2, 3}, one constant column): a = b jobs, equal keys."""
    rng = np.random.default_rng(4000 + 10 * m + seed)
    n = 12
    p = rng.integers(1, 4, size=(n, m)).astype(np.int32)
    if seed % 2 == 0:
        p[:, int(rng.integers(0, m))] = 2
    inst = pbb.Instance(n, m, p)
    perms, d1s, d2s = _nodes_small_f(n, 60, 9, seed)
    prob = orc.Problem(p, orc.LB2)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=128), bound="lb2") as pool:
        _, _, _, lf, lbw = pool.decompose_batch(perms, d1s, d2s, 10 ** 6)
    for i in range(len(d1s)):
        f = n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds_lb2_exact(perms[i], d1s[i], d2s[i])
        assert [int(x) for x in lf[i, :f]] == fw
        assert [int(x) for x in lbw[i, :f]] == bw


# ---------------------------------------------------------------- the reference's own steal policy

def _ref_instance(name):
    if name.startswith("gen:"):
        n, m, seed = (int(x) for x in name[4:].split(":"))
        return pbb.generate_taillard(n, m, seed)
    return pbb.taillard_named(name)


_STATS_KEYS = sorted(k for k in golden_io.ref_counts() if k.startswith("stats:"))


@pytest.mark.parametrize("key", _STATS_KEYS)
def test_reference_steal_policy_reproduces_pool_stats(key):
    """steal_policy = 1 (explorer.cpp:251-340 on the device) with the reference's round length
    (batch_steps) reproduces EVERY PoolStats counter of the compiled reference's pool_run:
    raw decomposed (replays included), leaves, local steals, steal phases, intervals
    initialized -- for K = 4^c (hypercube matching) and other K (largest eligible)."""
    g = golden_io.ref_counts()[key]
    inst = _ref_instance(g["instance"])
    nopr = bool(g["disable_pruning"])
    cfg = pbb.PoolConfig(explorers=g["explorers"], batch_steps=g["batch_steps"], steal_policy=1,
                         disable_pruning=nopr, record_census=nopr, rounds_per_sync=2)
    with pbb.GpuPool(inst, cfg, bound="lb1") as pool:
        pool.set_initial_bound(g["initial_ub"])
        pool.assign_fresh([(0, math.factorial(inst.n))])          # pool_run's default interval
        while pool.run_round():
            pass
        st = pool.stats()
        assert (st.decomposed, st.leaves, st.local_steals, st.steal_phases, st.intervals_initialized) == (
            g["decomposed"], g["leaves"], g["local_steals"], g["steal_phases"], g["intervals_initialized"])
        assert pool.best_value() == g["best_value"]
        if nopr:
            census = pool.take_census()
            assert len(census) == g["census_size"] and sorted(census) == list(range(math.factorial(inst.n)))


@pytest.mark.parametrize("policy", [0, 1])
def test_census_covers_every_leaf_under_any_partition(policy):
    """SPEC acceptance 4: pruning disabled, n <= 9, any partition into <= 16
    intervals: the census holds each of the n! leaves exactly once."""
    inst = pbb.generate_taillard(8, 5, 31337)
    nf = math.factorial(8)
    rng = np.random.default_rng(policy)
    cuts = sorted(set(int(x) for x in rng.integers(1, nf, 15)))
    ivs = list(zip([0] + cuts, cuts + [nf]))
    cfg = pbb.PoolConfig(explorers=64, disable_pruning=True, record_census=True, steal_policy=policy,
                         batch_steps=97 if policy else 0)
    with pbb.GpuPool(inst, cfg, bound="lb1") as pool:
        pool.set_initial_bound(10 ** 6)
        pool.assign_fresh(ivs)
        while pool.run_round():
            pass
        census = pool.take_census()
        assert pool.take_census() == []                             # taken: cleared
    assert sorted(census) == list(range(nf))


def test_census_requires_small_n_and_the_flag():
    with pytest.raises(ValueError):
        pbb.GpuPool(pbb.taillard_named("ta041"), pbb.PoolConfig(record_census=True))
    with pbb.GpuPool(pbb.taillard_named("ta001"), pbb.PoolConfig(explorers=32)) as pool:
        with pytest.raises(_lib.PbbError):
            pool.take_census()


# ---------------------------------------------------------------- the rest of the worker-facing surface

def _merged(ivs):
    out = []
    for a, b in sorted(ivs):
        if out and a <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


def test_apply_work_update_keeps_splits_and_reseats():
    """apply_work_update (explorer.cpp:162-199): echoing the snapshot keeps every explorer;
    splitting every interval in two keeps the left parts (ends shrink) and seats the right
    parts on idle explorers. The proof then completes with the reference's exact count."""
    ref = golden_io.ref_counts()["ta011@1582"]
    inst = pbb.taillard_named("ta011")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=1024, batch_steps=64, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(1582)
        pool.assign_split(200)
        for _ in range(2):
            pool.run_round()
        snap = pool.snapshot_intervals()
        act = pool.active_count()
        pool.apply_work_update(snap)                                # echo: nothing moves
        assert pool.snapshot_intervals() == snap and pool.active_count() == act
        halves = []
        for a, b in snap:
            mid = (a + b) // 2
            halves += [(a, mid), (mid, b)] if b - a >= 2 else [(a, b)]
        pool.apply_work_update(halves)
        assert _merged(pool.snapshot_intervals()) == _merged(snap)  # same remaining work
        assert pool.active_count() == len([h for h in halves if h[0] < h[1]])
        while pool.run_round():
            pass
        st = pool.stats()
    assert st.unique == ref["decomposed"] and st.leaves == ref["leaves"]


def test_apply_work_update_drops_work_and_errors():
    inst = pbb.taillard_named("ta011")
    nf = math.factorial(20)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=64, batch_steps=32, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(1582)
        pool.assign_split(64)
        pool.run_round()
        snap = pool.snapshot_intervals()
        keep = snap[: len(snap) // 2]
        pool.apply_work_update(keep)                                # the other half goes idle
        assert pool.snapshot_intervals() == keep
        with pytest.raises(ValueError):                             # more intervals than explorers
            pool.apply_work_update([(i, i + 1) for i in range(0, 2 * 65, 2)])
        pool.apply_work_update([])
        assert pool.active_count() == 0
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=8)) as pool:
        pool.set_initial_bound(1582)
        pool.assign_split(8)                                        # 8 explorers on [s_i, s_i+1)
        starts = [a for a, _ in pool.snapshot_intervals()]
        pool.apply_work_update([(a, a + 1024) for a in starts])     # all kept, ends shrink
        assert pool.snapshot_intervals() == [(a, a + 1024) for a in starts]
        with pytest.raises(_lib.PbbError):                          # 8 gaps, no idle explorer
            pool.apply_work_update([(0, nf)])


def test_marks_follow_the_reference():
    inst = pbb.taillard_named("ta001")
    neh = pbb.neh(inst)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=64, batch_steps=16, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(neh.cmax, neh.perm)
        assert not pool.improved_since_mark()                       # the seed is the mark
        pool.assign_split(4)
        saw = False
        while pool.run_round():
            saw |= pool.improved_since_mark()
        saw |= pool.improved_since_mark()
        assert saw and not pool.improved_since_mark()
        assert pool.best_schedule().cmax == pool.best_value() == 1278
        assert pool.steals_since_mark() > 0
        pool.reset_steal_mark()
        assert pool.steals_since_mark() == 0


def test_pool_timeline_csv(tmp_path):
    """PoolConfig.timeline_path: rows written by the pool at run_round (>= 50 ms apart, forced
    at exhaustion), exact floor(log2) remaining lengths, flush_timeline forces a sample."""
    import csv

    path = tmp_path / "pool_tl.csv"
    inst = pbb.taillard_named("ta011")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=96, rounds_per_sync=1, timeline_path=str(path))) as pool:
        pool.set_initial_bound(1582)
        pool.assign_fresh([(0, math.factorial(20))])
        while pool.run_round():
            pass
        pool.flush_timeline()
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["timestamp_ms", "explorer_id", "active", "interval_length_log2"]
    body = rows[1:]
    assert len(body) >= 2 * 96 and len(body) % 96 == 0
    first = body[:96]
    assert first[0][2] == "1" and int(first[0][3]) <= 61 and int(first[0][3]) >= 0   # log2(20!) = 61.07
    assert all(r[2] == "0" and r[3] == "-1" for r in body[-96:])


# ---------------------------------------------------------------- the reference's runtime driving GPU pools

GPU_WORKER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                          "gpu_worker")


def _gpu_worker(*args):
    if not os.path.exists(GPU_WORKER):
        pytest.skip("integration/_build/gpu_worker not built (make -C integration needs /root/reference)")
    out = subprocess.run([GPU_WORKER, *map(str, args)], capture_output=True, text=True, timeout=600, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("K", [16, 64, 48])
def test_reference_binding_pool_run_reproduces_pool_stats(K):
    """integration/pbb/gpu_pool.hpp (GpuExplorerPool, compiled against the reference's own
    headers) driven like pool_run with the reference steal policy: PoolStats equal the compiled
    reference's (tests/golden/ref_counts.json, made by oracle/_ref/ref_driver)."""
    g = golden_io.ref_counts()[f"stats:ta011@1582:K{K}:b1024:np0"]
    r = _gpu_worker("pool", "ta011", 1582, K, "lb1", 1, 1024)
    assert (r["decomposed"], r["leaves"], r["local_steals"], r["steal_phases"], r["intervals_initialized"]) == (
        g["decomposed"], g["leaves"], g["local_steals"], g["steal_phases"], g["intervals_initialized"])
    assert r["unique"] == golden_io.ref_counts()["ta011@1582"]["decomposed"]


@pytest.mark.parametrize("name,ub,leaves,unique", [("ta011", 1582, 54, 158049), ("ta021", 2297, 1440, 462443491)])
def test_reference_coordinator_drives_one_gpu_worker_exactly(name, ub, leaves, unique):
    """Coordinator::run (src/coordinator.cpp) over the reference's in-process transport and
    wire codec, one worker running worker_run's pool-role loop on a GpuExplorerPool
    (apply_work_update, marks, snapshots): the proof's counts equal pool_run's exactly."""
    r = _gpu_worker("cluster", name, ub, 1, "lb1")
    assert r["unique"] == unique and r["leaves"] == leaves
    assert r["coordinator_total_nodes"] == r["decomposed"]        # WORK checkpoints carried every node
    assert r["updates_applied"] >= 1 and r["splits"] == 0


def test_reference_coordinator_drives_several_gpu_workers():
    """Three GPU workers under the reference coordinator: work units are split by the
    coordinator (split_unit) and handed over with apply_work_update; every leaf is evaluated and
    nothing is lost (the protocol may redo work a stale snapshot had already covered, as it does
    with the reference's CPU workers)."""
    r = _gpu_worker("cluster", "ta011", 1582, 3, "lb1")
    assert r["splits"] > 0 and r["updates_applied"] > 3
    assert r["leaves"] >= 54 and r["unique"] >= 158049
    assert r["coordinator_total_nodes"] == r["decomposed"]


# ---------------------------------------------------------------- any machine count (m <= 20)

@pytest.mark.parametrize("m", [1, 2, 3, 4, 7, 9, 13, 15, 17, 19, 23, 40, 47, 60])
@pytest.mark.parametrize("bound", ["lb1", "lb2"])
def test_any_machine_count_bounds_match_oracle(m, bound):
    if m > 20 and bound == "lb2":
        with pytest.raises(ValueError):
            pbb.GpuPool(pbb.generate_taillard(12, m, 1), bound="lb2")
        return
    """m not in {5, 10, 20}: the pool pads the instance with zero-time machines; every child
    bound (LB2 over the real machine pairs only; m = 1: LB1) equals the oracle's."""
    n = 12
    inst = pbb.generate_taillard(n, m, 500 + m)
    perms, d1s, d2s = _random_nodes(n, 300, m)
    prob = orc.Problem(inst.p, orc.LB1 if bound == "lb1" else orc.LB2)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=128), bound=bound) as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, 10 ** 6)
    for i in range(len(d1s)):
        f = n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        assert [int(x) for x in lf[i, :f]] == fw and [int(x) for x in lbw[i, :f]] == bw
        d, clb, _ = prob.decompose(perms[i], d1s[i], d2s[i], 10 ** 6)
        assert int(dr[i]) == d and [int(x) for x in lb[i, :f]] == clb


@pytest.mark.parametrize("key", ["gen:30:15:4242@2490", "gen:16:13:1234@1512", "gen:18:3:77@926",
                                 "gen:14:40:2024@3124", "gen:12:60:606@4417", "gen:16:25:99@2282"])
def test_any_machine_count_fixed_trees_match_reference(key):
    """Fixed trees of instances with 15 (VFR-like 30 x 15), 13, 3, 25, 40 and 60 machines (LB1; m > 20
    runs the M = 40 / 60 kernels): unique node count, leaves and the per-f histogram equal the
    compiled reference's (ref_driver hist)."""
    g = golden_io.ref_counts()[key]
    name, ub = key.split("@")
    n, m, seed = (int(x) for x in name[4:].split(":"))
    inst = pbb.generate_taillard(n, m, seed)
    res = pbb.pool_run(inst, int(ub), cfg=pbb.PoolConfig())
    assert res.stats.unique == g["decomposed"] and res.stats.leaves == g["leaves"]
    assert res.best_value == int(ub)
    assert {str(k): v for k, v in res.hist.items()} == g["hist"]


# ---------------------------------------------------------------- wide processing times (LB1)

@pytest.mark.parametrize("n,m,pmax", [(12, 5, 50000), (12, 20, 9000), (14, 40, 20000), (40, 10, 30000),
                                      (64, 20, 300000)])
def test_wide_times_bounds_match_oracle(n, m, pmax):
    """(n+m)*max p >= 2^16: the explorers keep 32-bit front / tail / remain tables and the
    MinMin sums are reduced separately; every child bound, direction and prune flag equals the
    oracle's (int64, bound.cpp's types)."""
    rng = np.random.default_rng(n * 1000 + m)
    inst = pbb.Instance(n, m, rng.integers(1, pmax + 1, size=(n, m), dtype=np.int32))
    perms, d1s, d2s = _random_nodes(n, 300, m)
    prob = orc.Problem(inst.p, orc.LB1)
    inc = (n + m) * pmax // 3
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=128), bound="lb1") as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(perms, d1s, d2s, inc)
    for i in range(len(d1s)):
        f = n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        assert [int(x) for x in lf[i, :f]] == fw and [int(x) for x in lbw[i, :f]] == bw
        d, clb, prn = prob.decompose(perms[i], d1s[i], d2s[i], inc)
        assert int(dr[i]) == d and [int(x) for x in lb[i, :f]] == clb
        assert [bool(x) for x in pr[i, :f]] == [bool(x) for x in prn]


@pytest.mark.parametrize("key,scale", [("ta011@1582", 1000), ("gen:14:40:2024@3124", 700), ("ta061@5493", 100)])
def test_wide_times_scaled_fixed_trees_match_reference(key, scale):
    """Scaling every processing time by c scales every front, tail, bound and makespan by c and
    keeps every comparison and MinMin tie, so the fixed tree of c*p under c*ub is the
    reference's tree of p under ub: unique count, leaves and per-f histogram equal its golden
    counts (m = 40 runs the M = 40 wide kernels, ta061 the n > 64 explorer pool)."""
    g = golden_io.ref_counts()[key]
    name, ub = key.split("@")
    if name.startswith("gen:"):
        n, m, seed = (int(x) for x in name[4:].split(":"))
        base = pbb.generate_taillard(n, m, seed)
    else:
        base = pbb.taillard_named(name)
    inst = pbb.Instance(base.n, base.m, base.p.astype(np.int64) * scale)
    assert (inst.n + inst.m) * int(inst.p.max()) >= 1 << 16
    cfg = pbb.PoolConfig(explorers=1024) if inst.n > 64 else pbb.PoolConfig()
    res = pbb.pool_run(inst, int(ub) * scale, cfg=cfg)
    assert res.stats.unique == g["decomposed"] and res.stats.leaves == g["leaves"]
    assert res.best_value == int(ub) * scale
    assert {str(k): v for k, v in res.hist.items()} == {str(k): v for k, v in g["hist"].items()}


@pytest.mark.parametrize("seed", range(3))
def test_wide_times_optimum_matches_brute_force(seed):
    n, m = 8, 6
    rng = np.random.default_rng(77 + seed)
    inst = pbb.Instance(n, m, rng.integers(1, 200000, size=(n, m), dtype=np.int32))
    best = min(pbb.makespan(inst, perm) for perm in itertools.permutations(range(n)))
    res = pbb.pool_run(inst, 10 ** 9, cfg=pbb.PoolConfig(explorers=128))
    assert res.best_value == best and pbb.makespan(inst, res.best.perm) == best


def test_wide_times_limits():
    """LB2's pair tables stay 16-bit; LB1 takes n*(n+m)*max p < 2^31; a narrow pool refuses a
    wide instance in load_instance (its explorer tables are 16-bit)."""
    wide = pbb.Instance(10, 5, np.full((10, 5), 10000, dtype=np.int32))
    with pytest.raises(ValueError):
        pbb.GpuPool(wide, bound="lb2")
    with pytest.raises(ValueError):
        pbb.GpuPool(pbb.Instance(10, 5, np.full((10, 5), 20_000_000, dtype=np.int32)), bound="lb1")
    with pbb.GpuPool(pbb.generate_taillard(10, 5, 3), bound="lb1") as pool:
        with pytest.raises(RuntimeError):
            pool.load_instance(wide)
    with pbb.GpuPool(wide, bound="lb1") as pool:  # a wide pool takes narrow instances too
        pool.load_instance(pbb.generate_taillard(10, 5, 3))


@pytest.mark.parametrize("workers", [1, 2])
def test_product_worker_speaks_the_reference_protocol_over_tcp(workers):
    """libpbbgpu's own worker role and wire codec (pbbgpu_worker_run) connected over TCP to the
    reference's Coordinator and TcpListener: the proof completes; with one worker its counts
    are exactly pool_run's, and the coordinator's node total is the workers' WORK checkpoints."""
    r = _gpu_worker("tcp", "ta011", 1582, workers, "lb1")
    assert r["leaves"] >= 54 and r["unique"] >= 158049
    assert r["coordinator_total_nodes"] == r["decomposed"]
    assert r["messages"] == r["worker_messages"]               # every frame decoded by the reference
    if workers == 1:
        assert r["unique"] == 158049 and r["leaves"] == 54 and r["splits"] == 0
    else:
        assert r["splits"] > 0


# ---------------------------------------------------------------- explorer pools for n > 64

@pytest.mark.parametrize("key,bound,K", [("ta061@5493", "lb1", 1024), ("ta081@6070", "lb1", 4096),
                                         ("ta101@11150", "lb1", 8192), ("ta111@26000", "lb1", 2048),
                                         ("ta081@6070", "lb2", 4096), ("ta111@26000", "lb2", 1024)])
def test_large_n_explorer_pool_fixed_trees(key, bound, K):
    """64 < n <= 512: IVM explorers in HBM (int16 cells), one select -> bound (the large-n
    kernels) -> branch step at a time, log2-bucket interval stealing: unique counts, leaves and
    per-f histograms equal the reference's K = 1 fixed trees (LB1) / the oracle's (LB2)."""
    gold = golden_io.ref_counts()[key] if bound == "lb1" else golden_io.lb2_counts()[key]
    want = gold["decomposed"] if bound == "lb1" else gold["unique"]
    name, ub = key.split("@")
    inst = pbb.taillard_named(name)
    res = pbb.pool_run(inst, int(ub), cfg=pbb.PoolConfig(explorers=K), bound=bound)
    assert res.stats.K == K and res.stats.completed
    assert res.stats.unique == want and res.stats.leaves == gold["leaves"]
    assert res.best_value == int(ub)
    assert {str(k): v for k, v in res.hist.items()} == {str(k): v for k, v in gold["hist"].items()}


@pytest.mark.parametrize("key,bound,rounds", [("ta081@6070", "lb1", 2), ("ta081@6070", "lb1", 5),
                                              ("ta081@6070", "lb2", 3), ("ta101@11150", "lb1", 3)])
def test_large_n_snapshot_resume_preserves_count(key, bound, rounds):
    """snapshot_intervals on the n > 64 explorer pool (int16 IVMs): the remaining work after a
    few rounds, resumed in a fresh pool, completes the fixed tree with exact node accounting
    (nodes before - resume recount + nodes after == the reference's / the oracle's count)."""
    gold = golden_io.ref_counts()[key] if bound == "lb1" else golden_io.lb2_counts()[key]
    want = gold["decomposed"] if bound == "lb1" else gold["unique"]
    name, ub = key.split("@")
    inst = pbb.taillard_named(name)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=1024, rounds_per_sync=1), bound=bound) as pool:
        pool.set_initial_bound(int(ub))
        pool.assign_split(1024)
        for _ in range(rounds):
            pool.run_round()
        snap, recount = pool.snapshot()
        done = pool.stats()
    assert snap and not done.completed
    res = pbb.pool_run(inst, int(ub), intervals=snap, cfg=pbb.PoolConfig(explorers=max(1024, len(snap))), bound=bound)
    assert done.unique - recount + res.stats.unique == want
    assert done.leaves + res.stats.leaves == gold["leaves"]


def test_large_n_apply_work_update_keeps_splits_and_reseats():
    """apply_work_update on the n > 64 explorer pool: the echo keeps every explorer, halving
    every interval shrinks ends and seats the right halves; the proof completes exactly."""
    ref = golden_io.ref_counts()["ta081@6070"]
    inst = pbb.taillard_named("ta081")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=1024, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(6070)
        pool.assign_split(200)
        pool.run_round()
        snap = pool.snapshot_intervals()
        assert snap
        act = pool.active_count()
        pool.apply_work_update(snap)
        assert pool.snapshot_intervals() == snap and pool.active_count() == act
        halves = []
        for a, b in snap:
            mid = (a + b) // 2
            halves += [(a, mid), (mid, b)] if b - a >= 2 else [(a, b)]
        pool.apply_work_update(halves)
        assert _merged(pool.snapshot_intervals()) == _merged(snap)
        while pool.run_round():
            pass
        st = pool.stats()
    assert st.unique == ref["decomposed"] and st.leaves == ref["leaves"]


def test_large_n_checkpoint_restart_completes_the_proof(tmp_path):
    """Checkpoint / restart (reference format) of an n > 64 explorer pool: totals exact."""
    from paper_2012_09511_b200 import checkpoint as ck

    ref = golden_io.ref_counts()["ta101@11150"]
    inst = pbb.taillard_named("ta101")
    path = str(tmp_path / "ta101.ckpt")
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=2048, rounds_per_sync=1)) as pool:
        pool.set_initial_bound(11150)
        pool.assign_split()
        for _ in range(4):
            pool.run_round()
        first = pool.stats()
        d = ck.save_pool(pool, path)
    assert d.units[0].intervals and not first.completed
    with ck.resume_pool(path, inst, pbb.PoolConfig(explorers=2048)) as pool2:
        while pool2.run_round():
            pass
        rest = pool2.stats()
        assert pool2.best_value() == 11150
    assert first.leaves + rest.leaves == ref["leaves"]
    assert d.total_nodes + rest.unique == ref["decomposed"]


def test_large_n_timeline_and_explorer_lengths(tmp_path):
    """The pool-written activity timeline (PoolConfig.timeline_path) and explorer_lengths on an
    n > 64 explorer pool: reference CSV rows, work tracked while active, all idle at the end."""
    import csv

    inst = pbb.taillard_named("ta081")
    path = tmp_path / "tl_big.csv"
    K = 512
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=K, rounds_per_sync=1, timeline_path=str(path))) as pool:
        pool.set_initial_bound(6070)
        pool.assign_split()
        pool.run_round()
        lens = pool.explorer_lengths()
        assert len(lens) == K and max(lens) > 0
        while pool.run_round():
            pass
        pool.flush_timeline()
        assert max(pool.explorer_lengths()) == -3.0   # every explorer idle
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["timestamp_ms", "explorer_id", "active", "interval_length_log2"]
    body = rows[1:]
    assert len(body) >= 2 * K and len(body) % K == 0
    assert all(r[2] == "0" and r[3] == "-1" for r in body[-K:])
    assert any(r[2] == "1" and int(r[3]) > 0 for r in body[:-K])


def test_large_n_promote_and_offer_schedule():
    """promote_solutions on an n > 64 explorer pool: valid complete schedules (the explorers'
    paths completed in the incumbent's order), sorted by makespan; offers are taken."""
    inst = pbb.taillard_named("ta081")
    start = pbb.neh(inst)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=512), bound="lb1") as pool:
        pool.set_initial_bound(start.cmax, start.perm)
        pool.assign_split()
        pool.run_round()
        proms = pool.promote_solutions(5)
        assert 0 < len(proms) <= 5
        assert [p.cmax for p in proms] == sorted(p.cmax for p in proms)
        for p in proms:
            assert sorted(p.perm) == list(range(inst.n)) and pbb.makespan(inst, p.perm) == p.cmax
        better = pbb.insertion_local_search(inst, start, max_iterations=200, rng_seed=1)
        if better.cmax < start.cmax:
            assert pool.offer_schedule(better)
            pool.run_round()
            assert pool.best_value() <= better.cmax


def test_large_n_explorer_pool_finds_optimum_and_partitions():
    """An improving run from NEH on ta061 (100 x 5) proves the optimum 5493 with a verified
    schedule; a user partition of [0, n!) gives the same fixed-tree count."""
    inst = pbb.taillard_named("ta061")
    res = pbb.pool_run(inst, pbb.neh(inst).cmax, cfg=pbb.PoolConfig(explorers=1024))
    assert res.best_value == 5493 and pbb.makespan(inst, res.best.perm) == 5493
    nf = math.factorial(100)
    cuts = [0, nf // 7, nf // 3, nf // 2 + 12345, nf]
    res2 = pbb.pool_run(inst, 5493, intervals=list(zip(cuts[:-1], cuts[1:])), cfg=pbb.PoolConfig(explorers=1024))
    assert res2.stats.unique == golden_io.ref_counts()["ta061@5493"]["decomposed"]
