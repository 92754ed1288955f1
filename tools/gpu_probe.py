"""Quick GPU probe: correctness anchors + first timings (development tool)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb
from oracle import oracle as orc


def run(name, ub, bound="lb1", **kw):
    inst = pbb.taillard_named(name)
    cfg = pbb.PoolConfig(**kw)
    t0 = time.time()
    r = pbb.pool_run(inst, ub, cfg=cfg, bound=bound)
    dt = time.time() - t0
    s = r.stats
    print(json.dumps({"inst": name, "bound": bound, "ub": ub, "best": r.best_value, "unique": s.unique,
                      "raw": s.decomposed, "leaves": s.leaves, "wall": round(dt, 3), "kernel_ms": round(s.kernel_ms, 1),
                      "rounds": s.rounds, "steals": s.local_steals, "K": s.K, "G": s.group,
                      "Mnodes_s": round(s.unique / max(s.wall_s, 1e-9) / 1e6, 2), "completed": s.completed}), flush=True)
    return r


def parity(name, bound, count=2000, seed=1):
    inst = pbb.taillard_named(name)
    rng = np.random.default_rng(seed)
    n = inst.n
    perms, d1s, d2s = [], [], []
    for _ in range(count):
        perm = rng.permutation(n)
        f = int(rng.integers(1, n + 1))
        d1 = int(rng.integers(0, n - f + 1))
        d2 = n - f - d1
        perms.append(perm); d1s.append(d1); d2s.append(d2)
    prob = orc.Problem(inst.p, orc.LB1 if bound == "lb1" else orc.LB2)
    with pbb.GpuPool(inst, pbb.PoolConfig(explorers=1024), bound=bound) as pool:
        lb, dr, pr, lf, lbw = pool.decompose_batch(np.array(perms), d1s, d2s, 10**9)
    bad = 0
    for i in range(count):
        f = n - d1s[i] - d2s[i]
        fw, bw = prob.children_bounds(perms[i], d1s[i], d2s[i])
        d, clb, _ = prob.decompose(perms[i], d1s[i], d2s[i], 10**9)
        if list(lf[i, :f]) != fw or list(lbw[i, :f]) != bw or int(dr[i]) != d or list(lb[i, :f]) != clb:
            bad += 1
            if bad < 3:
                print("MISMATCH", name, bound, i, d1s[i], d2s[i], list(lf[i, :f]), fw, list(lbw[i, :f]), bw)
    print(json.dumps({"parity": name, "bound": bound, "count": count, "mismatches": bad}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "basic"
    if which == "basic":
        import __graft_entry__
        __graft_entry__.smoke()
        for nm, b in (("ta001", "lb1"), ("ta021", "lb1"), ("ta041", "lb1"), ("ta056", "lb1"), ("ta021", "lb2"), ("ta056", "lb2")):
            parity(nm, b, 500 if b == "lb2" else 2000)
        run("ta001", 1278)
        run("ta011", 1582)
        run("ta041", 2991)
        run("ta041", 3135)
        run("ta011", 1582, bound="lb2")
        run("ta021", 2297, time_limit_s=60)
    elif which == "ta021":
        run("ta021", 2297)
    elif which == "lb2":
        run("ta021", 2297, bound="lb2", time_limit_s=float(sys.argv[2]) if len(sys.argv) > 2 else 60)
