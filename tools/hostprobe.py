"""Development tool: host-side timing breakdown of a single-rank solve (outlier hunting)."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb

name, ub, bound, reps = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
kw = dict(kv.split("=") for kv in sys.argv[5].split(",")) if len(sys.argv) > 5 else {}
cfg = pbb.PoolConfig(**{k: int(v) for k, v in kw.items()})
inst = pbb.taillard_named(name)
with pbb.GpuPool(inst, cfg, bound=bound) as pool:
    K = pool.K()
    for rep in range(reps):
        t = [time.perf_counter()]
        pool.stats(); pool.histogram()
        t.append(time.perf_counter())
        pool.set_initial_bound(ub)
        t.append(time.perf_counter())
        pool.assign_split_range(0, K, K)
        t.append(time.perf_counter())
        rt = []
        while True:
            a = time.perf_counter()
            act = pool.run_round()
            rt.append(time.perf_counter() - a)
            if act == 0:
                break
        t.append(time.perf_counter())
        pool.stats(); pool.histogram()
        t.append(time.perf_counter())
        d = [round((t[i + 1] - t[i]) * 1e3, 2) for i in range(len(t) - 1)]
        rt.sort()
        print(json.dumps({"phases_ms": d, "rounds": len(rt), "round_max_ms": round(rt[-1] * 1e3, 2),
                          "round_2nd_ms": round(rt[-2] * 1e3, 2), "round_med_ms": round(rt[len(rt) // 2] * 1e3, 2)}), flush=True)
