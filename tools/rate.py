"""Time-bounded exploration rate (development tool): python tools/rate.py ta056 3679 lb2 5 [cfg]"""
import json, sys, time
sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200.multi import solve_distributed
name, ub, bound, secs = sys.argv[1], int(sys.argv[2]), sys.argv[3], float(sys.argv[4])
kw = dict(kv.split("=") for kv in sys.argv[5].split(",")) if len(sys.argv) > 5 else {}
cfg = pbb.PoolConfig(**{k: (float(v) if '.' in v else int(v)) for k, v in kw.items()})
with pbb.GpuPool(pbb.taillard_named(name), cfg, bound=bound) as pool:
    t = time.time()
    r = solve_distributed(pool, ub, time_limit_s=secs)
    dt = time.time() - t
    print(json.dumps({"inst": name, "bound": bound, "ub": ub, "cfg": kw, "K": pool.K(), "unique": r.unique,
                      "s": round(dt, 3), "Mnodes_s": round(r.unique / dt / 1e6, 2), "completed": r.completed}))
