"""Config sweep (development tool): time-to-proof for a few pool configurations."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb

name, ub, bound = sys.argv[1], int(sys.argv[2]), sys.argv[3]
import os
REPS = int(os.environ.get("REPS", "1"))
inst = pbb.taillard_named(name)
for spec in sys.argv[4:]:
    kw = dict(kv.split("=") for kv in spec.split(",")) if spec != "default" else {}
    cfg = pbb.PoolConfig(**{k: (float(v) if '.' in v else int(v)) for k, v in kw.items()})
    with pbb.GpuPool(inst, cfg, bound=bound) as pool:
        from paper_2012_09511_b200.multi import solve_distributed
        solve_distributed(pool, ub)  # warm
        for rep in range(REPS):
            s0 = pool.stats()
            t0 = time.time()
            r = solve_distributed(pool, ub)
            dt = time.time() - t0
            st = pool.stats()
            print(json.dumps({"cfg": spec, "K": st.K, "G": st.group, "unique": r.unique, "s": round(dt, 4),
                              "Mnodes_s": round(r.unique / dt / 1e6, 2), "rounds": r.rounds,
                              "steals": r.local_steals, "kernel_ms": round(st.kernel_ms - s0.kernel_ms, 1),
                              "steal_ms": round(st.steal_kernel_ms - s0.steal_kernel_ms, 1)}), flush=True)
