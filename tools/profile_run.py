"""Short run for ncu: ta021 LB2 (or LB1) pool rounds from the fresh split (development tool)."""
import sys

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb

bound = sys.argv[1] if len(sys.argv) > 1 else "lb2"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
inst = pbb.taillard_named("ta021")
with pbb.GpuPool(inst, pbb.PoolConfig(), bound=bound) as pool:
    pool.set_initial_bound(2297)
    pool.assign_split()
    for _ in range(rounds):
        if pool.run_round() == 0:
            break
    print(pool.stats())
