"""Development tool: cost of breadth-first seeding vs equal-range assignment."""
import sys
import time

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb

name, ub, bound, world = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
inst = pbb.taillard_named(name)
with pbb.GpuPool(inst, None, bound=bound) as pool:
    K = pool.K()
    for rep in range(3):
        pool.set_initial_bound(ub)
        t0 = time.perf_counter()
        pool.seed(ub, 0, world, world * K)
        t1 = time.perf_counter()
        pool.assign_split_strided(0, world, K, world * K)
        t2 = time.perf_counter()
        print(f"{name} {bound} W={world} K={K}: seed {1e3*(t1-t0):.1f} ms, equal split {1e3*(t2-t1):.1f} ms", flush=True)
