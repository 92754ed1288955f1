"""Development tool: host-side cost of pool create / solve / close (e2e breakdown)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200.multi import solve_distributed

name, ub, bound = sys.argv[1], int(sys.argv[2]), sys.argv[3]
inst = pbb.taillard_named(name)
for i in range(4):
    t0 = time.perf_counter()
    p = pbb.GpuPool(pbb.Instance(inst.n, inst.m, inst.p.copy()), None, bound=bound)
    t1 = time.perf_counter()
    r = solve_distributed(p, ub)
    t2 = time.perf_counter()
    st = p.stats()
    t3 = time.perf_counter()
    p.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms  stats {1e3*(t3-t2):.1f} ms  close {1e3*(t4-t3):.1f} ms", flush=True)
