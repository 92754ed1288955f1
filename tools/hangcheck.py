import sys, time
sys.path.insert(0, ".")
import paper_2012_09511_b200 as pbb
name, ub = sys.argv[1], int(sys.argv[2])
kw = dict(kv.split("=") for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 else {}
cfg = pbb.PoolConfig(**{k: int(v) for k, v in kw.items()})
t = time.time()
with pbb.GpuPool(pbb.taillard_named(name), cfg) as pool:
    pool.set_initial_bound(ub)
    pool.assign_split()
    r = 0
    while True:
        a = pool.run_round()
        r += 1
        if r <= 5 or r % 50 == 0 or a == 0:
            st = pool.stats()
            print(f"round {r} active {a} unique {st.unique} raw {st.decomposed} steps {st.steps} steals {st.local_steals} t {time.time()-t:.2f}", flush=True)
        if a == 0 or time.time() - t > 15:
            break
print(name, kw, "K", pool.K() if False else "", round(time.time() - t, 3), flush=True)
