"""ta111 (500x20) bounding-throughput sweep: batched decompose of sampled nodes by free-job count."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_09511_b200 as pbb

def w1(f, n, m): return (2*m-1)*(n-f) + 13*m*f + 9*f
def w2(f, n, m):
    P = m*(m-1)//2
    return (2*m-1)*(n-f) + 2*f*(2*m-1) + 8*P*f*f + 9*f

name = sys.argv[1] if len(sys.argv) > 1 else "ta111"
inst = pbb.taillard_named(name)
n, m = inst.n, inst.m
rng = np.random.default_rng(1)
peak = pbb.int32_peak()
for bound in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("lb1", "lb2")):
    with pbb.GpuPool(inst, bound=bound) as pool:
        for f in ((10, 50, 100, 200, 300, 400, 499) if n >= 500 else (10, 50, n - 1)):
            cnt = 32768 if bound == "lb1" else (2048 if f <= 100 else 1024)
            perms = rng.random((cnt, n)).argsort(axis=1).astype(np.int32)
            d1 = rng.integers(0, n - f + 1, cnt)
            d2 = n - f - d1
            pool.decompose_batch(perms[:64], d1[:64], d2[:64], 26670)
            s0 = pool.stats().batch_kernel_ms
            pool.decompose_batch(perms, d1, d2, 26670)
            ms = pool.stats().batch_kernel_ms - s0
            W = (w1 if bound == "lb1" else w2)(f, n, m)
            rate = cnt / (ms / 1e3)
            print(json.dumps({"inst": name, "bound": bound, "f": f, "nodes": cnt, "kernel_ms": round(ms, 3),
                              "nodes_per_s": round(rate), "alg_Tops": round(rate * W / 1e12, 3),
                              "frac_of_int32_peak": round(rate * W / peak, 3)}), flush=True)
