"""Short run for ncu: one ta111 decompose_batch launch per bound at a fixed free-job count
(development tool): python tools/profile_big.py lb1|lb2 f count"""
import sys

sys.path.insert(0, ".")
import numpy as np
import paper_2012_09511_b200 as pbb

bound, f, cnt = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = pbb.taillard_named("ta111")
n = inst.n
rng = np.random.default_rng(1)
perms = rng.random((cnt, n)).argsort(axis=1).astype(np.int32)
d1 = rng.integers(0, n - f + 1, cnt)
with pbb.GpuPool(inst, bound=bound) as pool:
    pool.decompose_batch(perms, d1, n - f - d1, 26670)
    print(pool.stats().batch_kernel_ms)
