import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2012_09511_b200 as pbb
from oracle import oracle as orc
inst = pbb.taillard_named("ta111")
prob = orc.Problem(inst.p, orc.LB2)
rng = np.random.default_rng(23)
with pbb.GpuPool(inst, bound="lb2") as pool:
    for f in (1, 2, 3, 5, 17):
        perm = rng.permutation(inst.n)
        for d1 in (0, 3, inst.n - f):
            d2 = inst.n - f - d1
            lb, dr, pr, lf, lbw = pool.decompose_batch(perm[None, :], [d1], [d2], 26670)
            fw, bw = prob.children_bounds(perm, d1, d2)
            g = [int(x) for x in lf[0, :f]], [int(x) for x in lbw[0, :f]]
            print(f, d1, d2, "OK" if (g[0] == fw and g[1] == bw) else "BAD", g, (fw, bw), flush=True)
