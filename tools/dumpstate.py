import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200 import _lib
name, ub, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = pbb.taillard_named(name)
n = inst.n
with pbb.GpuPool(inst, pbb.PoolConfig()) as pool:
    pool.set_initial_bound(ub); pool.assign_split()
    for r in range(rounds):
        a = pool.run_round()
    print("active", a, pool.stats())
    K = pool.K()
    buf = np.zeros(K * 4096, dtype=np.uint8)
    gs = ctypes.c_int(); off = (ctypes.c_int * 7)()
    _lib.check(_lib.load().pbbgpu_debug_state(pool._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), buf.size, ctypes.byref(gs), off))
    g = gs.value
    shown = 0
    for i in range(K):
        b = buf[i * g:(i + 1) * g]
        level = int(np.frombuffer(b[0:2].tobytes(), dtype=np.int16)[0]); state = b[2]; has_end = b[3]
        if state == 0:
            continue
        V = b[off[1]:off[1] + n].view(np.int8); E = b[off[3]:off[3] + n].view(np.int8); T = b[off[4]:off[4] + n].view(np.int8)
        rows = []
        for l in range(max(level, 0) + 1):
            o = off[0] + l * n - (l * (l - 1)) // 2
            rows.append(list(b[o:o + n - l].view(np.int8)))
        print(f"ivm {i} cta {i//16} state {state} level {level} d1 {b[4]} d2 {b[5]} rlev {b[6]} nrep {b[7]} has_end {has_end}")
        print("  V  ", list(V)); print("  end", list(E)); print("  tgt", list(T))
        for l, rw in enumerate(rows[:6]):
            print("  row", l, rw)
        shown += 1
        if shown > 8:
            break
