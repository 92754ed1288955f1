"""ctypes wrapper of oracle/liboracle.so — the CPU checker (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
Also locates the compiled reference (oracle/_ref/ref_driver) when it has been built.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
CLI = os.path.join(HERE, "pfsp_oracle")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

LB1, LB2 = 1, 2


class _Problem(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int), ("m", ctypes.c_int), ("p", ctypes.c_void_p), ("bound", ctypes.c_int),
        ("npairs", ctypes.c_int), ("pk", ctypes.c_void_p), ("pl", ctypes.c_void_p),
        ("order", ctypes.c_void_p), ("lag", ctypes.c_void_p),
    ]


class _Stats(ctypes.Structure):
    _fields_ = [
        ("decomposed", ctypes.c_uint64), ("unique", ctypes.c_uint64), ("leaves", ctypes.c_uint64),
        ("improvements", ctypes.c_uint64), ("best", ctypes.c_int64), ("best_perm", ctypes.c_int32 * 512),
        ("has_perm", ctypes.c_int), ("wall_s", ctypes.c_double), ("completed", ctypes.c_int),
        ("hist", ctypes.c_uint64 * 513),
    ]


_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE, "liboracle.so", "pfsp_oracle"], check=True, capture_output=True)
        _lib = ctypes.CDLL(LIB)
        _lib.or_problem_init.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int32), ctypes.c_int]
        _lib.or_problem_free.argtypes = [ctypes.POINTER(_Problem)]
        _lib.or_decompose.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_uint8)]
        _lib.or_children_bounds.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                            ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(ctypes.c_int64)]
        _lib.or_children_bounds_lb2_exact.argtypes = _lib.or_children_bounds.argtypes
        _lib.or_lb1_node.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int]
        _lib.or_lb1_node.restype = ctypes.c_int64
        _lib.or_taillard_named.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int32)]
        _lib.or_taillard.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
        _lib.or_makespan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int)]
        _lib.or_makespan.restype = ctypes.c_int64
        _lib.or_neh.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int)]
        _lib.or_neh.restype = ctypes.c_int64
        _lib.or_fact_midpoint.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_int)]
        _lib.or_solve.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_double, ctypes.POINTER(_Stats)]
    return _lib


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def taillard_named(name: str) -> np.ndarray:
    lib = load()
    p = np.zeros(500 * 20, dtype=np.int32)
    n, m = ctypes.c_int(), ctypes.c_int()
    if lib.or_taillard_named(name.encode(), ctypes.byref(n), ctypes.byref(m), p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))):
        raise ValueError(name)
    return p[: n.value * m.value].reshape(n.value, m.value).copy()


def generate_taillard(n: int, m: int, seed: int) -> np.ndarray:
    p = np.zeros(n * m, dtype=np.int32)
    if load().or_taillard(n, m, seed, p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))):
        raise ValueError("bad generator arguments")
    return p.reshape(n, m)


def makespan(p: np.ndarray, perm: Sequence[int]) -> int:
    p = np.ascontiguousarray(p, dtype=np.int32)
    pr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    return int(load().or_makespan(p.shape[0], p.shape[1], p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _ip(pr)))


def neh(p: np.ndarray) -> Tuple[int, List[int]]:
    p = np.ascontiguousarray(p, dtype=np.int32)
    out = np.zeros(p.shape[0], dtype=np.int32)
    v = load().or_neh(p.shape[0], p.shape[1], p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _ip(out))
    return int(v), [int(x) for x in out]


def midpoint(a: Sequence[int], b: Optional[Sequence[int]]) -> List[int]:
    n = len(a)
    aa = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    out = np.zeros(n, dtype=np.int32)
    if b is None:
        rc = load().or_fact_midpoint(n, _ip(aa), None, _ip(out))
    else:
        bb = np.ascontiguousarray(np.asarray(b, dtype=np.int32))
        rc = load().or_fact_midpoint(n, _ip(aa), _ip(bb), _ip(out))
    if rc:
        raise ValueError("midpoint requires a < b")
    return [int(x) for x in out]


class Problem:
    """Bounding data of one instance (LB1 or LB2)."""

    def __init__(self, p: np.ndarray, bound: int = LB1):
        self.p = np.ascontiguousarray(p, dtype=np.int32)
        self.n, self.m = self.p.shape
        self._pr = _Problem()
        if load().or_problem_init(ctypes.byref(self._pr), self.n, self.m,
                                  self.p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), bound):
            raise ValueError("bad problem")

    def __del__(self):
        try:
            load().or_problem_free(ctypes.byref(self._pr))
        except Exception:
            pass

    def decompose(self, perm, d1, d2, incumbent) -> Tuple[int, List[int], List[int]]:
        f = self.n - d1 - d2
        pr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
        lb = np.zeros(max(f, 1), dtype=np.int64)
        pruned = np.zeros(max(f, 1), dtype=np.uint8)
        d = ctypes.c_int()
        rc = load().or_decompose(ctypes.byref(self._pr), _ip(pr), d1, d2, incumbent,
                                 lb.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(d),
                                 pruned.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
        if rc:
            raise ValueError("decompose: no free jobs or bad incumbent")
        return d.value, [int(x) for x in lb[:f]], [int(x) for x in pruned[:f]]

    def children_bounds(self, perm, d1, d2) -> Tuple[List[int], List[int]]:
        f = self.n - d1 - d2
        pr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
        fw = np.zeros(f, dtype=np.int64)
        bw = np.zeros(f, dtype=np.int64)
        if load().or_children_bounds(ctypes.byref(self._pr), _ip(pr), d1, d2,
                                     fw.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                     bw.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))):
            raise ValueError("children_bounds: no free jobs")
        return [int(x) for x in fw], [int(x) for x in bw]

    def children_bounds_lb2_exact(self, perm, d1, d2) -> Tuple[List[int], List[int]]:
        """LB2 child bounds from the definition: per machine pair the optimum over ALL orders of
        the free jobs of the two-machine time-lag relaxation (subset DP; f <= 16)."""
        f = self.n - d1 - d2
        pr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
        fw = np.zeros(f, dtype=np.int64)
        bw = np.zeros(f, dtype=np.int64)
        if load().or_children_bounds_lb2_exact(ctypes.byref(self._pr), _ip(pr), d1, d2,
                                               fw.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                               bw.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))):
            raise ValueError("children_bounds_lb2_exact: needs 1 <= f <= 16 and m >= 2")
        return [int(x) for x in fw], [int(x) for x in bw]

    def lb1(self, perm, d1, d2) -> int:
        pr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
        return int(load().or_lb1_node(ctypes.byref(self._pr), _ip(pr), d1, d2))

    def solve(self, ub: int, threads: int = 1, prefix_depth: int = 0, pinned: bool = False,
              disable_pruning: bool = False, time_limit_s: float = 0.0) -> Dict:
        st = _Stats()
        if load().or_solve(ctypes.byref(self._pr), ub, threads, prefix_depth, int(pinned), int(disable_pruning),
                           time_limit_s, ctypes.byref(st)):
            raise ValueError("or_solve failed")
        return {
            "decomposed": st.decomposed, "unique": st.unique, "leaves": st.leaves,
            "improvements": st.improvements, "best": st.best,
            "best_perm": [int(st.best_perm[i]) for i in range(self.n)] if st.has_perm else [],
            "wall_s": st.wall_s, "completed": bool(st.completed),
            "hist": {f: int(st.hist[f]) for f in range(self.n + 1) if st.hist[f]},
        }


def ref_available() -> bool:
    return os.path.exists(REF_DRIVER)


def ref_run(*args: str, timeout: float = 600) -> Dict:
    """Run the compiled reference driver (oracle/_ref/ref_driver) and parse its JSON."""
    out = subprocess.run([REF_DRIVER, *map(str, args)], check=True, capture_output=True, text=True, timeout=timeout)
    return json.loads(out.stdout.strip().splitlines()[-1])
