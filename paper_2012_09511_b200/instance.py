"""PFSP instances (host side), mirroring include/pbb/instance.hpp.

All arithmetic runs in the C++ host code of libpbbgpu.so (src: csrc/pool.cu):
  generate_taillard / taillard_named   <- src/instance.cpp:80-163
  makespan                             <- src/instance.cpp:165-183
  neh                                  <- src/heuristic.cpp:73-103
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib


@dataclass
class Instance:
    n: int
    m: int
    p: np.ndarray  # int32 [n, m], p[j, k] = time of job j on machine k (job-major)
    label: str = ""

    def __post_init__(self):
        self.p = np.ascontiguousarray(np.asarray(self.p, dtype=np.int32).reshape(self.n, self.m))
        if self.n < 1 or self.m < 1:
            raise ValueError("instance needs n >= 1 and m >= 1")
        if (self.p < 0).any():
            raise ValueError("negative processing time")

    def pt(self, j: int, k: int) -> int:
        return int(self.p[j, k])

    def ptr(self):
        return self.p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


@dataclass
class Schedule:
    perm: List[int] = field(default_factory=list)
    cmax: int = -1

    def evaluated(self) -> bool:
        return self.cmax >= 0


def generate_taillard(n: int, m: int, seed: int) -> Instance:
    p = np.zeros((n, m), dtype=np.int32)
    _lib.check(_lib.load().pbbgpu_taillard(n, m, seed, p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return Instance(n, m, p, f"tai-{n}x{m}-{seed}")


def taillard_named(name: str) -> Instance:
    lib = _lib.load()
    n = ctypes.c_int()
    m = ctypes.c_int()
    _lib.check(lib.pbbgpu_taillard_named(name.encode(), ctypes.byref(n), ctypes.byref(m), None))
    p = np.zeros((n.value, m.value), dtype=np.int32)
    _lib.check(lib.pbbgpu_taillard_named(name.encode(), ctypes.byref(n), ctypes.byref(m),
                                         p.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return Instance(n.value, m.value, p, f"ta{int(name[2:]):03d}")


def parse_instance(text: str, machine_major: bool = False, label: str = "") -> Instance:
    """Plain-text format: "n m" then the matrix by job rows (or machine rows)."""
    toks = text.split()
    if len(toks) < 2:
        raise ValueError("instance header must hold n and m")
    n, m = int(toks[0]), int(toks[1])
    vals = [int(t) for t in toks[2:]]
    if len(vals) != n * m:
        raise ValueError(f"instance matrix has {len(vals)} entries, expected {n * m}")
    a = np.array(vals, dtype=np.int32)
    p = a.reshape(m, n).T if machine_major else a.reshape(n, m)
    return Instance(n, m, p, label)


def makespan(inst: Instance, perm: Sequence[int]) -> int:
    arr = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    if arr.size != inst.n:
        raise ValueError("schedule length does not match instance")
    v = _lib.load().pbbgpu_makespan(inst.n, inst.m, inst.ptr(), arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if v < 0:
        _lib.check(_lib.PBBGPU_ERR_ARG)
    return int(v)


def neh(inst: Instance) -> Schedule:
    out = np.zeros(inst.n, dtype=np.int32)
    v = _lib.load().pbbgpu_neh(inst.n, inst.m, inst.ptr(), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return Schedule([int(x) for x in out], int(v))


def insertion_local_search(inst: Instance, seed: Schedule, max_iterations: int = 0, max_seconds: float = 0.0,
                           rng_seed: int = 0) -> Schedule:
    """insertion_local_search (src/heuristic.cpp:105-155): first-improvement remove-and-reinsert
    descent, ties among equally good positions broken by a seeded mt19937_64."""
    sp = np.ascontiguousarray(np.asarray(seed.perm, dtype=np.int32))
    out = np.zeros(inst.n, dtype=np.int32)
    v = _lib.load().pbbgpu_insertion_ls(inst.n, inst.m, inst.ptr(), sp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                        int(max_iterations), float(max_seconds), int(rng_seed),
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if v < 0:
        _lib.check(_lib.PBBGPU_ERR_ARG)
    return Schedule([int(x) for x in out], int(v))
