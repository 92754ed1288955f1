"""paper_2012_09511_b200 — B200-native PFSP Branch-and-Bound (GPU IVM explorers, LB1/LB2).

Drop-in for the reference solver's solve/explore path (ExplorerPool / pool_run / decompose,
/root/reference/proj/include/pbb/explorer.hpp, bound.hpp). Compute runs only in
libpbbgpu.so (hand-written sm_100a kernels); see DESIGN.md.
"""
from .factoradic import compare, from_decimal, midpoint, to_decimal
from .instance import (Instance, Schedule, generate_taillard, insertion_local_search, makespan, neh, parse_instance,
                       taillard_named)
from .pool import (BACKWARD, FORWARD, NO_INCUMBENT, Decomposition, GpuPool, PoolConfig, PoolResult,
                   PoolStats, Subproblem, Timeline, int32_peak, normalize, pool_run, solve_pool, wire_reencode)

from .coop import CoopResult, solve_cooperative

__all__ = [
    "solve_cooperative", "CoopResult",
    "Instance", "Schedule", "generate_taillard", "taillard_named", "makespan", "neh", "parse_instance",
    "insertion_local_search",
    "GpuPool", "PoolConfig", "PoolStats", "PoolResult", "Subproblem", "Decomposition", "pool_run", "solve_pool",
    "normalize", "int32_peak", "wire_reencode", "Timeline", "to_decimal", "from_decimal", "compare", "midpoint", "FORWARD", "BACKWARD", "NO_INCUMBENT",
]
