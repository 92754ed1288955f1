"""Readers for the committed golden fixtures (tests/golden/, made by make_golden.py)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def ref_counts():
    with open(os.path.join(GOLDEN, "ref_counts.json")) as f:
        return json.load(f)


def ref_instances():
    out = {}
    name = None
    rows = []
    with open(os.path.join(GOLDEN, "ref_instances.txt")) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#"):
                if name:
                    out[name] = np.array(rows[1:], dtype=np.int32)
                name = line[2:]
                rows = []
            elif line:
                rows.append([int(x) for x in line.split()])
    if name:
        out[name] = np.array(rows[1:], dtype=np.int32)
    return out


def ref_nodes(name):
    """[(perm, d1, d2, direction, child_lb, pruned)], ub"""
    nodes = []
    ub = None
    with open(os.path.join(GOLDEN, f"ref_nodes_{name}.txt")) as f:
        for line in f:
            if line.startswith("#"):
                ub = int(line.split()[-1])
                continue
            parts = [p.split() for p in line.split("|")]
            perm = [int(x) for x in parts[0]]
            d1, d2 = (int(x) for x in parts[1])
            direction = int(parts[2][0])
            lbs = [int(x) for x in parts[3]]
            pruned = [int(x) for x in parts[4]]
            nodes.append((perm, d1, d2, direction, lbs, pruned))
    return nodes, ub


def lb2_counts():
    path = os.path.join(GOLDEN, "oracle_lb2_counts.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        return json.load(f)


# the reference's own K=1 run of ta021 at UB 2297 (534.8 s on one core),
# re-run in this container by oracle/_ref/ref_driver (see oracle_ref_ta021.json when present).
TA021_LB1 = {
    "decomposed": 462443491, "leaves": 1440,
    "hist": {2: 170427, 3: 1951223, 4: 9694463, 5: 30047941, 6: 61015202, 7: 89002719, 8: 96503761,
             9: 79699847, 10: 51645290, 11: 26785285, 12: 11126615, 13: 3653785, 14: 931916, 15: 183604,
             16: 27856, 17: 3250, 18: 287, 19: 20},
}
