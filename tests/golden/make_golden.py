"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs oracle/_ref/ref_driver (the unmodified reference sources compiled by oracle/Makefile,
`make -C oracle ref`) and stores its outputs. Needs /root/reference, i.e. runs in the build
container only; the fixtures are committed so the GPU box never reads the reference.

    python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def run(*args):
    out = subprocess.run([DRIVER, *map(str, args)], check=True, capture_output=True, text=True)
    return out.stdout


def main():
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    counts = {}
    # fixed trees (UB = optimum) and improving runs, K = 1 (pool_run semantics)
    for name, ub in (("ta001", 1278), ("ta011", 1582), ("ta031", 2724), ("ta041", 2991)):
        counts[f"{name}@{ub}"] = json.loads(run("hist", name, ub))
    # machine counts the compiled kernels do not have (padded with zero-time machines), incl. a
    # VFR-like 30 x 15 instance
    for name, ub in (("gen:30:15:4242", 2490), ("gen:16:13:1234", 1512), ("gen:18:3:77", 926),
                     ("gen:14:40:2024", 3124), ("gen:12:60:606", 4417), ("gen:16:25:99", 2282)):
        counts[f"{name}@{ub}"] = json.loads(run("hist", name, ub))
    # n > 64 fixed trees (explorer pools with IVM state in HBM)
    for name, ub in (("ta061", 5493), ("ta081", 6070), ("ta101", 11150), ("ta111", 26000)):
        counts[f"{name}@{ub}"] = json.loads(run("hist", name, ub))
    for name in ("ta001", "ta041"):
        counts[f"{name}@neh"] = json.loads(run("solve", name, "neh", 1, 1))
    for name in ("ta001", "ta011", "ta021", "ta031", "ta041", "ta056", "ta111"):
        counts[f"neh:{name}"] = json.loads(run("neh", name))
    for name, iters, seed in (("ta001", 2000, 7), ("ta021", 2000, 11), ("ta041", 500, 3), ("ta056", 300, 5)):
        counts[f"ils:{name}"] = json.loads(run("ils", name, iters, seed))
    # every PoolStats field of pool_run (K explorers, batch_steps, fixed tree or pruning disabled):
    # the reference steal policy on the GPU must reproduce these exactly
    for inst, ub, K, bs, nopr in (("ta011", 1582, 16, 1024, 0), ("ta011", 1582, 64, 1024, 0),
                                  ("ta011", 1582, 48, 1024, 0), ("ta011", 1582, 256, 1024, 0),
                                  ("ta011", 1582, 20, 256, 0), ("ta001", 1278, 16, 1024, 0),
                                  ("ta001", 1278, 4, 8, 0), ("gen:8:5:4242", 100000, 16, 64, 1),
                                  ("gen:9:5:77", 100000, 64, 128, 1), ("gen:9:10:78", 100000, 12, 200, 1)):
        counts[f"stats:{inst}@{ub}:K{K}:b{bs}:np{nopr}"] = json.loads(run("stats", inst, ub, K, 4, bs, nopr, nopr))
    with open(os.path.join(HERE, "ref_counts.json"), "w") as f:
        json.dump(counts, f, indent=1, sort_keys=True)
    # per-node decompose dumps (SURVEY.md §8(d) sampler): seed 42
    for name, ub, starts, per in (("ta001", 1278, 40, 10), ("ta021", 2297, 40, 10),
                                  ("ta041", 2991, 30, 10), ("ta056", 3679, 30, 10)):
        with open(os.path.join(HERE, f"ref_nodes_{name}.txt"), "w") as f:
            f.write(run("nodes", name, ub, 42, starts, per))
    # wire frames encoded by the reference (src/protocol.cpp encode)
    with open(os.path.join(HERE, "ref_frames.txt"), "w") as f:
        f.write(run("frames"))
    # coordinator checkpoint file written by the reference (checkpoint_save)
    subprocess.run([DRIVER, "ckpt", "ta021", os.path.join(HERE, "ref_checkpoint_ta021.ckpt")], check=True)
    # instance matrices as the reference generates them
    with open(os.path.join(HERE, "ref_instances.txt"), "w") as f:
        for name in ("ta001", "ta021", "ta041", "ta056", "ta111"):
            f.write(f"# {name}\n" + run("inst", name))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    sys.exit(main())
