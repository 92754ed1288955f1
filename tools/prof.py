"""Profiling / measurement driver (development tool; not product code).

  python tools/prof.py explore INST BOUND UB ROUNDS     pool rounds from the equal split (ncu target)
  python tools/prof.py rate INST UB BOUND SECONDS [k=v,...]  time-bounded exploration rate
  python tools/prof.py sweep INST [lb1,lb2]            large-n bounding sweep by free-job count
  python tools/prof.py summary REPORT.ncu-rep          key metrics of an ncu --set full capture
  python tools/prof.py src REPORT.ncu-rep [TOP]        per-source-line stall samples / instructions
  python tools/prof.py launches LAUNCHES.csv "CMD"     per-kernel shares of an ncu launch list
"""
import csv
import io
import json
import re
import subprocess
import sys
import time
from collections import OrderedDict

sys.path.insert(0, ".")

SUMMARY_KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def w1(f, n, m):
    return (2 * m - 1) * (n - f) + 13 * m * f + 9 * f


def w2(f, n, m):
    P = m * (m - 1) // 2
    return (2 * m - 1) * (n - f) + 2 * f * (2 * m - 1) + 8 * P * f * f + 9 * f


def cmd_explore(inst_name, bound, ub, rounds):
    """One explore launch per round (rounds_per_sync = 1); prints the raw decomposed nodes of
    every round, so an ncu capture of explore launch s + 1 (-s s -c 1) can be divided by its
    round's node count (profiles/ncu_summary.json: thread instructions per decomposed node)."""
    import paper_2012_09511_b200 as pbb
    inst = pbb.taillard_named(inst_name)
    with pbb.GpuPool(inst, pbb.PoolConfig(rounds_per_sync=1), bound=bound) as pool:
        pool.set_initial_bound(int(ub))
        pool.assign_split()
        per_round, last = [], 0
        for _ in range(int(rounds)):
            act = pool.run_round()
            d = pool.stats().decomposed
            per_round.append(d - last)
            last = d
            if act == 0:
                break
        print(json.dumps({"raw_decomposed_per_round": per_round}))
        print(pool.stats())


def cmd_rate(name, ub, bound, secs, kv=""):
    import paper_2012_09511_b200 as pbb
    from paper_2012_09511_b200.multi import solve_distributed
    kw = dict(x.split("=") for x in kv.split(",")) if kv else {}
    cfg = pbb.PoolConfig(**{k: (float(v) if "." in v else int(v)) for k, v in kw.items()})
    with pbb.GpuPool(pbb.taillard_named(name), cfg, bound=bound) as pool:
        t = time.time()
        r = solve_distributed(pool, int(ub), time_limit_s=float(secs))
        dt = time.time() - t
        print(json.dumps({"inst": name, "bound": bound, "ub": int(ub), "cfg": kw, "K": pool.K(), "unique": r.unique,
                          "s": round(dt, 3), "Mnodes_s": round(r.unique / dt / 1e6, 2), "completed": r.completed}))


def cmd_sweep(name, bounds="lb1,lb2"):
    import numpy as np
    import paper_2012_09511_b200 as pbb
    inst = pbb.taillard_named(name)
    n, m = inst.n, inst.m
    rng = np.random.default_rng(1)
    peak = pbb.int32_peak()
    for bound in bounds.split(","):
        with pbb.GpuPool(inst, bound=bound) as pool:
            for f in ((10, 50, 100, 200, 300, 400, 499) if n >= 500 else (10, 50, n - 1)):
                cnt = 32768 if bound == "lb1" else (8192 if f <= 128 else 1024)
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


def cmd_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        for k in SUMMARY_KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:85s} {v[i]:>24s} {units[i]}")
        print()


def cmd_src(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, fname, hdr = [], "", None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name" or r[2] != "-":
            continue
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        try:
            thr = int(r[hdr.index("Thread Instructions Executed")])
        except (ValueError, IndexError):
            thr = 0
        res.append((samp, inst, thr, fname, r[0], r[1].strip()[:100]))
    tot = sum(x[0] for x in res) or 1
    toti = sum(x[1] for x in res) or 1
    res.sort(reverse=True)
    # stall share, instruction share, active threads per executed instruction, line
    for samp, inst, thr, f, ln, src in res[:int(top)]:
        print(f"{100 * samp / tot:5.1f}% {100 * inst / toti:5.1f}%i {thr / inst if inst else 0:4.1f}t {f}:{ln:5s} {src}")


def cmd_launches(path, command="?"):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(pbbgpu::\w+\)|\(.*\)$", "", r["Kernel Name"])[:60]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values()) or 1.0
    print("# ncu launch list (gpu__time_duration.sum, --clock-control none)")
    print(f"# command: {command}")
    print("# cold-cache, serialised replays: compare SHARES, not absolute times")
    print(f"{'kernel':60s} {'launches':>9s} {'mean_us':>10s} {'total_ms':>10s} {'share':>7s}")
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:60s} {cnt:9d} {us / cnt:10.1f} {us / 1e3:10.2f} {100 * us / tot:6.1f}%")


if __name__ == "__main__":
    cmds = {"explore": cmd_explore, "rate": cmd_rate, "sweep": cmd_sweep, "summary": cmd_summary, "src": cmd_src,
            "launches": cmd_launches}
    if len(sys.argv) < 2 or sys.argv[1] not in cmds:
        print(__doc__)
        sys.exit(2)
    cmds[sys.argv[1]](*sys.argv[2:])
