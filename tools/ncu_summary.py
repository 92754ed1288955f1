"""Build profiles/ncu_summary.json (read by bench.py for roofline.traffic / executed_ops) from
`tools/prof.py summary` outputs of explore-kernel captures and the per-round node counts of the
same command (`tools/prof.py explore <inst> <bound> <ub> 60`, launch 41 = round index 40).

  python tools/ncu_summary.py OUT.json WORKLOAD=SUMMARY.txt:ROUNDS.txt [...]
"""
import json
import sys


def metric(txt, name):
    for line in txt.splitlines():
        if line.startswith(name + " "):
            parts = line.split()
            v = float(parts[1].replace(",", ""))
            unit = parts[2] if len(parts) > 2 else ""
            return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    raise KeyError(name)


def main(out, specs):
    res = {"source": "one ncu --set full capture per workload (explore launch 41 of tools/prof.py explore <inst> "
                     "<bound> <ub> 60, one launch per round); per-node figures divide by that launch's raw decomposed "
                     "nodes (round index 40 of the same command)"}
    for spec in specs:
        wl, files = spec.split("=", 1)
        summ, rounds = files.split(":")
        txt = open(summ).read()
        nodes = json.loads(open(rounds).read().splitlines()[0])["raw_decomposed_per_round"][40]
        res[f"{wl}:explore_kernel_dram_bytes_per_launch"] = metric(txt, "dram__bytes_read.sum") + metric(txt, "dram__bytes_write.sum")
        res[f"{wl}:explore_kernel_warp_inst_per_node"] = metric(txt, "smsp__inst_executed.sum") / nodes
        # thread instructions = warp instructions x active threads per instruction
        res[f"{wl}:explore_kernel_thread_inst_per_node"] = (metric(txt, "smsp__inst_executed.sum") * metric(
            txt, "smsp__thread_inst_executed_per_inst_executed.ratio") / nodes)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
