"""Development tool: summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launch_summary.py launches.csv "command line" > profiles/rNN_ncu_launches.txt"""
import csv
import io
import re
import sys
from collections import OrderedDict

txt = open(sys.argv[1]).read()
i = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[i:])))
agg = OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    name = re.sub(r"\(pbbgpu::ExploreParams\)|\(.*\)$", "", name)
    name = name.replace("(int)", "").replace("(bool)", "")[:60]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r["Metric Unit"], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v * scale
tot = sum(a[1] for a in agg.values()) or 1.0
print("# ncu launch list (gpu__time_duration.sum, --clock-control none)")
print(f"# command: {sys.argv[2] if len(sys.argv) > 2 else '?'}")
print("# cold-cache, serialised replays: compare SHARES, not absolute times")
print(f"{'kernel':60s} {'launches':>9s} {'mean_us':>10s} {'total_ms':>10s} {'share':>7s}")
for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:60s} {cnt:9d} {us / cnt:10.1f} {us / 1e3:10.2f} {100 * us / tot:6.1f}%")
