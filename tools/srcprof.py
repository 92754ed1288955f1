"""Development tool: per-source-line warp stall samples / instructions from an ncu report.
usage: python tools/srcprof.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[2] != "-":  # sass rows
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    res.append((samp, inst, fname, r[0], r[1].strip()[:110]))
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
res.sort(reverse=True)
for samp, inst, f, ln, src in res[:top]:
    print(f"{100 * samp / tot:5.1f}% {100 * inst / toti:5.1f}%i {f}:{ln:5s} {src}")
