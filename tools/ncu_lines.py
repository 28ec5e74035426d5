"""Per-source-line hotspots of an ncu report (needs -lineinfo and
--import-source on): warp-stall samples and executed instructions per CUDA
source line, top N.  usage: python tools/ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = ""
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    try:
        samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((samples, inst, f"{fname}:{r[0]}", r[1][:90]))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {loc:28s} {src}")

if len(sys.argv) > 3:
    # aggregate by file
    agg = {}
    for s_, i_, loc, _ in rows:
        f = loc.split(":")[0]
        a_ = agg.setdefault(f, [0, 0])
        a_[0] += s_
        a_[1] += i_
    print("by file:")
    for f, (s_, i_) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {f:28s} samp {100*s_/tot_s:5.1f}%  inst {100*i_/tot_i:5.1f}%")
    ranges = [tuple(map(int, r.split("-"))) for r in sys.argv[3].split(",")]
    print("by line range of the kernel file:")
    for lo, hi in ranges:
        s_ = sum(x[0] for x in rows if x[2].startswith("tc_step_kernel") and lo <= int(x[2].split(":")[1]) <= hi)
        i_ = sum(x[1] for x in rows if x[2].startswith("tc_step_kernel") and lo <= int(x[2].split(":")[1]) <= hi)
        print(f"  {lo}-{hi}: samp {100*s_/tot_s:5.1f}%  inst {100*i_/tot_i:5.1f}%")
