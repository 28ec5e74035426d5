"""Executed warp instructions per SASS opcode of an ncu report (needs
--import-source / source page): python tools/ncu_opcodes.py REPORT [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
agg = collections.Counter()
tot = 0
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    src = d.get("Source", "").split()
    try:
        n = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    agg[op] += n
    tot += n
print(f"total warp instructions {tot}")
for k, v in agg.most_common(top):
    print(f"{k:12s} {v:12d} {100 * v / tot:5.1f}%")
