"""Executed warp instructions of an ncu source page (cuda,sass CSV) attributed
to call sites of one kernel file: every SASS instruction is charged to the
last line of KERNEL_FILE seen at or before its address (inlined helpers from
other headers land on the line that called them).  Prints per-line totals and
the opcode mix of the top lines.
usage: python tools/ncu_callsite.py SRC.csv KERNEL_FILE [N] [lo-hi,lo-hi,...]
(SRC.csv from: ncu -i REP --page source --csv --print-source=cuda,sass)"""
import collections
import csv
import sys

path, kfile = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ranges = sys.argv[4] if len(sys.argv) > 4 else ""
ins = []  # (addr, file, line, n, op)
fname, line, hdr = "", None, None
with open(path, newline="") as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0] != "":
            line = int(r[0])
            continue
        if not r[2].startswith("0x"):
            continue
        try:
            n = int(r[7])
        except ValueError:
            continue
        src = r[3].split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "?")).split(".")[0]
        ins.append((int(r[2], 16), fname, line, n, op))
ins.sort()
cur = 0
per = collections.Counter()
ops = collections.defaultdict(collections.Counter)
tot = 0
for a, fn, ln, n, op in ins:
    if fn == kfile:
        cur = ln
    per[cur] += n
    ops[cur][op] += n
    tot += n
print(f"total warp instructions {tot}")
for ln, n in per.most_common(top):
    mix = ", ".join(f"{o} {100 * c / n:.0f}%" for o, c in ops[ln].most_common(5))
    print(f"{kfile}:{ln:<5d} {100 * n / tot:5.1f}%  {n:11d}  {mix}")
if ranges:
    print("by line range:")
    for rg in ranges.split(","):
        lo, hi = map(int, rg.split("-"))
        n = sum(v for k, v in per.items() if lo <= k <= hi)
        c = collections.Counter()
        for k in per:
            if lo <= k <= hi:
                c.update(ops[k])
        mix = ", ".join(f"{o} {100 * v / max(n, 1):.0f}%" for o, v in c.most_common(6))
        print(f"  {lo:5d}-{hi:<5d} {100 * n / tot:5.1f}%  {n:11d}  {mix}")
