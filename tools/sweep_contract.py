"""Sweep the standalone warp-per-cell contraction's warps per CTA and ring
depth (VPINN_CW_WARPS, VPINN_CW_STAGES) on the C5 gear workload; prints
ms/launch and GB/s (configurations that do not fit fall back to the
row-chunked kernel)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys; sys.path.insert(0, %r)
import bench
from paper_2404_12063_b200 import gpu as G
hp, _ = bench.build_problem()
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
ms, b = g.time_contract(50)
print(ms, b / (ms * 1e-3) / 1e9)
''' % ROOT
import itertools
for warps, stages in itertools.product([8, 12, 16], [2, 3]):
    env = dict(os.environ, VPINN_CW_STAGES=str(stages), VPINN_CW_WARPS=str(warps))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    out = r.stdout.strip().split()
    print(json.dumps({"warps": warps, "stages": stages, "ms": float(out[0]) if out else None,
                      "GBs": float(out[1]) if out else None,
                      "err": r.stderr.strip()[-300:] if r.returncode else ""}), flush=True)
