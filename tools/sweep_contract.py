"""Sweep the standalone warp-per-cell contraction's ring depth (env var
VPINN_CW_STAGES) on the C5 gear workload; prints ms/launch and GB/s."""
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
for stages in [2, 3, 4]:
    env = dict(os.environ, VPINN_CW_STAGES=str(stages))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    out = r.stdout.strip().split()
    print(json.dumps({"stages": stages, "ms": float(out[0]) if out else None,
                      "GBs": float(out[1]) if out else None,
                      "err": r.stderr.strip()[-300:] if r.returncode else ""}), flush=True)
