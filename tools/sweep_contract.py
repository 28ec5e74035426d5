"""Sweep the standalone contraction's chunk/ring configuration (env vars)."""
import itertools
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
ms, b = g.time_contract(20)
print(ms, b / (ms * 1e-3) / 1e9)
''' % ROOT
for ldg, cells, stages, one in itertools.product([1, 0], [5, 3, 2], [2, 3, 4], [0, 1]):
    if ldg == 0 and (stages != 2 or one):
        continue
    env = dict(os.environ, VPINN_CC_CELLS=str(cells), VPINN_CC_STAGES=str(stages), VPINN_CC_ONE_CTA=str(one),
               VPINN_CC_LDGSTS=str(ldg))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    out = r.stdout.strip().split()
    print(json.dumps({"ldgsts": ldg, "cells": cells, "stages": stages, "one_cta_budget": one,
                      "ms": float(out[0]) if out else None, "GBs": float(out[1]) if out else None,
                      "err": r.stderr.strip()[-200:] if r.returncode else ""}), flush=True)
