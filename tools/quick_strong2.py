"""Strong-form gear epoch (L2-flushed), kernel time and name.  usage: python tools/quick_strong2.py"""
import copy
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
cfg = copy.deepcopy(bench.GEAR_CFG)
cfg["discretization"]["form"] = "strong"
hp = host.HostProblem(cfg, mesh=mesh)
g = G.GpuStep.from_problem(hp.view(0), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(5, 1e-3)
g.synchronize()
fl = []
for _ in range(20):
    g.flush_l2()
    fl.append(g.time_steps(1, 1e-3))
k, r, a = g.profile_step(10)
print(json.dumps({"strong_flushed_ms": round(float(np.median(fl)), 4), "kernel_ms": round(k, 4),
                  "kernel": g.step_kernel()}))
