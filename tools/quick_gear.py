"""C5 gear epoch times for the headline network and the paper's
[2,50,50,50,1] variant: L2-flushed single epochs (median), the step kernel's
share, kernel name.  usage: python tools/quick_gear.py [which ...] (c5, paper, inverse)"""
import copy
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
which = sys.argv[1:] or ["c5", "paper"]
out = {}
for w in which:
    cfg = copy.deepcopy(bench.GEAR_CFG)
    if w == "paper":
        cfg["discretization"]["n_test_per_dim"] = 4
        cfg["problem"]["n_boundary_points"] = 6096
        cfg["network"]["layers"] = [2, 50, 50, 50, 1]
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
    out[w] = {"flushed_ms": round(float(np.median(fl)), 4), "step_kernel_ms": round(k, 4),
              "reduce_ms": round(r, 4), "adam_ms": round(a, 4), "kernel": g.step_kernel()}
    g.close()
print(json.dumps(out))
