"""Weak (bench gear) and strong epoch times: L2-flushed single epochs and
warm back-to-back epochs (graph replay).  usage: python tools/quick_epoch.py"""
import copy
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
out = {}
for form in ("weak", "strong"):
    cfg = copy.deepcopy(bench.GEAR_CFG)
    cfg["discretization"]["form"] = form
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
    warm = g.time_steps(100, 1e-3) / 100
    rep = g.train(60, lr0=1e-3)
    out[form] = {"flushed_ms": round(float(np.median(fl)), 4), "warm_ms": round(warm, 4),
                 "train_median_ms": round(1e3 * float(np.median(rep.records["seconds"][10:])), 4)}
    g.close()
print(json.dumps(out))
