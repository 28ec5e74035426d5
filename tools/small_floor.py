"""Small-problem epoch floor (C2 sweep end): per-kernel times for 1..64 cells."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

cfg = {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 400},
       "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
       "network": {"layers": [2, 30, 30, 30, 1]},
       "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
for e in (1, 8, 32):
    hp = host.HostProblem(cfg, mesh=host.Mesh.structured(e, e))
    g = G.GpuStep.from_problem(hp.view(0), keepalive=hp)
    g.set_params(hp.init_params())
    g.adam_reset()
    g.run_steps(10, 1e-3)
    g.synchronize()
    k, r, a = g.profile_step(20)
    warm = g.time_steps(200, 1e-3) / 200
    rep = g.train(60, lr0=1e-3)
    print(json.dumps({"cells": e * e, "kernel": g.step_kernel()[:40], "step_ms": round(k, 4), "reduce_ms": round(r, 4),
                      "adam_ms": round(a, 4), "graph_epoch_ms": round(warm, 4),
                      "train_median_ms": round(1e3 * float(np.median(rep.records["seconds"][10:])), 4)}))
    g.close()
