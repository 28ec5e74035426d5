"""Quick iteration timer: C5 gear fused step kernel (warm and L2-flushed),
reduce/adam, the standalone contraction, and the tc-vs-ffma kernel names.
usage: python tools/quick_step.py [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
hp, _ = bench.build_problem()
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(5, 1e-3)
g.synchronize()
ms_mlp, ms_red, ms_adam = g.profile_step(reps)
flushed = []
for _ in range(reps):
    g.flush_l2()
    flushed.append(g.time_steps(1, 1e-3))
ms_c, b_c = g.time_contract(reps)
print(json.dumps({"kernel": g.step_kernel(), "step_ms": ms_mlp, "reduce_ms": ms_red, "adam_ms": ms_adam,
                  "epoch_flushed_ms": float(np.median(flushed)), "contract_ms": ms_c,
                  "contract_GBs": b_c / (ms_c * 1e-3) / 1e9}))
