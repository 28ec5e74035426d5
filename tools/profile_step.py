"""Minimal driver for ncu: build the C5 gear problem and run a few epochs
(+ one standalone contraction launch) through the C-ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
hp, _ = bench.build_problem()
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(steps, 1e-3)
g.synchronize()
g.time_contract(1)
print("done", g.launch_count())
