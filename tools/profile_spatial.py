"""Minimal driver for ncu: the paper's spatial-coefficient inverse on C4's
disk (two-output network, tc2 two-output variant), a few epochs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

cfg = {"problem": {"pde": {"type": "cd2d_variable_eps", "b": [1.0, 0.0]}, "forcing": "one",
                   "boundary_g": "zero", "exact_solution": "sinpi_u", "n_boundary_points": 400,
                   "sensors": {"count": 50, "seed": 7}},
       "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
       "network": {"layers": [2, 30, 30, 30, 2]},
       "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
hp = host.HostProblem(cfg, mesh=host.Mesh.disk(32))
g = G.GpuStep.from_problem(hp.view(0), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(4, 1e-3)
g.synchronize()
print("kernel", g.step_kernel())
