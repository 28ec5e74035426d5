"""C3 p/q-refinement point (8x8 cells, 10x10 test functions, 40x40 Gauss
points: the split path) for ncu launch lists: python tools/profile_c3.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t, q = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (10, 40)
cfg = {"problem": {"forcing": "sin4pi_f", "boundary_g": "sin4pi_u", "n_boundary_points": 400},
       "discretization": {"n_test_per_dim": t, "n_quad_per_dim": q},
       "network": {"layers": [2, 30, 30, 30, 1]},
       "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
hp = host.HostProblem(cfg, mesh=host.Mesh.structured(8, 8))
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(steps, 1e-3)
g.synchronize()
print("kernel", g.step_kernel(), "profile ms (step, reduce, adam):", g.profile_step(5))
