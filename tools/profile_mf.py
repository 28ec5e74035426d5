"""Gear problem with device assembly: one launch each of the tensor and the
matrix-free contraction (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(16, 887)
dp = host.HostProblem(bench.GEAR_CFG, mesh=mesh, device_assembly=True)
g = G.GpuStep.from_problem(dp.view(0, 0, 1), keepalive=dp)
print("tensor", g.time_contract(3), "matrix-free", g.time_contract_matrix_free(3))
