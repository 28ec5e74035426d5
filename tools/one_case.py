"""One parity case (debugging): python tools/one_case.py NT NQ NX NY [layers...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from tests.gpu_helpers import make_pair  # noqa: E402

nt, nq, nx, ny = map(int, sys.argv[1:5])
layers = tuple(map(int, sys.argv[5:])) or (2, 30, 30, 30, 1)
spec = po.ProblemSpec(*po.structured_mesh(nx, ny), n_test_1d=nt, n_quad_1d=nq, forcing="sin2pi_f",
                      boundary_g="sin2pi_u", n_boundary=37, layers=layers, seed=5)
ob, g, p0 = make_pair(spec)
print(g.step_kernel())
po_, _ = ob.loss_and_grad(p0)
pg, gg = g.loss_and_grad()
print("loss rel", abs(pg[0] - po_[0]) / abs(po_[0]))
