import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import pyoracle as po
from tests.gpu_helpers import make_pair
for layers in [(2, 7, 13, 5, 1), (2, 30, 13, 30, 1), (2, 13, 30, 30, 1), (2, 30, 30, 13, 1), (2, 7, 7, 7, 1), (2, 20, 20, 1), (2, 20, 9, 1), (2, 9, 20, 1)]:
    spec = po.ProblemSpec(*po.structured_mesh(3, 4), n_test_1d=4, n_quad_1d=6, forcing="sin2pi_f", boundary_g="sin2pi_u",
                          n_boundary=50, layers=layers, bx=0.4, seed=11)
    try:
        ob, g, p0 = make_pair(spec)
        po_, _ = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        print(layers, g.step_kernel()[:30], abs(pg[0] - po_[0]) / abs(po_[0]))
    except Exception as e:
        print(layers, "ERR", e)
