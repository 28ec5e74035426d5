import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as po
from tests.gpu_helpers import make_pair
for nt, nq in ((2, 2), (3, 3), (2, 3)):
    for mesh in ((9, 7), (4, 4), (8, 8), (6, 6)):
        for layers in ((2, 30, 30, 1), (2, 20, 20, 1), (2, 24, 11, 1), (2, 30, 30, 30, 1)):
            spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing="sin2pi_f",
                                  boundary_g="sin2pi_u", n_boundary=37, layers=layers, seed=5)
            ob, g, p0 = make_pair(spec)
            po_, _ = ob.loss_and_grad(p0)
            pg, gg = g.loss_and_grad()
            r = abs(pg[0] - po_[0]) / abs(po_[0])
            rv = abs(pg[1] - po_[1]) / abs(po_[1])
            if r > 1e-5:
                print("BAD", (nt, nq), mesh, layers, g.step_kernel()[:28], r, rv, pg, po_)
print("done")
