"""Parity over a grid of discretisations and network shapes (the GPU kernel
the context selects for each: tensor-core step, CUDA-core step, split path):
n_test x n_quad per dimension from 1x1 to 8x13 (Q > 128 takes the split
path), 1 to 63 cells, uniform / ragged / one-layer / two-output networks,
tanh and sigmoid, with and without convection.  Found: ragged widths on the
tensor-core step, a loss race for many small cells per tile, a misaligned
mbarrier in the row-chunked contraction, the bf16 kernel at Q = 1."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.gpu_helpers import make_pair

pytestmark = pytest.mark.gpu

PAIRS = [(1, 1), (1, 3), (2, 2), (3, 7), (6, 6), (2, 12), (8, 13)]
MESHES = [(1, 1), (2, 3), (9, 7)]
NETS = [(2, 30, 30, 30, 1), (2, 17, 1), (2, 24, 11, 1), (2, 16, 16, 16, 2)]


@pytest.mark.parametrize("pair", PAIRS)
def test_shape_grid_matches_oracle(pair):
    nt, nq = pair
    fails = []
    for mesh, layers, sig, conv in itertools.product(MESHES, NETS, [False, True], [False, True]):
        if layers[-1] == 2 and sig:
            continue  # no sigmoid two-output variant instantiated
        kw = dict(eps_source=2, bx=0.5) if layers[-1] == 2 else dict(bx=0.3 if conv else 0.0)
        fx = "sinpi_vareps_f" if layers[-1] == 2 else "sin2pi_f"
        spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing=fx,
                              boundary_g="sin2pi_u", n_boundary=37, layers=layers, sigmoid=sig, seed=5, **kw)
        ob, g, p0 = make_pair(spec)
        po_, _ = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        ge = np.abs(gg - g64).max() / max(np.abs(g64).max(), 1e-30)
        if lr > 1e-5 or ge > 2e-4:
            fails.append((mesh, layers, sig, conv, g.step_kernel(), lr, ge))
        g.close()
    assert not fails, fails
