"""Strong-form parity over a grid of shapes: 1-4 hidden layers of widths
1..32 (ragged), tanh / sigmoid, point counts that leave partial 16-point warp
tiles, convection and a trainable coefficient."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.test_strong_form import make_strong_pair

pytestmark = pytest.mark.gpu

NETS = [(2, 1, 1), (2, 32, 1), (2, 5, 32, 1), (2, 32, 3, 17, 1), (2, 9, 9, 9, 9, 1)]


@pytest.mark.parametrize("layers", NETS)
def test_strong_shape_grid_matches_oracle(layers):
    fails = []
    for (nt, nq), mesh, sig, inv in itertools.product([(1, 1), (2, 3), (3, 7)], [(1, 1), (3, 2)],
                                                       [False, True], [False, True]):
        kw = dict(eps_source=1, scalars=(1.7,), bx=0.4, by=-0.2, n_sensors=5,
                  sensor_field="sin2pi_u") if inv else {}
        spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing="sin2pi_f",
                              boundary_g="sin2pi_u", n_boundary=23, layers=layers, sigmoid=sig, seed=3,
                              strong=True, **kw)
        ob, g, p0 = make_strong_pair(spec)
        po_, go32 = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        ge = np.abs(gg - g64).max() / max(np.abs(g64).max(), 1e-30)
        # gradient: 1e-5 of max|g| against fp64, or 4x the fp32 oracle's own
        # distance from fp64 where that noise floor is higher (tiny problems)
        e32 = np.abs(go32 - g64).max() / max(np.abs(g64).max(), 1e-30)
        if lr > 1e-5 or ge > max(1e-5, 4.0 * e32):
            fails.append(((nt, nq), mesh, sig, inv, lr, ge))
        g.close()
    assert not fails, fails
