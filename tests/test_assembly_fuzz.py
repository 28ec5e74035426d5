"""Device-side assembly against the host arrays over a grid of rules, meshes
and both loss forms, including rank partitions and the split path (Q > 128):
the objective and gradient of a context the device assembled match the one
built from host arrays (bit-identical for the weak form's tensors, tolerance
for the strong form's device-evaluated forcing)."""
import itertools

import numpy as np
import pytest

from paper_2404_12063_b200 import host

pytestmark = pytest.mark.gpu


def _cfg(form, nt, nq):
    return {"problem": {"pde": {"type": "cd2d", "eps": 0.9, "b": [0.4, -0.1]}, "forcing": "sin2pi_f",
                        "boundary_g": "sin2pi_u", "n_boundary_points": 29},
            "discretization": {"form": form, "n_test_per_dim": nt, "n_quad_per_dim": nq},
            "network": {"layers": [2, 18, 18, 1]},
            "training": {"learning_rate": 1e-3, "seed": 13, "precision": "single"}}


@pytest.mark.parametrize("form", ["weak", "strong"])
def test_device_assembly_grid(form):
    fails = []
    for (nt, nq), (nx, ny, skew), world in itertools.product(
            [(1, 2), (3, 4), (5, 5), (4, 12)], [(1, 1, 0.0), (3, 2, 0.25), (7, 5, 0.1)], [1, 2]):
        mesh = host.Mesh.structured(nx, ny, skew=skew)
        hp = host.HostProblem(_cfg(form, nt, nq), mesh=mesh)
        dp = host.HostProblem(_cfg(form, nt, nq), mesh=mesh, device_assembly=True)
        for r in range(world):
            gh, gd = hp.gpu(0, r, world), dp.gpu(0, r, world)
            ph, grh = gh.loss_and_grad()
            pd, grd = gd.loss_and_grad()
            tol = 0.0 if form == "weak" else 1e-6
            bad_parts = np.abs(ph - pd).max() > tol * max(1.0, np.abs(ph).max())
            bad_grad = np.abs(grh - grd).max() > tol * max(1e-30, np.abs(grh).max())
            if bad_parts or bad_grad:
                fails.append(((nt, nq), (nx, ny, skew), world, r, gh.step_kernel(), ph, pd))
            gh.close()
            gd.close()
    assert not fails, fails
