"""North-star accuracy criterion: the final L2 / L-infinity solution error of
a trained network within 1% of the CPU reference's (oracle) on the same mesh,
seed and schedule.  The reference computes the metrics with evaluate(order 0)
on a uniform grid over the mesh bounding box (trainer.hpp:403-446); the GPU
run goes through the C++ host trainer (vpinn_host_train: vpinn_gpu_train +
device evaluate), weak form and strong form."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2404_12063_b200 import host

ITERS = 800
# the reference default rate: at this rate the fp32 and fp64 oracles end
# within 1e-5 of each other, so the comparison is well posed (at 2e-3-5e-3
# Adam amplifies fp32 rounding and even fp32 vs fp64 oracles end up to 10x
# apart in final error)
LR = 1e-3
GRID = 41


def _cfg(form):
    return {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "exact_solution": "sin2pi_u",
                        "n_boundary_points": 120, "domain": {"nx": 4, "ny": 4}},
            "discretization": {"form": form, "n_test_per_dim": 3, "n_quad_per_dim": 6},
            "network": {"layers": [2, 30, 30, 30, 1]},
            "training": {"iterations": ITERS, "learning_rate": LR, "seed": 42, "precision": "single",
                         "log_every": 400},
            "output": {"grid_nx": GRID, "grid_ny": GRID}}


def _oracle_metrics(form):
    nodes, cells = po.structured_mesh(4, 4)
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=3, n_quad_1d=6,
                                         forcing="sin2pi_f", boundary_g="sin2pi_u", n_boundary=120,
                                         layers=(2, 30, 30, 30, 1), seed=42, strong=form == "strong"),
                          double=False)
    out = ob.train(ob.init_params(), ITERS, lr0=LR, log_every=400)
    xs = np.linspace(0.0, 1.0, GRID)
    pts = np.array([(x, y) for y in xs for x in xs])  # x fastest (trainer.hpp:409-418)
    u = ob.evaluate(out["params"], pts, 0)[0].astype(np.float64)
    ue = po.field("sin2pi_u", pts[:, 0], pts[:, 1])
    d = u - ue
    return {"rel_l2": float(np.sqrt(np.sum(d * d) / np.sum(ue * ue))), "max_err": float(np.abs(d).max())}


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["weak", "strong"])
def test_final_solution_error_within_one_percent_of_reference(form):
    hp = host.HostProblem(_cfg(form))
    rep, _ = hp.train(device=0)
    assert rep["steps_run"] == ITERS
    ref = _oracle_metrics(form)
    # a trained solution, not the initial guess (rel. L2 ~1): weak ~3%,
    # strong (the PINN baseline learns slower) ~51% after 800 epochs
    assert ref["rel_l2"] < 0.6
    for k in ("rel_l2", "max_err"):
        assert abs(rep["metrics"][k] - ref[k]) <= 0.01 * ref[k], (k, rep["metrics"][k], ref[k])
