"""GPU parity on every BASELINE.json config at full size (the C5 headline
included): the C-ABI path against the CPU oracle on the same mesh, seed and
fp32 arithmetic.

* loss parts at the initial parameters within 1e-5 relative of the fp32
  oracle (north star);
* the parameter gradient within 1e-5 of max|g| of the fp64 oracle (the
  fp32-vs-fp64 noise floor of the oracle itself is printed beside it);
* 100 Adam epochs (lr 1e-3): every epoch's total loss within 1e-5 relative
  of the fp32 oracle's (north star: "per-epoch loss within 1e-5 relative over
  the first 100 epochs"), each loss component within 1e-5 of the total,
  final parameters within 1e-4; where the fp64 oracle's own trajectory is
  farther than 1e-5 from the fp32 oracle's (the fp32 noise floor), twice
  that floor.

The large configs compare against committed oracle fixtures
(tests/golden/parity/*.npz, made by tests/golden/make_parity_fixtures.py and
pinned to the oracle by tests/test_oracle_golden.py); the two reference
configs that run in seconds (forward_sine.json, inverse_eps.json) run the
oracle live.
"""
import os
import sys

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.gpu_helpers import gpu_from_oracle

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import parity_cases as pc  # noqa: E402

pytestmark = pytest.mark.gpu

FIX = os.path.join(os.path.dirname(__file__), "golden", "parity")
LIVE = ("forward_sine", "inverse_eps")
_cache = {}


def _ref(case):
    """(spec, oracle32, fixture dict) — the fixture, or the live oracle run."""
    if case in _cache:
        return _cache[case]
    spec = pc.CASES[case]()
    ob = po.OracleProblem(spec, double=False)
    if case in LIVE:
        p0 = ob.init_params().astype(np.float32)
        run = ob.train(p0, pc.EPOCHS, lr0=pc.LR, log_every=1)
        o64 = po.OracleProblem(spec, double=True)
        parts64, grad64 = o64.loss_and_grad(p0.astype(np.float64))
        run64 = o64.train(p0.astype(np.float64), pc.EPOCHS, lr0=pc.LR, log_every=1)
        _, grad32 = ob.loss_and_grad(p0)
        fx = {"p0": p0, "traj32": run["every_step"], "params32": run["params"], "parts64": parts64,
              "grad64": grad64, "grad32": grad32, "traj64": run64["every_step"]}
    else:
        fx = dict(np.load(os.path.join(FIX, case + ".npz")))
    _cache[case] = (spec, ob, fx)
    return _cache[case]


CASES = list(pc.FIXTURE_CASES) + list(LIVE)


@pytest.mark.parametrize("case", CASES)
def test_loss_parts_and_gradient(case):
    spec, ob, fx = _ref(case)
    g = gpu_from_oracle(ob, spec)
    g.set_params(fx["p0"])
    parts, grad = g.loss_and_grad()
    ref = fx["traj32"][0]  # the fp32 oracle's epoch-1 record = the loss at p0
    for k in range(4):
        if ref[k] != 0.0:
            assert abs(parts[k] - ref[k]) / abs(ref[k]) < 1e-5, (k, parts, ref)
    g64 = fx["grad64"]
    scale = np.abs(g64).max()
    err = np.abs(grad - g64).max() / scale
    floor = np.abs(fx["grad32"] - g64).max() / scale
    print(f"{case}: gradient error vs fp64 {err:.2e} (fp32 oracle {floor:.2e}), kernel {g.step_kernel()}")
    assert err < 1e-5, (err, floor)


@pytest.mark.parametrize("case", CASES)
def test_hundred_epoch_trajectory(case):
    spec, ob, fx = _ref(case)
    g = gpu_from_oracle(ob, spec)
    g.set_params(fx["p0"])
    rep = g.train(pc.EPOCHS, lr0=pc.LR)
    assert rep.steps_run == pc.EPOCHS
    ref = fx["traj32"]
    tot = np.abs(ref[:, 0])
    # the total loss per epoch within 1e-5 relative (the north star); each
    # component within 1e-5 of the total it contributes to (a component's own
    # relative error is noise-dominated when it is small, e.g. the boundary
    # mismatch of a zero-boundary problem).  Where fp32 itself cannot meet
    # 1e-5 -- the fp64 oracle's trajectory is farther than that from the fp32
    # oracle's (Adam's +-lr first steps flip with the sign of gradients below
    # fp32 rounding: the paper's [2,50,50,50,1] gear, ~5e-5) -- the bound is
    # twice that fp32 noise floor
    floor = np.abs(fx["traj64"][:, 0] - ref[:, 0]) / tot
    tol = max(1e-5, 2.0 * float(floor.max()))
    for k, name in enumerate(("total", "variational", "boundary", "sensor")):
        if np.all(ref[:, k] == 0.0):
            continue
        r = np.abs(rep.records[name] - ref[:, k]) / tot
        print(f"{name}: max rel {r.max():.2e} (fp32 noise floor {floor.max():.2e}, bound {tol:.1e})")
        assert r.max() < tol, (name, r.max(), int(r.argmax()), floor.max())
    assert np.abs(g.get_params() - fx["params32"]).max() < 1e-4
    if spec.eps_source == 1:
        assert abs(rep.final_eps - float(fx["params32"][-1])) < 1e-5
