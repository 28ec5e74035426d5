"""Accuracy margins of the strong-form kernel against the oracle (the
quantities tests/test_strong_form.py bounds): loss rel. error, gradient error
vs fp64, 100-epoch trajectory max rel. error."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as po  # noqa: E402
from tests.test_strong_form import CASES, make_strong_pair  # noqa: E402

out = {}
for name in ("poisson_d3", "cd2d_sensors_scalar_eps", "gear_many_tiles"):
    spec = CASES[name]()
    ob, g, p0 = make_strong_pair(spec)
    po_, _ = ob.loss_and_grad(p0)
    pg, gg = g.loss_and_grad()
    _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
    r = {"loss_rel": abs(pg[0] - po_[0]) / abs(po_[0]),
         "grad_err": float(np.abs(gg - g64).max() / np.abs(g64).max())}
    if name == "cd2d_sensors_scalar_eps":
        ref = ob.train(p0, 100, lr0=1e-3, log_every=1)
        rep = g.train(100, lr0=1e-3)
        tot = ref["every_step"][:, 0]
        r["traj_max_rel"] = float((np.abs(rep.records["total"] - tot) / np.abs(tot)).max())
    out[name] = r
print(json.dumps(out))
