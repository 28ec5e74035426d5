"""Loss / gradient parity of the default GPU kernel against the oracle over a
grid of discretisations and network shapes (quick fuzz; prints failures)."""
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as po  # noqa: E402
from tests.gpu_helpers import make_pair  # noqa: E402

PAIRS = [(1, 1), (1, 3), (2, 2), (3, 7), (6, 6), (2, 12), (8, 13)]
# one (n_test, n_quad) pair per process: a device fault poisons the context
sel = [PAIRS[int(sys.argv[1])]] if len(sys.argv) > 1 else PAIRS
bad = 0
n = 0
for (nt, nq), mesh, layers, sig, conv in itertools.product(
        sel,
        [(1, 1), (2, 3), (9, 7)],
        [(2, 30, 30, 30, 1), (2, 17, 1), (2, 24, 11, 1), (2, 16, 16, 16, 2)],
        [False, True], [False, True]):
    if layers[-1] == 2 and sig:
        continue
    kw = dict(eps_source=2, bx=0.5) if layers[-1] == 2 else dict(bx=0.3 if conv else 0.0)
    if os.environ.get("FUZZ_SCALAR") and layers[-1] == 1:  # trainable eps + sensors
        kw.update(eps_source=1, scalars=(1.3,), n_sensors=11, sensor_field="sin2pi_u")
    fx = "sinpi_vareps_f" if layers[-1] == 2 else "sin2pi_f"
    spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing=fx,
                          boundary_g="sin2pi_u", n_boundary=37, layers=layers, sigmoid=sig, seed=5, **kw)
    n += 1
    try:
        ob, g, p0 = make_pair(spec)
        po_, _ = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        ge = np.abs(gg - g64).max() / max(np.abs(g64).max(), 1e-30)
        if lr > 1e-5 or ge > 2e-4:
            bad += 1
            print("FAIL", (nt, nq), mesh, layers, sig, conv, g.step_kernel()[:32], lr, ge)
    except Exception as e:  # noqa: BLE001
        msg = str(e)
        if "not instantiated" not in msg:
            bad += 1
        print("ERR ", (nt, nq), mesh, layers, sig, conv, msg[:90])
        if "illegal" in msg or "unspecified launch failure" in msg:
            break
print(f"{n} cases, {bad} failures")
