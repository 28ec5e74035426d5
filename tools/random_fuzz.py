"""Randomised parity fuzz of the default GPU path against the oracle: random
structured meshes, test / quadrature orders (Q > 128 takes the split path),
served networks (2-3 hidden layers of width <= 62, one or two outputs,
ragged), tanh / sigmoid, fixed / trainable / spatial coefficient,
convection, sensors.  Loss within 1e-5, gradient within 1e-5 of max|g| of
the fp64 oracle (or 4x the fp32 oracle's own distance), 5-epoch history
within 1e-5 (or twice the fp32 noise floor; the loss likewise).
usage: python tools/random_fuzz.py N [seed]   (FUZZ_MODE=wide | strong)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as po  # noqa: E402
from tests.gpu_helpers import make_pair  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
# FUZZ_MODE=wide: depth 1-4 (the CUDA-core step's shapes too); =strong: the strong form
WIDE = os.environ.get("FUZZ_MODE", "")
ONLY = int(os.environ["FUZZ_ONLY"]) if os.environ.get("FUZZ_ONLY") else None  # re-run one case (diagnostics)
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
for case in range(n):
    nx, ny = (int(v) for v in rng.integers(1, 13, size=2))
    nt = int(rng.integers(1, 8))
    nq = int(rng.choice([2, 3, 4, 5, 6, 8, 10, 11, 12, 13, 15, 20]))
    strong = WIDE == "strong"
    depth = int(rng.integers(1, 5)) if WIDE else int(rng.integers(2, 4))
    outs = 1 if strong else int(rng.integers(1, 3))
    if strong:
        wmax = 32
    elif depth <= 2:
        wmax = 64
    elif depth == 3:
        wmax = 50 if outs == 2 else 62
    else:
        wmax = 36
    hidden = tuple(int(v) for v in rng.integers(2, wmax + 1, size=depth))
    if rng.random() < 0.5:
        hidden = (hidden[0],) * depth
    layers = (2,) + hidden + (outs,)
    sig = bool(rng.random() < 0.3)
    kw = {}
    if outs == 2:
        kw.update(eps_source=2, forcing="sinpi_vareps_f")
    else:
        kw.update(forcing=str(rng.choice(["sin2pi_f", "sin4pi_f", "one"])))
        if rng.random() < 0.3:
            kw.update(eps_source=1, scalars=(float(rng.uniform(0.5, 2.0)),))
    if rng.random() < 0.4:
        kw.update(bx=float(rng.uniform(-1, 1)), by=float(rng.uniform(-1, 1)))
    if rng.random() < 0.4:
        kw.update(n_sensors=int(rng.integers(1, 40)), sensor_field="sin2pi_u")
    if strong:
        kw.pop("forcing", None)
        kw.update(forcing="sin2pi_f", strong=True)
    spec = po.ProblemSpec(*po.structured_mesh(nx, ny, skew=float(rng.uniform(0, 0.2))), n_test_1d=nt,
                          n_quad_1d=nq, boundary_g="sin2pi_u", n_boundary=int(rng.integers(1, 300)),
                          layers=layers, sigmoid=sig, seed=int(rng.integers(1, 1000)), **kw)
    desc = f"{case}: mesh {nx}x{ny} nt {nt} nq {nq} layers {layers} sig {sig} {kw}"
    if ONLY is not None and case != ONLY:
        continue
    try:
        if strong:
            from tests.test_strong_form import make_strong_pair
            ob, g, p0 = make_strong_pair(spec)
        else:
            ob, g, p0 = make_pair(spec)
        po_, go32 = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        o64 = po.OracleProblem(spec, double=True)
        _, g64 = o64.loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        lfloor = abs(o64.loss_and_grad(p0.astype(np.float64))[0][0] - po_[0]) / abs(po_[0])
        scale = max(np.abs(g64).max(), 1e-30)
        ge = np.abs(gg - g64).max() / scale
        e32 = np.abs(go32 - g64).max() / scale
        ref = ob.train(p0, 5, lr0=1e-3, log_every=1)["every_step"][:, 0]
        ref64 = o64.train(p0.astype(np.float64), 5, lr0=1e-3, log_every=1)["every_step"][:, 0]
        rep = g.train(5, lr0=1e-3)
        tr = np.abs(rep.records["total"] - ref) / np.abs(ref)
        floor = np.abs(ref64 - ref) / np.abs(ref)
        ok = lr < max(1e-5, 2 * lfloor) and ge < max(1e-5, 4 * e32) and tr.max() < max(1e-5, 2 * floor.max())
        if ONLY is not None:
            k = int(np.abs(gg - g64).argmax())
            print("worst parameter", k, "gpu", gg[k], "fp64", g64[k], "fp32", go32[k], "max|g|", scale,
                  "n_int", ob.n_int, "n_bnd", ob.n_bnd, "n_sen", ob.n_sen, "kernel", g.step_kernel())
        if not ok:
            bad += 1
            print("FAIL", desc, g.step_kernel()[:48], f"loss {lr:.1e} grad {ge:.1e} (fp32 {e32:.1e}) "
                  f"hist {tr.max():.1e} (floor {floor.max():.1e})", flush=True)
        g.close()
    except Exception as e:  # noqa: BLE001
        msg = str(e)
        if "not instantiated" in msg:
            continue
        bad += 1
        print("ERR ", desc, msg[:120], flush=True)
        if "illegal" in msg or "unspecified launch failure" in msg:
            break
print(f"{n} cases, {bad} failures")
