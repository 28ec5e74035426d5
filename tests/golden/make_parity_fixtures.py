"""Generates tests/golden/parity/<case>.npz: the CPU oracle's answers on the
large BASELINE configs (parity_cases.FIXTURE_CASES), so the GPU tests do not
rerun minutes of oracle epochs on the GPU box.  Per case:

  p0        initial parameters (float32, reference init, network.hpp:66-96)
  traj32    [EPOCHS][4] fp32 oracle history: total, L_v, L_b, L_s per epoch
            (trainer.hpp:316-341, every step logged), Adam lr 1e-3
  params32  fp32 oracle parameters after EPOCHS epochs
  parts64   fp64 oracle loss parts at p0
  grad64    fp64 oracle gradient at p0 (the noise-floor reference)
  grad32    fp32 oracle gradient at p0
  traj64    [EPOCHS][4] fp64 oracle history from the same p0: |traj64 -
            traj32| is the fp32 noise floor of the trajectory (Adam's first
            steps are +-lr per parameter, so parameters whose gradient sits
            below fp32 rounding flip with it; on the paper's [2,50,50,50,1]
            gear the fp64 and fp32 oracles differ by ~5e-5 at epochs 2-4)

Run (CPU, ~30 min, one process per case):
    python tests/golden/make_parity_fixtures.py [case ...]
    python tests/golden/make_parity_fixtures.py --add64 [case ...]   (traj64 only)
tests/test_oracle_golden.py re-derives traj32[0] / grad32 from the oracle to
pin each fixture to the current oracle build.
"""
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

OUT = os.path.join(HERE, "parity")


def add64(name):
    """Adds traj64 to an existing fixture (the fp32 entries are unchanged)."""
    from oracle import pyoracle as po
    import parity_cases as pc
    t0 = time.time()
    path = os.path.join(OUT, name + ".npz")
    fx = dict(np.load(path))
    o64 = po.OracleProblem(pc.CASES[name](), double=True)
    run = o64.train(fx["p0"].astype(np.float64), pc.EPOCHS, lr0=pc.LR, log_every=1)
    fx["traj64"] = run["every_step"]
    np.savez_compressed(path, **fx)
    r = np.abs(fx["traj64"][:, 0] - fx["traj32"][:, 0]) / np.abs(fx["traj32"][:, 0])
    return f"{name}: {time.time() - t0:.0f} s, fp64-vs-fp32 oracle trajectory max rel {r.max():.2e}"


def make(name):
    from oracle import pyoracle as po
    import parity_cases as pc
    t0 = time.time()
    spec = pc.CASES[name]()
    o32 = po.OracleProblem(spec, double=False)
    p0 = o32.init_params().astype(np.float32)
    _, grad32 = o32.loss_and_grad(p0)
    run = o32.train(p0, pc.EPOCHS, lr0=pc.LR, log_every=1)
    o64 = po.OracleProblem(spec, double=True)
    parts64, grad64 = o64.loss_and_grad(p0.astype(np.float64))
    os.makedirs(OUT, exist_ok=True)
    run64 = o64.train(p0.astype(np.float64), pc.EPOCHS, lr0=pc.LR, log_every=1)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), p0=p0, traj32=run["every_step"],
                        params32=run["params"].astype(np.float32), parts64=parts64, grad64=grad64,
                        grad32=grad32.astype(np.float32), traj64=run64["every_step"])
    e32 = np.abs(grad32 - grad64).max() / np.abs(grad64).max()
    return f"{name}: {time.time() - t0:.0f} s, steps {run['steps_run']}, fp32-oracle grad err {e32:.2e}"


if __name__ == "__main__":
    import parity_cases as pc
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    fn = add64 if "--add64" in sys.argv else make
    names = args or list(pc.FIXTURE_CASES)
    with mp.Pool(len(names)) as pool:
        for line in pool.imap_unordered(fn, names):
            print(line, flush=True)
