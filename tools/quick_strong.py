"""Strong-form epoch time on the C5 gear (bench workload with form=strong):
ms/epoch L2-flushed and warm, kernel name.  VPINN_SF_WARPS picks warps/CTA."""
import copy
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402


def main():
    cfg = copy.deepcopy(bench.GEAR_CFG)
    cfg["discretization"]["form"] = "strong"
    mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
    hp = host.HostProblem(cfg, mesh=mesh)
    g = G.GpuStep.from_problem(hp.view(0), keepalive=hp)
    g.set_params(hp.init_params())
    g.adam_reset()
    g.run_steps(5, 1e-3)
    g.synchronize()
    times = []
    for _ in range(20):
        g.flush_l2()
        times.append(g.time_steps(1, 1e-3))
    warm = g.time_steps(50, 1e-3) / 50
    parts, _ = g.loss_and_grad()
    out = {"kernel": g.step_kernel(), "flushed_ms": float(np.median(times)), "warm_ms": warm,
           "n_int": hp.n_int, "n_bnd": hp.n_bnd, "loss": parts.tolist(),
           "pts_per_s": (hp.n_int + hp.n_bnd) / (np.median(times) * 1e-3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
