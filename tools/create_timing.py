"""Phase times of vpinn_gpu_create for the bench gear (host arrays path),
repeated, from pageable and from page-locked inputs:
VPINN_CREATE_TIMING=1 python tools/create_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
hp = host.HostProblem(bench.GEAR_CFG, mesh=mesh)
pv, keep = G.pin_problem(hp.view(0))
for rep in range(8):
    pinned = rep % 2 == 1
    t0 = time.perf_counter()
    g = G.GpuStep.from_problem(pv if pinned else hp.view(0), keepalive=hp)
    t1 = time.perf_counter()
    g.set_params(hp.init_params())
    g.train(50)
    t2 = time.perf_counter()
    g.close()
    print(f"rep {rep} {'pinned' if pinned else 'pageable'}: create {1e3*(t1-t0):.2f} ms, train(50) {1e3*(t2-t1):.2f} ms", file=sys.stderr, flush=True)
