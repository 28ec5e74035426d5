"""Phase wall times of the from-mesh end-to-end path on the C5 gear
(HostProblem(device_assembly) -> create -> train(K) -> get_params), five
fresh contexts after one warm-up; VPINN_CREATE_TIMING=1 adds create's phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import gpu as G, host  # noqa: E402

mesh = host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for it in range(6):
    t0 = time.perf_counter()
    dp = host.HostProblem(bench.GEAR_CFG, mesh=mesh, device_assembly=True)
    t1 = time.perf_counter()
    g = G.GpuStep.from_problem(dp.view(0, 0, 1), keepalive=dp)
    t2 = time.perf_counter()
    g.set_params(dp.init_params())
    g.train(K, lr0=1e-3)
    t3 = time.perf_counter()
    g.get_params()
    t4 = time.perf_counter()
    g.close()
    print(f"run {it}: build {1e3*(t1-t0):.2f} create {1e3*(t2-t1):.2f} train {1e3*(t3-t2):.2f} "
          f"get {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms", flush=True)
