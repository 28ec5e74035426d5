import time, sys, os
sys.path.insert(0, os.getcwd())
import bench
from paper_2404_12063_b200 import host, gpu as G
mesh = host.Mesh.gear(16, 887)
for rep in range(3):
    t0 = time.perf_counter(); dp = host.HostProblem(bench.GEAR_CFG, mesh=mesh, device_assembly=True); t1 = time.perf_counter()
    v = dp.view(0, 0, 1); t2 = time.perf_counter()
    g = G.GpuStep.from_problem(v, keepalive=dp); t3 = time.perf_counter()
    g.set_params(dp.init_params()); g.train(50); t4 = time.perf_counter(); g.close(); t5 = time.perf_counter()
    hp = host.HostProblem(bench.GEAR_CFG, mesh=mesh); t6 = time.perf_counter()
    vv = hp.view(0, 0, 1); t7 = time.perf_counter()
    g2 = G.GpuStep.from_problem(vv, keepalive=hp); t8 = time.perf_counter()
    print(f"dev: build {1e3*(t1-t0):.1f} view {1e3*(t2-t1):.1f} create {1e3*(t3-t2):.1f} train {1e3*(t4-t3):.1f} close {1e3*(t5-t4):.1f} | host: build {1e3*(t6-t5):.1f} view {1e3*(t7-t6):.1f} create {1e3*(t8-t7):.1f} ms")
    g2.close()
