"""Per-phase cycle breakdown of the tensor-core step (CTA 0, first tiles) on
the C5 gear problem: VPINN_PHASE_CLOCK=1 makes thread 0 of CTA 0 record
clock64() at the phase marks of tc_step_kernel.cuh (mark(i))."""
import os
import sys

os.environ["VPINN_PHASE_CLOCK"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2404_12063_b200 import _capi, gpu as G  # noqa: E402

NAMES2 = ["start", "L0+store+sync+issue", "epi1(+store,issue L2)", "epi2(last)", "out layer+sync",
          "sync+tma wait", "phase A+resid", "phase B+cells", "adjoint sync", "out rev+G+issue", "G2+X1+issue",
          "G1+W0", "bar_w+readout"]
NAMES = ["start", "L0+store+sync", "L1 mma+epi", "store B+sync", "L2 mma+epi", "out layer+sync",
         "sEx sync+tma wait", "phase A+sync", "residual+sync", "phase B+sync", "adjoint sync",
         "out rev+colsum+G+sync", "state+L0+adj2", "bar_w+G1/X1+sync", "adj1", "bar_w", "colsum W0"]
hp, _ = bench.build_problem()
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(3, 1e-3)
g.synchronize()
buf = np.zeros(8 * 32, np.int64)
_capi.check(_capi.lib().vpinn_gpu_phase_clock(g.h, buf.ctypes.data_as(C.c_void_p), buf.size))
tc2 = g.step_kernel().startswith("tc2")
nm = 13 if tc2 else 17
if tc2:
    NAMES = NAMES2
t = buf.reshape(8, 32)[:, :nm].astype(np.float64)
d = np.diff(t, axis=1)
per_tile = t[1:, 0] - t[:-1, 0]
print(g.step_kernel())
print("tile cycles:", per_tile.astype(int).tolist())
for i in range(nm - 1):
    print(f"{NAMES[i+1]:24s} " + " ".join(f"{int(x):6d}" for x in d[:, i]) + f"   mean {d[1:, i].mean():7.0f}")
print("sum of marks per tile", d.sum(axis=1).astype(int).tolist())
