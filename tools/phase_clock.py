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
if len(sys.argv) > 1 and sys.argv[1].startswith("c2"):
    # C2 sweep point: e x e unit-square cells, T=25, Q=100 (a lone tile per CTA)
    from paper_2404_12063_b200 import host  # noqa: E402
    e = int(sys.argv[1][3:] or 1)
    cfg = {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 400},
           "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
           "network": {"layers": [2, 30, 30, 30, 1]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    hp = host.HostProblem(cfg, mesh=host.Mesh.structured(e, e))
else:
    hp, _ = bench.build_problem()
g = G.GpuStep.from_problem(hp.view(0, 0, 1), keepalive=hp)
g.set_params(hp.init_params())
g.adam_reset()
g.run_steps(3, 1e-3)
g.synchronize()
buf = np.zeros(8 * 32 + 3 * 1024, np.int64)
_capi.check(_capi.lib().vpinn_gpu_phase_clock(g.h, buf.ctypes.data_as(C.c_void_p), buf.size))
tc2 = g.step_kernel().startswith("tc2")
nm = 13 if tc2 else 17
if tc2:
    NAMES = NAMES2
ctas = buf[256:].reshape(1024, 3)
t = buf[:256].reshape(8, 32)[:, :nm].astype(np.float64)
d = np.diff(t, axis=1)
per_tile = t[1:, 0] - t[:-1, 0]
print(g.step_kernel())
print("tile cycles:", per_tile.astype(int).tolist())
for i in range(nm - 1):
    print(f"{NAMES[i+1]:24s} " + " ".join(f"{int(x):6d}" for x in d[:, i]) + f"   mean {d[1:, i].mean():7.0f}")
allv = buf[:256]
sm = buf[7 * 32 + 20: 7 * 32 + 26]
if sm[0]:
    print("setup marks (cycles from entry):", [int(x - allv[-1]) for x in sm])
tt = buf[:256].reshape(8, 32)
if tt[1, 15]:
    print("MMA issue (cycles): prop", (tt[1:, 14] - tt[1:, 13]).tolist(), "param", (tt[1:, 15] - tt[1:, 14]).tolist())
if allv[-1]:
    print(f"CTA 0: entry -> first tile {int(t[0, 0] - allv[-1])} cycles; entry -> exit {int(allv[-2] - allv[-1])} cycles "
          f"({(allv[-2] - allv[-1]) / 1.965e3:.1f} us at 1965 MHz); tiles {int(allv[-3])}")
print("sum of marks per tile", d.sum(axis=1).astype(int).tolist())

cta = ctas[ctas[:, 0] > 0]
if len(cta):
    t0 = cta[:, 0].min()
    st, en = (cta[:, 0] - t0) / 1e3, (cta[:, 1] - t0) / 1e3
    print(f"CTAs {len(cta)}: start spread {st.max():.1f} us; end min/median/max {en.min():.1f} / {np.median(en):.1f} / "
          f"{en.max():.1f} us; SMs used {len(set(cta[:, 2].tolist()))}")
    order = np.argsort(-en)[:6]
    print("latest CTAs (block, sm, start, end us):", [(int(i), int(cta[i, 2]), round(float(st[i]), 1),
                                                        round(float(en[i]), 1)) for i in order])
