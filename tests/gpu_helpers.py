"""Builds matched (oracle, GPU) problem pairs from one ProblemSpec."""
import numpy as np

from oracle import pyoracle as po


def gpu_from_oracle(ob: "po.OracleProblem", spec: "po.ProblemSpec", **kw):
    from paper_2404_12063_b200.gpu import GpuStep
    pts = ob.array("points")
    return GpuStep(
        grad_x=ob.array("grad_x"), grad_y=ob.array("grad_y"), test=ob.array("test"),
        forcing=ob.array("forcing"), n_elem=ob.E, n_test=ob.T, n_quad=ob.Q, points=pts,
        n_interior=ob.n_int, n_boundary=ob.n_bnd, n_sensors=ob.n_sen,
        boundary_values=ob.array("boundary_values"), sensor_values=ob.array("sensor_values"),
        layer_sizes=spec.layers, sigmoid=spec.sigmoid, n_scalars=len(spec.scalars),
        eps=spec.eps, bx=spec.bx, by=spec.by, eps_source=spec.eps_source,
        eps_scalar_index=spec.eps_scalar_index, tau=spec.tau, gamma=spec.gamma, **kw)


def make_pair(spec, **kw):
    ob = po.OracleProblem(spec, double=False)
    g = gpu_from_oracle(ob, spec, **kw)
    p0 = ob.init_params().astype(np.float32)
    g.set_params(p0)
    return ob, g, p0


def c1_spec(**over):
    """BASELINE config C1: 8x8 unit square, 5x5 test fns, 10x10 Gauss, [2,30,30,30,1]."""
    nodes, cells = po.structured_mesh(8, 8)
    kw = dict(n_test_1d=5, n_quad_1d=10, forcing="sin2pi_f", boundary_g="sin2pi_u", n_boundary=400,
              boundary_seed=1, layers=(2, 30, 30, 30, 1), seed=42)
    kw.update(over)
    return po.ProblemSpec(nodes=nodes, cells=cells, **kw)
