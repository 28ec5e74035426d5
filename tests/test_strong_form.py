"""Strong-form collocation on the GPU against the oracle.

The oracle's strong form is pinned by the reference's order-2 / strong-residual
known answers (tests/test_oracle_golden.py).  Here the B200 kernels -- the
tcgen05 step (sf2_step_kernel.cuh, fp16 split) for 2-3 hidden layers of width
<= 31 and the warp-tiled mma.sync one (sf_step_kernel.cuh, 3xTF32) for the
other shapes -- must reproduce, on the same inputs:
order-2 evaluate(), the composite objective and its gradient, and a 100-epoch
training trajectory (loss within 1e-5 relative per epoch, the north-star
tolerance).  CPU-side tests check the host plumbing only.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.refutil import read_msh

GOLD = os.path.join(os.path.dirname(__file__), "golden", "meshes")


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-30)


def strong_spec(mesh=(4, 4), **over):
    nodes, cells = po.structured_mesh(*mesh)
    kw = dict(n_test_1d=3, n_quad_1d=5, forcing="sin2pi_f", boundary_g="sin2pi_u", n_boundary=120,
              layers=(2, 30, 30, 30, 1), seed=42, strong=True)
    kw.update(over)
    return po.ProblemSpec(nodes=nodes, cells=cells, **kw)


def make_strong_pair(spec, **kw):
    from paper_2404_12063_b200.gpu import GpuStep
    ob = po.OracleProblem(spec, double=False)
    g = GpuStep(grad_x=None, grad_y=None, test=None, forcing=None, n_elem=ob.E, n_test=ob.T,
                n_quad=ob.Q, points=ob.array("points"), n_interior=ob.n_int, n_boundary=ob.n_bnd,
                n_sensors=ob.n_sen, boundary_values=ob.array("boundary_values"),
                sensor_values=ob.array("sensor_values"), layer_sizes=spec.layers,
                sigmoid=spec.sigmoid, n_scalars=len(spec.scalars), eps=spec.eps, bx=spec.bx,
                by=spec.by, eps_source=spec.eps_source, eps_scalar_index=spec.eps_scalar_index,
                tau=spec.tau, gamma=spec.gamma,
                strong_forcing=ob.array("strong_forcing").astype(np.float32), **kw)
    p0 = ob.init_params().astype(np.float32)
    g.set_params(p0)
    return ob, g, p0


def expected_kernel(spec):
    hidden = spec.layers[1:-1]
    return "sf2_step_kernel" if len(hidden) in (2, 3) and max(hidden) <= 31 else "sf_step_kernel<"


CASES = {
    "poisson_d3": lambda: strong_spec(),
    "acceptance_case4": lambda: strong_spec(mesh=(2, 2), n_test_1d=3, n_quad_1d=4, forcing="one",
                                            boundary_g="zero", n_boundary=40, layers=(2, 12, 12, 1)),
    "cd2d_sensors_scalar_eps": lambda: strong_spec(bx=0.7, by=-0.4, eps_source=1, scalars=(1.5,),
                                                   n_sensors=37, sensor_field="sin2pi_u",
                                                   layers=(2, 20, 20, 1)),
    "sigmoid_d3_ragged": lambda: strong_spec(mesh=(3, 5), layers=(2, 7, 13, 5, 1), sigmoid=True,
                                             n_boundary=33, eps=0.6),
    "one_hidden": lambda: strong_spec(layers=(2, 24, 1), bx=0.3),
    "four_hidden": lambda: strong_spec(layers=(2, 16, 16, 16, 16, 1), forcing="one",
                                       boundary_g="zero"),
    "gear_many_tiles": lambda: po.ProblemSpec(
        *read_msh(os.path.join(GOLD, "gearlike_v41.msh")), n_test_1d=5, n_quad_1d=5, forcing="gear_f",
        boundary_g="zero", n_boundary=800, eps=1.0, bx=0.1, layers=(2, 30, 30, 30, 1), seed=42,
        strong=True),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_strong_loss_and_gradient_match_oracle(name):
    spec = CASES[name]()
    ob, g, p0 = make_strong_pair(spec)
    assert expected_kernel(spec) in g.step_kernel()
    parts_o, go32 = ob.loss_and_grad(p0)
    parts_g, grad_g = g.loss_and_grad()
    assert rel(parts_g[0], parts_o[0]) < 1e-5, (parts_g, parts_o)
    for k in (1, 2, 3):
        if parts_o[k] != 0.0:
            assert rel(parts_g[k], parts_o[k]) < 1e-5, (k, parts_g, parts_o)
    o64 = po.OracleProblem(spec, double=True)
    _, g64 = o64.loss_and_grad(p0.astype(np.float64))
    err = np.abs(grad_g - g64).max() / np.abs(g64).max()
    e32 = np.abs(go32 - g64).max() / np.abs(g64).max()
    assert err < max(1e-5, 4.0 * e32), (err, e32)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["poisson_d3", "sigmoid_d3_ragged", "four_hidden"])
def test_order2_evaluate_matches_oracle(name):
    spec = CASES[name]()
    ob, g, p0 = make_strong_pair(spec)
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1.2, 1.2, size=(2001, 2))
    ref = ob.evaluate2(p0, pts)
    got = g.forward2(pts)
    for a, b in zip(got, ref):
        assert np.abs(a - b).max() <= 3e-5 * max(1.0, np.abs(b).max())
    # order 0/1 through the same kernel
    u, ux, uy, _ = g.forward(pts, 1)
    assert np.array_equal(u, got[0]) and np.array_equal(ux, got[1]) and np.array_equal(uy, got[2])


@pytest.mark.gpu
def test_strong_training_trajectory_matches_oracle():
    """Per-epoch loss within 1e-5 relative over 100 epochs (north-star tolerance)."""
    spec = CASES["cd2d_sensors_scalar_eps"]()
    ob, g, p0 = make_strong_pair(spec)
    ref = ob.train(p0, 100, lr0=1e-3, log_every=1)
    rep = g.train(100, lr0=1e-3)
    assert rep.steps_run == 100
    tot_o = ref["every_step"][:, 0]
    r = np.abs(rep.records["total"] - tot_o) / np.abs(tot_o)
    assert r.max() < 1e-5, (r.max(), int(r.argmax()))
    assert np.abs(g.get_params() - ref["params"]).max() < 1e-4
    assert abs(rep.final_eps - ref["final_eps"]) < 1e-5


@pytest.mark.gpu
def test_strong_fresh_contexts_are_bitwise_identical():
    spec = CASES["gear_many_tiles"]()
    _, g1, _ = make_strong_pair(spec)
    _, g2, _ = make_strong_pair(spec)
    a, ga = g1.loss_and_grad()
    b, gb = g2.loss_and_grad()
    assert np.array_equal(a, b) and np.array_equal(ga, gb)


@pytest.mark.gpu
def test_strong_rank_partition_sums_to_whole():
    """Two rank sub-contexts on one device: parts and gradients add up."""
    spec = CASES["cd2d_sensors_scalar_eps"]()
    ob, g, p0 = make_strong_pair(spec)
    whole, gw = g.loss_and_grad()
    acc = np.zeros(4)
    gacc = np.zeros_like(gw)
    for r in range(2):
        _, gr, _ = make_strong_pair(spec, rank=r, world_size=2)
        pr, grr = gr.loss_and_grad()
        acc += pr
        gacc += grr
    assert np.allclose(acc, whole, rtol=1e-5)
    assert np.abs(gacc - gw).max() <= 1e-5 * np.abs(gw).max()


@pytest.mark.gpu
def test_strong_rejects_unsupported_shapes():
    from paper_2404_12063_b200._capi import VpinnError
    with pytest.raises(VpinnError) as e:
        make_strong_pair(strong_spec(layers=(2, 40, 1)))
    assert e.value.code == 2
    with pytest.raises(VpinnError) as e:
        make_strong_pair(strong_spec(layers=(2, 16, 2), eps_source=2))
    assert e.value.code == 4


@pytest.mark.gpu
def test_strong_form_through_host_pipeline_and_device_assembly():
    """form: strong from a config (the C++ host pipeline's view) against the
    same problem with the device assembling the points and f at them."""
    from paper_2404_12063_b200 import host
    cfg = {"problem": {"pde": {"type": "cd2d", "eps": 0.8, "b": [0.3, -0.2]}, "forcing": "sin2pi_f",
                       "boundary_g": "sin2pi_u", "n_boundary_points": 96},
           "discretization": {"form": "strong", "n_test_per_dim": 3, "n_quad_per_dim": 5},
           "network": {"layers": [2, 24, 24, 1]},
           "training": {"learning_rate": 1e-3, "seed": 3, "precision": "single"}}
    mesh = host.Mesh.structured(6, 5, skew=0.2)
    hp = host.HostProblem(cfg, mesh=mesh)
    dp = host.HostProblem(cfg, mesh=mesh, device_assembly=True)
    gh, gd = hp.gpu(), dp.gpu()
    assert "step_kernel" in gh.step_kernel() and gh.step_kernel() == gd.step_kernel()
    ph, grh = gh.loss_and_grad()
    pd, grd = gd.loss_and_grad()
    assert np.abs(ph - pd).max() <= 1e-6 * np.abs(ph).max(), (ph, pd)
    assert np.abs(grh - grd).max() <= 1e-6 * np.abs(grh).max()
    # the host view against the oracle on the same mesh
    nodes, cells, _ = mesh.arrays()
    spec = po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=3, n_quad_1d=5, forcing="sin2pi_f",
                          boundary_g="sin2pi_u", n_boundary=96, eps=0.8, bx=0.3, by=-0.2,
                          layers=(2, 24, 24, 1), seed=3, strong=True)
    ob = po.OracleProblem(spec, double=False)
    po_, _ = ob.loss_and_grad(hp.init_params())
    assert rel(ph[0], po_[0]) < 1e-5
    rep = gd.train(20, lr0=1e-3)
    ref = ob.train(hp.init_params(), 20, lr0=1e-3, log_every=1)
    r = np.abs(rep.records["total"] - ref["every_step"][:, 0]) / np.abs(ref["every_step"][:, 0])
    assert r.max() < 1e-5


@pytest.mark.gpu
def test_weak_only_entry_points_reject_strong_contexts():
    from paper_2404_12063_b200._capi import VpinnError
    _, g, _ = make_strong_pair(CASES["acceptance_case4"]())
    with pytest.raises(VpinnError) as e:
        g.contract(np.zeros(g.n_elem * g.n_quad, np.float32), np.zeros(g.n_elem * g.n_quad, np.float32))
    assert e.value.code == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["poisson_d3", "cd2d_sensors_scalar_eps", "gear_many_tiles"])
@pytest.mark.parametrize("mode", ["mma_sync", "tc_spill"])
def test_strong_alternate_kernels_match_oracle(name, mode):
    """The warp-tiled mma.sync strong-form kernel on shapes the tcgen05 one
    serves, and the tcgen05 kernel's accumulator spill path forced every
    tile (vpinn_gpu_set_test_hooks): same parity bar."""
    from paper_2404_12063_b200 import _capi
    L = _capi.lib()
    _capi.check(L.vpinn_gpu_set_test_hooks(1 if mode == "mma_sync" else 2))
    try:
        spec = CASES[name]()
        ob, g, p0 = make_strong_pair(spec)
        assert ("sf2_step" in g.step_kernel()) == (mode == "tc_spill"), g.step_kernel()
        parts_o, go32 = ob.loss_and_grad(p0)
        parts_g, grad_g = g.loss_and_grad()
        assert rel(parts_g[0], parts_o[0]) < 1e-5, (parts_g, parts_o)
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        err = np.abs(grad_g - g64).max() / np.abs(g64).max()
        e32 = np.abs(go32 - g64).max() / np.abs(g64).max()
        assert err < max(1e-5, 4.0 * e32), (err, e32)
    finally:
        _capi.check(L.vpinn_gpu_set_test_hooks(0))


@pytest.mark.gpu
@pytest.mark.parametrize("layers", [(2, 30, 1), (2, 17, 7, 8, 9, 1), (2, 32, 32, 1)])
def test_strong_training_on_the_mma_sync_step_matches_oracle(layers):
    """train() through the mma.sync strong-form step (1 or 4 hidden layers,
    width 32): every epoch runs (the epoch tail reads the trainer state it
    updates; a step kernel that released the tail before its own wait once
    let it read a stale step count and skip epochs) and the history follows
    the oracle's."""
    spec = strong_spec(mesh=(6, 5), n_test_1d=2, n_quad_1d=6, layers=layers, bx=0.3, n_boundary=80)
    ob, g, p0 = make_strong_pair(spec)
    assert "sf_step_kernel<" in g.step_kernel(), g.step_kernel()
    ref = ob.train(p0, 12, lr0=1e-3, log_every=1)["every_step"][:, 0]
    ref64 = po.OracleProblem(spec, double=True).train(p0.astype(np.float64), 12, lr0=1e-3,
                                                       log_every=1)["every_step"][:, 0]
    rep = g.train(12, lr0=1e-3)
    assert rep.steps_run == 12
    r = np.abs(rep.records["total"] - ref) / np.abs(ref)
    floor = np.abs(ref64 - ref) / np.abs(ref)
    assert r.max() < max(1e-5, 2.0 * floor.max()), (r.max(), floor.max())
