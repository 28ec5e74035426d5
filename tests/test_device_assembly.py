"""Device-side premultiplier assembly: a context built
from the mesh (vpinn_gpu_create with a vpinn_gpu_assembly input) must hold
byte-identical tensors / forcing / points to a context uploaded from the
host assembly (reference assembly.hpp:58-135), and therefore compute the
same bits."""
import ctypes as C

import numpy as np
import pytest

from paper_2404_12063_b200 import _capi, host

pytestmark = pytest.mark.gpu

GEAR_CFG = {
    "problem": {"pde": {"type": "cd2d", "eps": 1.0, "b": [0.1, 0.0]}, "forcing": "gear_f",
                "boundary_g": "zero", "n_boundary_points": 800},
    "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 5},
    "network": {"layers": [2, 30, 30, 30, 1]},
    "training": {"iterations": 10, "learning_rate": 1e-3, "seed": 42, "precision": "single"},
}
C1_CFG = {
    "problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 400},
    "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
    "network": {"layers": [2, 30, 30, 30, 1]},
    "training": {"iterations": 10, "learning_rate": 1e-3, "seed": 42, "precision": "single"},
}
CASES = {
    "gear_cd2d": (GEAR_CFG, lambda: host.Mesh.gear(4, 120)),
    "c1_square": (C1_CFG, lambda: host.Mesh.structured(8, 8)),
    "skewed_sigmoid": ({**C1_CFG, "network": {"layers": [2, 16, 1], "activation": "sigmoid"},
                        "discretization": {"n_test_per_dim": 3, "n_quad_per_dim": 6}},
                       lambda: host.Mesh.structured(12, 12, skew=0.2)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_device_assembly_is_bit_identical_to_host(name):
    cfg, mk = CASES[name]
    mesh = mk()
    hp = host.HostProblem(cfg, mesh=mesh)
    dp = host.HostProblem(cfg, mesh=mesh, device_assembly=True)
    assert (hp.E, hp.T, hp.Q, hp.n_int, hp.n_bnd) == (dp.E, dp.T, dp.Q, dp.n_int, dp.n_bnd)
    g_host, g_dev = hp.gpu(), dp.gpu()
    E, T, Q = hp.E, hp.T, hp.Q
    for which, n in ((0, E * T * Q), (1, E * T * Q), (3, E * T)):
        a, b = g_host.download_tensor(which, n), g_dev.download_tensor(which, n)
        assert a.tobytes() == b.tobytes(), (which, int(np.sum(a != b)))
    pa, ga = g_host.loss_and_grad()
    pb, gb = g_dev.loss_and_grad()
    assert np.array_equal(pa, pb) and np.array_equal(ga, gb)


def test_device_assembly_convection_test_tensor_and_training():
    """cd2d keeps the test tensor on the device; 20 epochs trained from a
    device-assembled context follow the host-assembled one bit for bit."""
    cfg, mk = CASES["gear_cd2d"]
    mesh = mk()
    hp = host.HostProblem(cfg, mesh=mesh)
    dp = host.HostProblem(cfg, mesh=mesh, device_assembly=True)
    g_host, g_dev = hp.gpu(), dp.gpu()
    n = hp.E * hp.T * hp.Q
    assert g_host.download_tensor(2, n).tobytes() == g_dev.download_tensor(2, n).tobytes()
    ra, rb = g_host.train(20), g_dev.train(20)
    assert np.array_equal(ra.records["total"], rb.records["total"])
    assert np.array_equal(g_host.get_params(), g_dev.get_params())


def test_device_assembly_rejects_degenerate_cell():
    """A clockwise cell has a negative Jacobian determinant: mesh error (3),
    like DegenerateElementError (assembly.hpp:75-81)."""
    nodes = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    cells = np.array([[0, 3, 2, 1]], np.int32)  # clockwise
    xi = np.array([0.0]); eta = np.array([0.0]); w = np.array([4.0])
    basis = (np.ones(1), np.zeros(1), np.zeros(1))
    from paper_2404_12063_b200.gpu import GpuStep
    with pytest.raises(_capi.VpinnError) as e:
        GpuStep.assemble(nodes, cells, (xi, eta, w), basis, "one")
    assert e.value.code == 3
    cells = np.array([[0, 1, 2, 3]], np.int32)
    out = GpuStep.assemble(nodes, cells, (xi, eta, w), basis, "one")
    # unit square, one point at the centre: det = 1/4, w det v = 1, forcing = 1 * f(0.5, 0.5) = 1
    assert out["test"][0] == 1.0 and out["forcing"][0] == 1.0
    assert np.allclose(out["quad_points"][0], [0.5, 0.5])


@pytest.mark.parametrize("world", [2, 3])
def test_device_assembly_partitions_like_the_upload(world):
    """Rank r of W assembles only its contiguous cells [floor(rE/W), floor((r+1)E/W))."""
    from paper_2404_12063_b200.gpu import GpuStep
    cfg, mk = CASES["gear_cd2d"]
    mesh = mk()
    hp = host.HostProblem(cfg, mesh=mesh)
    dp = host.HostProblem(cfg, mesh=mesh, device_assembly=True)
    for r in range(world):
        a = GpuStep.from_problem(hp.view(0, r, world), keepalive=hp)
        b = GpuStep.from_problem(dp.view(0, r, world), keepalive=dp)
        part = _capi.partition(hp.E, hp.n_bnd, hp.n_sen, r, world)
        E = part[1] - part[0]
        for which, n in ((0, E * hp.T * hp.Q), (2, E * hp.T * hp.Q), (3, E * hp.T)):
            assert a.download_tensor(which, n).tobytes() == b.download_tensor(which, n).tobytes()
        a.set_params(hp.init_params())
        b.set_params(hp.init_params())
        pa, ga = a.loss_and_grad()
        pb, gb = b.loss_and_grad()
        assert np.array_equal(pa, pb) and np.array_equal(ga, gb)


@pytest.mark.parametrize("name", ["gear_cd2d", "c1_square"])
def test_matrix_free_contraction_matches_the_tensor_contraction(name):
    """Algorithm 3 from the basis tables + per-cell
    geometry equals Algorithm 3 on the premultiplier tensors to fp32
    rounding (loss 1e-5 relative; residuals / adjoints 1e-5 of their max)."""
    cfg, mk = CASES[name]
    dp = host.HostProblem(cfg, mesh=mk(), device_assembly=True)
    g = dp.gpu()
    rng = np.random.default_rng(3)
    ni = dp.E * dp.Q
    ux = rng.standard_normal(ni).astype(np.float32)
    uy = rng.standard_normal(ni).astype(np.float32)
    l1, r1, xb1, yb1, _, _ = g.contract(ux, uy)
    l2, r2, xb2, yb2, _ = g.contract_matrix_free(ux, uy)
    assert abs(l1 - l2) / abs(l1) < 1e-5
    for a, b in ((r1, r2), (xb1, xb2), (yb1, yb2)):
        assert np.abs(a - b).max() / np.abs(a).max() < 1e-5
    ms, nbytes = g.time_contract_matrix_free(3)
    assert ms > 0 and nbytes > 0


@pytest.mark.parametrize("name", ["gear_cd2d", "c1_square"])
def test_matrix_free_contraction_matches_the_oracle(name):
    """SURVEY 8f rank 3 against the CPU oracle's variational_loss_tensor
    (losses.hpp:91-168) on the same cells and derivatives: loss 1e-5
    relative, residuals / adjoints within 1e-5 of their max (fp32 rounding of
    a different factorisation of the same sums)."""
    from oracle import pyoracle as po
    cfg, mk = CASES[name]
    mesh = mk()
    nodes, cells, _ = mesh.arrays()
    pde = cfg["problem"].get("pde", {})
    b = pde.get("b", [0.0, 0.0])
    disc = cfg["discretization"]
    spec = po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=disc["n_test_per_dim"],
                          n_quad_1d=disc["n_quad_per_dim"], forcing=cfg["problem"]["forcing"],
                          boundary_g=cfg["problem"]["boundary_g"],
                          n_boundary=cfg["problem"]["n_boundary_points"], eps=pde.get("eps", 1.0),
                          bx=b[0], by=b[1], layers=(2, 30, 30, 30, 1), seed=42)
    ob = po.OracleProblem(spec, double=False)
    dp = host.HostProblem(cfg, mesh=mesh, device_assembly=True)
    g = dp.gpu()
    rng = np.random.default_rng(5)
    ni = dp.E * dp.Q
    assert ni == ob.E * ob.Q
    ux = rng.standard_normal(ni).astype(np.float32)
    uy = rng.standard_normal(ni).astype(np.float32)
    lo, ro, xbo, ybo, _, _ = ob.var_loss(ux, uy, None, (), weight=1.0)
    lm, rm, xbm, ybm, _ = g.contract_matrix_free(ux, uy)
    assert abs(lm - lo) / abs(lo) < 1e-5
    for a, r in ((rm, ro), (xbm, xbo), (ybm, ybo)):
        a = np.asarray(a).reshape(-1)
        r = np.asarray(r).reshape(-1)
        assert np.abs(a - r).max() / np.abs(r).max() < 1e-5


def test_matrix_free_contraction_needs_the_geometry():
    cfg, mk = CASES["c1_square"]
    hp = host.HostProblem(cfg, mesh=mk())
    g = hp.gpu()
    ni = hp.E * hp.Q
    with pytest.raises(_capi.VpinnError) as e:
        g.contract_matrix_free(np.zeros(ni), np.zeros(ni))
    assert e.value.code == 2


def test_pinned_input_upload_is_bit_identical():
    """vpinn_gpu_create DMAs page-locked caller arrays directly (no staging
    ring): the uploaded bytes, the loss / gradient and a 10-epoch history are
    identical to the staged upload of the same pageable arrays.  The gear is
    large enough (3 x 9.4 MB tensors) that both go through the chunked path."""
    from paper_2404_12063_b200 import gpu as G
    cfg = GEAR_CFG
    hp = host.HostProblem(cfg, mesh=host.Mesh.gear(8, 470))
    E, T, Q = hp.E, hp.T, hp.Q
    assert 4 * E * T * Q >= 4 << 20
    pv, keep = G.pin_problem(hp.view(0))
    g_page = G.GpuStep.from_problem(hp.view(0), keepalive=hp)
    g_pin = G.GpuStep.from_problem(pv, keepalive=(hp, keep))
    for which, n in ((0, E * T * Q), (1, E * T * Q), (2, E * T * Q), (3, E * T)):
        a, b = g_page.download_tensor(which, n), g_pin.download_tensor(which, n)
        assert a.tobytes() == b.tobytes(), (which, int(np.sum(a != b)))
    p0 = hp.init_params()
    for g in (g_page, g_pin):
        g.set_params(p0)
    la, ga = g_page.loss_and_grad()
    lb, gb = g_pin.loss_and_grad()
    assert np.array_equal(la, lb) and np.array_equal(ga, gb)
    ra, rb = g_page.train(10), g_pin.train(10)
    assert np.array_equal(ra.records["total"], rb.records["total"])
    assert np.array_equal(g_page.get_params(), g_pin.get_params())
    # rank 1 of 2: the upload starts inside the page-locked allocation
    pv1, keep1 = G.pin_problem(hp.view(0, 1, 2))
    r_page = G.GpuStep.from_problem(hp.view(0, 1, 2), keepalive=hp)
    r_pin = G.GpuStep.from_problem(pv1, keepalive=(hp, keep1))
    e0, e1 = _capi.partition(E, hp.n_bnd, hp.n_sen, 1, 2)[:2]
    n = (e1 - e0) * T * Q
    for which in (0, 1, 2):
        assert r_page.download_tensor(which, n).tobytes() == r_pin.download_tensor(which, n).tobytes()
