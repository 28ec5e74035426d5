"""Pins the CPU oracle against the reference's own known-answer tests.

Each test names the reference Catch2 case it restates (paths relative to
reference proj/tests/).  The oracle is only trusted as a checker for the
GPU path because these pass.
"""
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.refutil import SplitMix, read_msh, synthetic_eval


def spec_for(nodes, cells, **kw):
    kw.setdefault("layers", (2, 4, 1))
    kw.setdefault("n_boundary", 8)
    return po.ProblemSpec(nodes=nodes, cells=cells, **kw)


def rel_diff(a, b):
    return abs(a - b) / max(1.0, abs(a), abs(b))


# --- quadrature: test_quadrature.cpp ---------------------------------------
def test_gauss_rules_integrate_monomials_exactly():
    for n in range(1, 12):
        x, w = po.gauss_rule(n, False)
        assert abs(w.sum() - 2.0) < 1e-13
        for d in range(2 * n):
            exact = 0.0 if d % 2 else 2.0 / (d + 1)
            assert abs((w * x ** d).sum() - exact) < 1e-12
    for n in range(2, 12):
        x, w = po.gauss_rule(n, True)
        assert x[0] == -1.0 and x[-1] == 1.0
        for d in range(2 * n - 2):
            exact = 0.0 if d % 2 else 2.0 / (d + 1)
            assert abs((w * x ** d).sum() - exact) < 1e-12


def test_test_functions_vanish_on_reference_boundary():
    # commands.hpp:437-445 / quadrature.hpp:58-67
    for k in range(1, 16):
        assert abs(po.test_fn(k, 1.0)[0]) < 1e-12
        assert abs(po.test_fn(k, -1.0)[0]) < 1e-12
    # v_1 = P2 - P0 = (3x^2-1)/2 - 1, v_1' = 3x
    v, d = po.test_fn(1, 0.5)
    assert abs(v - (-0.125 - 1.0)) < 1e-15 and abs(d - 1.5) < 1e-14


# --- fields: test_fields.cpp:68-119 ----------------------------------------
def test_frozen_field_values():
    pts = [(0.3, -0.7), (-0.9, 0.4), (0.123, 0.456), (0.5, 0.5)]
    x = np.array([p[0] for p in pts]); y = np.array([p[1] for p in pts])
    bu = [0.83795465658142076, 4.4005113640348021, 0.14947240275824694, 2.0554228099169483]
    bf = [-3.6748120922657339, 3.6892444093997918, -5.5722692578450213, -0.63394844031749031]
    vf = [-7.1487815397273984, -2.4163385481941435, 5.2475576570710274, 13.393133120955175]
    np.testing.assert_allclose(po.field("bump_u", x, y), bu, rtol=1e-14)
    np.testing.assert_allclose(po.field("bump_f", x, y), bf, rtol=1e-13)
    np.testing.assert_allclose(po.field("sinpi_vareps_f", x, y), vf, rtol=1e-13)
    assert abs(po.field("gear_f", 0.0, 9.0)[0] - 1.0) < 1e-15
    assert abs(po.field("gear_f", 0.7, -3.0)[0] - (50 * math.sin(0.7) + math.cos(0.7))) < 1e-13
    with pytest.raises(po.OracleError) as e:
        po.field("nope", 0.0, 0.0)
    assert e.value.code == 2


# --- network: test_network.cpp ---------------------------------------------
def test_parameter_count_and_glorot_bound():
    p = po.init_params_f64([2, 30, 30, 30, 1], 0)
    assert p.size == 1981
    a = po.init_params_f64([2, 30, 30, 1], 42)
    b = po.init_params_f64([2, 30, 30, 1], 42)
    c = po.init_params_f64([2, 30, 30, 1], 43)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    w0 = a[:60]
    assert np.abs(w0).max() <= math.sqrt(6.0 / 32) and np.abs(w0).max() > 0
    assert np.all(a[60:90] == 0.0)  # biases zero


def _one_unit(w11, w12, b1, w2, b2, double=True):
    nodes, cells = po.structured_mesh(1, 1)
    pb = po.OracleProblem(spec_for(nodes, cells, layers=(2, 1, 1), n_test_1d=1, n_quad_1d=2),
                          double=double)
    return pb, np.array([w11, w12, b1, w2, b2])


def test_one_unit_closed_form_values_and_derivatives():
    w11, w12, b1, w2, b2 = 0.7, -0.4, 0.2, 1.3, -0.5
    pb, par = _one_unit(w11, w12, b1, w2, b2)
    pts = np.array([[0.3, -0.8], [-1.1, 0.45], [2.0, 1.0]])
    u, ux, uy, _ = pb.evaluate(par, pts, 1)
    for i, (x, y) in enumerate(pts):
        z = math.tanh(w11 * x + w12 * y + b1)
        s1 = 1 - z * z
        assert abs(u[i] - (w2 * z + b2)) < 1e-14
        assert abs(ux[i] - w2 * s1 * w11) < 1e-14
        assert abs(uy[i] - w2 * s1 * w12) < 1e-14


def test_chunk_transparency_and_determinism():
    # test_network.cpp:238-255 — 1,300 points over three 512-point chunks
    nodes, cells = po.structured_mesh(1, 1)
    pb = po.OracleProblem(spec_for(nodes, cells, layers=(2, 16, 1), n_test_1d=1, n_quad_1d=2,
                                   seed=31), double=True)
    par = pb.init_params()
    r = SplitMix(7)
    pts = np.array([[r.uniform(-2, 2), r.uniform(-2, 2)] for _ in range(1300)])
    a = pb.evaluate(par, pts, 1)
    b = pb.evaluate(par, pts, 1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    s = pb.evaluate(par, pts[700:701], 1)
    assert abs(a[0][700] - s[0][0]) <= 4 * np.spacing(abs(s[0][0]))


# --- losses: test_losses.cpp ---------------------------------------------
def test_single_element_residual_hand_computation():
    # test_losses.cpp:48-87: residual -2, loss 4
    nodes, cells = po.structured_mesh(1, 1)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=1, n_quad_1d=2, forcing="const:3",
                                   eps=5.0, bx=1.0), double=True)
    Q = pb.Q
    for loop in (False, True):
        loss, res, *_ = pb.var_loss(np.full(Q, 1.0), np.full(Q, 2.0), loop=loop)
        assert res.shape == (1, 1)
        assert abs(res[0, 0] - (-2.0)) < 1e-12
        assert abs(loss - 4.0) < 1e-12


SCENARIOS = {
    "poisson": dict(eps=0.7),
    "cd2d": dict(eps=0.01, bx=0.8, by=-0.3),
    "scalar coefficient": dict(eps_source=1, eps_scalar_index=0, bx=0.4),
    "spatial coefficient": dict(eps_source=2, by=0.9),
}


@pytest.mark.parametrize("name", list(SCENARIOS))
def test_tensor_equals_loop_regular_mesh(name):
    # test_losses.cpp:89-156 (tensor vs general loop, 1e-12)
    sc = SCENARIOS[name]
    nodes, cells = po.structured_mesh(3, 3)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=3, n_quad_1d=4,
                                   forcing="tc_sin2x_plus_y", **sc), double=True)
    n = pb.E * pb.Q
    u, ux, uy, eps, scal = synthetic_eval(n, 99, sc.get("eps_source") == 2,
                                          1 if sc.get("eps_source") == 1 else 0)
    rt = pb.var_loss(ux, uy, eps, scal)
    rl = pb.var_loss(ux, uy, eps, scal, loop=True)
    assert rel_diff(rt[0], rl[0]) < 1e-12
    d = np.abs(rt[1] - rl[1]) / np.maximum(1.0, np.maximum(np.abs(rt[1]), np.abs(rl[1])))
    assert d.max() < 1e-12


def test_tensor_equals_loop_on_skewed_fixture(golden_dir):
    # test_losses.cpp:158-193 on the reference's skewed_12x12 fixture
    nodes, cells = read_msh(os.path.join(golden_dir, "meshes", "skewed_12x12_v22.msh"))
    assert cells.shape[0] == 144
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=2, n_quad_1d=3,
                                   forcing="tc_x2_minus_3y", eps=0.3, bx=1.1, by=0.2),
                          double=True)
    u, ux, uy, _, _ = synthetic_eval(pb.E * pb.Q, 7)
    rt = pb.var_loss(ux, uy)
    rg = pb.var_loss(ux, uy, loop=True)
    assert rel_diff(rt[0], rg[0]) < 1e-12
    d = np.abs(rt[1] - rg[1]) / np.maximum(1.0, np.maximum(np.abs(rt[1]), np.abs(rg[1])))
    assert d.max() < 1e-12
    # adjoints of the two kernels agree too
    np.testing.assert_allclose(rt[2], rg[2], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("kind", ["fixed", "scalar", "spatial"])
def test_variational_adjoints_match_finite_differences(kind):
    # test_losses.cpp:195-318 (weight 1.7, h=1e-6, tolerance 1e-6)
    sc = {"fixed": dict(eps=0.9, bx=-0.5, by=0.25),
          "scalar": dict(eps_source=1, eps_scalar_index=1),
          "spatial": dict(eps_source=2, bx=0.6)}[kind]
    nodes, cells = po.structured_mesh(2, 2, (-1.0, 1.0), (0.0, 1.0))
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=2, n_quad_1d=3,
                                   forcing="tc_cosx_plus_y", **sc), double=True)
    n = pb.E * pb.Q
    w, h = 1.7, 1e-6
    _, ux, uy, eps, scal = synthetic_eval(n, 1234, kind == "spatial", 2 if kind == "scalar" else 0)
    base = pb.var_loss(ux, uy, eps, scal, weight=w)
    pick = SplitMix(5)
    ok = lambda a, fd: abs(a - fd) <= 1e-6 or abs(a - fd) <= 1e-6 * abs(fd)
    for _ in range(8):
        p = pick.integer(n)
        for arr, adj in ((ux, base[2]), (uy, base[3])):
            ap, am = arr.copy(), arr.copy()
            ap[p] += h; am[p] -= h
            args_p = (ap, uy) if arr is ux else (ux, ap)
            args_m = (am, uy) if arr is ux else (ux, am)
            fd = (pb.var_loss(*args_p, eps, scal)[0] - pb.var_loss(*args_m, eps, scal)[0]) / (2 * h) * w
            assert ok(adj[p], fd)
        if kind == "spatial":
            ep, em = eps.copy(), eps.copy()
            ep[p] += h; em[p] -= h
            fd = (pb.var_loss(ux, uy, ep, scal)[0] - pb.var_loss(ux, uy, em, scal)[0]) / (2 * h) * w
            assert ok(base[4][p], fd)
    if kind == "scalar":
        sp, sm = list(scal), list(scal)
        sp[1] += h; sm[1] -= h
        fd = (pb.var_loss(ux, uy, None, sp)[0] - pb.var_loss(ux, uy, None, sm)[0]) / (2 * h) * w
        assert ok(base[5][1], fd) and base[5][0] == 0.0


def test_composite_parameter_gradient_matches_finite_differences():
    # test_losses.cpp:460-531: weak residual + boundary penalty, every param
    nodes, cells = po.structured_mesh(2, 2)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=2, n_quad_1d=3,
                                   forcing="tc_sin3x_minus_y", boundary_g="tc_sinx_times_y",
                                   n_boundary=16, boundary_seed=11, eps=0.8, bx=0.3,
                                   layers=(2, 8, 1), seed=21), double=True)
    p0 = pb.init_params()
    parts, g = pb.loss_and_grad(p0)
    assert abs(parts[0] - (parts[1] + 10 * parts[2])) <= 1e-13 * abs(parts[0])
    h = 1e-6
    for i in range(p0.size):
        pp, pm = p0.copy(), p0.copy()
        pp[i] += h; pm[i] -= h
        fd = (pb.loss_and_grad(pp)[0][0] - pb.loss_and_grad(pm)[0][0]) / (2 * h)
        assert abs(g[i] - fd) <= 1e-5 or abs(g[i] - fd) <= 1e-5 * abs(fd), i


def test_penalty_values_and_adjoints():
    # test_losses.cpp:320-345 via the composite objective: boundary-only batch
    nodes, cells = po.structured_mesh(2, 2)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=1, n_quad_1d=2,
                                   forcing="zero", boundary_g="tc_x_minus_y", n_boundary=8,
                                   boundary_seed=7), double=True)
    pts = pb.array("points")[pb.n_int:]
    vals = pb.array("boundary_values")
    np.testing.assert_array_equal(vals, pts[:, 0] - pts[:, 1])
    on_edge = (np.abs(pts[:, 0]) < 1e-12) | (np.abs(pts[:, 0] - 1) < 1e-12) | \
              (np.abs(pts[:, 1]) < 1e-12) | (np.abs(pts[:, 1] - 1) < 1e-12)
    assert on_edge.all()


# --- trainer: test_trainer.cpp ---------------------------------------------
def test_adam_scalar_trajectory():
    # test_trainer.cpp:85-106 (1e-15)
    g = np.array([[math.sin(0.9 * t) + 0.2] for t in range(1, 26)])
    pref, m, v = 0.7, 0.0, 0.0
    for t in range(1, 26):
        gt = g[t - 1, 0]
        m = 0.9 * m + 0.1 * gt
        v = 0.999 * v + 0.001 * gt * gt
        pref -= 3e-3 * (m / (1 - 0.9 ** t)) / (math.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        p = po.adam_f64([0.7], g[:t], 3e-3)
        assert abs(p[0] - pref) < 1e-15


def test_adam_first_step_is_signed_lr():
    # test_trainer.cpp:51-72
    for c in (1.0, 0.01, 3.0, 1e4):
        p = po.adam_f64([0.0], [[5.0 * c]], 1e-3)
        assert p[0] < 0 and 1e-3 * (1 - 1e-6) <= abs(p[0]) <= 1e-3
    p = po.adam_f64([1.0, 1.0], [[2.0, 0.0]], 1e-2)
    assert p[0] != 1.0 and p[1] == 1.0
    with pytest.raises(po.OracleError) as e:
        po.adam_f64([0.0, 0.0], [[1.0, float("nan")]], 1e-3)
    assert e.value.code == 4


def test_learning_rate_schedule():
    # test_trainer.cpp:126-143
    assert po.lr_at(1e-3, 0) == 1e-3 and po.lr_at(1e-3, 123456) == 1e-3
    assert abs(po.lr_at(0.005, 0, 0.99, 1000, True) - 0.005) < 1e-18
    assert abs(po.lr_at(0.005, 999, 0.99, 1000, True) - 0.005) < 1e-18
    assert abs(po.lr_at(0.005, 1000, 0.99, 1000, True) / 0.00495 - 1) < 1e-12
    assert abs(po.lr_at(0.005, 2000, 0.99, 1000, True) / 0.0049005 - 1) < 1e-12


def _tiny(nx=2, ny=2, nq=3, nt=2, layers=(2, 6, 1), seed=17, double=True, **kw):
    # test_trainer.cpp:13-35 tiny_problem (boundary seed 5, 40 points)
    nodes, cells = po.structured_mesh(nx, ny)
    return po.OracleProblem(spec_for(nodes, cells, n_test_1d=nt, n_quad_1d=nq,
                                     forcing="sin2pi_f", boundary_g="sin2pi_u", n_boundary=40,
                                     boundary_seed=5, layers=layers, seed=seed, **kw),
                            double=double)


def test_batch_layout():
    # test_trainer.cpp:154-162
    pb = _tiny()
    assert (pb.n_int, pb.n_bnd, pb.n_sen) == (36, 40, 0)
    pts = pb.array("points")
    assert pts.shape == (76, 2)


def test_training_history_bitwise_deterministic_and_decreasing():
    # test_trainer.cpp:201-218 and 220-238
    pb = _tiny()
    a = pb.train(pb.init_params(), 40, log_every=1)
    b = pb.train(pb.init_params(), 40, log_every=1)
    assert np.array_equal(a["every_step"], b["every_step"])
    pb2 = _tiny(nq=5, layers=(2, 10, 1), seed=29)
    r = pb2.train(pb2.init_params(), 400, lr0=5e-3)
    tot = r["every_step"][:, 0]
    assert tot[-50:].mean() < tot[:50].mean()
    # components compose to the total under the default weights
    np.testing.assert_allclose(tot, r["every_step"][:, 1] + 10 * r["every_step"][:, 2], rtol=1e-12)


def test_inverse_and_plateau_stops():
    # test_trainer.cpp:260-310 (validation stop; plateau stop)
    pb = _tiny(1, 1, 3, 1, layers=(2, 4, 1), seed=3, eps_source=1, scalars=(2.0,),
               n_sensors=10, sensor_seed=9, sensor_field="sin2pi_u")
    r = pb.train(pb.init_params(), 50, eps_abs_tol=10.0, eps_actual=0.3)
    assert r["steps_run"] == 1 and r["stop_reason"] == 1 and math.isfinite(r["final_eps"])
    pb2 = _tiny(1, 1, 3, 1, layers=(2, 4, 1), seed=3)
    r2 = pb2.train(pb2.init_params(), 200, loss_tol=0.999999, plateau_window=5)
    assert r2["stop_reason"] == 2 and r2["steps_run"] <= 10


# --- assembly: test_assembly.cpp ------------------------------------------
def test_constant_forcing_reaches_only_lowest_test_function():
    # test_assembly.cpp:107-121
    nodes, cells = po.structured_mesh(1, 1)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=4, n_quad_1d=8, forcing="one"),
                          double=True)
    f = pb.array("forcing")
    assert abs(f[0] - 1.0) < 1e-13 and np.abs(f[1:]).max() < 1e-13


def test_element_tensors_match_direct_evaluation():
    # test_assembly.cpp:50-83 on the single skewed element
    nodes = np.array([[0.0, 0.0], [1.0, 0.0], [1.5, 1.0], [0.0, 1.0]])
    cells = np.array([[0, 1, 2, 3]], dtype=np.int32)
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=3, n_quad_1d=4, forcing="one"),
                          double=True)
    assert (pb.E, pb.T, pb.Q) == (1, 9, 16)
    xi, eta, w = pb.array("rule")
    gx = pb.array("grad_x").reshape(9, 16)
    tv = pb.array("test").reshape(9, 16)
    n = nodes
    xc1 = 0.25 * (-n[0, 0] + n[1, 0] + n[2, 0] - n[3, 0]); xc2 = 0.25 * (-n[0, 0] - n[1, 0] + n[2, 0] + n[3, 0])
    xc3 = 0.25 * (n[0, 0] - n[1, 0] + n[2, 0] - n[3, 0]); yc1 = 0.25 * (-n[0, 1] + n[1, 1] + n[2, 1] - n[3, 1])
    yc2 = 0.25 * (-n[0, 1] - n[1, 1] + n[2, 1] + n[3, 1]); yc3 = 0.25 * (n[0, 1] - n[1, 1] + n[2, 1] - n[3, 1])
    for q in range(16):
        j11 = xc1 + xc3 * eta[q]; j12 = yc1 + yc3 * eta[q]
        j21 = xc2 + xc3 * xi[q]; j22 = yc2 + yc3 * xi[q]
        det = j11 * j22 - j12 * j21
        for j in range(9):
            jx, jy = j % 3, j // 3
            vx, dvx = po.test_fn(jx + 1, xi[q]); vy, dvy = po.test_fn(jy + 1, eta[q])
            a, e = dvx * vy, vx * dvy
            dvdx = (j22 * a - j12 * e) / det
            assert abs(gx[j, q] - w[q] * det * dvdx) <= 1e-14 * max(1.0, abs(gx[j, q]))
            assert abs(tv[j, q] - w[q] * det * vx * vy) <= 1e-14 * max(1.0, abs(tv[j, q]))


def test_tensor_layout_contract_k_j_q():
    # assembly.hpp:83-85,106 / test_assembly.cpp:308-341: entry (k,j,q) at (k*T+j)*Q+q
    nodes, cells = po.structured_mesh(2, 1, (0.0, 1.0), (0.0, 2.0))
    pb = po.OracleProblem(spec_for(nodes, cells, n_test_1d=2, n_quad_1d=3, forcing="one"),
                          double=True)
    gx = pb.array("grad_x")
    assert gx.size == 2 * 4 * 9
    # cell 1 is the translate of cell 0 on a uniform grid: identical slices
    np.testing.assert_array_equal(gx[:36], gx[36:])
    pts = pb.array("points")[: pb.n_int]
    assert pts[9, 0] >= 0.5 and pts[8, 0] < 0.5  # element-major point order


def test_sensor_sampling_deterministic():
    # test_assembly.cpp:288-306 — points inside the domain, seeded
    nodes, cells = po.structured_mesh(3, 3, (-1.0, 1.0), (-1.0, 1.0))
    mk = lambda s: po.OracleProblem(spec_for(nodes, cells, n_test_1d=1, n_quad_1d=2,
                                             forcing="one", n_sensors=50, sensor_seed=s,
                                             sensor_field="sin2pi_u"), double=True)
    a, b, c = mk(11), mk(11), mk(12)
    pa = a.array("points")[a.n_int + a.n_bnd:]
    assert pa.shape == (50, 2) and (np.abs(pa) < 1.0).all()
    assert np.array_equal(pa, b.array("points")[b.n_int + b.n_bnd:])
    assert not np.array_equal(pa, c.array("points")[c.n_int + c.n_bnd:])


# --- strong form (order 2): test_network.cpp, test_losses.cpp, acceptance --
def test_one_unit_closed_form_second_derivatives():
    # test_network.cpp:74-92 at order 2 (1e-14)
    w11, w12, b1, w2, b2 = 0.7, -0.4, 0.2, 1.3, -0.5
    pb, par = _one_unit(w11, w12, b1, w2, b2)
    pts = np.array([[0.3, -0.8], [-1.1, 0.45], [2.0, 1.0]])
    u, ux, uy, uxx, uyy = pb.evaluate2(par, pts)
    for i, (x, y) in enumerate(pts):
        z = math.tanh(w11 * x + w12 * y + b1)
        s1 = 1 - z * z
        s2 = -2.0 * z * s1
        assert abs(u[i] - (w2 * z + b2)) < 1e-14
        assert abs(ux[i] - w2 * s1 * w11) < 1e-14
        assert abs(uy[i] - w2 * s1 * w12) < 1e-14
        assert abs(uxx[i] - w2 * s2 * w11 * w11) < 1e-14
        assert abs(uyy[i] - w2 * s2 * w12 * w12) < 1e-14


def test_second_derivatives_match_finite_differences_of_u():
    # test_network.cpp:137-157 (1e-7 first, 1e-3 second derivatives)
    nodes, cells = po.structured_mesh(1, 1)
    pb = po.OracleProblem(spec_for(nodes, cells, layers=(2, 10, 8, 1), n_test_1d=1, n_quad_1d=2,
                                   seed=5), double=True)
    par = pb.init_params()
    h = 1e-6
    for x, y in ((0.2, 0.7), (-0.5, 0.1)):
        u, ux, uy, uxx, uyy = (a[0] for a in pb.evaluate2(par, [[x, y]]))
        f = lambda a, b: pb.evaluate(par, [[a, b]], 0)[0][0]
        assert abs(ux - (f(x + h, y) - f(x - h, y)) / (2 * h)) < 1e-7
        assert abs(uy - (f(x, y + h) - f(x, y - h)) / (2 * h)) < 1e-7
        assert abs(uxx - (f(x + h, y) - 2 * u + f(x - h, y)) / (h * h)) < 1e-3
        assert abs(uyy - (f(x, y + h) - 2 * u + f(x, y - h)) / (h * h)) < 1e-3


def test_strong_residual_value_and_adjoints():
    # test_losses.cpp:344-412: six points from Rng(42), scalar eps 0.8,
    # b = (0.5, -0.4), segment [1, 5)
    r = SplitMix(42)
    n = 6
    cols = {k: np.zeros(n) for k in ("u", "ux", "uy", "uxx", "uyy")}
    for i in range(n):
        for k in ("u", "ux", "uy", "uxx", "uyy"):
            cols[k][i] = r.uniform(-1, 1)
    fs = np.array([0.1, -0.2, 0.3, 0.0])
    args = dict(bx=0.5, by=-0.4, eps_source=1, eps_scalar_index=0, scalars=(0.8,))
    ev = [cols[k] for k in ("u", "ux", "uy", "uxx", "uyy")]
    got, uxb, uyb, uxxb, uyyb, sb = po.strong_loss(*ev, 1, 4, fs, **args)
    expect = 0.0
    for i in range(4):
        p = 1 + i
        P = -0.8 * (cols["uxx"][p] + cols["uyy"][p]) + 0.5 * cols["ux"][p] - 0.4 * cols["uy"][p] - fs[i]
        expect += P * P / 4.0
    assert abs(got - expect) <= 1e-14 * abs(expect)
    assert uxb[0] == 0.0  # outside the segment
    h = 1e-6
    for p in range(1, 5):
        ep = [a.copy() for a in ev]
        em = [a.copy() for a in ev]
        ep[3][p] += h
        em[3][p] -= h
        fd = (po.strong_loss(*ep, 1, 4, fs, **args)[0] - po.strong_loss(*em, 1, 4, fs, **args)[0]) / (2 * h)
        assert abs(uxxb[p] - fd) <= 1e-7
    ap = dict(args, scalars=(0.8 + h,))
    am = dict(args, scalars=(0.8 - h,))
    fd = (po.strong_loss(*ev, 1, 4, fs, **ap)[0] - po.strong_loss(*ev, 1, 4, fs, **am)[0]) / (2 * h)
    assert abs(sb[0] - fd) <= 1e-7
    with pytest.raises(po.OracleError):  # spatial coefficient rejected
        po.strong_loss(*ev, 1, 4, fs, eps_source=2)


def _strong_problem(**kw):
    # acceptance_main.cpp:111-160, case 4: 2x2 mesh, 4 quad / 3 test per dim,
    # 40 boundary points, weights 10/10, forcing 'one', g = 0, [2,12,12,1]
    nodes, cells = po.structured_mesh(2, 2)
    base = dict(n_test_1d=3, n_quad_1d=4, forcing="one", boundary_g="zero", n_boundary=40,
                layers=(2, 12, 12, 1), strong=True)
    base.update(kw)
    return po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells, **base), double=True)


@pytest.mark.parametrize("variant", ["acceptance", "convection_scalar_eps", "sigmoid"])
def test_strong_form_parameter_gradient_matches_finite_differences(variant):
    # acceptance_main.cpp:171-214 criterion 2 (rel 1e-4, floor 1e-8) on the
    # strong-form case, plus convection / trainable eps / sigmoid variants
    kw = {"acceptance": {},
          # constant forcing keeps P = O(1), above the finite-difference
          # noise floor (acceptance_main.cpp:156-157)
          "convection_scalar_eps": dict(bx=0.6, by=-0.3, eps_source=1, scalars=(1.3,),
                                        n_sensors=6, sensor_field="sin2pi_u"),
          "sigmoid": dict(sigmoid=True, layers=(2, 7, 6, 5, 1))}[variant]
    pb = _strong_problem(**kw)
    f = pb.array("strong_forcing")
    pts = pb.array("points")[: pb.n_int]
    np.testing.assert_array_equal(f, po.field("one", pts[:, 0], pts[:, 1]))
    p0 = pb.init_params()
    parts, g = pb.loss_and_grad(p0)
    assert abs(parts[0] - (parts[1] + 10 * parts[2] + 10 * parts[3])) <= 1e-13 * abs(parts[0])
    worst = 0.0
    for i in range(p0.size):
        step = 1e-6 * max(1.0, abs(p0[i]))
        pp, pm = p0.copy(), p0.copy()
        pp[i] += step
        pm[i] -= step
        fd = (pb.loss_and_grad(pp)[0][0] - pb.loss_and_grad(pm)[0][0]) / (2 * step)
        allowed = max(1e-4 * max(abs(g[i]), abs(fd)), 1e-8)
        worst = max(worst, abs(g[i] - fd) / allowed)
    assert worst <= 1.0, worst


def test_strong_residual_is_mean_square_of_pointwise_operator():
    # trainer.hpp:246-248 + losses.hpp:446-455 recomputed from evaluate(order 2)
    pb = _strong_problem(bx=0.6, by=-0.3, eps=0.7, forcing="sin2pi_f")
    p0 = pb.init_params()
    parts, _ = pb.loss_and_grad(p0)
    pts = pb.array("points")[: pb.n_int]
    u, ux, uy, uxx, uyy = pb.evaluate2(p0, pts)
    f = pb.array("strong_forcing")
    P = -0.7 * (uxx + uyy) + 0.6 * ux - 0.3 * uy - f
    assert abs(parts[1] - np.mean(P * P)) <= 1e-12 * parts[1]


# ---------------------------------------------------------------------------
# the committed parity fixtures (tests/golden/parity/*.npz) belong to this
# oracle: the epoch-1 record of each fixture's 100-epoch run is the loss at
# p0, and the fp32 gradient is the oracle's, bit for bit
@pytest.mark.parametrize("case", ["c5_gear", "c5_inverse", "c5_paper", "c2_4096", "c3_t10_q40"])
def test_parity_fixture_is_this_oracles_output(case):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import parity_cases as pc
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "parity", case + ".npz"))
    ob = po.OracleProblem(pc.CASES[case](), double=False)
    p0 = ob.init_params().astype(np.float32)
    assert np.array_equal(p0.view(np.uint32), fx["p0"].view(np.uint32))
    parts, grad = ob.loss_and_grad(p0)
    assert np.array_equal(parts, fx["traj32"][0])
    assert np.array_equal(grad.view(np.uint32), fx["grad32"].view(np.uint32))
    assert fx["traj32"].shape == (pc.EPOCHS, 4) and np.all(np.isfinite(fx["traj32"]))
    assert fx["traj64"].shape == (pc.EPOCHS, 4) and np.all(np.isfinite(fx["traj64"]))
    assert np.allclose(fx["traj64"][0], fx["parts64"], rtol=1e-14, atol=0.0)  # epoch 1 = the loss at p0
    assert fx["traj32"][-1, 0] < fx["traj32"][0, 0]


def test_pure_python_gear_is_the_reference_recipe(golden_dir):
    """oracle/pyoracle.gear_mesh (used by bench.py's CPU legs so they load no
    product code) writes the reference generator's bytes (SHA-256 pinned from
    proj/data/gen_fixtures.py) and parses to the 14,192-cell C5 gear."""
    import hashlib
    import json
    info = json.load(open(os.path.join(golden_dir, "gear_14192.json")))["gear_14192"]
    text = po.gear_msh41_text(16, 887)
    assert hashlib.sha256(text.encode()).hexdigest() == info["sha256"]
    nodes, cells = po.gear_mesh(16, 887)
    assert nodes.shape == (17 * 887, 2) and cells.shape == (14192, 4)
    assert cells.min() == 0 and cells.max() == 17 * 887 - 1
    small_n, small_c = po.gear_mesh(6, 96)
    ref_n, ref_c = read_msh(os.path.join(golden_dir, "meshes", "gearlike_v41.msh"))
    assert np.array_equal(small_n.view(np.uint64), ref_n.view(np.uint64))
    assert np.array_equal(small_c, ref_c)
