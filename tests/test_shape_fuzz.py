"""Parity over a grid of discretisations and network shapes (the GPU kernel
the context selects for each: tensor-core step, CUDA-core step, split path):
n_test x n_quad per dimension from 1x1 to 8x13 (Q > 128 takes the split
path), 1 to 63 cells, uniform / ragged / one-layer / two-output networks,
tanh and sigmoid, with and without convection.  Found: ragged widths on the
tensor-core step, a loss race for many small cells per tile, a misaligned
mbarrier in the row-chunked contraction, the bf16 kernel at Q = 1."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.gpu_helpers import make_pair

pytestmark = pytest.mark.gpu

PAIRS = [(1, 1), (1, 3), (2, 2), (3, 7), (6, 6), (2, 12), (8, 13)]
MESHES = [(1, 1), (2, 3), (9, 7)]
NETS = [(2, 30, 30, 30, 1), (2, 17, 1), (2, 24, 11, 1), (2, 16, 16, 16, 2)]


@pytest.mark.parametrize("scalar", [False, True])
@pytest.mark.parametrize("pair", PAIRS)
def test_shape_grid_matches_oracle(pair, scalar):
    """scalar: a trainable coefficient and sensors on the one-output networks"""
    nt, nq = pair
    fails = []
    for mesh, layers, sig, conv in itertools.product(MESHES, NETS, [False, True], [False, True]):
        kw = dict(eps_source=2, bx=0.5) if layers[-1] == 2 else dict(bx=0.3 if conv else 0.0)
        if scalar and layers[-1] == 1:
            kw.update(eps_source=1, scalars=(1.3,), n_sensors=11, sensor_field="sin2pi_u")
        fx = "sinpi_vareps_f" if layers[-1] == 2 else "sin2pi_f"
        spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing=fx,
                              boundary_g="sin2pi_u", n_boundary=37, layers=layers, sigmoid=sig, seed=5, **kw)
        ob, g, p0 = make_pair(spec)
        po_, go32 = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        ge = np.abs(gg - g64).max() / max(np.abs(g64).max(), 1e-30)
        # gradient: 1e-5 of max|g| against fp64, or 4x the fp32 oracle's own
        # distance from fp64 where that noise floor is higher (tiny problems)
        e32 = np.abs(go32 - g64).max() / max(np.abs(g64).max(), 1e-30)
        if lr > 1e-5 or ge > max(1e-5, 4.0 * e32):
            fails.append((mesh, layers, sig, conv, g.step_kernel(), lr, ge))
        g.close()
    assert not fails, fails


@pytest.mark.parametrize("layers", NETS + [(2, 7, 13, 5, 1), (2, 50, 50, 50, 1)])
@pytest.mark.parametrize("sig", [False, True])
def test_evaluate_grid_matches_oracle(layers, sig):
    """evaluate(order 0 / 1) at arbitrary points through whichever forward
    kernel the context selects (tensor-core forward mode or CUDA cores)."""
    kw = dict(eps_source=2, bx=0.5, forcing="sinpi_vareps_f") if layers[-1] == 2 else {}
    spec = po.ProblemSpec(*po.structured_mesh(2, 2), n_test_1d=3, n_quad_1d=4, boundary_g="sin2pi_u",
                          n_boundary=20, layers=layers, sigmoid=sig, seed=8, **kw)
    ob, g, p0 = make_pair(spec)
    pts = np.random.default_rng(1).uniform(-1.5, 1.5, size=(777, 2))
    for order in (0, 1):
        ref = ob.evaluate(p0, pts, order)
        got = g.forward(pts, order)
        for k in range(1 + 2 * order):
            assert np.abs(got[k] - ref[k]).max() <= 3e-5 * max(1.0, np.abs(ref[k]).max()), (order, k)
        if layers[-1] == 2:
            assert np.abs(got[3] - ref[3]).max() <= 3e-5 * max(1.0, np.abs(ref[3]).max())


def test_ragged_training_with_schedule_and_plateau_matches_oracle():
    """train() (trainer.hpp:275-382) on a ragged network through the tensor-core
    step: exponential lr schedule, plateau stop, per-epoch loss within 1e-5."""
    spec = po.ProblemSpec(*po.structured_mesh(3, 3), n_test_1d=3, n_quad_1d=5, forcing="sin2pi_f",
                          boundary_g="sin2pi_u", n_boundary=60, layers=(2, 25, 12, 25, 1), bx=0.2, seed=4)
    ob, g, p0 = make_pair(spec)
    kw = dict(lr0=3e-3, lr_exponential=True, decay=0.9, every=7, loss_tol=0.2, plateau_window=6)
    ref = ob.train(p0, 80, log_every=1, **kw)
    rep = g.train(80, **kw)
    assert "tc2" in g.step_kernel()
    assert rep.steps_run == ref["steps_run"] and rep.stop_reason == ref["stop_reason"]
    r = np.abs(rep.records["total"] - ref["every_step"][:, 0]) / np.abs(ref["every_step"][:, 0])
    assert r.max() < 1e-5, r.max()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("layers", [(2, 30, 30, 30, 1), (2, 16, 16, 16, 2), (2, 24, 11, 1)])
def test_rank_partitions_sum_to_the_whole(world, layers):
    """vpinn_gpu_create(rank, world) sub-contexts on one device (the multi-GPU
    partition): their loss parts and gradients add up to the
    single-rank ones; the per-epoch all-reduce of the device path is that sum."""
    kw = dict(eps_source=2, bx=0.5, forcing="sinpi_vareps_f") if layers[-1] == 2 else dict(bx=0.3)
    spec = po.ProblemSpec(*po.structured_mesh(5, 4), n_test_1d=4, n_quad_1d=5, boundary_g="sin2pi_u",
                          n_boundary=41, n_sensors=9, sensor_field="sin2pi_u", layers=layers, seed=6, **kw)
    _, g, _ = make_pair(spec)
    whole, gw = g.loss_and_grad()
    acc, gacc = np.zeros(4), np.zeros_like(gw)
    for r in range(world):
        _, gr, _ = make_pair(spec, rank=r, world_size=world)
        pr, grr = gr.loss_and_grad()
        acc += pr
        gacc += grr
    assert np.allclose(acc, whole, rtol=2e-6)
    assert np.abs(gacc - gw).max() <= 2e-5 * np.abs(gw).max()


def test_single_rank_nccl_communicator_path():
    """The NCCL plumbing of the multi-GPU path (dlopen'd libnccl, communicator
    from a unique id, the per-epoch all-reduce inside the captured epoch graph)
    exercised with a one-rank communicator: results equal the plain context."""
    from paper_2404_12063_b200 import gpu as G
    spec = po.ProblemSpec(*po.structured_mesh(4, 4), n_test_1d=3, n_quad_1d=5, forcing="sin2pi_f",
                          boundary_g="sin2pi_u", n_boundary=40, layers=(2, 30, 30, 30, 1), seed=12)
    _, g0, p0 = make_pair(spec)
    _, g1, _ = make_pair(spec)
    g1.attach_comm(G.nccl_unique_id(), 1, 0)
    a, ga = g0.loss_and_grad()
    b, gb = g1.loss_and_grad()
    assert np.array_equal(a, b) and np.array_equal(ga, gb)
    r0 = g0.train(15, lr0=1e-3)
    r1 = g1.train(15, lr0=1e-3)
    assert np.array_equal(r0.records["total"], r1.records["total"])
    assert np.array_equal(g0.get_params(), g1.get_params())


@pytest.mark.parametrize("spg", [1, 7, 64])
def test_stop_inside_a_multi_step_graph(spg):
    """The epoch loop is replayed as CUDA graphs of steps_per_graph epochs; a
    coefficient-tolerance stop inside a graph must end the run at the same
    step as the reference, whatever the graph length (trainer.hpp:344-356)."""
    spec = po.ProblemSpec(*po.structured_mesh(2, 2, (-1.0, 1.0), (-1.0, 1.0)), n_test_1d=5, n_quad_1d=10,
                          forcing="bump_f", boundary_g="bump_u", n_boundary=400, n_sensors=50, sensor_seed=7,
                          sensor_field="bump_u", eps_source=1, scalars=(2.0,), layers=(2, 20, 20, 1), seed=42)
    ob, g, p0 = make_pair(spec)
    ref = ob.train(p0, 60, lr0=1e-3, eps_abs_tol=1.6955, eps_actual=0.3)
    rep = g.train(60, lr0=1e-3, eps_abs_tol=1.6955, eps_actual=0.3, steps_per_graph=spg)
    assert rep.steps_run == ref["steps_run"] < 60 and rep.stop_reason == ref["stop_reason"] == 1
    assert abs(rep.final_eps - ref["final_eps"]) < 1e-5
    assert np.abs(g.get_params() - ref["params"]).max() < 1e-4


def test_contexts_created_and_driven_from_two_threads():
    """Distinct contexts may be driven from distinct host threads (the C-ABI
    contract): concurrent creates share the staged-upload path and the block
    cache, results equal a serial run."""
    import threading
    # 1,800 cells: each 4.5 MB premultiplier tensor goes through the staged uploader
    spec = po.ProblemSpec(*po.structured_mesh(45, 40), n_test_1d=5, n_quad_1d=5, forcing="sin2pi_f",
                          boundary_g="sin2pi_u", n_boundary=80, layers=(2, 30, 30, 30, 1), bx=0.2, seed=21)
    ob = po.OracleProblem(spec, double=False)
    _, g0, _ = make_pair(spec)
    serial = g0.train(10, lr0=1e-3).records["total"].copy()
    g0.close()
    out = [None, None]

    def run(i):
        _, g, _ = make_pair(spec)
        out[i] = g.train(10, lr0=1e-3).records["total"].copy()
        g.close()

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert ob.n_int > 0
    assert np.array_equal(out[0], serial) and np.array_equal(out[1], serial)


# the network shapes the GPU path serves (variant.h): depth 1-4, widths up to
# 64 (62 for three hidden layers with one output, 50 with two, 36 for four),
# one or two outputs, tanh and sigmoid -- each through the kernel the context
# selects (tensor-core step in its 32- or 64-wide class, or the CUDA-core step)
WIDE_NETS = [(2, 64, 1), (2, 64, 2), (2, 60, 60, 1), (2, 33, 1, 1), (2, 64, 64, 1), (2, 48, 64, 2),
             (2, 55, 40, 55, 1), (2, 62, 62, 62, 1), (2, 40, 40, 40, 2), (2, 50, 50, 50, 2),
             (2, 36, 36, 36, 36, 1), (2, 20, 30, 36, 10, 2), (2, 8, 8, 8, 8, 1)]


@pytest.mark.parametrize("layers", WIDE_NETS)
@pytest.mark.parametrize("sig", [False, True])
def test_served_network_shapes_match_oracle(layers, sig):
    kw = dict(eps_source=2, bx=0.5, forcing="sinpi_vareps_f") if layers[-1] == 2 else dict(bx=0.3)
    fails = []
    for (nt, nq), mesh in ((3, 4), (2, 3)), ((5, 10), (1, 1)), ((4, 5), (9, 7)):
        spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, boundary_g="sin2pi_u",
                              n_boundary=37, layers=layers, sigmoid=sig, seed=11, **kw)
        ob, g, p0 = make_pair(spec)
        po_, go32 = ob.loss_and_grad(p0)
        pg, gg = g.loss_and_grad()
        _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
        lr = abs(pg[0] - po_[0]) / abs(po_[0])
        ge = np.abs(gg - g64).max() / max(np.abs(g64).max(), 1e-30)
        e32 = np.abs(go32 - g64).max() / max(np.abs(g64).max(), 1e-30)
        if lr > 1e-5 or ge > max(1e-5, 4.0 * e32):
            fails.append(((nt, nq), mesh, g.step_kernel(), lr, ge, e32))
        pts = np.random.default_rng(2).uniform(-1.2, 1.2, size=(300, 2))
        ref = ob.evaluate(p0, pts, 1)
        got = g.forward(pts, 1)
        for k in range(4 if layers[-1] == 2 else 3):  # u, u_x, u_y (, eps = softplus(y1))
            if np.abs(got[k] - ref[k]).max() > 3e-5 * max(1.0, np.abs(ref[k]).max()):
                fails.append(("evaluate", k, g.step_kernel()))
        g.close()
    assert not fails, fails


@pytest.mark.parametrize("layers", [(2, 64, 64, 64, 1), (2, 60, 60, 60, 2), (2, 40, 40, 40, 40, 1)])
def test_unserved_network_shapes_fail_with_a_config_error(layers):
    from paper_2404_12063_b200._capi import VpinnError
    kw = dict(eps_source=2, forcing="sinpi_vareps_f") if layers[-1] == 2 else {}
    spec = po.ProblemSpec(*po.structured_mesh(1, 1), n_test_1d=2, n_quad_1d=3, boundary_g="sin2pi_u",
                          n_boundary=5, layers=layers, seed=1, **kw)
    with pytest.raises(VpinnError) as e:
        make_pair(spec)
    assert e.value.code == 2


# the split path's row contraction (Q > 128 points per cell): the warp-owned-row
# kernel in its float4 (Q % 4 == 0, 4 / 8 / 13 float4 per lane) and scalar
# (Q % 4 != 0) layouts, CTA row ranges spanning several small cells, fewer rows
# than SMs, a trainable and a spatial coefficient, and the row-block kernel
# beyond 1,664 points (or with convection)
ROW_CASES = {
    "vec4_many_cells": dict(mesh=(15, 14), nt=2, nq=12),
    "scalar_many_cells": dict(mesh=(15, 14), nt=2, nq=13, eps_source=1, scalars=(1.3,), n_sensors=11,
                              sensor_field="sin2pi_u"),
    "vec8_3x3": dict(mesh=(3, 3), nt=3, nq=24),
    "vec13_one_cell": dict(mesh=(1, 1), nt=6, nq=40),
    "scalar52_spatial": dict(mesh=(2, 1), nt=4, nq=35, layers=(2, 16, 16, 16, 2), eps_source=2, bx=0.0,
                             forcing="sinpi_vareps_f"),
    "rows_kernel_q1681": dict(mesh=(1, 2), nt=5, nq=41),
    "fewer_rows_than_warps": dict(mesh=(1, 1), nt=2, nq=12),
    "rows_spanning_cells_scalar": dict(mesh=(7, 5), nt=3, nq=17, bx=0.0),
    "rows_kernel_conv": dict(mesh=(2, 2), nt=4, nq=20, bx=0.4, by=-0.3),
}


@pytest.mark.parametrize("case", list(ROW_CASES))
def test_row_contraction_layouts_match_oracle(case):
    kw = dict(ROW_CASES[case])
    mesh, nt, nq = kw.pop("mesh"), kw.pop("nt"), kw.pop("nq")
    kw.setdefault("layers", (2, 30, 30, 30, 1))
    kw.setdefault("forcing", "sin2pi_f")
    spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, boundary_g="sin2pi_u",
                          n_boundary=37, seed=9, **kw)
    ob, g, p0 = make_pair(spec)
    assert ob.Q > 128  # the split path
    po_, go32 = ob.loss_and_grad(p0)
    pg, gg = g.loss_and_grad()
    _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
    assert abs(pg[0] - po_[0]) / abs(po_[0]) < 1e-5, (pg, po_)
    e32 = np.abs(go32 - g64).max() / np.abs(g64).max()
    assert np.abs(gg - g64).max() / np.abs(g64).max() < max(1e-5, 4.0 * e32)
    # bitwise reproducible (fixed summation order everywhere)
    pg2, gg2 = g.loss_and_grad()
    assert np.array_equal(np.asarray(pg2), np.asarray(pg)) and np.array_equal(gg2, gg)
    g.close()


# served-shape gaps the randomised fuzz (tools/random_fuzz.py) found: the
# 64-wide class with many small cells per tile (more than 128 test rows at
# 112 points: fewer cells per tile) and with 112 < Q <= 128 (cells larger than
# its tile: the split path)
@pytest.mark.parametrize("mesh,nt,nq,layers", [((12, 8), 5, 3, (2, 53, 10, 13, 1)),
                                               ((1, 1), 7, 5, (2, 53, 53, 53, 1)),
                                               ((6, 6), 4, 11, (2, 62, 62, 62, 1)),
                                               ((12, 2), 3, 11, (2, 15, 51, 59, 1))])
def test_wide_class_tiling_gaps_match_oracle(mesh, nt, nq, layers):
    spec = po.ProblemSpec(*po.structured_mesh(*mesh), n_test_1d=nt, n_quad_1d=nq, forcing="sin4pi_f",
                          boundary_g="sin2pi_u", n_boundary=60, layers=layers, bx=0.3, seed=3)
    ob, g, p0 = make_pair(spec)
    assert "tc2_step" in g.step_kernel(), g.step_kernel()
    po_, go32 = ob.loss_and_grad(p0)
    pg, gg = g.loss_and_grad()
    _, g64 = po.OracleProblem(spec, double=True).loss_and_grad(p0.astype(np.float64))
    assert abs(pg[0] - po_[0]) / abs(po_[0]) < 1e-5
    e32 = np.abs(go32 - g64).max() / np.abs(g64).max()
    assert np.abs(gg - g64).max() / np.abs(g64).max() < max(1e-5, 4.0 * e32)
    g.close()
