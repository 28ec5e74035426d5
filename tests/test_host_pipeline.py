"""The product's C++ host pipeline (config -> mesh -> assembly -> sampling ->
init) against the independent oracle restatement, bit for bit, plus the
reference's mesh-reader / config contracts.  CPU only."""
import hashlib
import json
import os
import shutil

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2404_12063_b200 import host
from paper_2404_12063_b200._capi import VpinnError
from tests.refutil import read_msh

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MESHES = os.path.join(GOLD, "meshes")


def bits(a, dt):
    a = np.ascontiguousarray(a, dtype=dt)
    return a.view(np.uint32 if dt == np.float32 else np.uint64)


def assert_same_problem(hp: "host.HostProblem", ob: "po.OracleProblem"):
    assert (hp.E, hp.T, hp.Q, hp.n_int, hp.n_bnd, hp.n_sen, hp.n_params) == \
        (ob.E, ob.T, ob.Q, ob.n_int, ob.n_bnd, ob.n_sen, ob.n_params)
    ha = hp.arrays()
    for name in ("grad_x", "grad_y", "test", "forcing"):
        assert np.array_equal(bits(ha[name], np.float32), bits(ob.array(name), np.float32)), name
    assert np.array_equal(bits(ha["points"], np.float64), bits(ob.array("points"), np.float64))
    assert np.array_equal(bits(ha["boundary_values"], np.float64), bits(ob.array("boundary_values"), np.float64))
    if hp.n_sen:
        assert np.array_equal(bits(ha["sensor_values"], np.float64), bits(ob.array("sensor_values"), np.float64))
    assert np.array_equal(bits(hp.init_params(), np.float32), bits(ob.init_params(), np.float32))
    xi, eta, w = hp.rule()
    r = ob.array("rule")
    assert np.array_equal(xi, r[0]) and np.array_equal(eta, r[1]) and np.array_equal(w, r[2])


def cfg(**kw):
    c = {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "domain": {"nx": 8, "ny": 8},
                     "n_boundary_points": 400},
         "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
         "network": {"layers": [2, 30, 30, 30, 1]},
         "training": {"iterations": 10, "learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    for k, v in kw.items():
        c[k].update(v)
    return c


def test_c1_assembly_bit_exact_against_oracle():
    hp = host.HostProblem(cfg())
    nodes, cells = po.structured_mesh(8, 8)
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells), double=False)
    assert_same_problem(hp, ob)


def test_gear_fixture_mesh_and_assembly_bit_exact():
    m = host.Mesh.read_gmsh(os.path.join(MESHES, "gearlike_v41.msh"))
    assert (m.n_elements, m.n_boundary_nodes) == (576, 192)  # test_mesh_io.cpp:32-42
    assert m.health() == (0, 0)
    nodes_h, cells_h, _ = m.arrays()
    nodes_r, cells_r = read_msh(os.path.join(MESHES, "gearlike_v41.msh"))
    assert np.array_equal(nodes_h.view(np.uint64), nodes_r.view(np.uint64))
    assert np.array_equal(cells_h, cells_r)
    c = cfg(problem={"pde": {"type": "cd2d", "eps": 1.0, "b": [0.1, 0.0]}, "forcing": "gear_f",
                     "boundary_g": "zero", "n_boundary_points": 800},
            discretization={"n_test_per_dim": 5, "n_quad_per_dim": 5})
    hp = host.HostProblem(c, mesh=m)
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes_r, cells=cells_r, n_test_1d=5, n_quad_1d=5,
                                         forcing="gear_f", boundary_g="zero", n_boundary=800,
                                         eps=1.0, bx=0.1), double=False)
    assert_same_problem(hp, ob)


def test_gear_14192_generator_reproduces_reference_recipe_bytes():
    info = json.load(open(os.path.join(GOLD, "gear_14192.json")))["gear_14192"]
    text = host.gear_msh_text(16, 887)
    assert len(text.encode()) == info["n_bytes"]
    assert hashlib.sha256(text.encode()).hexdigest() == info["sha256"]
    small = host.gear_msh_text(6, 96)
    assert small == open(os.path.join(MESHES, "gearlike_v41.msh")).read()
    g = host.Mesh.gear(16, 887)
    assert (g.n_elements, g.n_nodes) == (14192, 15079)
    assert g.health() == (0, 0)
    # the oracle's pure-Python generator (bench.py's CPU legs) gives the same mesh
    nodes, cells, _ = g.arrays()
    pn, pcells = po.gear_mesh(16, 887)
    assert np.array_equal(nodes.view(np.uint64), pn.view(np.uint64)) and np.array_equal(cells, pcells)


def test_skewed_bench_mesh_and_disk_with_sensors_bit_exact():
    src = host.structured_source(6, 6, skew=0.2, skew_seed=1234)
    c = cfg(discretization={"n_test_per_dim": 4, "n_quad_per_dim": 6})
    hp = host.HostProblem(c, mesh=src)
    nodes, cells = po.structured_mesh(6, 6, skew=0.2, skew_seed=1234)
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=4, n_quad_1d=6), double=False)
    assert_same_problem(hp, ob)
    disk = host.Mesh.disk(8)
    assert disk.n_elements == 64 and disk.health() == (0, 0)
    c = cfg(problem={"pde": {"type": "cd2d", "eps": 0.5, "b": [1.0, 0.0]}, "forcing": "one",
                     "boundary_g": "zero", "exact_solution": "sinpi_u",
                     "sensors": {"count": 20, "seed": 7}},
            network={"layers": [2, 20, 20, 1], "eps_scalar_init": 2.0})
    hp = host.HostProblem(c, mesh=disk)
    nodes, cells, _ = disk.arrays()
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells, forcing="one", boundary_g="zero",
                                         eps=0.5, bx=1.0, n_sensors=20, sensor_seed=7,
                                         sensor_field="sinpi_u", eps_source=1, scalars=(2.0,),
                                         layers=(2, 20, 20, 1)), double=False)
    assert_same_problem(hp, ob)


def test_strong_form_config_builds_the_collocation_problem():
    # commands.hpp:147-152: form "strong" -> f at the quadrature points, cast
    # to float at use (losses.hpp:450); same batch as the weak form
    c = cfg(problem={"forcing": "sin2pi_f", "boundary_g": "sin2pi_u"},
            discretization={"form": "strong", "n_test_per_dim": 3, "n_quad_per_dim": 5},
            network={"layers": [2, 12, 12, 1]})
    hp = host.HostProblem(c, mesh=host.structured_source(3, 3))
    a = hp.arrays()
    assert a["form"] == 1
    nodes, cells = po.structured_mesh(3, 3)
    ob = po.OracleProblem(po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=3, n_quad_1d=5,
                                         layers=(2, 12, 12, 1), strong=True), double=False)
    assert np.array_equal(bits(a["points"], np.float64), bits(ob.array("points"), np.float64))
    assert np.array_equal(bits(a["strong_forcing"], np.float32),
                          bits(ob.array("strong_forcing").astype(np.float32), np.float32))
    weak = host.HostProblem(cfg(problem={"forcing": "sin2pi_f", "boundary_g": "sin2pi_u"}),
                            mesh=host.structured_source(3, 3))
    assert weak.arrays()["form"] == 0 and weak.arrays()["strong_forcing"] is None


def test_reference_configs_build_unchanged(tmp_path):
    # gear_cd2d.json points at data/meshes/gearlike_v41.msh relative to proj/
    (tmp_path / "data" / "meshes").mkdir(parents=True)
    shutil.copy(os.path.join(MESHES, "gearlike_v41.msh"), tmp_path / "data" / "meshes")
    sizes = {}
    for name in ("forward_sine.json", "gear_cd2d.json", "inverse_eps.json", "benchmark_sweep.json"):
        text = open(os.path.join(GOLD, "configs", name)).read()
        hp = host.HostProblem(text, base_dir=str(tmp_path))
        sizes[name] = (hp.E, hp.T, hp.Q, hp.n_bnd, hp.n_sen, hp.n_params)
        assert hp.precision_downgraded  # reference default precision is double
    assert sizes["forward_sine.json"] == (4, 225, 1600, 400, 0, 1981)
    assert sizes["gear_cd2d.json"] == (576, 25, 25, 800, 0, 1981)
    assert sizes["inverse_eps.json"] == (4, 25, 1600, 400, 50, 20 * 2 + 20 + 20 * 20 + 20 + 20 + 1 + 1)
    assert sizes["benchmark_sweep.json"][:3] == (1, 25, 100)


@pytest.mark.parametrize("text,code,needle", [
    ('{"problem": {"forcing": "one", "boundary_g": "zero", "bogus": 1}}', 2, "problem.bogus: unknown key"),
    ('{"problem": {"forcing": "nope", "boundary_g": "zero"}}', 2, "problem.forcing: unknown field 'nope'"),
    ('{"problem": {"forcing": "one", "boundary_g": "zero", "pde": {"b": [1, 0]}}}', 2, "poisson mode requires zero convection"),
    ('{"problem": {"forcing": "one", "boundary_g": "zero"}, "discretization": {"kernel": "loop"}}', 2, "kernel 'tensor'"),
    ('{"discretization": {}}', 2, "missing required section 'problem'"),
    ('{"problem": {"forcing": "one", "boundary_g": "zero"}, "training": {"lr_schedule": {"type": "cos"}}}', 2, "lr_schedule.type"),
    ('{not json', 2, "<config>"),
])
def test_config_strictness_and_modes(text, code, needle):
    with pytest.raises(VpinnError) as e:
        host.HostProblem(text)
    assert e.value.code == code and needle in str(e.value), str(e.value)


def test_gmsh_reader_contracts():
    m = host.Mesh.read_gmsh(os.path.join(MESHES, "square_2x2_v22.msh"))
    assert (m.n_nodes, m.n_elements, m.n_boundary_nodes) == (9, 4, 8)
    m = host.Mesh.read_gmsh(os.path.join(MESHES, "square_1x1_v41.msh"))
    assert (m.n_nodes, m.n_elements, m.n_boundary_nodes) == (4, 1, 4)
    m = host.Mesh.read_gmsh(os.path.join(MESHES, "skewed_12x12_v22.msh"))
    assert m.n_elements == 144 and m.health() == (0, 0)
    for bad in ("bad_triangle_v22.msh", "bad_dangling_v22.msh", "bad_binary_v22.msh"):
        with pytest.raises(VpinnError) as e:
            host.Mesh.read_gmsh(os.path.join(MESHES, bad))
        assert e.value.code == 3, bad
    with pytest.raises(VpinnError) as e:
        host.Mesh.read_gmsh("/nonexistent/path.msh")
    assert e.value.code == 5
    cw = ("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n4\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n"
          "$EndNodes\n$Elements\n1\n1 3 2 0 2 1 4 3 2\n$EndElements\n")
    m = host.Mesh.parse_gmsh(cw)
    _, cells, _ = m.arrays()
    assert cells[0, 0] == 0 and m.health() == (0, 0)
    for txt in ("$MeshFormat\n3.0 0 8\n$EndMeshFormat\n", ""):
        with pytest.raises(VpinnError) as e:
            host.Mesh.parse_gmsh(txt)
        assert e.value.code == 3


def _msh22(nodes, cells):
    """gmsh 2.2 ASCII text of a quad mesh (node ids 1-based in file order)."""
    out = ["$MeshFormat", "2.2 0 8", "$EndMeshFormat", "$Nodes", str(len(nodes))]
    out += [f"{i + 1} {float(x)!r} {float(y)!r} 0" for i, (x, y) in enumerate(nodes)]
    out += ["$EndNodes", "$Elements", str(len(cells))]
    out += [f"{k + 1} 3 2 0 1 " + " ".join(str(int(v) + 1) for v in c) for k, c in enumerate(cells)]
    out += ["$EndElements", ""]
    return "\n".join(out)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_boundary_samples_on_renumbered_meshes_match_oracle(seed):
    """The host's boundary-edge pass (counting sort by min node id) walks the
    single-incidence edges in the reference's (min id, max id) map order:
    with node ids shuffled, the arc-length samples must still equal the
    oracle's bit for bit (mesh.hpp boundary edges, problem.hpp sampling)."""
    rng = np.random.default_rng(seed)
    nx, ny = (int(v) for v in rng.integers(2, 9, size=2))
    nodes, cells = po.structured_mesh(nx, ny, skew=0.2, skew_seed=seed)
    perm = rng.permutation(len(nodes))  # new id of old node i is perm[i]
    pn = np.empty_like(nodes)
    pn[perm] = nodes
    pc = perm[np.asarray(cells)]
    m = host.Mesh.parse_gmsh(_msh22(pn, pc))
    c = cfg(problem={"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 97},
            discretization={"n_test_per_dim": 2, "n_quad_per_dim": 3})
    hp = host.HostProblem(c, mesh=m)
    ob = po.OracleProblem(po.ProblemSpec(nodes=pn, cells=pc, n_test_1d=2, n_quad_1d=3, forcing="sin2pi_f",
                                         boundary_g="sin2pi_u", n_boundary=97), double=False)
    assert_same_problem(hp, ob)
    dp = host.HostProblem(c, mesh=m, device_assembly=True)
    assert np.array_equal(bits(dp.arrays()["boundary_values"], np.float64), bits(ob.array("boundary_values"), np.float64))
