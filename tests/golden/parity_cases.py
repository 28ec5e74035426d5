"""The BASELINE.json configs as oracle ProblemSpecs, shared by the fixture
generator (make_parity_fixtures.py) and the GPU parity tests
(tests/test_baseline_parity.py).  Test infrastructure only.

  c5_gear       C5: the 14,192-cell gear (gen_fixtures.py recipe, n_r=16,
                n_t=887), gear_cd2d.json settings (proj/configs/gear_cd2d.json):
                cd2d eps=1, b=(0.1,0), gear_f, T=25, Q=25, P_b=800, [2,30,30,30,1]
  c5_inverse    C5 inverse: the same gear, trainable scalar eps (init 2.0),
                50 sensors (seed 7) of sin2pi_u (config.hpp:37-41 defaults)
  c5_paper      the paper's gear variant: T=16, Q=25,
                P_b=6,096, [2,50,50,50,1]
  c2_4096       C2's largest point: 64x64 unit square, T=25, Q=100
  c3_t10_q40    C3's largest point: 8x8 cells, T=100 (10x10), Q=1,600 (40x40),
                sin4pi (omega = 4 pi)
  forward_sine  proj/configs/forward_sine.json (2x2 cells, T=225, Q=1,600)
  inverse_eps   proj/configs/inverse_eps.json (2x2 on [-1,1]^2, T=25,
                Q=1,600, [2,20,20,1], scalar eps init 2.0, 50 sensors seed 7)
"""
from oracle import pyoracle as po


def _gear(**over):
    nodes, cells = po.gear_mesh(16, 887)
    kw = dict(n_test_1d=5, n_quad_1d=5, forcing="gear_f", boundary_g="zero", n_boundary=800,
              eps=1.0, bx=0.1, by=0.0, layers=(2, 30, 30, 30, 1), seed=42)
    kw.update(over)
    return po.ProblemSpec(nodes=nodes, cells=cells, **kw)


def _square(n, t, q, forcing, g, **over):
    nodes, cells = po.structured_mesh(n, n)
    kw = dict(n_test_1d=t, n_quad_1d=q, forcing=forcing, boundary_g=g, n_boundary=400,
              boundary_seed=1, layers=(2, 30, 30, 30, 1), seed=42)
    kw.update(over)
    return po.ProblemSpec(nodes=nodes, cells=cells, **kw)


CASES = {
    "c5_gear": lambda: _gear(),
    "c5_inverse": lambda: _gear(n_sensors=50, sensor_seed=7, sensor_field="sin2pi_u", eps_source=1,
                                scalars=(2.0,)),
    "c5_paper": lambda: _gear(n_test_1d=4, n_boundary=6096, layers=(2, 50, 50, 50, 1)),
    "c2_4096": lambda: _square(64, 5, 10, "sin2pi_f", "sin2pi_u"),
    "c3_t10_q40": lambda: _square(8, 10, 40, "sin4pi_f", "sin4pi_u"),
    "forward_sine": lambda: _square(2, 15, 40, "sin2pi_f", "sin2pi_u"),
    "inverse_eps": lambda: po.ProblemSpec(
        *po.structured_mesh(2, 2, (-1.0, 1.0), (-1.0, 1.0)), n_test_1d=5, n_quad_1d=40,
        forcing="bump_f", boundary_g="bump_u", n_boundary=400, n_sensors=50, sensor_seed=7,
        sensor_field="bump_u", eps_source=1, scalars=(2.0,), layers=(2, 20, 20, 1), seed=42),
}

# cases whose 100-epoch oracle run is too slow to repeat at test time
# (>= ~0.5 s per oracle epoch): their trajectories are committed fixtures
FIXTURE_CASES = ("c5_gear", "c5_inverse", "c5_paper", "c2_4096", "c3_t10_q40")
EPOCHS = 100
LR = 1e-3
