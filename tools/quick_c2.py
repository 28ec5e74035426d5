"""C2 small-problem epoch times through the reference bench_case protocol
(10 warm-ups, median of 15 single timed epochs), cell counts e*e from argv.
usage: python tools/quick_c2.py 1 2 4 8"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import host  # noqa: E402

cfg = {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 400},
       "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
       "network": {"layers": [2, 30, 30, 30, 1]},
       "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
out = {}
for e in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    r = host.bench_case(cfg, e, 5, 10, 0.0, 15, 0)
    out[e * e] = round(1e3 * r["median_s"], 4)
print(json.dumps(out))
