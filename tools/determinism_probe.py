"""Repeat loss_and_grad on the parity cases and report any run-to-run
difference (the device path is deterministic by construction; a difference
means a race).  Usage: python tools/determinism_probe.py [reps] [case ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests.test_gpu_parity import CASES, make_pair  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
names = sys.argv[2:] or list(CASES)
bad = 0
for name in names:
    spec = CASES[name]()
    ob, g, p0 = make_pair(spec)
    parts_o, _ = ob.loss_and_grad(p0)
    ref_parts, ref_grad = g.loss_and_grad()
    diffs = 0
    for r in range(reps):
        parts, grad = g.loss_and_grad()
        if not (np.array_equal(parts, ref_parts) and np.array_equal(grad, ref_grad)):
            diffs += 1
            print(f"  {name} rep {r}: parts {parts} vs {ref_parts}; max grad diff "
                  f"{np.abs(grad - ref_grad).max():.3e}", flush=True)
    rel = abs(ref_parts[0] - parts_o[0]) / abs(parts_o[0])
    print(f"{name}: {diffs}/{reps} differing runs; rel loss vs oracle {rel:.2e}; parts {ref_parts} oracle {parts_o}",
          flush=True)
    bad += diffs
sys.exit(1 if bad else 0)
