"""The bench's C2 cell-count and C3 p/q sweeps alone (median ms/epoch).
usage: python tools/quick_sweeps.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps({"sweep_c3": bench._sweep_c3(0), "sweep_c2": bench._sweep(0)}))
