"""The paper's gear variant ([2,50,50,50,1], T=16, P_b=6,096) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_12063_b200 import host  # noqa: E402

print(bench._c5_paper(host.Mesh.gear(bench.GEAR_NR, bench.GEAR_NT), 0))
