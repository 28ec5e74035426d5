"""Where does a cta_group::1 M=64 tcgen05.mma put its 64 rows in TMEM?
(tc_probe mode 4: D[r][i] = sum_p Apart_{r/32}[p][r%32] H_h[p][i])"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import _capi  # noqa: E402


def bf16_hi(x):
    b = x.astype(np.float32).view(np.uint32)
    return ((b + np.uint32(0x8000)) & np.uint32(0xFFFF0000)).view(np.float32)


rng = np.random.default_rng(5)
A = rng.standard_normal((128, 32)).astype(np.float32)
W = rng.standard_normal((32, 32)).astype(np.float32)
H = rng.standard_normal((128, 32)).astype(np.float32)
out = np.zeros(128 * 32 + 128 * 96, np.float32)
ptr = lambda a: a.ctypes.data_as(C.c_void_p)
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 4
_capi.check(_capi.lib().vpinn_gpu_tc_probe(0, mode, ptr(A), ptr(W), ptr(H), ptr(out)))
raw = out[128 * 32:].reshape(128, 96)[:, :32].astype(np.float64)
ah = bf16_hi(A)
am = ((A - ah).view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
hh = bf16_hi(H).astype(np.float64)
rows = np.concatenate([ah.astype(np.float64).T @ hh, am.astype(np.float64).T @ hh])  # [64][32]
for lane in range(128):
    d = np.abs(rows - raw[lane][None, :]).max(axis=1) / (np.abs(rows).max(axis=1) + 1e-30)
    r = int(np.argmin(d))
    tag = f"row {r:2d} (err {d[r]:.1e})" if d[r] < 1e-3 else f"-- (max {np.abs(raw[lane]).max():.2e})"
    print(f"lane {lane:3d}: {tag}")
