"""Diagnose the tcgen05 probe: run each mode on structured inputs and
compare the raw output against candidate products."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12063_b200 import _capi  # noqa: E402

L = _capi.lib()
ptr = lambda a: a.ctypes.data_as(C.c_void_p)
rng = np.random.default_rng(1)
A = rng.standard_normal((128, 32)).astype(np.float32)
W = rng.standard_normal((32, 32)).astype(np.float32)
H = rng.standard_normal((128, 32)).astype(np.float32)
np.set_printoptions(precision=3, suppress=True, linewidth=160)
for mode in (0, 1, 2):
    out = np.zeros((128 * 32 + 128 * 96,), np.float32)
    rc = L.vpinn_gpu_tc_probe(0, mode, ptr(A), ptr(W), ptr(H), ptr(out))
    print("mode", mode, "rc", rc, _capi.lib().vpinn_gpu_last_error() if rc else "")
    if mode < 2:
        got = out[:128 * 32].reshape(128, 32)
        cands = {"A@W.T": A @ W.T, "A@W": A @ W}
    else:
        got = out[:32 * 32].reshape(32, 32)
        cands = {"A.T@H": A.T @ H, "A.T@A": A.T @ A, "H.T@H": H.T @ H, "A.T@H.T?": (A.T @ H).T}
    print("  got: nonzero", np.count_nonzero(got), "absmax", np.abs(got).max(), "nan", np.isnan(got).sum())
    for k, v in cands.items():
        print("  vs", k, "relerr", np.abs(got - v).max() / np.abs(v).max())
    print("  got[0,:8]", got[0, :8])
    print("  got[1,:8]", got[1, :8])
    if mode == 2:
        raw = out[128 * 32:].reshape(128, 96)
        print("  raw nonzero", np.count_nonzero(raw), "row0", raw[0, :8], "row32", raw[32, :8])
