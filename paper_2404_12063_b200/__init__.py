"""B200-native FastVPINNs training step (arXiv 2404.12063) behind the
reference's C++ loss/trainer boundary.

Layout:
  csrc/gpu/   sm_100a kernels + the C-ABI of include/vpinn_gpu.h
  csrc/host/  Eigen-free C++ mirror of the reference host path (config, mesh,
              quadrature, assembly, train loop) calling the C-ABI
  _capi.py / gpu.py  thin ctypes binding used by tests/ and bench.py
"""
__version__ = "0.1.0"
