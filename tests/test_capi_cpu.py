"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and refuses to run without an sm_100 device (no fallback)."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from paper_2404_12063_b200 import _capi


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    names = _capi.declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = {l.split(".")[-2] for l in out.splitlines() if ".cubin" in l}
    assert archs == {"sm_100a"}, archs


@pytest.mark.skipif(_capi.lib().vpinn_gpu_device_ok() == 1, reason="a B200 is present")
def test_create_fails_loudly_without_device():
    from paper_2404_12063_b200.gpu import GpuStep
    T, Q = 1, 4
    with pytest.raises(_capi.VpinnError) as e:
        GpuStep(grad_x=np.zeros(T * Q), grad_y=np.zeros(T * Q), test=None, forcing=np.zeros(T),
                n_elem=1, n_test=T, n_quad=Q, points=np.zeros((Q + 1, 2)), n_interior=Q,
                n_boundary=1, n_sensors=0, boundary_values=np.zeros(1),
                layer_sizes=(2, 30, 30, 30, 1))
    assert e.value.code == 6


def test_contract_violations_are_config_or_numeric_errors():
    from paper_2404_12063_b200.gpu import GpuStep
    with pytest.raises(_capi.VpinnError) as e:
        GpuStep(grad_x=np.zeros(4), grad_y=np.zeros(4), test=None, forcing=np.zeros(1),
                n_elem=1, n_test=1, n_quad=4, points=np.zeros((4, 2)), n_interior=3,
                n_boundary=1, n_sensors=0, boundary_values=np.zeros(1))
    assert e.value.code == 4  # interior count does not cover the quadrature points
    with pytest.raises(_capi.VpinnError) as e:
        GpuStep(grad_x=np.zeros(4), grad_y=np.zeros(4), test=None, forcing=np.zeros(1),
                n_elem=1, n_test=1, n_quad=4, points=np.zeros((5, 2)), n_interior=4,
                n_boundary=1, n_sensors=0, boundary_values=np.zeros(1), layer_sizes=(3, 4, 1))
    assert e.value.code == 2  # input dimension must be 2
