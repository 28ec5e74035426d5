"""ctypes binding of include/vpinn_host.h: the C++ host pipeline
(config -> mesh -> assembly -> sampling -> init) that feeds the B200 step."""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Union

import numpy as np

from . import _capi
from .gpu import GpuStep

MESH_FROM_CONFIG, MESH_STRUCTURED, MESH_GEAR, MESH_DISK, MESH_HANDLE = 0, 1, 2, 3, 4


class MeshSource(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("skew", C.c_double), ("skew_seed", C.c_uint64), ("mesh", C.c_void_p)]


_declared = False


def _lib():
    global _declared
    L = _capi.lib()
    if not _declared:
        vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
        sig = {
            "vpinn_host_last_error": (C.c_char_p, []),
            "vpinn_host_mesh_read_gmsh": (i32, [C.c_char_p, C.POINTER(vp)]),
            "vpinn_host_mesh_parse_gmsh": (i32, [C.c_char_p, C.POINTER(vp)]),
            "vpinn_host_mesh_make": (i32, [C.POINTER(MeshSource), C.POINTER(vp)]),
            "vpinn_host_mesh_counts": (None, [vp, vp]),
            "vpinn_host_mesh_arrays": (None, [vp, vp, vp, vp]),
            "vpinn_host_mesh_health": (None, [vp, C.POINTER(i64), C.POINTER(i64)]),
            "vpinn_host_mesh_free": (None, [vp]),
            "vpinn_host_gear_msh_text": (i32, [i32, i32, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
            "vpinn_host_problem_from_config": (i32, [C.c_char_p, C.c_char_p, C.POINTER(MeshSource),
                                                     C.POINTER(vp)]),
            "vpinn_host_problem_from_config_ex": (i32, [C.c_char_p, C.c_char_p, C.POINTER(MeshSource), i32,
                                                        C.POINTER(vp)]),
            "vpinn_host_problem_counts": (None, [vp, vp]),
            "vpinn_host_problem_view": (i32, [vp, i32, i32, i32, C.POINTER(_capi.Problem)]),
            "vpinn_host_problem_params": (None, [vp, vp]),
            "vpinn_host_problem_rule": (None, [vp, vp, vp, vp]),
            "vpinn_host_problem_free": (None, [vp]),
            "vpinn_host_train": (i32, [vp, i32, vp, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
            "vpinn_host_bench_case": (i32, [C.c_char_p, i32, i32, i32, C.c_double, i32, i32, vp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _declared = True
    return L


def _check(rc):
    if rc != 0:
        raise _capi.VpinnError(rc, _lib().vpinn_host_last_error().decode(errors="replace"))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Mesh:
    def __init__(self, handle):
        self.h = handle
        c = np.zeros(3, dtype=np.int64)
        _lib().vpinn_host_mesh_counts(self.h, _p(c))
        self.n_nodes, self.n_elements, self.n_boundary_nodes = map(int, c)

    def __del__(self):
        if getattr(self, "h", None):
            _lib().vpinn_host_mesh_free(self.h)
            self.h = None

    @classmethod
    def read_gmsh(cls, path):
        h = C.c_void_p()
        _check(_lib().vpinn_host_mesh_read_gmsh(os.fsencode(path), C.byref(h)))
        return cls(h)

    @classmethod
    def parse_gmsh(cls, text: str):
        h = C.c_void_p()
        _check(_lib().vpinn_host_mesh_parse_gmsh(text.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def make(cls, src: MeshSource):
        h = C.c_void_p()
        _check(_lib().vpinn_host_mesh_make(C.byref(src), C.byref(h)))
        return cls(h)

    @classmethod
    def structured(cls, nx, ny, x_range=(0.0, 1.0), y_range=(0.0, 1.0), skew=0.0, skew_seed=1234):
        return cls.make(structured_source(nx, ny, x_range, y_range, skew, skew_seed))

    @classmethod
    def gear(cls, n_r=16, n_t=887):
        return cls.make(MeshSource(kind=MESH_GEAR, nx=n_r, ny=n_t))

    @classmethod
    def disk(cls, n=32):
        return cls.make(MeshSource(kind=MESH_DISK, nx=n, ny=n))

    def arrays(self):
        nodes = np.zeros((self.n_nodes, 2))
        cells = np.zeros((self.n_elements, 4), dtype=np.int32)
        bnd = np.zeros(self.n_boundary_nodes, dtype=np.int32)
        _lib().vpinn_host_mesh_arrays(self.h, _p(nodes), _p(cells), _p(bnd))
        return nodes, cells, bnd

    def health(self):
        d, m = C.c_int64(), C.c_int64()
        _lib().vpinn_host_mesh_health(self.h, C.byref(d), C.byref(m))
        return d.value, m.value

    def source(self) -> MeshSource:
        return MeshSource(kind=MESH_HANDLE, mesh=self.h)


def structured_source(nx, ny, x_range=(0.0, 1.0), y_range=(0.0, 1.0), skew=0.0, skew_seed=1234):
    return MeshSource(kind=MESH_STRUCTURED, nx=nx, ny=ny, x0=x_range[0], x1=x_range[1],
                      y0=y_range[0], y1=y_range[1], skew=skew, skew_seed=skew_seed)


def gear_msh_text(n_r: int, n_t: int) -> str:
    n = C.c_size_t()
    _check(_lib().vpinn_host_gear_msh_text(n_r, n_t, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(_lib().vpinn_host_gear_msh_text(n_r, n_t, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class HostProblem:
    """build_problem(config[, premade mesh]) on the C++ host side.
    device_assembly=True skips the host premultiplier assembly: the device
    context builds the tensors, the forcing and the interior points itself."""

    def __init__(self, config: Union[dict, str], base_dir: Optional[str] = None,
                 mesh: Optional[Union[MeshSource, Mesh]] = None, device_assembly: bool = False):
        text = config if isinstance(config, str) else json.dumps(config)
        src = mesh.source() if isinstance(mesh, Mesh) else mesh
        self._mesh_keep = mesh
        self.device_assembly = device_assembly
        h = C.c_void_p()
        _check(_lib().vpinn_host_problem_from_config_ex(text.encode(), (base_dir or "").encode(),
                                                        C.byref(src) if src is not None else None,
                                                        1 if device_assembly else 0, C.byref(h)))
        self.h = h
        c = np.zeros(8, dtype=np.int64)
        _lib().vpinn_host_problem_counts(h, _p(c))
        (self.E, self.T, self.Q, self.n_int, self.n_bnd, self.n_sen, self.n_params,
         downgraded) = map(int, c)
        self.precision_downgraded = bool(downgraded)

    def __del__(self):
        if getattr(self, "h", None):
            _lib().vpinn_host_problem_free(self.h)
            self.h = None

    def view(self, device=0, rank=0, world=1) -> _capi.Problem:
        pb = _capi.Problem()
        _check(_lib().vpinn_host_problem_view(self.h, device, rank, world, C.byref(pb)))
        return pb

    def arrays(self):
        """Host arrays (copies) in the reference layouts."""
        pb = self.view()
        E, T, Q = self.E, self.T, self.Q
        n_pts = self.n_int + self.n_bnd + self.n_sen

        def f32(ptr, n):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), (n,)).copy() if ptr else None

        def f64(ptr, n):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), (n,)).copy() if ptr and n else np.zeros(0)

        return {
            "grad_x": f32(pb.grad_x, E * T * Q), "grad_y": f32(pb.grad_y, E * T * Q),
            "test": f32(pb.test, E * T * Q), "forcing": f32(pb.forcing, E * T),
            "points": f64(pb.points, 2 * n_pts).reshape(-1, 2),
            "boundary_values": f64(pb.boundary_values, self.n_bnd),
            "sensor_values": f64(pb.sensor_values, self.n_sen),
            "form": int(pb.form),
            "strong_forcing": f32(pb.strong_forcing, self.n_int),
        }

    def init_params(self):
        out = np.zeros(self.n_params, dtype=np.float32)
        _lib().vpinn_host_problem_params(self.h, _p(out))
        return out

    def rule(self):
        xi, eta, w = (np.zeros(self.Q) for _ in range(3))
        _lib().vpinn_host_problem_rule(self.h, _p(xi), _p(eta), _p(w))
        return xi, eta, w

    def gpu(self, device=0, rank=0, world=1) -> GpuStep:
        """Device context straight from the host view (no Python copies)."""
        g = GpuStep.from_problem(self.view(device, rank, world), keepalive=self)
        g.set_params(self.init_params())
        return g

    def train(self, device=0):
        n = C.c_size_t()
        params = np.zeros(self.n_params, dtype=np.float32)
        cap = 1 << 24
        buf = C.create_string_buffer(cap)
        _check(_lib().vpinn_host_train(self.h, device, _p(params), buf, cap, C.byref(n)))
        return json.loads(buf.value.decode()), params


def bench_case(config: Union[dict, str], e_per_dim, n_test_per_dim, n_quad_per_dim, skew=0.0,
               reps=15, device=0):
    text = config if isinstance(config, str) else json.dumps(config)
    out = np.zeros(3)
    _check(_lib().vpinn_host_bench_case(text.encode(), e_per_dim, n_test_per_dim, n_quad_per_dim,
                                        skew, reps, device, _p(out)))
    return {"median_s": out[0], "p10_s": out[1], "p90_s": out[2]}
