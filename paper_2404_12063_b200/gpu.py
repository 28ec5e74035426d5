"""Python handle over the C-ABI step (vpinn_gpu_*), numpy in / numpy out.

This is the binding the tests and bench.py use; the reference-facing host
side is the C++ layer in csrc/host (vpinn::gpu::train etc.).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi

EPS_FIXED, EPS_SCALAR, EPS_SPATIAL = 0, 1, 2


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class TrainReport:
    records: np.ndarray  # structured: total, variational, boundary, sensor, lr, eps, seconds
    steps_run: int
    converged: bool
    stop_reason: int
    abort_step: int
    final_eps: float


def pin_problem(pb: "_capi.Problem"):
    """A copy of a filled vpinn_gpu_problem whose premultiplier tensors,
    forcing, points and strong-form forcing live in page-locked host memory
    (the caller's pinned input buffers): vpinn_gpu_create then DMAs them
    straight from there instead of staging them.  Returns (problem, keepalive)."""
    import torch
    out = _capi.Problem()
    C.pointer(out)[0] = pb
    E, T, Q = pb.n_elem, pb.n_test, pb.n_quad
    n_pts = pb.n_interior + pb.n_boundary + pb.n_sensors
    keep = []
    for name, nbytes in (("grad_x", 4 * E * T * Q), ("grad_y", 4 * E * T * Q), ("test", 4 * E * T * Q),
                         ("forcing", 4 * E * T), ("points", 16 * n_pts), ("strong_forcing", 4 * pb.n_interior)):
        src = getattr(pb, name)
        if not src:
            continue
        buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        C.memmove(buf.data_ptr(), src, nbytes)
        keep.append(buf)
        setattr(out, name, buf.data_ptr())
    return out, keep


class GpuStep:
    """One device context: the uploaded ProblemAssembly + network parameters."""

    def __init__(self, *, grad_x, grad_y, test, forcing, n_elem, n_test, n_quad, points,
                 n_interior, n_boundary, n_sensors, boundary_values=None, sensor_values=None,
                 layer_sizes: Sequence[int] = (2, 30, 30, 30, 1), sigmoid=False, n_scalars=0,
                 eps=1.0, bx=0.0, by=0.0, eps_source=EPS_FIXED, eps_scalar_index=0,
                 tau=10.0, gamma=10.0, device=0, rank=0, world_size=1, strong_forcing=None):
        """strong_forcing (f at the n_interior points) selects LossForm::strong
        (trainer.hpp:246-248); the tensors and forcing may then be None."""
        L = _capi.lib()
        f32 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
        f64 = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        self._keep = [f32(grad_x), f32(grad_y), f32(test), f32(forcing), f64(points),
                      f64(boundary_values), f64(sensor_values),
                      np.ascontiguousarray(layer_sizes, dtype=np.int32), f32(strong_forcing)]
        gx, gy, tv, fc, pts, bv, sv, ls, sf = self._keep
        pb = _capi.Problem()
        pb.n_elem, pb.n_test, pb.n_quad = n_elem, n_test, n_quad
        pb.grad_x, pb.grad_y, pb.test, pb.forcing, pb.points = _p(gx), _p(gy), _p(tv), _p(fc), _p(pts)
        pb.n_interior, pb.n_boundary, pb.n_sensors = n_interior, n_boundary, n_sensors
        pb.boundary_values, pb.sensor_values = _p(bv), _p(sv)
        pb.n_layer_sizes, pb.layer_sizes = len(ls), _p(ls)
        pb.activation = 1 if sigmoid else 0
        pb.n_scalars = n_scalars
        pb.eps, pb.bx, pb.by = eps, bx, by
        pb.eps_source, pb.eps_scalar_index = eps_source, eps_scalar_index
        pb.tau, pb.gamma = tau, gamma
        pb.device, pb.rank, pb.world_size = device, rank, world_size
        if sf is not None:
            pb.form, pb.strong_forcing = _capi.FORM_STRONG, _p(sf)
        h = C.c_void_p()
        _capi.check(L.vpinn_gpu_create(C.byref(pb), C.byref(h)))
        self.h = h
        self.n_elem, self.n_test, self.n_quad = n_elem, n_test, n_quad
        self.n_params = L.vpinn_gpu_param_count(h)
        self.layer_sizes = tuple(layer_sizes)

    @classmethod
    def from_problem(cls, pb: "_capi.Problem", keepalive=None) -> "GpuStep":
        """Create from an already filled vpinn_gpu_problem (e.g. the C++ host view)."""
        self = cls.__new__(cls)
        self._keep = [keepalive, pb]
        h = C.c_void_p()
        _capi.check(_capi.lib().vpinn_gpu_create(C.byref(pb), C.byref(h)))
        self.h = h
        self.n_elem, self.n_test, self.n_quad = pb.n_elem, pb.n_test, pb.n_quad
        self.n_params = _capi.lib().vpinn_gpu_param_count(h)
        sizes = C.cast(pb.layer_sizes, C.POINTER(C.c_int32))
        self.layer_sizes = tuple(sizes[i] for i in range(pb.n_layer_sizes))
        return self

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().vpinn_gpu_destroy(self.h)
            self.h = None

    __del__ = close

    # ---- parameters ----
    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        _capi.check(_capi.lib().vpinn_gpu_set_params(self.h, _p(p), p.size))

    def get_params(self):
        p = np.zeros(self.n_params, dtype=np.float32)
        _capi.check(_capi.lib().vpinn_gpu_get_params(self.h, _p(p), p.size))
        return p

    # ---- probes ----
    def loss_and_grad(self):
        parts = np.zeros(4)
        g = np.zeros(self.n_params)
        _capi.check(_capi.lib().vpinn_gpu_loss_and_grad(self.h, _p(parts), _p(g)))
        return parts, g

    def forward(self, points, order=1):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        n = pts.shape[0]
        u, ux, uy, e = (np.zeros(n, dtype=np.float32) for _ in range(4))
        _capi.check(_capi.lib().vpinn_gpu_forward(self.h, _p(pts), n, order, _p(u), _p(ux), _p(uy), _p(e)))
        return u, ux, uy, (e if self.layer_sizes[-1] >= 2 else None)

    def forward2(self, points):
        """evaluate(order 2): u, u_x, u_y, u_xx, u_yy (strong-form contexts)."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        n = pts.shape[0]
        outs = [np.zeros(n, dtype=np.float32) for _ in range(5)]
        _capi.check(_capi.lib().vpinn_gpu_forward2(self.h, _p(pts), n, *[_p(o) for o in outs]))
        return tuple(outs)

    def contract(self, ux, uy, eps=None, scalars=None, weight=1.0):
        ni = self.n_elem * self.n_quad
        ux = np.ascontiguousarray(ux, dtype=np.float32)
        uy = np.ascontiguousarray(uy, dtype=np.float32)
        e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float32)
        sc = None if scalars is None else np.ascontiguousarray(scalars, dtype=np.float32)
        loss = C.c_double()
        res = np.zeros(self.n_elem * self.n_test, dtype=np.float32)
        uxb = np.zeros(ni, dtype=np.float32)
        uyb = np.zeros(ni, dtype=np.float32)
        eb = np.zeros(ni, dtype=np.float32)
        sb = np.zeros(max(1, 0 if scalars is None else len(scalars)))
        _capi.check(_capi.lib().vpinn_gpu_contract(self.h, _p(ux), _p(uy), _p(e), _p(sc), weight,
                                                   C.byref(loss), _p(res), _p(uxb), _p(uyb), _p(eb), _p(sb)))
        return loss.value, res.reshape(self.n_elem, self.n_test), uxb, uyb, eb, sb

    def contract_matrix_free(self, ux, uy, scalars=None, weight=1.0):
        """vpinn_gpu_contract_matrix_free (device-assembly contexts)."""
        ni = self.n_elem * self.n_quad
        ux = np.ascontiguousarray(ux, dtype=np.float32)
        uy = np.ascontiguousarray(uy, dtype=np.float32)
        sc = None if scalars is None else np.ascontiguousarray(scalars, dtype=np.float32)
        loss = C.c_double()
        res = np.zeros(self.n_elem * self.n_test, dtype=np.float32)
        uxb = np.zeros(ni, dtype=np.float32)
        uyb = np.zeros(ni, dtype=np.float32)
        sb = np.zeros(max(1, 0 if scalars is None else len(scalars)))
        _capi.check(_capi.lib().vpinn_gpu_contract_matrix_free(self.h, _p(ux), _p(uy), _p(sc), weight, C.byref(loss),
                                                               _p(res), _p(uxb), _p(uyb), _p(sb)))
        return loss.value, res.reshape(self.n_elem, self.n_test), uxb, uyb, sb

    def time_contract_matrix_free(self, reps=20):
        ms, b = C.c_double(), C.c_double()
        _capi.check(_capi.lib().vpinn_gpu_time_contract_matrix_free(self.h, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    @staticmethod
    def assemble(nodes, cells, rule, basis, forcing="zero", device=0):
        """Device-side assembly (vpinn_gpu_assemble): nodes [n][2], cells
        [E][4], rule = (xi, eta, w), basis = (val, dxi, deta) [T][Q] ->
        dict of grad_x, grad_y, test ([E][T][Q] flat), forcing ([E][T] flat),
        quad_points [E*Q][2] (double)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        cells = np.ascontiguousarray(cells, dtype=np.int32)
        xi, eta, w = (np.ascontiguousarray(a, dtype=np.float64) for a in rule)
        val, dxi, deta = (np.ascontiguousarray(a, dtype=np.float64) for a in basis)
        E, Q, T = cells.shape[0], xi.size, val.size // xi.size
        a = _capi.Assembly()
        a.n_nodes = nodes.shape[0]
        a.nodes, a.elements, a.xi, a.eta, a.weights = _p(nodes), _p(cells), _p(xi), _p(eta), _p(w)
        a.basis_val, a.basis_dxi, a.basis_deta = _p(val), _p(dxi), _p(deta)
        a.forcing = forcing.encode()
        out = {k: np.zeros(E * T * Q, np.float32) for k in ("grad_x", "grad_y", "test")}
        out["forcing"] = np.zeros(E * T, np.float32)
        out["quad_points"] = np.zeros((E * Q, 2))
        _capi.check(_capi.lib().vpinn_gpu_assemble(device, E, T, Q, C.byref(a), _p(out["grad_x"]),
                                                   _p(out["grad_y"]), _p(out["test"]), _p(out["forcing"]),
                                                   _p(out["quad_points"])))
        return out

    def download_tensor(self, which: int, n: int):
        out = np.zeros(n, dtype=np.float32)
        _capi.check(_capi.lib().vpinn_gpu_download_tensor(self.h, which, _p(out), n))
        return out

    # ---- training ----
    def train(self, iterations, lr0=1e-3, lr_exponential=False, decay=0.99, every=1000,
              eps_abs_tol=None, eps_actual=None, loss_tol=None, plateau_window=2000,
              steps_per_graph=0) -> TrainReport:
        s = _capi.TrainSpec()
        s.iterations, s.lr_exponential, s.lr0, s.decay, s.every = iterations, int(lr_exponential), lr0, decay, every
        s.has_eps_abs_tol, s.eps_abs_tol = int(eps_abs_tol is not None), eps_abs_tol or 0.0
        s.has_eps_actual, s.eps_actual = int(eps_actual is not None), eps_actual or 0.0
        s.has_loss_tol, s.loss_tol = int(loss_tol is not None), loss_tol or 0.0
        s.plateau_window, s.steps_per_graph = plateau_window, steps_per_graph
        recs = (_capi.StepRecord * iterations)()
        res = _capi.TrainResult()
        rc = _capi.lib().vpinn_gpu_train(self.h, C.byref(s), recs, C.byref(res))
        arr = np.ctypeslib.as_array(recs)[: res.steps_run].copy() if res.steps_run else np.zeros(0)
        rep = TrainReport(arr, res.steps_run, bool(res.converged), res.stop_reason, res.abort_step,
                          res.final_eps)
        if rc != 0:
            err = _capi.VpinnError(rc, _capi.lib().vpinn_gpu_last_error().decode())
            err.report = rep
            raise err
        return rep

    def adam_reset(self):
        _capi.check(_capi.lib().vpinn_gpu_adam_reset(self.h))

    def run_steps(self, n, lr=1e-3):
        _capi.check(_capi.lib().vpinn_gpu_run_steps(self.h, n, lr))

    def synchronize(self):
        _capi.check(_capi.lib().vpinn_gpu_synchronize(self.h))

    def time_steps(self, n, lr=1e-3):
        ms = C.c_double()
        _capi.check(_capi.lib().vpinn_gpu_time_steps(self.h, n, lr, C.byref(ms)))
        return ms.value

    def time_contract(self, reps=20):
        ms, b = C.c_double(), C.c_double()
        _capi.check(_capi.lib().vpinn_gpu_time_contract(self.h, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def time_contract_kernels(self, reps=20):
        """(ms per launch, ms of the streaming kernel alone, algorithmic bytes)."""
        ms, ms1, b = C.c_double(), C.c_double(), C.c_double()
        _capi.check(_capi.lib().vpinn_gpu_time_contract_kernels(self.h, reps, C.byref(ms), C.byref(ms1), C.byref(b)))
        return ms.value, ms1.value, b.value

    def step_kernel(self) -> str:
        """Name of the kernel running this context's fused epoch step."""
        return _capi.lib().vpinn_gpu_step_kernel(self.h).decode()

    def profile_step(self, reps=10):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _capi.check(_capi.lib().vpinn_gpu_profile_step(self.h, reps, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def flush_l2(self):
        _capi.check(_capi.lib().vpinn_gpu_flush_l2(self.h))

    def launch_count(self):
        return _capi.lib().vpinn_gpu_launch_count(self.h)

    def attach_comm(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        _capi.check(_capi.lib().vpinn_gpu_attach_comm(self.h, buf, nranks, rank))

    def peer_handle(self) -> bytes:
        """This rank's mailbox as a 64-byte CUDA IPC handle (vpinn_gpu_peer_handle)."""
        buf = C.create_string_buffer(64)
        _capi.check(_capi.lib().vpinn_gpu_peer_handle(self.h, buf))
        return buf.raw

    def attach_peers(self, handles, nranks: int, rank: int):
        """Every rank's handle in rank order (vpinn_gpu_attach_peers)."""
        blob = b"".join(handles)
        assert len(blob) == 64 * nranks
        buf = C.create_string_buffer(blob, len(blob))
        _capi.check(_capi.lib().vpinn_gpu_attach_peers(self.h, buf, nranks, rank))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _capi.check(_capi.lib().vpinn_gpu_nccl_unique_id(buf))
    return buf.raw


def device_ok() -> bool:
    return bool(_capi.lib().vpinn_gpu_device_ok())
