"""ctypes front end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  It wraps oracle/_build/liboracle.so (built by
oracle/Makefile from oracle/vpinn_oracle.hpp, a plain-C++ restatement of the
reference hot path; see that header for the file:line map).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


_NATIVE_PATH = os.path.join(_HERE, "_build", "liboracle_native.so")
_NATIVE_STAMP = _NATIVE_PATH + ".cpu"
_native = None


def _cpu_id() -> str:
    try:
        first = open("/proc/cpuinfo").read().split("\n\n")[0]
    except OSError:
        return "unknown"
    keep = ("vendor_id", "cpu family", "model", "model name", "flags")
    return "\n".join(ln for ln in first.splitlines() if ln.split(":")[0].strip() in keep)


def lib_native():
    """The TIMING build (Makefile target 'native': the reference's
    -O3 -march=native flags + the Eigen-style float tanh).  Compiled on the
    machine that runs it (the stamp holds that CPU's /proc/cpuinfo entry), so
    -march=native never meets a different CPU.  Only bench.py's CPU-baseline
    legs use it; every check runs on lib()."""
    global _native
    if _native is None:
        cpu = _cpu_id()
        stale = not os.path.exists(_NATIVE_PATH) or not os.path.exists(_NATIVE_STAMP) or \
            open(_NATIVE_STAMP).read() != cpu
        if stale:
            if os.path.exists(_NATIVE_PATH):
                os.remove(_NATIVE_PATH)
            subprocess.run(["make", "-s", "-C", _HERE, "native"], check=True)
            with open(_NATIVE_STAMP, "w") as fh:
                fh.write(cpu)
        _native = C.CDLL(_NATIVE_PATH)
        _declare(_native)
    return _native


class OracleSpec(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int), ("nodes_xy", C.POINTER(C.c_double)),
        ("n_cells", C.c_int), ("cells", C.POINTER(C.c_int)),
        ("n_test_1d", C.c_int), ("n_quad_1d", C.c_int), ("lobatto", C.c_int),
        ("forcing", C.c_char_p), ("boundary_g", C.c_char_p), ("sensor_field", C.c_char_p),
        ("n_boundary", C.c_int), ("boundary_seed", C.c_ulonglong),
        ("n_sensors", C.c_int), ("sensor_seed", C.c_ulonglong),
        ("eps", C.c_double), ("bx", C.c_double), ("by", C.c_double),
        ("eps_source", C.c_int), ("eps_scalar_index", C.c_int),
        ("tau", C.c_double), ("gamma", C.c_double),
        ("n_sizes", C.c_int), ("sizes", C.POINTER(C.c_int)), ("sigmoid", C.c_int),
        ("n_scalars", C.c_int), ("scalar_init", C.POINTER(C.c_double)),
        ("seed", C.c_ulonglong), ("use_double", C.c_int), ("strong", C.c_int),
    ]


class OracleTrainSpec(C.Structure):
    _fields_ = [
        ("iterations", C.c_longlong), ("lr_exponential", C.c_int),
        ("lr0", C.c_double), ("decay", C.c_double), ("every", C.c_int), ("log_every", C.c_int),
        ("has_eps_tol", C.c_int), ("has_eps_actual", C.c_int), ("has_loss_tol", C.c_int),
        ("eps_abs_tol", C.c_double), ("eps_actual", C.c_double), ("loss_tol", C.c_double),
        ("plateau_window", C.c_int),
    ]


def _declare(L):
    vp = C.c_void_p
    L.vo_last_error.restype = C.c_char_p
    L.vo_build.restype = vp
    L.vo_build.argtypes = [C.POINTER(OracleSpec)]
    L.vo_free.argtypes = [vp]
    L.vo_is_double.argtypes = [vp]
    L.vo_counts.argtypes = [vp, C.POINTER(C.c_longlong)]
    L.vo_get_array.argtypes = [vp, C.c_int, vp]
    L.vo_loss_and_grad.argtypes = [vp, vp, C.POINTER(C.c_double), vp]
    L.vo_evaluate.argtypes = [vp, vp, vp, C.c_longlong, C.c_int, vp, vp, vp, vp]
    ll = C.c_longlong
    L.vo_loss_and_grad_part.argtypes = [vp, vp, ll, ll, ll, ll, ll, ll, C.POINTER(C.c_double), vp]
    L.vo_var_loss.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, C.c_double,
                              C.POINTER(C.c_double), vp, vp, vp, vp, vp]
    L.vo_train.argtypes = [vp, vp, C.POINTER(OracleTrainSpec), vp, C.POINTER(C.c_longlong),
                           C.POINTER(C.c_int), C.POINTER(C.c_double)]
    L.vo_time_steps.argtypes = [vp, vp, C.c_double, C.c_int, C.c_int, vp]
    L.vo_adam_f64.argtypes = [vp, vp, C.c_int, C.c_int, C.c_double]
    L.vo_adam_f32.argtypes = [vp, vp, C.c_int, C.c_int, vp]
    L.vo_lr_at.restype = C.c_double
    L.vo_lr_at.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_longlong]
    L.vo_gauss_rule.argtypes = [C.c_int, C.c_int, vp, vp]
    L.vo_test_fn.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.vo_field.argtypes = [C.c_char_p, vp, vp, C.c_longlong, vp]
    L.vo_structured_mesh.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_double, C.c_ulonglong, vp, vp]
    L.vo_init_params_f64.argtypes = [vp, C.c_int, C.c_ulonglong, vp]
    L.vo_evaluate2.argtypes = [vp, vp, vp, C.c_longlong, vp, vp, vp, vp, vp]
    L.vo_strong_loss.argtypes = [vp, vp, vp, vp, vp, ll, ll, ll, C.c_double, C.c_double,
                                 C.c_double, C.c_int, C.c_int, vp, C.c_int, vp, C.c_double,
                                 C.POINTER(C.c_double), vp, vp, vp, vp, vp]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().vo_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# small free functions
def gauss_rule(n: int, lobatto: bool = False):
    x = np.zeros(n)
    w = np.zeros(n)
    _check(lib().vo_gauss_rule(n, int(lobatto), _p(x), _p(w)))
    return x, w


def test_fn(k: int, x: float):
    v = C.c_double()
    d = C.c_double()
    lib().vo_test_fn(k, x, C.byref(v), C.byref(d))
    return v.value, d.value


def field(name: str, x, y):
    x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
    y = np.ascontiguousarray(np.atleast_1d(y), dtype=np.float64)
    out = np.zeros_like(x)
    _check(lib().vo_field(name.encode(), _p(x), _p(y), x.size, _p(out)))
    return out


def lr_at(lr0, step, decay=0.99, every=1000, exponential=False):
    return lib().vo_lr_at(int(exponential), lr0, decay, every, step)


def structured_mesh(nx, ny, x_range=(0.0, 1.0), y_range=(0.0, 1.0), skew=0.0, skew_seed=1234):
    nodes = np.zeros(((nx + 1) * (ny + 1), 2))
    cells = np.zeros((nx * ny, 4), dtype=np.int32)
    _check(lib().vo_structured_mesh(nx, ny, x_range[0], x_range[1], y_range[0], y_range[1],
                                    skew, skew_seed, _p(nodes), _p(cells)))
    return nodes, cells


def gear_msh41_text(n_r: int, n_t: int, teeth: int = 12, amp: float = 0.06, r_in: float = 0.35,
                    r_out: float = 1.0) -> str:
    """The reference fixture generator's gear recipe (proj/data/gen_fixtures.py
    main(), lines 158-179: ring of n_t x n_r quads, radius modulated by
    amp*sin(teeth*theta), inner and outer boundary lines) written as Gmsh 4.1
    text the way its msh41() writer does (lines 40-75: one entity block per
    dimension, '%.16g' coordinates).  Pure Python: the reference arm of
    bench.py builds the C5 gear with it without loading the product library.
    The SHA-256 at n_r=16, n_t=887 is pinned in tests/golden/gear_14192.json."""
    out = ["$MeshFormat", "4.1 0 8", "$EndMeshFormat"]
    nodes = []
    for j in range(n_r + 1):
        s = j / n_r
        for i in range(n_t):
            th = 2 * math.pi * i / n_t
            r = r_in + s * (r_out + amp * math.sin(teeth * th) - r_in)
            nodes.append((r * math.cos(th), r * math.sin(th)))
    nid = lambda i, j: j * n_t + (i % n_t) + 1  # noqa: E731
    n = len(nodes)
    out += ["$Nodes", f"1 {n} 1 {n}", f"2 1 0 {n}"]
    out += [str(i) for i in range(1, n + 1)]
    out += [f"{x:.16g} {y:.16g} 0" for x, y in nodes]
    out.append("$EndNodes")
    lines = [(nid(i, 0), nid(i + 1, 0)) for i in range(n_t)]
    lines += [(nid(i, n_r), nid(i + 1, n_r)) for i in range(n_t)]
    quads = [(nid(i, j), nid(i, j + 1), nid(i + 1, j + 1), nid(i + 1, j)) for j in range(n_r) for i in range(n_t)]
    total = len(lines) + len(quads)
    out += ["$Elements", f"2 {total} 1 {total}", f"1 1 1 {len(lines)}"]
    out += [f"{e + 1} {a} {b}" for e, (a, b) in enumerate(lines)]
    out.append(f"2 1 3 {len(quads)}")
    out += [f"{len(lines) + e + 1} {' '.join(map(str, q))}" for e, q in enumerate(quads)]
    out.append("$EndElements")
    return "\n".join(out) + "\n"


def gear_mesh(n_r: int = 16, n_t: int = 887):
    """(nodes [N][2] double, cells [E][4] 0-based) of gear_msh41_text, as the
    Gmsh reader sees them (coordinates parsed back from the '%.16g' text)."""
    lines = gear_msh41_text(n_r, n_t).split("\n")
    n = (n_r + 1) * n_t
    k = lines.index("$Nodes") + 3 + n  # past the block header and the node tags
    nodes = np.array([[float(v) for v in ln.split()[:2]] for ln in lines[k:k + n]], dtype=np.float64)
    k = lines.index("$Elements") + 3 + 2 * n_t + 1  # past the boundary-line block
    cells = np.array([[int(v) - 1 for v in ln.split()[1:5]] for ln in lines[k:k + n_r * n_t]], dtype=np.int32)
    return nodes, cells


def init_params_f64(sizes: Sequence[int], seed: int):
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    n = sum(sizes[i + 1] * sizes[i] + sizes[i + 1] for i in range(len(sizes) - 1))
    out = np.zeros(n)
    lib().vo_init_params_f64(_p(sz), len(sizes), seed, _p(out))
    return out


def adam_f64(p0, grads, lr):
    p = np.array(p0, dtype=np.float64)
    g = np.ascontiguousarray(grads, dtype=np.float64)
    _check(lib().vo_adam_f64(_p(p), _p(g), p.size, g.shape[0], lr))
    return p


def adam_f32(p0, grads, lrs):
    p = np.array(p0, dtype=np.float32)
    g = np.ascontiguousarray(grads, dtype=np.float32)
    lr = np.ascontiguousarray(lrs, dtype=np.float64)
    _check(lib().vo_adam_f32(_p(p), _p(g), p.size, g.shape[0], _p(lr)))
    return p


def strong_loss(u, ux, uy, uxx, uyy, begin, count, f, eps=1.0, bx=0.0, by=0.0, eps_source=0,
                eps_scalar_index=0, scalars=(), weight=1.0):
    """strong_residual_loss (losses.hpp:422-467) in double on given derivatives:
    returns (loss, uxb, uyb, uxxb, uyyb, scalar_bar)."""
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (u, ux, uy, uxx, uyy)]
    n = arrs[0].size
    fv = np.ascontiguousarray(f, dtype=np.float64)
    sc = np.ascontiguousarray(list(scalars) or [0.0], dtype=np.float64)
    outs = [np.zeros(n) for _ in range(4)]
    sb = np.zeros(max(1, len(scalars)))
    loss = C.c_double()
    _check(lib().vo_strong_loss(*[_p(a) for a in arrs], n, begin, count, eps, bx, by, eps_source,
                                eps_scalar_index, _p(sc), len(scalars), _p(fv), weight,
                                C.byref(loss), *[_p(o) for o in outs], _p(sb)))
    return (loss.value, *outs, sb[: len(scalars)])


# ---------------------------------------------------------------------------
@dataclass
class ProblemSpec:
    """Arguments of build_problem (commands.hpp:123-178) for a given mesh."""
    nodes: np.ndarray
    cells: np.ndarray
    n_test_1d: int = 5
    n_quad_1d: int = 10
    lobatto: bool = False
    forcing: str = "sin2pi_f"
    boundary_g: str = "sin2pi_u"
    sensor_field: Optional[str] = None
    n_boundary: int = 400
    boundary_seed: int = 1
    n_sensors: int = 0
    sensor_seed: int = 7
    eps: float = 1.0
    bx: float = 0.0
    by: float = 0.0
    eps_source: int = 0  # 0 fixed, 1 scalar, 2 spatial
    eps_scalar_index: int = 0
    tau: float = 10.0
    gamma: float = 10.0
    layers: Sequence[int] = (2, 30, 30, 30, 1)
    sigmoid: bool = False
    scalars: Sequence[float] = dc_field(default_factory=tuple)
    seed: int = 42
    strong: bool = False  # LossForm::strong (trainer.hpp:178)


class OracleProblem:
    def __init__(self, spec: ProblemSpec, double: bool = False, timing_build: bool = False):
        """timing_build: run on lib_native() (bench.py's CPU-baseline legs only)."""
        self._L = lib_native() if timing_build else lib()
        self.spec = spec
        self.double = double
        self.dtype = np.float64 if double else np.float32
        self._nodes = np.ascontiguousarray(spec.nodes, dtype=np.float64)
        self._cells = np.ascontiguousarray(spec.cells, dtype=np.int32)
        self._sizes = np.ascontiguousarray(spec.layers, dtype=np.int32)
        self._scal = np.ascontiguousarray(list(spec.scalars) or [0.0], dtype=np.float64)
        s = OracleSpec()
        s.n_nodes = self._nodes.shape[0]
        s.nodes_xy = self._nodes.ctypes.data_as(C.POINTER(C.c_double))
        s.n_cells = self._cells.shape[0]
        s.cells = self._cells.ctypes.data_as(C.POINTER(C.c_int))
        s.n_test_1d, s.n_quad_1d, s.lobatto = spec.n_test_1d, spec.n_quad_1d, int(spec.lobatto)
        s.forcing = spec.forcing.encode()
        s.boundary_g = spec.boundary_g.encode()
        s.sensor_field = (spec.sensor_field or "zero").encode()
        s.n_boundary, s.boundary_seed = spec.n_boundary, spec.boundary_seed
        s.n_sensors, s.sensor_seed = spec.n_sensors, spec.sensor_seed
        s.eps, s.bx, s.by = spec.eps, spec.bx, spec.by
        s.eps_source, s.eps_scalar_index = spec.eps_source, spec.eps_scalar_index
        s.tau, s.gamma = spec.tau, spec.gamma
        s.n_sizes = len(spec.layers)
        s.sizes = self._sizes.ctypes.data_as(C.POINTER(C.c_int))
        s.sigmoid = int(spec.sigmoid)
        s.n_scalars = len(spec.scalars)
        s.scalar_init = self._scal.ctypes.data_as(C.POINTER(C.c_double))
        s.seed = spec.seed
        s.use_double = int(double)
        s.strong = int(spec.strong)
        self._spec_c = s
        h = self._L.vo_build(C.byref(s))
        if not h:
            raise OracleError(-1, self._L.vo_last_error().decode())
        self.h = h
        cnt = (C.c_longlong * 7)()
        self._L.vo_counts(h, cnt)
        self.E, self.T, self.Q, self.n_int, self.n_bnd, self.n_sen, self.n_params = list(cnt)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self._L.vo_free(h)
            self.h = None

    @property
    def n_points(self):
        return self.n_int + self.n_bnd + self.n_sen

    def array(self, which: str) -> np.ndarray:
        idx = {"grad_x": 0, "grad_y": 1, "test": 2, "forcing": 3, "points": 4,
               "boundary_values": 5, "sensor_values": 6, "init_params": 7, "rule": 8,
               "strong_forcing": 9}[which]
        if idx <= 2:
            out = np.zeros(self.E * self.T * self.Q, dtype=self.dtype)
        elif idx == 3:
            out = np.zeros(self.E * self.T, dtype=self.dtype)
        elif idx == 4:
            out = np.zeros((self.n_points, 2))
        elif idx == 5:
            out = np.zeros(self.n_bnd)
        elif idx == 6:
            out = np.zeros(self.n_sen)
        elif idx == 7:
            out = np.zeros(self.n_params)
        elif idx == 9:
            out = np.zeros(self.n_int)
        else:
            out = np.zeros((3, self.Q))
        _check(self._L.vo_get_array(self.h, idx, _p(out)))
        return out

    def init_params(self) -> np.ndarray:
        return self.array("init_params").astype(self.dtype)

    def loss_and_grad(self, params):
        par = np.ascontiguousarray(params, dtype=self.dtype)
        parts = (C.c_double * 4)()
        grad = np.zeros(self.n_params, dtype=self.dtype)
        _check(self._L.vo_loss_and_grad(self.h, _p(par), parts, _p(grad)))
        return np.array(list(parts)), grad

    def loss_and_grad_part(self, params, e0, e1, b0, b1, s0, s1):
        """Rank sub-problem objective (global penalty normalisation)."""
        par = np.ascontiguousarray(params, dtype=self.dtype)
        parts = (C.c_double * 4)()
        grad = np.zeros(self.n_params, dtype=self.dtype)
        _check(self._L.vo_loss_and_grad_part(self.h, _p(par), e0, e1, b0, b1, s0, s1, parts, _p(grad)))
        return np.array(list(parts)), grad

    def evaluate(self, params, points, order=1):
        par = np.ascontiguousarray(params, dtype=self.dtype)
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        n = pts.shape[0]
        u, ux, uy = (np.zeros(n, dtype=self.dtype) for _ in range(3))
        eps = np.zeros(n, dtype=self.dtype) if self.spec.layers[-1] >= 2 else None
        _check(self._L.vo_evaluate(self.h, _p(par), _p(pts), n, order, _p(u),
                                 _p(ux) if order >= 1 else None, _p(uy) if order >= 1 else None,
                                 _p(eps) if eps is not None else None))
        return u, ux, uy, eps

    def evaluate2(self, params, points):
        """evaluate(order=2): u, u_x, u_y, u_xx, u_yy (network.hpp:414-449)."""
        par = np.ascontiguousarray(params, dtype=self.dtype)
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        n = pts.shape[0]
        outs = [np.zeros(n, dtype=self.dtype) for _ in range(5)]
        _check(self._L.vo_evaluate2(self.h, _p(par), _p(pts), n, *[_p(o) for o in outs]))
        return tuple(outs)

    def var_loss(self, ux, uy, eps=None, scalars=(), weight=1.0, loop=False):
        n = self.E * self.Q
        ux = np.ascontiguousarray(ux, dtype=self.dtype)
        uy = np.ascontiguousarray(uy, dtype=self.dtype)
        e = None if eps is None else np.ascontiguousarray(eps, dtype=self.dtype)
        sc = np.ascontiguousarray(list(scalars) or [0.0], dtype=np.float64)
        loss = C.c_double()
        res = np.zeros(self.E * self.T, dtype=self.dtype)
        uxb = np.zeros(n, dtype=self.dtype)
        uyb = np.zeros(n, dtype=self.dtype)
        eb = np.zeros(n, dtype=self.dtype)
        sb = np.zeros(max(1, len(scalars)))
        _check(self._L.vo_var_loss(self.h, int(loop), _p(ux), _p(uy), None if e is None else _p(e),
                                 _p(sc), len(scalars), weight, C.byref(loss), _p(res), _p(uxb),
                                 _p(uyb), _p(eb), _p(sb)))
        return loss.value, res.reshape(self.E, self.T), uxb, uyb, eb, sb[: len(scalars)]

    def train(self, params, iterations, lr0=1e-3, log_every=100, lr_exponential=False, decay=0.99,
              every=1000, eps_abs_tol=None, eps_actual=None, loss_tol=None, plateau_window=2000):
        par = np.array(params, dtype=self.dtype)
        ts = OracleTrainSpec()
        ts.iterations, ts.lr_exponential, ts.lr0, ts.decay = iterations, int(lr_exponential), lr0, decay
        ts.every, ts.log_every = every, log_every
        ts.has_eps_tol, ts.eps_abs_tol = int(eps_abs_tol is not None), eps_abs_tol or 0.0
        ts.has_eps_actual, ts.eps_actual = int(eps_actual is not None), eps_actual or 0.0
        ts.has_loss_tol, ts.loss_tol = int(loss_tol is not None), loss_tol or 0.0
        ts.plateau_window = plateau_window
        hist = np.zeros((iterations, 4))
        steps = C.c_longlong()
        reason = C.c_int()
        feps = C.c_double()
        _check(self._L.vo_train(self.h, _p(par), C.byref(ts), _p(hist), C.byref(steps),
                              C.byref(reason), C.byref(feps)))
        return {"params": par, "every_step": hist[: steps.value], "steps_run": steps.value,
                "stop_reason": reason.value, "final_eps": feps.value}

    def time_steps(self, params, lr=1e-3, warmup=1, reps=3):
        par = np.array(params, dtype=self.dtype)
        sec = np.zeros(reps)
        _check(self._L.vo_time_steps(self.h, _p(par), lr, warmup, reps, _p(sec)))
        return sec
