"""ctypes/numpy binding of the CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module, and only as the checker or the timed CPU
baseline.  The product package ``paper_1810_05628_b200`` never imports it.

Two libraries are bound (both built by ``oracle/Makefile`` into
``oracle/_ref/``):

* ``libptgo.so``        — our plain-C restatement (``oracle/ptgo.c``) of the
  reference hot path, generalised to the patch model (complex probe, M x M
  frames, free positions).
* ``libptycho_ref.so``  — the UNMODIFIED reference library
  (/root/reference/proj/src/*.cpp) plus a C veneer (``oracle/ref_capi.cpp``).
  Present only where /root/reference exists at build time.

Arrays: complex fields are numpy ``complex128`` (layout-identical to
``std::complex<double>``); patterns are ``float64``; positions ``int32 [N,2]``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)

DISTANCE, INTENSITY = 0, 1
STOP_NAMES = {0: "tolerance", 1: "budget", 2: "maxiters", 3: "stall"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr(a: Optional[np.ndarray], typ=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(typ)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- libptgo.so
class _Problem(C.Structure):
    _fields_ = [("n", C.c_int), ("M", C.c_int), ("w", C.c_int), ("N", C.c_int),
                ("pos", _ip), ("probe", _dp), ("data", _dp), ("metric", C.c_int)]


class _Counter(C.Structure):
    _fields_ = [("weighted", C.c_double), ("per_level", C.c_long * 16)]


class _Hist(C.Structure):
    _fields_ = [("weighted", C.c_double), ("value", C.c_double), ("gnorm", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("hist", C.POINTER(_Hist)), ("len", C.c_int), ("cap", C.c_int), ("reason", C.c_int)]


class _SolverCfg(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("grad_tol_rel", C.c_double), ("grad_tol_abs", C.c_double),
                ("lbfgs_memory", C.c_int), ("linesearch_max", C.c_int), ("max_weighted", C.c_double),
                ("cg_max_iters", C.c_int), ("cg_rel_tol", C.c_double)]


class _MgCfg(C.Structure):
    _fields_ = [("k1", C.c_int), ("k2", C.c_int), ("coarsest_max_iters", C.c_int),
                ("coarsest_grad_tol_rel", C.c_double), ("intermediate_grad_tol_rel", C.c_double),
                ("lbfgs_memory", C.c_int), ("linesearch_max", C.c_int), ("grad_tol_abs", C.c_double)]


class _DriverCfg(C.Structure):
    _fields_ = [("budget", C.c_double), ("grad_tol_rel", C.c_double), ("grad_tol_abs", C.c_double),
                ("max_cycles", C.c_int)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(REF_DIR, "libptgo.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.ptgo_last_error.restype = C.c_char_p
        L.ptgo_norm2sq.restype = C.c_double
        L.ptgo_norm2sq.argtypes = [_dp, C.c_size_t]
        L.ptgo_dot_real.restype = C.c_double
        L.ptgo_dot_real.argtypes = [_dp, _dp, C.c_size_t]
        L.ptgo_set_fft_hook.argtypes = [C.c_void_p]
        L.ptgo_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def has_reference() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libptycho_ref.so"))


def ref():
    global _ref
    if _ref is None:
        path = os.path.join(REF_DIR, "libptycho_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (reference sources absent at build time)")
        L = C.CDLL(path)
        L.ptref_last_error.restype = C.c_char_p
        L.ptref_norm2sq.restype = C.c_double
        L.ptref_dot_real.restype = C.c_double
        _ref = L
    return _ref


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().ptgo_last_error().decode())


def _check_ref(rc: int):
    if rc != 0:
        raise OracleError(rc, ref().ptref_last_error().decode())


def set_threads(t: int):
    lib().ptgo_set_threads(int(t))


def use_reference_fft(on: bool = True):
    """Route the oracle's 2-D FFTs through the reference's own OpenMP
    ``kernels::fft2_inplace`` (kernels.cpp:126) — the CPU-baseline setting."""
    if on:
        addr = C.cast(ref().ptref_fft2, C.c_void_p).value
        lib().ptgo_set_fft_hook(C.c_void_p(addr))
    else:
        lib().ptgo_set_fft_hook(None)


@dataclass
class Problem:
    """Patch-model problem; probe None = the reference's binary window."""
    n: int
    M: int
    w: int
    pos: np.ndarray                # int32 [N, 2]
    data: np.ndarray               # float64 [N, M, M]
    probe: Optional[np.ndarray] = None   # complex128 [M, M]
    metric: int = DISTANCE

    def __post_init__(self):
        self.pos = np.ascontiguousarray(self.pos, dtype=np.int32).reshape(-1, 2)
        self.data = _f64(self.data).reshape(-1, self.M, self.M)
        if self.probe is not None:
            self.probe = _c128(self.probe).reshape(self.M, self.M)

    @property
    def N(self) -> int:
        return self.pos.shape[0]

    def _c(self) -> _Problem:
        return _Problem(self.n, self.M, self.w, self.N, _ptr(self.pos, _ip),
                        _ptr(self.probe.view(np.float64)) if self.probe is not None else None,
                        _ptr(self.data), self.metric)


def fft2(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    out = _c128(a).copy()
    _check(lib().ptgo_fft2(_ptr(out.view(np.float64)), C.c_int(out.shape[0]), C.c_int(int(inverse))))
    return out


def norm2sq(a) -> float:
    a = _c128(a)
    return lib().ptgo_norm2sq(_ptr(a.view(np.float64)), a.size)


def dot_real(a, b) -> float:
    a, b = _c128(a), _c128(b)
    return lib().ptgo_dot_real(_ptr(a.view(np.float64)), _ptr(b.view(np.float64)), a.size)


def evaluate(p: Problem, z, v=None):
    z = _c128(z)
    v = _c128(v) if v is not None else None
    grad = np.zeros((p.n, p.n), np.complex128)
    val = C.c_double()
    prob = p._c()
    _check(lib().ptgo_evaluate(C.byref(prob), _ptr(z.view(np.float64)),
                               _ptr(v.view(np.float64)) if v is not None else None,
                               C.byref(val), _ptr(grad.view(np.float64))))
    return val.value, grad


def project_modulus(p: Problem, z, k: int) -> np.ndarray:
    z = _c128(z)
    out = np.zeros((p.M, p.M), np.complex128)
    prob = p._c()
    _check(lib().ptgo_project_modulus(C.byref(prob), _ptr(z.view(np.float64)), C.c_int(k),
                                      _ptr(out.view(np.float64))))
    return out


def simulate(n: int, M: int, w: int, pos, z, probe=None) -> np.ndarray:
    pos = np.ascontiguousarray(pos, dtype=np.int32).reshape(-1, 2)
    z = _c128(z)
    N = pos.shape[0]
    out = np.zeros((N, M, M), np.float64)
    p = Problem(n, M, w, pos, np.zeros((0, M, M)), probe)
    prob = _Problem(n, M, w, N, _ptr(p.pos, _ip),
                    _ptr(p.probe.view(np.float64)) if p.probe is not None else None, None, 0)
    _check(lib().ptgo_simulate(C.byref(prob), _ptr(z.view(np.float64)), _ptr(out)))
    return out


def philox4x64(ctr, key) -> np.ndarray:
    """One Philox4x64-10 block (4 uint64 words)."""
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    out = np.zeros(4, np.uint64)
    u64p = C.POINTER(C.c_uint64)
    lib().ptgo_philox4x64(c.ctypes.data_as(u64p), k.ctypes.data_as(u64p), out.ctypes.data_as(u64p))
    return out


def add_noise(d, level: float, seed: int = 0, uniforms=None) -> np.ndarray:
    """addNoise (forward.cpp:56-86) on a stack d [N, m, m]; uniforms None = Philox stream."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    N, mm = d.shape[0], int(np.prod(d.shape[1:]))
    out = np.empty_like(d)
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    _check(lib().ptgo_add_noise(C.c_int(N), C.c_size_t(mm), _ptr(d), C.c_double(level), C.c_uint64(seed),
                                _ptr(u) if u is not None else None, _ptr(out)))
    return out


def add_poisson(d, photons: float, seed: int = 4) -> np.ndarray:
    """Poisson photon noise, the GPU's sampler restated (Philox uniforms)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    N, mm = d.shape[0], int(np.prod(d.shape[1:]))
    out = np.empty_like(d)
    _check(lib().ptgo_add_poisson(C.c_int(N), C.c_size_t(mm), _ptr(d), C.c_double(photons), C.c_uint64(seed),
                                  _ptr(out)))
    return out


def ref_add_noise(d, level: float, seed: int) -> np.ndarray:
    """The reference's own addNoise (std::mt19937_64 stream)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    out = np.empty_like(d)
    _check_ref(ref().ptref_add_noise(C.c_int(d.shape[0]), C.c_int(d.shape[1]), _ptr(d), C.c_double(level),
                                     C.c_uint64(seed), _ptr(out)))
    return out


def ref_uniform_stream(seed: int, count: int) -> np.ndarray:
    """The first `count` rng::uniform01 draws of std::mt19937_64(seed) (rng.hpp:14-16)."""
    out = np.empty(count, np.float64)
    _check_ref(ref().ptref_uniform_stream(C.c_uint64(seed), C.c_size_t(count), _ptr(out)))
    return out


def restrict_field(f) -> np.ndarray:
    f = _c128(f)
    out = np.zeros((f.shape[0] // 2, f.shape[0] // 2), np.complex128)
    _check(lib().ptgo_restrict_field(_ptr(f.view(np.float64)), C.c_int(f.shape[0]),
                                     _ptr(out.view(np.float64))))
    return out


def prolong_field(f) -> np.ndarray:
    f = _c128(f)
    out = np.zeros((2 * f.shape[0], 2 * f.shape[0]), np.complex128)
    _check(lib().ptgo_prolong_field(_ptr(f.view(np.float64)), C.c_int(f.shape[0]),
                                    _ptr(out.view(np.float64))))
    return out


def restrict_data(d) -> np.ndarray:
    d = _f64(d)
    N, M = d.shape[0], d.shape[1]
    out = np.zeros((N, M // 2, M // 2), np.float64)
    _check(lib().ptgo_restrict_data(_ptr(d), C.c_int(N), C.c_int(M), _ptr(out)))
    return out


def _report(rep: _Report):
    hist = np.array([[rep.hist[i].weighted, rep.hist[i].value, rep.hist[i].gnorm]
                     for i in range(rep.len)], dtype=np.float64).reshape(-1, 3)
    reason = rep.reason
    lib().ptgo_report_free(C.byref(rep))
    return hist, reason


@dataclass
class SolveResult:
    z: np.ndarray
    value: float
    grad: Optional[np.ndarray]
    history: np.ndarray            # [iters+1, 3] = (weighted evals, value, |grad|)
    reason: int
    weighted: float
    per_level: list


def pie(p: Problem, z0, gamma: float = 0.0, sweeps: int = 1,
        max_weighted: float = float("inf")) -> SolveResult:
    z0 = _c128(z0)
    z = np.zeros_like(z0)
    ctr = _Counter()
    rep = _Report()
    fv = C.c_double()
    prob = p._c()
    _check(lib().ptgo_pie(C.byref(prob), _ptr(z0.view(np.float64)), C.c_double(gamma), C.c_int(sweeps),
                          C.c_double(max_weighted), C.byref(ctr), _ptr(z.view(np.float64)),
                          C.byref(fv), C.byref(rep)))
    hist, reason = _report(rep)
    return SolveResult(z, fv.value, None, hist, reason, ctr.weighted, list(ctr.per_level[:1]))


def solver_cfg(**kw) -> _SolverCfg:
    c = _SolverCfg()
    lib().ptgo_solver_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, _dp, _dp)


def _solver(fname: str, p: Problem, z0, v, cfg) -> SolveResult:
    z0 = _c128(z0)
    v = _c128(v) if v is not None else None
    n = p.n
    prob = p._c()

    def fn(_user, zp, valp, gp):
        return lib().ptgo_evaluate(C.byref(prob), zp, _ptr(v.view(np.float64)) if v is not None else None,
                                   valp, gp)

    cfn = _FN(fn)

    class _Counted(C.Structure):
        _fields_ = [("fn", _FN), ("user", C.c_void_p), ("len", C.c_size_t), ("level", C.c_int),
                    ("weight", C.c_double)]

    obj = _Counted(cfn, None, n * n, 0, 1.0)
    c = solver_cfg(**cfg)
    ctr = _Counter()
    rep = _Report()
    z = np.zeros_like(z0)
    g = np.zeros_like(z0)
    val = C.c_double()
    f = getattr(lib(), fname)
    f.argtypes = [C.c_void_p, _dp, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _dp, C.c_void_p, _dp,
                  C.c_void_p]
    _check(f(C.byref(obj), _ptr(z0.view(np.float64)), C.byref(c), C.byref(ctr), None, None,
             _ptr(z.view(np.float64)), C.byref(val), _ptr(g.view(np.float64)), C.byref(rep)))
    hist, reason = _report(rep)
    return SolveResult(z, val.value, g, hist, reason, ctr.weighted, [ctr.per_level[0]])


def lbfgs(p: Problem, z0, v=None, **cfg) -> SolveResult:
    """solvers.cpp:87-141 on the (v-shifted) objective of ``p``."""
    return _solver("ptgo_lbfgs", p, z0, v, cfg)


def truncated_newton(p: Problem, z0, v=None, **cfg) -> SolveResult:
    """solvers.cpp:143-227 on the (v-shifted) objective of ``p``."""
    return _solver("ptgo_truncated_newton", p, z0, v, cfg)


class Hierarchy:
    def __init__(self, p: Problem, depth: int, **mg):
        self.p = p
        self._prob = p._c()
        self.cfg = _MgCfg()
        lib().ptgo_mg_cfg_default(C.byref(self.cfg))
        for k, v in mg.items():
            setattr(self.cfg, k, v)
        self._h = C.c_void_p()
        _check(lib().ptgo_hierarchy_build(C.byref(self._prob), C.c_int(depth), C.byref(self.cfg),
                                          C.byref(self._h)))
        self.depth = depth

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().ptgo_hierarchy_free(self._h)
                self._h = None
        except Exception:
            pass

    def level(self, l: int) -> Problem:
        L = lib()
        L.ptgo_hierarchy_level.restype = C.POINTER(_Problem)
        pp = L.ptgo_hierarchy_level(self._h, C.c_int(l)).contents
        n, M, w, N = pp.n, pp.M, pp.w, pp.N
        pos = np.ctypeslib.as_array(pp.pos, shape=(N, 2)).copy()
        data = np.ctypeslib.as_array(pp.data, shape=(N, M, M)).copy()
        probe = None
        if pp.probe:
            probe = np.ctypeslib.as_array(pp.probe, shape=(M, M, 2)).copy().view(np.complex128)[..., 0]
        return Problem(n, M, w, pos, data, probe, pp.metric)

    def coarsest_iters(self) -> int:
        return lib().ptgo_hierarchy_coarsest_iters(self._h)

    def driver(self, z0, budget=100.0, grad_tol_rel=0.0, grad_tol_abs=1e-13,
               max_cycles=1000000) -> SolveResult:
        z0 = _c128(z0)
        dc = _DriverCfg(budget, grad_tol_rel, grad_tol_abs, max_cycles)
        ctr = _Counter()
        rep = _Report()
        z = np.zeros_like(z0)
        g = np.zeros_like(z0)
        val = C.c_double()
        _check(lib().ptgo_mgopt_driver(self._h, _ptr(z0.view(np.float64)), C.byref(dc), C.byref(ctr),
                                       _ptr(z.view(np.float64)), C.byref(val), _ptr(g.view(np.float64)),
                                       C.byref(rep)))
        hist, reason = _report(rep)
        return SolveResult(z, val.value, g, hist, reason, ctr.weighted,
                           [int(ctr.per_level[l]) for l in range(self.depth)])

    def cycle(self, level: int, z, v, warm=None):
        """One mgoptCycle (multigrid.cpp:117-169); returns (z, value, grad, weighted)."""
        z = _c128(z)
        v = _c128(v)
        ctr = _Counter()
        zo = np.zeros_like(z)
        go = np.zeros_like(z)
        val = C.c_double()
        wv = C.c_double(warm[0]) if warm is not None else None
        wg = _c128(warm[1]) if warm is not None else None
        _check(lib().ptgo_mgopt_cycle(self._h, C.c_int(level), _ptr(z.view(np.float64)),
                                      _ptr(v.view(np.float64)), C.byref(ctr),
                                      C.byref(wv) if wv is not None else None,
                                      _ptr(wg.view(np.float64)) if wg is not None else None,
                                      _ptr(zo.view(np.float64)), C.byref(val), _ptr(go.view(np.float64))))
        return zo, val.value, go, ctr.weighted


# ------------------------------------------------------ the reference itself
def ref_raster(n: int, w: int, s: int) -> np.ndarray:
    cap = max(1, ((n - w) // max(s, 1) + 1) ** 2)
    win = np.zeros((cap, 3), np.int32)
    cnt = C.c_int()
    _check_ref(ref().ptref_raster(n, w, s, _ptr(win, _ip), cap, C.byref(cnt)))
    return win[: cnt.value].copy()


def _win(pos, w) -> np.ndarray:
    pos = np.ascontiguousarray(pos, dtype=np.int32).reshape(-1, 2)
    out = np.zeros((pos.shape[0], 3), np.int32)
    out[:, :2] = pos
    out[:, 2] = w
    return out


def ref_simulate(n: int, w: int, pos, z) -> np.ndarray:
    win = _win(pos, w)
    z = _c128(z)
    out = np.zeros((win.shape[0], n, n), np.float64)
    _check_ref(ref().ptref_simulate(n, win.shape[0], _ptr(win, _ip), _ptr(z.view(np.float64)), _ptr(out)))
    return out


def ref_evaluate(metric: int, n: int, w: int, pos, data, z, v=None):
    win = _win(pos, w)
    data = _f64(data)
    z = _c128(z)
    v = _c128(v) if v is not None else None
    grad = np.zeros((n, n), np.complex128)
    val = C.c_double()
    _check_ref(ref().ptref_evaluate(metric, n, win.shape[0], _ptr(win, _ip), _ptr(data),
                                    _ptr(z.view(np.float64)),
                                    _ptr(v.view(np.float64)) if v is not None else None,
                                    C.byref(val), _ptr(grad.view(np.float64))))
    return val.value, grad


def ref_project_modulus(n: int, window, d, z) -> np.ndarray:
    win = np.ascontiguousarray(window, dtype=np.int32)
    d = _f64(d)
    z = _c128(z)
    out = np.zeros((n, n), np.complex128)
    _check_ref(ref().ptref_project_modulus(n, _ptr(win, _ip), _ptr(d), _ptr(z.view(np.float64)),
                                           _ptr(out.view(np.float64))))
    return out


def ref_fft2(a, inverse=False) -> np.ndarray:
    out = _c128(a).copy()
    _check_ref(ref().ptref_fft2_checked(_ptr(out.view(np.float64)), out.shape[0], int(inverse)))
    return out


def ref_restrict_field(f):
    f = _c128(f)
    out = np.zeros((f.shape[0] // 2,) * 2, np.complex128)
    _check_ref(ref().ptref_restrict_field(_ptr(f.view(np.float64)), f.shape[0], _ptr(out.view(np.float64))))
    return out


def ref_prolong_field(f):
    f = _c128(f)
    out = np.zeros((2 * f.shape[0],) * 2, np.complex128)
    _check_ref(ref().ptref_prolong_field(_ptr(f.view(np.float64)), f.shape[0], _ptr(out.view(np.float64))))
    return out


def ref_restrict_data(d):
    d = _f64(d)
    N, n = d.shape[0], d.shape[1]
    out = np.zeros((N, n // 2, n // 2), np.float64)
    _check_ref(ref().ptref_restrict_data(_ptr(d), N, n, _ptr(out)))
    return out


def ref_pie(n, w, pos, data, z0, gamma=0.0, sweeps=1, max_weighted=float("inf")) -> SolveResult:
    win = _win(pos, w)
    data = _f64(data)
    z0 = _c128(z0)
    z = np.zeros_like(z0)
    cap = sweeps + 2
    hist = np.zeros((cap, 3))
    nh = C.c_int()
    fv, wt = C.c_double(), C.c_double()
    reason = C.c_int()
    _check_ref(ref().ptref_pie(n, win.shape[0], _ptr(win, _ip), _ptr(data), _ptr(z0.view(np.float64)),
                               C.c_double(gamma), sweeps, C.c_double(max_weighted),
                               _ptr(z.view(np.float64)), C.byref(fv), _ptr(hist), cap, C.byref(nh),
                               C.byref(wt), C.byref(reason)))
    return SolveResult(z, fv.value, None, hist[: nh.value].copy(), reason.value, wt.value, [])


def ref_lbfgs(metric, n, w, pos, data, z0, v=None, max_iters=100, grad_tol_rel=0.0,
              grad_tol_abs=1e-13, lbfgs_memory=25, linesearch_max=50,
              max_weighted=float("inf")) -> SolveResult:
    win = _win(pos, w)
    data = _f64(data)
    z0 = _c128(z0)
    v = _c128(v) if v is not None else None
    z = np.zeros_like(z0)
    g = np.zeros_like(z0)
    cap = max_iters + 2
    hist = np.zeros((cap, 3))
    nh = C.c_int()
    val, wt = C.c_double(), C.c_double()
    reason = C.c_int()
    _check_ref(ref().ptref_lbfgs(metric, n, win.shape[0], _ptr(win, _ip), _ptr(data),
                                 _ptr(v.view(np.float64)) if v is not None else None,
                                 _ptr(z0.view(np.float64)), max_iters, C.c_double(grad_tol_rel),
                                 C.c_double(grad_tol_abs), lbfgs_memory, linesearch_max,
                                 C.c_double(max_weighted), _ptr(z.view(np.float64)), C.byref(val),
                                 _ptr(g.view(np.float64)), _ptr(hist), cap, C.byref(nh), C.byref(wt),
                                 C.byref(reason)))
    return SolveResult(z, val.value, g, hist[: nh.value].copy(), reason.value, wt.value, [])


def ref_truncated_newton(metric, n, w, pos, data, z0, v=None, max_iters=100, grad_tol_rel=0.0,
                         grad_tol_abs=1e-13, linesearch_max=50, cg_max_iters=20, cg_rel_tol=0.1,
                         max_weighted=float("inf")) -> SolveResult:
    win = _win(pos, w)
    data = _f64(data)
    z0 = _c128(z0)
    v = _c128(v) if v is not None else None
    z = np.zeros_like(z0)
    g = np.zeros_like(z0)
    cap = max_iters + 2
    hist = np.zeros((cap, 3))
    nh = C.c_int()
    val, wt = C.c_double(), C.c_double()
    reason = C.c_int()
    _check_ref(ref().ptref_truncated_newton(
        metric, n, win.shape[0], _ptr(win, _ip), _ptr(data), _ptr(v.view(np.float64)) if v is not None else None,
        _ptr(z0.view(np.float64)), max_iters, C.c_double(grad_tol_rel), C.c_double(grad_tol_abs), linesearch_max,
        cg_max_iters, C.c_double(cg_rel_tol), C.c_double(max_weighted), _ptr(z.view(np.float64)), C.byref(val),
        _ptr(g.view(np.float64)), _ptr(hist), cap, C.byref(nh), C.byref(wt), C.byref(reason)))
    return SolveResult(z, val.value, g, hist[: nh.value].copy(), reason.value, wt.value, [])


def ref_mgopt(metric, n, w, s, data, z0, depth, k1=1, k2=1, coarsest_max_iters=0, budget=100.0,
              grad_tol_rel=0.0, grad_tol_abs=1e-13, max_cycles=1000000) -> SolveResult:
    data = _f64(data)
    z0 = _c128(z0)
    z = np.zeros_like(z0)
    cap = max_cycles + 2 if max_cycles < 100000 else 100000
    hist = np.zeros((cap, 3))
    nh = C.c_int()
    val, wt = C.c_double(), C.c_double()
    per = (C.c_long * 16)()
    reason = C.c_int()
    _check_ref(ref().ptref_mgopt(metric, n, w, s, _ptr(data), depth, k1, k2, coarsest_max_iters,
                                 C.c_double(budget), C.c_double(grad_tol_rel), C.c_double(grad_tol_abs),
                                 max_cycles, _ptr(z0.view(np.float64)), _ptr(z.view(np.float64)),
                                 C.byref(val), _ptr(hist), cap, C.byref(nh), C.byref(wt), per,
                                 C.byref(reason)))
    return SolveResult(z, val.value, None, hist[: min(nh.value, cap)].copy(), reason.value, wt.value,
                       [int(per[l]) for l in range(depth)])


def ref_metrics(z, z_true):
    """metrics.cpp:67-136 via the reference: (relativeError, magnitudeRelError, phaseSSIM)."""
    z = _c128(z)
    zt = _c128(z_true)
    out = np.zeros(3)
    _check_ref(ref().ptref_metrics(z.shape[0], _ptr(z.view(np.float64)), _ptr(zt.view(np.float64)), _ptr(out)))
    return tuple(out)


def ref_canonical_phase(z):
    z = _c128(z)
    out = np.zeros(z.shape)
    _check_ref(ref().ptref_canonical_phase(z.shape[0], _ptr(z.view(np.float64)), _ptr(out)))
    return out
