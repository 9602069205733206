"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle (oracle/_build/libttsw_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module;
the product package (paper_2408_03483_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import traceback
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("TTSW_ORACLE_LIB") or os.path.join(_HERE, "_build", "libttsw_oracle.so")

OK, INPUT, SHAPE, STATE, DEGENERACY, CONVERGENCE, EVALUATION, INTERNAL, DEADLINE = 0, 1, 2, 3, 4, 5, 6, 8, 9


class OracleError(Exception):
    def __init__(self, code, msg, residual=0.0, iterations=0, row=-1, col=-1):
        super().__init__(msg)
        self.code, self.residual, self.iterations, self.row, self.col = code, residual, iterations, row, col


class InputError(OracleError): pass
class ShapeError(OracleError): pass
class StateError(OracleError): pass
class DegeneracyError(OracleError): pass
class ConvergenceError(OracleError): pass
class EvaluationError(OracleError): pass
class DeadlineReached(OracleError): pass  # bench-only bounded CPU sample ran out of time


_EXC = {INPUT: InputError, SHAPE: ShapeError, STATE: StateError, DEGENERACY: DegeneracyError,
        CONVERGENCE: ConvergenceError, EVALUATION: EvaluationError, DEADLINE: DeadlineReached}


class CrossCfg(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_rank", C.c_long), ("max_sweeps", C.c_int),
                ("rank_increment", C.c_long), ("validation_sample", C.c_int), ("seed", C.c_ulonglong)]

    @staticmethod
    def make(eps=1e-10, max_rank=128, max_sweeps=30, rank_increment=2, validation_sample=1000,
             seed=0x5EED5EED):
        return CrossCfg(eps, max_rank, max_sweeps, rank_increment, validation_sample, seed)


class CrossStats(C.Structure):
    _fields_ = [("evaluations", C.c_long), ("sweeps", C.c_int), ("residual", C.c_double)]


class SolverDesc(C.Structure):
    _fields_ = [("model", C.c_int), ("scheme", C.c_int), ("n", C.c_long), ("g", C.c_double),
                ("f", C.c_double), ("H", C.c_double), ("dt", C.c_double), ("tol", C.c_double),
                ("lambda_eps_floor", C.c_double), ("cross", CrossCfg)]


# RhsHooks callbacks (ttsw_oracle.h): borrowed q3 handles in, three owned handles out.
GHOST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_double, C.POINTER(C.c_void_p))
SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.POINTER(C.c_void_p))


def _borrow(h):
    t = TT.__new__(TT)
    t.h = C.c_void_p(h)
    return t


def _release(t):
    h = t.h.value
    t.h = None
    return h


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        D = C.POINTER(C.c_double)
        L.ttor_tt_new.restype = P
        L.ttor_tt_new.argtypes = [C.c_long, C.c_long, C.c_long, D, D]
        L.ttor_tt_free.argtypes = [P]
        L.ttor_set_sample_deadline.argtypes = [C.c_double]
        L.ttor_solver_set_eps_policy.argtypes = [P, C.c_double, C.c_int, C.c_double, C.c_double]
        L.ttor_solver_eps.argtypes = [P, D]
        L.ttor_tt_dims.argtypes = [P, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_long)]
        L.ttor_tt_get.argtypes = [P, D, D]
        L.ttor_solver_new.restype = P
        L.ttor_solver_new.argtypes = [C.POINTER(SolverDesc)]
        L.ttor_solver_free.argtypes = [P]
        L.ttor_solver_get_state.restype = P
        L.ttor_solver_get_state.argtypes = [P, C.c_int]
        L.ttor_solver_set_state.argtypes = [P, C.c_int, P]
        L.ttor_solver_step.argtypes = [P, C.c_long]
        L.ttor_solver_rhs.argtypes = [P, C.POINTER(C.c_void_p)]
        L.ttor_solver_set_hooks.argtypes = [P, GHOST_FN, SOURCE_FN, P]
        L.ttor_solver_set_time.argtypes = [P, C.c_double]
        L.ttor_solver_time.restype = C.c_double
        L.ttor_solver_time.argtypes = [P]
        L.ttor_solver_trace_len.restype = C.c_long
        L.ttor_solver_trace_len.argtypes = [P]
        L.ttor_solver_trace.argtypes = [P, C.POINTER(C.c_long), D, D]
        L.ttor_solver_trace_clear.argtypes = [P]
        L.ttor_rng_new.restype = P
        L.ttor_rng_new.argtypes = [C.c_ulonglong]
        L.ttor_rng_free.argtypes = [P]
        L.ttor_rng_normal.argtypes = [P, C.c_long, D]
        L.ttor_rng_uniform_int.argtypes = [P, C.c_long, C.c_long, C.c_long, C.POINTER(C.c_long)]
        L.ttor_rng_uniform_real.argtypes = [P, C.c_double, C.c_double, C.c_long, D]
        L.ttor_rng_raw.restype = C.c_ulonglong
        L.ttor_rng_raw.argtypes = [P]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(code):
    if code != OK:
        buf = C.create_string_buffer(4096)
        res, it, row, col = C.c_double(), C.c_int(), C.c_long(), C.c_long()
        lib().ttor_last_error(buf, 4096, C.byref(res), C.byref(it), C.byref(row), C.byref(col))
        cls = _EXC.get(code, OracleError)
        raise cls(code, buf.value.decode(), res.value, it.value, row.value, col.value)


class TT:
    """Owning handle of an oracle TTMatrix (core_x m x r, core_y r x n, column-major)."""

    def __init__(self, handle):
        if not handle:
            _check(INPUT if True else OK)
        self.h = C.c_void_p(handle)

    @staticmethod
    def from_cores(cx, cy):
        cx = np.asfortranarray(cx, dtype=np.float64)
        cy = np.asfortranarray(cy, dtype=np.float64)
        if cx.ndim != 2 or cy.ndim != 2:
            raise ValueError("cores must be 2-D")
        h = lib().ttor_tt_new(cx.shape[0], cy.shape[1], cx.shape[1], _dp(cx), _dp(cy))
        if not h:
            _check(INPUT)
        return TT(h)

    @staticmethod
    def constant(m, n, v):
        return TT.from_cores(np.full((m, 1), float(v)), np.ones((1, n)))

    @staticmethod
    def zero(m, n):
        return TT.from_cores(np.zeros((m, 1)), np.zeros((1, n)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ttor_tt_free(self.h)
            self.h = None

    @property
    def shape(self):
        m, n, r = C.c_long(), C.c_long(), C.c_long()
        lib().ttor_tt_dims(self.h, C.byref(m), C.byref(n), C.byref(r))
        return m.value, n.value, r.value

    @property
    def rank(self):
        return self.shape[2]

    def cores(self):
        m, n, r = self.shape
        cx = np.zeros((m, r), order="F")
        cy = np.zeros((r, n), order="F")
        lib().ttor_tt_get(self.h, _dp(cx), _dp(cy))
        return cx, cy

    def full(self):
        cx, cy = self.cores()
        return cx @ cy


def _out():
    return C.c_void_p()


def from_full(a, eps):
    a = np.asfortranarray(a, dtype=np.float64)
    o = _out()
    _check(lib().ttor_from_full(C.c_long(a.shape[0]), C.c_long(a.shape[1]), _dp(a), C.c_double(eps), C.byref(o)))
    return TT(o.value)


def round_(x, eps, with_margin=False):
    o, k, mg, ka = _out(), C.c_long(), C.c_double(), C.c_double()
    _check(lib().ttor_round(x.h, C.c_double(eps), C.byref(o), C.byref(k), C.byref(mg), C.byref(ka)))
    t = TT(o.value)
    return (t, mg.value, ka.value) if with_margin else t


def add(x, y):
    o = _out()
    _check(lib().ttor_add(x.h, y.h, C.byref(o)))
    return TT(o.value)


def scale(x, a):
    o = _out()
    _check(lib().ttor_scale(x.h, C.c_double(a), C.byref(o)))
    return TT(o.value)


def axpy(a, x, b, y, eps):
    o = _out()
    _check(lib().ttor_axpy(C.c_double(a), x.h, C.c_double(b), y.h, C.c_double(eps), C.byref(o)))
    return TT(o.value)


def hadamard(x, y):
    o = _out()
    _check(lib().ttor_hadamard(x.h, y.h, C.byref(o)))
    return TT(o.value)


def norm_fro(x):
    v = C.c_double()
    _check(lib().ttor_norm_fro(x.h, C.byref(v)))
    return v.value


def sum_entries(x):
    v = C.c_double()
    _check(lib().ttor_sum_entries(x.h, C.byref(v)))
    return v.value


def core_map(x, axis, op, scheme=0, side=0, n=0, a0=0, a1=0):
    o = _out()
    _check(lib().ttor_core_map(x.h, C.c_int(axis), C.c_int(op), C.c_int(scheme), C.c_int(side), C.c_long(n),
                               C.c_long(a0), C.c_long(a1), C.byref(o)))
    return TT(o.value)


def core_map_dense(x, axis, m):
    m = np.asfortranarray(m, dtype=np.float64)
    o = _out()
    _check(lib().ttor_core_map_dense(x.h, C.c_int(axis), C.c_long(m.shape[0]), C.c_long(m.shape[1]), _dp(m),
                                     C.byref(o)))
    return TT(o.value)


def recip(x, eps, max_iterations=200):
    o, it = _out(), C.c_int()
    try:
        _check(lib().ttor_recip(x.h, C.c_double(eps), C.c_int(max_iterations), C.byref(it), C.byref(o)))
    except OracleError as e:
        e.recip_iterations = it.value
        raise
    return TT(o.value), it.value


FN_IDENTITY, FN_PRODUCT, FN_SQRT, FN_AFFINE, FN_SQUARE = 0, 1, 2, 3, 4
FN_WENO5_S1_MINUS, FN_WENO5_S1_PLUS, FN_WENO5_S2_QUAD = 10, 11, 12
FN_LLF_LAMBDA, FN_WAVE_SPEED = 20, 21


def cross(fn, ops, guess, cfg=None, param=0.0):
    arr = (C.c_void_p * len(ops))(*[o.h.value for o in ops])
    p = (C.c_double * 1)(param)
    o, st = _out(), CrossStats()
    cfg = cfg or CrossCfg.make()
    _check(lib().ttor_cross(C.c_int(fn), p, arr, C.c_int(len(ops)), guess.h, C.byref(cfg), C.byref(o), C.byref(st)))
    return TT(o.value), st


def maxvol(m):
    m = np.asfortranarray(m, dtype=np.float64)
    rows = (C.c_long * m.shape[1])()
    _check(lib().ttor_maxvol(C.c_long(m.shape[0]), C.c_long(m.shape[1]), _dp(m), rows))
    return list(rows)


def svd_values(a):
    a = np.asfortranarray(a, dtype=np.float64)
    s = np.zeros(min(a.shape))
    _check(lib().ttor_svd_values(C.c_long(a.shape[0]), C.c_long(a.shape[1]), _dp(a), _dp(s)))
    return s


def truncation_rank(sv, eps):
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    k, mg = C.c_long(), C.c_double()
    _check(lib().ttor_truncation_rank(_dp(sv), C.c_long(len(sv)), C.c_double(eps), C.byref(k), C.byref(mg)))
    return k.value, mg.value


def tables(scheme):
    out = np.zeros(96)
    _check(lib().ttor_tables(C.c_int(scheme), _dp(out)))
    k = int(out[83])
    nq = int(out[84])
    return {
        "step1_c": out[0:9].reshape(3, 3)[: k + 1, : k + 1].copy(),
        "step1_ideal": out[9:9 + k + 1].copy(),
        "step1_row": out[12:12 + 2 * k + 1].copy(),
        "c": [out[17 + m * 9:26 + m * 9].reshape(3, 3)[: k + 1, : k + 1].copy() for m in range(nq)],
        "gamma": [out[44 + m * 3:44 + m * 3 + k + 1].copy() for m in range(nq)],
        "point_row": [out[53 + m * 5:53 + m * 5 + 2 * k + 1].copy() for m in range(nq)],
        "gamma_plus": out[68:71].copy(), "gamma_minus": out[71:74].copy(), "weno_d": out[74:77].copy(),
        "offset": out[77:77 + nq].copy(), "weight": out[80:80 + nq].copy(), "radius": k, "nq": nq,
        "sigma_plus": out[85], "sigma_minus": out[86],
    }


def weno_step1(v5, eps):
    v = np.ascontiguousarray(v5, dtype=np.float64)
    o = C.c_double()
    _check(lib().ttor_weno_step1(_dp(v), C.c_double(eps), C.byref(o)))
    return o.value


def weno_step2(v5, m, eps):
    v = np.ascontiguousarray(v5, dtype=np.float64)
    o = C.c_double()
    _check(lib().ttor_weno_step2(_dp(v), C.c_int(m), C.c_double(eps), C.byref(o)))
    return o.value


def smoothness(v5):
    v = np.ascontiguousarray(v5, dtype=np.float64)
    b = np.zeros(3)
    _check(lib().ttor_smoothness(_dp(v), _dp(b)))
    return b


def weno_weights(beta, ideal, eps):
    b = np.ascontiguousarray(beta, dtype=np.float64)
    i = np.ascontiguousarray(ideal, dtype=np.float64)
    o = np.zeros(3)
    _check(lib().ttor_weno_weights(_dp(b), _dp(i), C.c_double(eps), _dp(o)))
    return o


def periodic_ghost(x):
    o = _out()
    _check(lib().ttor_periodic_ghost(x.h, C.byref(o)))
    return TT(o.value)


def ghosted(x, bc_x, bc_y, strip_x=None, strip_y=None, eps_tt=-1.0):
    sx = np.asfortranarray(strip_x, dtype=np.float64) if bc_x else None
    sy = np.asfortranarray(strip_y, dtype=np.float64) if bc_y else None
    o = _out()
    _check(lib().ttor_ghosted(x.h, int(bc_x), int(bc_y), _dp(sx) if sx is not None else None,
                              _dp(sy) if sy is not None else None, C.c_double(eps_tt), C.byref(o)))
    return TT(o.value)


def reconstruct_faces(g, axis, scheme, eps_tt=1e-12, cfg=None, dx=1.0, dy=1.0):
    mi, pl = _out(), _out()
    cfg = cfg or CrossCfg.make()
    _check(lib().ttor_reconstruct_faces(g.h, C.c_int(axis), C.c_int(scheme), C.c_double(eps_tt), C.byref(cfg),
                                        C.c_double(dx), C.c_double(dy), C.byref(mi), C.byref(pl)))
    return TT(mi.value), TT(pl.value)


def physical_flux(u3, axis, model, g, f, H, eps):
    arr = (C.c_void_p * 3)(*[u.h.value for u in u3])
    out = (C.c_void_p * 3)()
    _check(lib().ttor_physical_flux(arr, C.c_int(axis), C.c_int(model), C.c_double(g), C.c_double(f),
                                    C.c_double(H), C.c_double(eps), out))
    return [TT(out[c]) for c in range(3)]


class Solver:
    """Oracle SSP-RK3 driver: fixed EpsSchedule, periodic ghosts (swe.hpp:362-454)."""

    def __init__(self, model, scheme, n, g, f, H, dt, tol, cross_cfg=None, lambda_eps_floor=1e-6):
        cfg = cross_cfg or CrossCfg.make(seed=1)
        self.desc = SolverDesc(model, scheme, n, g, f, H, dt, tol, lambda_eps_floor, cfg)
        self.h = C.c_void_p(lib().ttor_solver_new(C.byref(self.desc)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ttor_solver_free(self.h)
            self.h = None

    def set_hooks(self, fill_ghost=None, extra_source=None):
        """RhsHooks (swe.hpp:276-282): fill_ghost([q0, q1, q2], t) -> 3 ghosted TTs,
        extra_source(t) -> 3 TTs (None keeps the periodic ghosts / no extra source)."""

        def ghost(user, q3, t, out):
            qs = [_borrow(q3[c]) for c in range(3)]
            try:
                res = fill_ghost(qs, t)
                for c in range(3):
                    out[c] = _release(res[c])
                return 0
            except Exception:
                traceback.print_exc()
                return 1
            finally:  # borrowed: owned by the library
                for q in qs:
                    q.h = None

        def source(user, t, out):
            try:
                res = extra_source(t)
                for c in range(3):
                    out[c] = _release(res[c])
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        self._hooks = (GHOST_FN(ghost) if fill_ghost else GHOST_FN(), SOURCE_FN(source) if extra_source else SOURCE_FN())
        _check(lib().ttor_solver_set_hooks(self.h, self._hooks[0], self._hooks[1], None))

    @property
    def time(self):
        return lib().ttor_solver_time(self.h)

    @time.setter
    def time(self, t):
        _check(lib().ttor_solver_set_time(self.h, float(t)))

    def set_state(self, tts):
        for c, t in enumerate(tts):
            _check(lib().ttor_solver_set_state(self.h, c, t.h))

    def state(self):
        return [TT(lib().ttor_solver_get_state(self.h, c)) for c in range(3)]

    def rhs(self):
        out = (C.c_void_p * 3)()
        _check(lib().ttor_solver_rhs(self.h, out))
        return [TT(out[c]) for c in range(3)]

    def step(self, nsteps=1):
        _check(lib().ttor_solver_step(self.h, C.c_long(nsteps)))

    def set_eps_policy(self, c_eps, order=3, volume=1.0, clip=1e-3):
        _check(lib().ttor_solver_set_eps_policy(self.h, float(c_eps), int(order), float(volume), float(clip)))

    def eps(self):
        out = np.zeros(4)
        lib().ttor_solver_eps(self.h, _dp(out))
        return out

    def step_sample(self, seconds):
        """Bench only: one step bounded by `seconds` of wall time. Returns True when the step
        completed; otherwise the rounding trace holds the completed roundings."""
        lib().ttor_set_sample_deadline(float(seconds))
        try:
            self.step(1)
            return True
        except DeadlineReached:
            return False
        finally:
            lib().ttor_set_sample_deadline(0.0)

    def trace(self, clear=True):
        n = lib().ttor_solver_trace_len(self.h)
        ints = np.zeros(6 * n, dtype=np.int64)
        mg = np.zeros(n)
        ka = np.zeros(n)
        if n:
            lib().ttor_solver_trace(self.h, ints.ctypes.data_as(C.POINTER(C.c_long)), _dp(mg), _dp(ka))
        if clear:
            lib().ttor_solver_trace_clear(self.h)
        return ints.reshape(n, 6), mg, ka

    def cross_trace(self, clear=True):
        L = lib()
        L.ttor_solver_cross_trace_len.restype = C.c_long
        n = L.ttor_solver_cross_trace_len(self.h)
        ints = np.zeros(3 * n, dtype=np.int64)
        res = np.zeros(n)
        L.ttor_solver_cross_trace(self.h, ints.ctypes.data_as(C.POINTER(C.c_long)), _dp(res), C.c_int(1 if clear else 0))
        return ints.reshape(n, 3), res


class Rng:
    """std::mt19937_64 + libstdc++ distributions, mirroring tests/support.hpp."""

    def __init__(self, seed):
        self.h = C.c_void_p(lib().ttor_rng_new(C.c_ulonglong(seed)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ttor_rng_free(self.h)
            self.h = None

    def random_matrix(self, rows, cols):
        out = np.zeros(rows * cols)
        lib().ttor_rng_normal(self.h, rows * cols, _dp(out))
        return out.reshape((rows, cols), order="F")

    def random_tt(self, rows, cols, rank):
        return TT.from_cores(self.random_matrix(rows, rank), self.random_matrix(rank, cols))

    def random_orthonormal(self, rows, cols):
        a = self.random_matrix(rows, cols)
        q, r = np.linalg.qr(a)
        # Householder QR sign convention (Eigen): R diagonal has sign -sign(a_kk...) — any
        # orthonormal basis serves the tests that use it.
        return q

    def uniform_int(self, lo, hi, count):
        out = np.zeros(count, dtype=np.int64)
        lib().ttor_rng_uniform_int(self.h, lo, hi, count, out.ctypes.data_as(C.POINTER(C.c_long)))
        return out

    def uniform_real(self, lo, hi, count):
        out = np.zeros(count)
        lib().ttor_rng_uniform_real(self.h, lo, hi, count, _dp(out))
        return out
