"""ctypes binding of the C ABI in include/ttsw_capi.h (libttsw_cuda.so, sm_100a).

This is the Python mirror of the reference's `Rep` plugin surface
(/root/reference/proj/include/ttsw/swe.hpp:84-119) and its step-level callers
(`rhs<Rep>` swe.hpp:362-423, `ssprk3<Rep>` swe.hpp:428-454). There is no CPU
fallback: loading fails loudly when the CUDA library or a GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import traceback

# Independent work runs on several streams at once (concurrent crosses, ensemble members);
# more hardware work queues than the default 8 avoid false serialisation. Read by CUDA at
# context creation, so it is set before any CUDA use in this process.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libttsw_cuda.so")

OK, INPUT, SHAPE, STATE, DEGENERACY, CONVERGENCE, EVALUATION, CUDA, INTERNAL = 0, 1, 2, 3, 4, 5, 6, 7, 8
AXIS_X, AXIS_Y = 0, 1
UPWIND3, UPWIND5, WENO5 = 0, 1, 2
MINUS, PLUS = 0, 1
LINEAR, NONLINEAR = 0, 1
MAP_PERIODIC_PAD, MAP_STEP1, MAP_QPOINT, MAP_QSUM, MAP_DIFF, MAP_ROW_SLICE, MAP_QSLICE = range(7)
FN_IDENTITY, FN_PRODUCT, FN_SQRT, FN_AFFINE, FN_SQUARE = 0, 1, 2, 3, 4
FN_WENO5_S1_MINUS, FN_WENO5_S1_PLUS, FN_WENO5_S2_QUAD = 10, 11, 12
FN_LLF_LAMBDA, FN_WAVE_SPEED = 20, 21

# Every symbol include/ttsw_capi.h declares (checked by the CPU test suite).
EXPORTS = [
    "ttsw_ctx_create", "ttsw_ctx_destroy", "ttsw_last_error", "ttsw_ctx_sync", "ttsw_ctx_stream",
    "ttsw_ctx_launches", "ttsw_ctx_time_rounds", "ttsw_ctx_round_stats", "ttsw_ctx_set_sketch", "ttsw_ctx_sketch_stats", "ttsw_tt_from_host", "ttsw_tt_from_full", "ttsw_tt_to_host", "ttsw_tt_dims", "ttsw_tt_free",
    "ttsw_tt_constant", "ttsw_round", "ttsw_add", "ttsw_scale", "ttsw_axpy", "ttsw_hadamard", "ttsw_mul",
    "ttsw_core_map", "ttsw_core_map_csr", "ttsw_norm_fro", "ttsw_sum_entries", "ttsw_recip_taylor", "ttsw_cross", "ttsw_maxvol",
    "ttsw_periodic_ghost", "ttsw_ghosted", "ttsw_reconstruct_faces", "ttsw_solver_create", "ttsw_solver_destroy",
    "ttsw_solver_set_state", "ttsw_solver_get_state", "ttsw_solver_rhs", "ttsw_solver_step",
    "ttsw_solver_trace_len", "ttsw_solver_trace", "ttsw_solver_trace_clear", "ttsw_solver_set_tracing", "ttsw_solver_set_hooks", "ttsw_solver_set_time", "ttsw_solver_time",
    "ttsw_solver_set_eps_policy", "ttsw_solver_eps",
    "ttsw_solver_cross_trace_len", "ttsw_solver_cross_trace", "ttsw_solver_set_dt",
    "ttsw_dense_create", "ttsw_dense_destroy", "ttsw_dense_set_state", "ttsw_dense_get_state",
    "ttsw_dense_device_state", "ttsw_dense_set_dt", "ttsw_dense_set_time", "ttsw_dense_time", "ttsw_dense_set_hooks",
    "ttsw_dense_step", "ttsw_dense_rhs",
    "ttsw_ensemble_create", "ttsw_ensemble_destroy", "ttsw_ensemble_set_state_host", "ttsw_ensemble_step",
    "ttsw_ensemble_records", "ttsw_ensemble_last_error",
]


class TTSWError(Exception):
    def __init__(self, code, msg, residual=0.0, iterations=0, row=-1, col=-1):
        super().__init__(msg)
        self.code, self.residual, self.iterations, self.row, self.col = code, residual, iterations, row, col


class InputError(TTSWError): pass
class ShapeError(TTSWError): pass
class StateError(TTSWError): pass
class DegeneracyError(TTSWError): pass
class ConvergenceError(TTSWError): pass
class EvaluationError(TTSWError): pass
class CudaError(TTSWError): pass


_EXC = {INPUT: InputError, SHAPE: ShapeError, STATE: StateError, DEGENERACY: DegeneracyError,
        CONVERGENCE: ConvergenceError, EVALUATION: EvaluationError, CUDA: CudaError}


class ErrInfo(C.Structure):
    _fields_ = [("residual", C.c_double), ("iterations", C.c_int), ("row", C.c_long), ("col", C.c_long)]


class CrossCfg(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_rank", C.c_long), ("max_sweeps", C.c_int),
                ("rank_increment", C.c_long), ("validation_sample", C.c_int), ("seed", C.c_ulonglong)]

    @staticmethod
    def make(eps=1e-10, max_rank=128, max_sweeps=30, rank_increment=2, validation_sample=1000,
             seed=0x5EED5EED):
        return CrossCfg(eps, max_rank, max_sweeps, rank_increment, validation_sample, seed)


class CrossStats(C.Structure):
    _fields_ = [("evaluations", C.c_long), ("sweeps", C.c_int), ("residual", C.c_double)]


class RoundInfo(C.Structure):
    _fields_ = [("m", C.c_long), ("n", C.c_long), ("r_in", C.c_long), ("k_out", C.c_long), ("margin", C.c_double),
                ("kappa", C.c_double)]


class SolverDesc(C.Structure):
    _fields_ = [("model", C.c_int), ("scheme", C.c_int), ("n", C.c_long), ("g", C.c_double),
                ("f", C.c_double), ("H", C.c_double), ("dt", C.c_double), ("tol", C.c_double),
                ("lambda_eps_floor", C.c_double), ("cross", CrossCfg)]


_lib = None


# RhsHooks callbacks (include/ttsw_capi.h): borrowed q3 handles in, three owned handles out.
GHOST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.c_double, C.POINTER(C.c_void_p))
SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.POINTER(C.c_void_p))
# Dense-path callbacks: exact ghost strips of one component, the cell-average extra source.
DENSE_STRIP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double))
DENSE_SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.POINTER(C.c_double))


def load_library():
    """Load libttsw_cuda.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA library {LIB_PATH} is missing: run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, D = C.c_void_p, C.POINTER(C.c_double)
    L.ttsw_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.ttsw_ctx_destroy.argtypes = [P]
    L.ttsw_last_error.argtypes = [P, C.c_char_p, C.c_long, C.POINTER(ErrInfo)]
    L.ttsw_ctx_sync.argtypes = [P]
    L.ttsw_ctx_stream.restype = P
    L.ttsw_ctx_stream.argtypes = [P]
    L.ttsw_ctx_launches.restype = C.c_long
    L.ttsw_ctx_launches.argtypes = [P]
    L.ttsw_ctx_time_rounds.argtypes = [P, C.c_int]
    L.ttsw_ctx_round_stats.argtypes = [P, D, C.c_int]
    L.ttsw_ctx_set_sketch.argtypes = [P, C.c_int, C.c_int, C.c_int]
    L.ttsw_ctx_sketch_stats.argtypes = [P, C.POINTER(C.c_long), C.POINTER(C.c_long)]
    L.ttsw_tt_from_host.argtypes = [P, C.c_long, C.c_long, C.c_long, D, D, C.POINTER(C.c_void_p)]
    L.ttsw_tt_from_full.argtypes = [P, C.c_long, C.c_long, D, C.c_double, C.POINTER(C.c_void_p), C.POINTER(RoundInfo)]
    L.ttsw_tt_to_host.argtypes = [P, P, D, D]
    L.ttsw_tt_dims.argtypes = [P, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_long)]
    L.ttsw_tt_free.argtypes = [P]
    L.ttsw_tt_constant.argtypes = [P, C.c_long, C.c_long, C.c_double, C.POINTER(C.c_void_p)]
    L.ttsw_round.argtypes = [P, P, C.c_double, C.POINTER(C.c_void_p), C.POINTER(RoundInfo)]
    L.ttsw_add.argtypes = [P, P, P, C.POINTER(C.c_void_p)]
    L.ttsw_scale.argtypes = [P, P, C.c_double, C.POINTER(C.c_void_p)]
    L.ttsw_axpy.argtypes = [P, C.c_double, P, C.c_double, P, C.c_double, C.POINTER(C.c_void_p)]
    L.ttsw_hadamard.argtypes = [P, P, P, C.POINTER(C.c_void_p)]
    L.ttsw_mul.argtypes = [P, P, P, C.c_double, C.POINTER(C.c_void_p)]
    L.ttsw_core_map.argtypes = [P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, C.c_long,
                                C.POINTER(C.c_void_p)]
    L.ttsw_core_map_csr.argtypes = [P, P, C.c_int, C.c_long, C.c_long, C.POINTER(C.c_long), C.POINTER(C.c_long), D,
                                    C.POINTER(C.c_void_p)]
    L.ttsw_norm_fro.argtypes = [P, P, D]
    L.ttsw_sum_entries.argtypes = [P, P, D]
    L.ttsw_recip_taylor.argtypes = [P, P, C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]
    L.ttsw_cross.argtypes = [P, C.c_int, D, C.POINTER(C.c_void_p), C.c_int, P, C.POINTER(CrossCfg),
                             C.POINTER(C.c_void_p), C.POINTER(CrossStats)]
    L.ttsw_maxvol.argtypes = [P, C.c_long, C.c_long, D, C.POINTER(C.c_long)]
    L.ttsw_periodic_ghost.argtypes = [P, P, C.POINTER(C.c_void_p)]
    L.ttsw_ghosted.argtypes = [P, P, C.c_int, C.c_int, D, D, C.c_double, C.POINTER(C.c_void_p)]
    L.ttsw_reconstruct_faces.argtypes = [P, P, C.c_int, C.c_int, C.c_double, C.POINTER(CrossCfg), C.c_double,
                                         C.c_double, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    L.ttsw_solver_create.argtypes = [P, C.POINTER(SolverDesc), C.POINTER(C.c_void_p)]
    L.ttsw_solver_destroy.argtypes = [P]
    L.ttsw_solver_set_state.argtypes = [P, C.c_int, P]
    L.ttsw_solver_get_state.argtypes = [P, C.c_int, C.POINTER(C.c_void_p)]
    L.ttsw_solver_rhs.argtypes = [P, C.POINTER(C.c_void_p)]
    L.ttsw_solver_step.argtypes = [P, C.c_long]
    L.ttsw_solver_trace_len.restype = C.c_long
    L.ttsw_solver_trace_len.argtypes = [P]
    L.ttsw_solver_trace.argtypes = [P, C.POINTER(C.c_long), D, D]
    L.ttsw_solver_trace_clear.argtypes = [P]
    L.ttsw_solver_set_tracing.argtypes = [P, C.c_int]
    L.ttsw_solver_set_hooks.argtypes = [P, GHOST_FN, SOURCE_FN, P]
    L.ttsw_solver_set_time.argtypes = [P, C.c_double]
    L.ttsw_solver_time.restype = C.c_double
    L.ttsw_solver_time.argtypes = [P]
    L.ttsw_solver_set_eps_policy.argtypes = [P, C.c_double, C.c_int, C.c_double, C.c_double]
    L.ttsw_solver_eps.argtypes = [P, D]
    L.ttsw_solver_set_dt.argtypes = [P, C.c_double]
    L.ttsw_dense_create.argtypes = [P, C.POINTER(SolverDesc), C.POINTER(C.c_void_p)]
    L.ttsw_dense_destroy.argtypes = [P]
    L.ttsw_dense_set_state.argtypes = [P, C.c_int, D]
    L.ttsw_dense_get_state.argtypes = [P, C.c_int, D]
    L.ttsw_dense_device_state.restype = P
    L.ttsw_dense_device_state.argtypes = [P, C.c_int]
    L.ttsw_dense_set_dt.argtypes = [P, C.c_double]
    L.ttsw_dense_set_time.argtypes = [P, C.c_double]
    L.ttsw_dense_time.restype = C.c_double
    L.ttsw_dense_time.argtypes = [P]
    L.ttsw_dense_set_hooks.argtypes = [P, C.c_int, C.c_int, DENSE_STRIP_FN, DENSE_SOURCE_FN, P]
    L.ttsw_dense_step.argtypes = [P, C.c_long]
    L.ttsw_dense_rhs.argtypes = [P, D]
    L.ttsw_ensemble_create.argtypes = [C.c_int, C.c_int, C.POINTER(SolverDesc), C.c_int, C.POINTER(C.c_void_p)]
    L.ttsw_ensemble_destroy.argtypes = [P]
    L.ttsw_ensemble_set_state_host.argtypes = [P, C.c_int, C.c_int, C.c_long, C.c_long, C.c_long, D, D, C.c_double]
    L.ttsw_ensemble_step.argtypes = [P, C.c_long]
    L.ttsw_ensemble_records.argtypes = [P, D]
    L.ttsw_ensemble_last_error.argtypes = [P, C.c_char_p, C.c_long]
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Context:
    """One CUDA stream + memory pool on one device (ttsw_ctx)."""

    def __init__(self, device=0):
        L = load_library()
        h = C.c_void_p()
        code = L.ttsw_ctx_create(device, C.byref(h))
        self.h = h
        if code != OK:
            self._raise(code)

    def close(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ttsw_ctx_destroy(self.h)
        self.h = C.c_void_p() if C is not None else None  # ctypes may be gone at interpreter shutdown

    def __del__(self):
        self.close()

    def _raise(self, code):
        buf = C.create_string_buffer(4096)
        info = ErrInfo()
        _lib.ttsw_last_error(self.h, buf, 4096, C.byref(info))
        raise _EXC.get(code, TTSWError)(code, buf.value.decode(), info.residual, info.iterations, info.row, info.col)

    def check(self, code):
        if code != OK:
            self._raise(code)

    def sync(self):
        self.check(_lib.ttsw_ctx_sync(self.h))

    @property
    def stream(self):
        return _lib.ttsw_ctx_stream(self.h)

    @property
    def launches(self):
        return _lib.ttsw_ctx_launches(self.h)

    def time_rounds(self, on=True):
        _lib.ttsw_ctx_time_rounds(self.h, 1 if on else 0)

    def set_sketch(self, on=True, min_rank=0, default_columns=0):
        """Sketched pre-compression of large-rank roundings (ttsw_ctx_set_sketch)."""
        _lib.ttsw_ctx_set_sketch(self.h, 1 if on else 0, int(min_rank), int(default_columns))

    def sketch_stats(self):
        u, f = C.c_long(), C.c_long()
        _lib.ttsw_ctx_sketch_stats(self.h, C.byref(u), C.byref(f))
        return {"used": u.value, "fallback": f.value}

    def round_stats(self, reset=False):
        """{ms, flops, bytes, count} of the roundings timed since the last reset."""
        s = np.zeros(4)
        _lib.ttsw_ctx_round_stats(self.h, _dp(s), 1 if reset else 0)
        return {"ms": s[0], "flops": s[1], "bytes": s[2], "count": int(s[3])}

    # --- fields ---------------------------------------------------------------------
    def tt(self, cx, cy):
        cx = np.asfortranarray(cx, dtype=np.float64)
        cy = np.asfortranarray(cy, dtype=np.float64)
        if cx.ndim != 2 or cy.ndim != 2 or cx.shape[1] != cy.shape[0]:
            raise ShapeError(SHAPE, "TTMatrix: core inner dimensions do not match")
        o = C.c_void_p()
        self.check(_lib.ttsw_tt_from_host(self.h, cx.shape[0], cy.shape[1], cx.shape[1], _dp(cx), _dp(cy),
                                          C.byref(o)))
        return TT(self, o)

    def from_full(self, a, eps, with_info=False):
        """tt_from_full (tt.hpp:82-97) on the device."""
        a = np.asfortranarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ShapeError(SHAPE, "tt_from_full: expected a matrix")
        o = C.c_void_p()
        info = RoundInfo()
        self.check(_lib.ttsw_tt_from_full(self.h, a.shape[0], a.shape[1], _dp(a), float(eps), C.byref(o),
                                          C.byref(info)))
        return (TT(self, o), info) if with_info else TT(self, o)

    def constant(self, m, n, v):
        o = C.c_void_p()
        self.check(_lib.ttsw_tt_constant(self.h, m, n, float(v), C.byref(o)))
        return TT(self, o)

    def zero(self, m, n):
        return self.tt(np.zeros((m, 1)), np.zeros((1, n)))

    def _op(self, fn, *args):
        o = C.c_void_p()
        self.check(fn(self.h, *args, C.byref(o)))
        return TT(self, o)

    def round(self, x, eps, with_info=False):
        o, info = C.c_void_p(), RoundInfo()
        self.check(_lib.ttsw_round(self.h, x.h, float(eps), C.byref(o), C.byref(info)))
        t = TT(self, o)
        return (t, info) if with_info else t

    def add(self, x, y):
        return self._op(_lib.ttsw_add, x.h, y.h)

    def scale(self, x, a):
        return self._op(_lib.ttsw_scale, x.h, C.c_double(a))

    def axpy(self, a, x, b, y, eps):
        return self._op(_lib.ttsw_axpy, C.c_double(a), x.h, C.c_double(b), y.h, C.c_double(eps))

    def hadamard(self, x, y):
        return self._op(_lib.ttsw_hadamard, x.h, y.h)

    def mul(self, x, y, eps):
        return self._op(_lib.ttsw_mul, x.h, y.h, C.c_double(eps))

    def core_map(self, x, axis, op, scheme=0, side=0, n=0, a0=0, a1=0):
        return self._op(_lib.ttsw_core_map, x.h, axis, op, scheme, side, n, a0, a1)

    def core_map_dense(self, x, axis, m):
        """apply_core_map with an arbitrary operator matrix (passed by its nonzeros, CSR)."""
        m = np.asarray(m, dtype=np.float64)
        rows, cols = m.shape
        nz = [np.nonzero(m[i])[0] for i in range(rows)]
        rowptr = np.zeros(rows + 1, dtype=np.int64)
        rowptr[1:] = np.cumsum([len(z) for z in nz])
        colidx = np.concatenate(nz).astype(np.int64) if rowptr[-1] else np.zeros(1, dtype=np.int64)
        vals = np.ascontiguousarray(np.concatenate([m[i, z] for i, z in enumerate(nz)])) if rowptr[-1] \
            else np.zeros(1)
        lp = C.POINTER(C.c_long)
        return self._op(_lib.ttsw_core_map_csr, x.h, axis, rows, cols, rowptr.ctypes.data_as(lp),
                        colidx.ctypes.data_as(lp), _dp(vals))

    def norm_fro(self, x):
        v = C.c_double()
        self.check(_lib.ttsw_norm_fro(self.h, x.h, C.byref(v)))
        return v.value

    def sum_entries(self, x):
        v = C.c_double()
        self.check(_lib.ttsw_sum_entries(self.h, x.h, C.byref(v)))
        return v.value

    def recip(self, x, eps, max_iterations=200):
        o, it = C.c_void_p(), C.c_int()
        try:
            self.check(_lib.ttsw_recip_taylor(self.h, x.h, float(eps), max_iterations, C.byref(it), C.byref(o)))
        except TTSWError as e:
            e.recip_iterations = it.value
            raise
        return TT(self, o), it.value

    def cross(self, fn, ops, guess, cfg=None, param=0.0):
        arr = (C.c_void_p * len(ops))(*[o.h.value for o in ops])
        p = (C.c_double * 1)(param)
        o, st = C.c_void_p(), CrossStats()
        cfg = cfg or CrossCfg.make()
        self.check(_lib.ttsw_cross(self.h, fn, p, arr, len(ops), guess.h, C.byref(cfg), C.byref(o), C.byref(st)))
        return TT(self, o), st

    def maxvol(self, m):
        m = np.asfortranarray(m, dtype=np.float64)
        rows = (C.c_long * m.shape[1])()
        self.check(_lib.ttsw_maxvol(self.h, m.shape[0], m.shape[1], _dp(m), rows))
        return list(rows)

    def periodic_ghost(self, x):
        return self._op(_lib.ttsw_periodic_ghost, x.h)

    def ghosted(self, x, bc_x, bc_y, strip_x=None, strip_y=None, eps_tt=-1.0):
        """tt_ghosted (cases.cpp:298-344); bc 0 = Periodic, 1 = DirichletExact with the given
        exact ghost strips (6 x (ny+6) for x, (nx+6) x 6 for y)."""
        if bc_x not in (0, 1) or bc_y not in (0, 1):
            raise InputError(INPUT, "tt_ghosted: unknown boundary kind")
        nx, ny, _ = x.shape
        sx = sy = None
        if bc_x:
            sx = np.asfortranarray(strip_x, dtype=np.float64)
            if sx.shape != (6, ny + 6):
                raise ShapeError(SHAPE, "tt_ghosted: x strip must be 6 x (ny+6)")
        if bc_y:
            sy = np.asfortranarray(strip_y, dtype=np.float64)
            if sy.shape != (nx + 6, 6):
                raise ShapeError(SHAPE, "tt_ghosted: y strip must be (nx+6) x 6")
        return self._op(_lib.ttsw_ghosted, x.h, int(bc_x), int(bc_y), _dp(sx) if sx is not None else None,
                        _dp(sy) if sy is not None else None, float(eps_tt))

    def reconstruct_faces(self, g, axis, scheme, eps_tt=1e-12, cfg=None, dx=1.0, dy=1.0):
        mi, pl = C.c_void_p(), C.c_void_p()
        cfg = cfg or CrossCfg.make()
        self.check(_lib.ttsw_reconstruct_faces(self.h, g.h, axis, scheme, float(eps_tt), C.byref(cfg), dx, dy,
                                               C.byref(mi), C.byref(pl)))
        return TT(self, mi), TT(self, pl)


class TT:
    """Caller-owned device TT handle (ttsw_tt)."""

    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ttsw_tt_free(self.h)
            self.h = C.c_void_p()

    @property
    def shape(self):
        m, n, r = C.c_long(), C.c_long(), C.c_long()
        _lib.ttsw_tt_dims(self.h, C.byref(m), C.byref(n), C.byref(r))
        return m.value, n.value, r.value

    @property
    def rank(self):
        return self.shape[2]

    def cores(self):
        m, n, r = self.shape
        cx = np.zeros((m, r), order="F")
        cy = np.zeros((r, n), order="F")
        self.ctx.check(_lib.ttsw_tt_to_host(self.ctx.h, self.h, _dp(cx), _dp(cy)))
        return cx, cy

    def full(self):
        cx, cy = self.cores()
        return cx @ cy


class _BorrowedTT(TT):
    """A hook's view of a handle the library owns (never freed from Python)."""

    def __del__(self):
        self.h = None


def _release3(res, out):
    """Hand three TTs over to the library (it takes ownership of every non-NULL slot, also
    when the hook then fails); the same TT may fill several slots."""
    res = list(res)
    if len(res) != 3:
        raise ValueError("a hook must return three fields")
    given = {}
    for c, t in enumerate(res):
        if id(t) not in given:
            given[id(t)] = t.h.value
            t.h = None
        out[c] = given[id(t)]


class Solver:
    """Step-level driver: ssprk3<CudaTTRep> with a fixed EpsSchedule and periodic ghosts."""

    def __init__(self, ctx, model, scheme, n, g, f, H, dt, tol, cross_cfg=None, lambda_eps_floor=1e-6):
        self.ctx = ctx
        cfg = cross_cfg or CrossCfg.make(seed=1)
        self.desc = SolverDesc(model, scheme, n, g, f, H, dt, tol, lambda_eps_floor, cfg)
        h = C.c_void_p()
        ctx.check(_lib.ttsw_solver_create(ctx.h, C.byref(self.desc), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ttsw_solver_destroy(self.h)
            self.h = C.c_void_p()

    def set_state(self, tts):
        for c, t in enumerate(tts):
            self.ctx.check(_lib.ttsw_solver_set_state(self.h, c, t.h))

    def state(self):
        out = []
        for c in range(3):
            o = C.c_void_p()
            self.ctx.check(_lib.ttsw_solver_get_state(self.h, c, C.byref(o)))
            out.append(TT(self.ctx, o))
        return out

    def rhs(self):
        out = (C.c_void_p * 3)()
        self.ctx.check(_lib.ttsw_solver_rhs(self.h, out))
        return [TT(self.ctx, C.c_void_p(out[c])) for c in range(3)]

    def step(self, nsteps=1):
        self.ctx.check(_lib.ttsw_solver_step(self.h, nsteps))

    def set_tracing(self, on):
        _lib.ttsw_solver_set_tracing(self.h, 1 if on else 0)

    def set_dt(self, dt):
        self.ctx.check(_lib.ttsw_solver_set_dt(self.h, float(dt)))

    def set_hooks(self, fill_ghost=None, extra_source=None):
        """RhsHooks (swe.hpp:276-282): fill_ghost([q0, q1, q2], t) -> 3 ghosted TTs (e.g.
        Context.ghosted with exact strips), extra_source(t) -> 3 TTs. None = periodic / none."""
        ctx = self.ctx

        def borrow(h):
            t = _BorrowedTT.__new__(_BorrowedTT)
            t.ctx, t.h = ctx, C.c_void_p(h)
            return t

        def ghost(user, q3, t, out):
            qs = [borrow(q3[c]) for c in range(3)]
            try:
                _release3(fill_ghost(qs, t), out)
                return 0
            except Exception:
                traceback.print_exc()
                return 1
            finally:  # the q3 handles live on the library's stack: never freed here
                for q in qs:
                    q.h = None

        def source(user, t, out):
            try:
                _release3(extra_source(t), out)
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        self._hooks = (GHOST_FN(ghost) if fill_ghost else GHOST_FN(), SOURCE_FN(source) if extra_source else SOURCE_FN())
        self.ctx.check(_lib.ttsw_solver_set_hooks(self.h, self._hooks[0], self._hooks[1], None))

    @property
    def time(self):
        return _lib.ttsw_solver_time(self.h)

    @time.setter
    def time(self, t):
        self.ctx.check(_lib.ttsw_solver_set_time(self.h, float(t)))

    def set_eps_policy(self, c_eps, order=3, volume=1.0, clip=1e-3):
        """Policy-mode tolerances recomputed from the state before every step (swe.hpp:134-183)."""
        self.ctx.check(_lib.ttsw_solver_set_eps_policy(self.h, float(c_eps), int(order), float(volume), float(clip)))

    def eps(self):
        out = np.zeros(4)
        _lib.ttsw_solver_eps(self.h, _dp(out))
        return out

    def trace(self, clear=True):
        n = _lib.ttsw_solver_trace_len(self.h)
        ints = np.zeros(6 * n, dtype=np.int64)
        mg = np.zeros(n)
        ka = np.zeros(n)
        if n:
            _lib.ttsw_solver_trace(self.h, ints.ctypes.data_as(C.POINTER(C.c_long)), _dp(mg), _dp(ka))
        if clear:
            _lib.ttsw_solver_trace_clear(self.h)
        return ints.reshape(n, 6), mg, ka

    def cross_trace(self, clear=True):
        _lib.ttsw_solver_cross_trace_len.restype = C.c_long
        n = _lib.ttsw_solver_cross_trace_len(self.h)
        ints = np.zeros(3 * n, dtype=np.int64)
        res = np.zeros(n)
        _lib.ttsw_solver_cross_trace(self.h, ints.ctypes.data_as(C.POINTER(C.c_long)), _dp(res), 1 if clear else 0)
        return ints.reshape(n, 3), res


class DenseSolver:
    """Full-tensor DenseRep path on the device (swe.hpp:45-80 through rhs/ssprk3): three
    n x n cell-average fields resident in HBM."""

    def __init__(self, ctx, model, scheme, n, g, f, H, dt):
        self.ctx, self.n = ctx, n
        self.desc = SolverDesc(model, scheme, n, g, f, H, dt, 0.0, 1e-6, CrossCfg.make())
        h = C.c_void_p()
        ctx.check(_lib.ttsw_dense_create(ctx.h, C.byref(self.desc), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ttsw_dense_destroy(self.h)
            self.h = C.c_void_p()

    def set_state(self, fields):
        for c, a in enumerate(fields):
            a = np.asfortranarray(a, dtype=np.float64)
            if a.shape != (self.n, self.n):
                raise ValueError("dense state must be n x n")
            self.ctx.check(_lib.ttsw_dense_set_state(self.h, c, _dp(a)))

    def state(self):
        out = []
        for c in range(3):
            a = np.zeros((self.n, self.n), order="F")
            self.ctx.check(_lib.ttsw_dense_get_state(self.h, c, _dp(a)))
            out.append(a)
        return out

    def step(self, nsteps=1):
        self.ctx.check(_lib.ttsw_dense_step(self.h, nsteps))

    def rhs(self):
        out = np.zeros(3 * self.n * self.n)
        self.ctx.check(_lib.ttsw_dense_rhs(self.h, _dp(out)))
        return [out[c * self.n * self.n:(c + 1) * self.n * self.n].reshape(self.n, self.n, order="F")
                for c in range(3)]

    def set_dt(self, dt):
        self.ctx.check(_lib.ttsw_dense_set_dt(self.h, float(dt)))

    @property
    def time(self):
        return _lib.ttsw_dense_time(self.h)

    @time.setter
    def time(self, t):
        self.ctx.check(_lib.ttsw_dense_set_time(self.h, float(t)))

    def set_hooks(self, bc_x=0, bc_y=0, strips=None, source=None):
        """strips(t, c) -> (strip_x 6 x (n+6) or None, strip_y (n+6) x 6 or None);
        source(t) -> three n x n arrays. Exceptions become StateError at the step."""
        n = self.n

        def fs(user, t, c, sx, sy):
            try:
                a, b = strips(t, c)
                if a is not None:
                    np.ctypeslib.as_array(sx, shape=(6 * (n + 6),))[:] = np.asarray(a, dtype=float).ravel(order="F")
                if b is not None:
                    np.ctypeslib.as_array(sy, shape=(6 * (n + 6),))[:] = np.asarray(b, dtype=float).ravel(order="F")
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        def fsrc(user, t, out):
            try:
                res = source(t)
                o = np.ctypeslib.as_array(out, shape=(3 * n * n,))
                for c in range(3):
                    o[c * n * n:(c + 1) * n * n] = np.asarray(res[c], dtype=float).ravel(order="F")
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        self._hooks = (DENSE_STRIP_FN(fs) if strips else DENSE_STRIP_FN(),
                       DENSE_SOURCE_FN(fsrc) if source else DENSE_SOURCE_FN())
        self.ctx.check(_lib.ttsw_dense_set_hooks(self.h, int(bc_x), int(bc_y), self._hooks[0], self._hooks[1], None))


class Ensemble:
    """Native ensemble runtime (ttsw_ensemble_*): independent members on one device, stepped
    by library worker threads with one context (stream) each."""

    def __init__(self, device, descs, threads=16):
        load_library()
        arr = (SolverDesc * len(descs))(*descs)
        h = C.c_void_p()
        st = _lib.ttsw_ensemble_create(int(device), len(descs), arr, int(threads), C.byref(h))
        if st != OK:
            raise _EXC.get(st, TTSWError)(st, "ensemble creation failed")
        self.h, self.members = h, len(descs)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.ttsw_ensemble_destroy(self.h)
            self.h = C.c_void_p()

    def _check(self, st):
        if st != OK:
            buf = C.create_string_buffer(4096)
            _lib.ttsw_ensemble_last_error(self.h, buf, 4096)
            raise _EXC.get(st, TTSWError)(st, buf.value.decode())

    def set_state(self, member, c, cx, cy, round_eps=-1.0):
        cx = np.asfortranarray(cx, dtype=np.float64)
        cy = np.asfortranarray(cy, dtype=np.float64)
        m, r = cx.shape
        self._check(_lib.ttsw_ensemble_set_state_host(self.h, int(member), int(c), m, cy.shape[1], r, _dp(cx), _dp(cy),
                                                      float(round_eps)))

    def step(self, nsteps=1):
        self._check(_lib.ttsw_ensemble_step(self.h, int(nsteps)))

    def records(self):
        out = np.zeros(10 * self.members)
        self._check(_lib.ttsw_ensemble_records(self.h, _dp(out)))
        return out.reshape(self.members, 10)
