"""ctypes binding of ``libparafrac_b200.so`` (include/parafrac_b200.h).

Loads the in-tree shared library built by ``__graft_entry__.build()``; if it
is missing the import fails loudly — there is no CPU fallback.  ``Context``
wraps one ``pf_ctx`` (device tables, buffers, stream) and translates C-ABI
error codes into the reference's exceptions (``errors.py:8-34``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from collections import OrderedDict

import numpy as np

from .errors import CoefficientError, DeviceError, DivergenceError, SolverFailure
from .l1 import gamma_2_minus, weights_for
from .spaces import ChebyshevOperator, SineOperator

LIB_NAME = "libparafrac_b200.so"
# PARAFRAC_B200_LIB selects another in-tree build of the same library (the
# -DPF_JITTER protocol-stress build of tests/test_protocol_jitter.py)
LIB_PATH = os.environ.get("PARAFRAC_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

PF_OK, PF_ERR_ARGUMENT, PF_ERR_SOLVER, PF_ERR_COEFFICIENT = 0, 1, 2, 3
PF_ERR_DIVERGENCE, PF_ERR_CUDA, PF_ERR_UNSUPPORTED = 4, 5, 6

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class pf_problem(C.Structure):
    _fields_ = [("functor", C.c_int), ("p", C.c_double * 6), ("alpha", C.c_double),
                ("t_final", C.c_double), ("a", C.c_double), ("b", C.c_double)]


class pf_grid(C.Structure):
    _fields_ = [("nt", C.c_int), ("m", C.c_int)]


class pf_space(C.Structure):
    _fields_ = [("kind", C.c_int), ("modes", C.c_int), ("nodes", _dp), ("d1", _dp),
                ("quad_weights", _dp), ("pcg_tol", C.c_double), ("pcg_maxit", C.c_int)]


class pf_weights(C.Structure):
    _fields_ = [("b_fine", _dp), ("len_fine", C.c_long), ("b_frac", _dp), ("len_frac", C.c_long),
                ("gamma_2_minus", C.c_double)]


class pf_error(C.Structure):
    _fields_ = [("code", C.c_int), ("step_n", C.c_int), ("step_r", C.c_int), ("node", C.c_int),
                ("iteration", C.c_int), ("interval", C.c_int), ("cuda_error", C.c_int),
                ("message", C.c_char * 256)]


class pf_stats(C.Structure):
    _fields_ = [("fine_launches", C.c_longlong), ("coarse_launches", C.c_longlong),
                ("pcg_iterations", C.c_longlong), ("solves", C.c_longlong),
                ("last_fine_ms", C.c_double), ("last_coarse_ms", C.c_double),
                ("helper_launches", C.c_longlong), ("kernel_launches", C.c_longlong)]


# name -> (restype, argtypes); every symbol include/parafrac_b200.h declares
SIGNATURES = {
    "pf_create": (C.c_int, [C.POINTER(pf_problem), C.POINTER(pf_grid), C.POINTER(pf_space),
                            C.POINTER(pf_weights), C.c_int, C.POINTER(C.c_void_p)]),
    "pf_destroy": (None, [C.c_void_p]),
    "pf_last_error": (C.c_int, [C.c_void_p, C.POINTER(pf_error)]),
    "pf_state_size": (C.c_int, [C.c_void_p]),
    "pf_get_stats": (C.c_int, [C.c_void_p, C.POINTER(pf_stats)]),
    "pf_reset_stats": (C.c_int, [C.c_void_p]),
    "pf_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pf_version": (C.c_char_p, []),
    "pf_debug_phases": (C.c_int, [C.POINTER(C.c_longlong), C.c_int]),
    "pf_debug_trace": (C.c_int, [C.POINTER(C.c_longlong)]),
    "pf_debug_looptop": (C.c_int, [C.POINTER(C.c_longlong), C.c_int]),
    "pf_debug_slice_times_ns": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]),
    "pf_coarse_step": (C.c_int, [C.c_void_p, _dp, C.c_int, C.c_int, _dp]),
    "pf_run_coarse": (C.c_int, [C.c_void_p, _dp, _dp]),
    "pf_fine_sweep": (C.c_int, [C.c_void_p, _dp, C.c_int, C.c_int, C.c_int, _dp]),
    "pf_fine_propagate": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int, _dp, _dp]),
    "pf_chain_fine": (C.c_int, [C.c_void_p, _dp, _dp]),
    "pf_fine_sequential": (C.c_int, [C.c_void_p, _dp, _dp]),
    "pf_parareal": (C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                              _dp, _dp, _ip, _ip]),
    "pf_dev_fine_sweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "pf_dev_fine_sweep_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "pf_dev_check": (C.c_int, [C.c_void_p]),
    "pf_dev_parareal_init": (C.c_int, [C.c_void_p, _dp]),
    "pf_dev_parareal_states": (C.c_void_p, [C.c_void_p]),
    "pf_dev_parareal_correct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp]),
    "pf_dev_parareal_read": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "pf_dev_parareal_frozen": (C.c_int, [C.c_void_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the solver has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def ptr(a):
    """float64 C-contiguous numpy array -> double* (None passes NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def f64(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and out.shape != shape:
        out = out.reshape(shape)
    return out


def raise_for(err, default_step=None):
    code = err.code
    msg = err.message.decode(errors="replace") or "parafrac_b200 failure"
    if code == PF_ERR_SOLVER:
        step = (err.step_n, err.step_r) if err.step_r >= 0 else err.step_n
        if default_step is not None and err.step_r < 0:
            step = default_step
        raise SolverFailure(step, msg)
    if code == PF_ERR_COEFFICIENT:
        raise CoefficientError(err.node, msg)
    if code == PF_ERR_DIVERGENCE:
        raise DivergenceError(err.iteration, err.interval, msg)
    if code in (PF_ERR_ARGUMENT, PF_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise DeviceError(f"{msg} (code {code}, cuda error {err.cuda_error})")


class Context:
    """One device context for (problem functor, operator, grids)."""

    def __init__(self, problem, op, grids, device=0):
        fid, params = problem.device_functor()
        alpha = float(problem.alpha)
        prob = pf_problem(fid, (C.c_double * 6)(*params), alpha, float(grids.t_final),
                          float(op.a), float(op.b))
        grid = pf_grid(int(grids.nt), int(grids.m))
        self._keep = []
        if isinstance(op, ChebyshevOperator):
            nodes = f64(op.nodes)
            d1 = f64(op.d1)
            qw = f64(op.quad_weights)
            self._keep += [nodes, d1, qw]
            space = pf_space(1, int(op.degree), ptr(nodes), ptr(d1), ptr(qw), 0.0, 0)
        elif isinstance(op, SineOperator):
            space = pf_space(2 if op.dims == 1 else 3, int(op.modes), None, None, None, float(op.pcg_tol),
                             int(op.pcg_maxit))
        else:
            raise ValueError(f"unsupported operator type {type(op).__name__}")
        wt = weights_for(alpha)
        nt, m = int(grids.nt), int(grids.m)
        b_fine = f64(wt.on_grid(1, max(nt * m + 1, max(m, nt) + 2)))
        b_frac = f64(wt.on_grid(m, max(nt - 1, 0) * m + m + 1))
        self._keep += [b_fine, b_frac]
        weights = pf_weights(ptr(b_fine), b_fine.size, ptr(b_frac), b_frac.size, gamma_2_minus(alpha))
        self.lock = threading.Lock()
        handle = C.c_void_p()
        rc = lib.pf_create(C.byref(prob), C.byref(grid), C.byref(space), C.byref(weights), int(device),
                           C.byref(handle))
        self.handle = handle
        self.size = op.interior_size
        self.nt, self.m = nt, m
        if rc != PF_OK:
            err = self.last_error()
            self.close()
            raise_for(err)

    def last_error(self):
        err = pf_error()
        if self.handle:
            lib.pf_last_error(self.handle, C.byref(err))
        return err

    def check(self, rc, default_step=None):
        if rc != PF_OK:
            raise_for(self.last_error(), default_step)

    def stats(self):
        s = pf_stats()
        lib.pf_get_stats(self.handle, C.byref(s))
        return {k: getattr(s, k) for k, _ in pf_stats._fields_}

    def close(self):
        lock = getattr(self, "lock", None)
        if lock is None:
            self._destroy()
            return
        with lock:  # never free device buffers under a call in flight
            self._destroy()

    def _destroy(self):
        if getattr(self, "handle", None):
            lib.pf_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_CACHE: "OrderedDict[tuple, Context]" = OrderedDict()
_CACHE_LOCK = threading.Lock()
_CACHE_MAX = 8


def _op_key(op):
    if isinstance(op, ChebyshevOperator):
        return ("cheb", op.degree, op.a, op.b, op.d1.tobytes(), op.nodes.tobytes())
    return ("sine", op.modes, op.dims, op.pcg_tol, op.pcg_maxit)


def context_for(problem, op, grids, device=0):
    """Cached context: device tables are built once per (functor, order, op, grids)."""
    fid, params = problem.device_functor()
    key = (fid, params, float(problem.alpha), _op_key(op), float(grids.t_final), int(grids.nt),
           int(grids.m), int(device))
    with _CACHE_LOCK:
        ctx = _CACHE.get(key)
        if ctx is not None:
            _CACHE.move_to_end(key)
            return ctx
    ctx = Context(problem, op, grids, device)
    with _CACHE_LOCK:
        _CACHE[key] = ctx
        # eviction only drops the cache's reference: a caller (or another
        # thread mid-call under ctx.lock) may still hold the context, which
        # is destroyed by Context.__del__ once the last reference goes
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    return ctx
