"""Oracle package — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package; the product (paper_1311_1753_b200) never does.

  Oracle     — oracle/pf_oracle.c, the C restatement of the reference path
  Reference  — oracle/_ref/libparfit_ref.so, the unmodified reference headers
               compiled from /root/reference (absent => Reference.available()
               is False)
Both consume the same pf_graph / pf_data description as the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(_HERE, "_build", "libpf_oracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libparfit_ref.so")

_oracle = None
_ref = None


def build():
    """make -C oracle (the C restatement always; _ref when /root/reference exists)"""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", _HERE], stdout=subprocess.DEVNULL)


def _olib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_LIB):
            build()
        L = C.CDLL(ORACLE_LIB)
        L.po_create.restype = C.c_void_p
        L.po_create.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_char_p]
        L.po_destroy.argtypes = [C.c_void_p]
        L.po_eval.restype = C.c_int
        L.po_eval.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int,
                              C.POINTER(C.c_double), C.c_char_p]
        L.po_eval_mt.restype = C.c_int
        L.po_eval_mt.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_int,
                                 C.POINTER(C.c_double), C.c_char_p]
        L.po_n_params.argtypes = [C.c_void_p]
        L.po_param_variable.argtypes = [C.c_void_p, C.c_int]
        L.po_n_nodes.argtypes = [C.c_void_p]
        L.po_floor_count.restype = C.c_uint64
        L.po_floor_count.argtypes = [C.c_void_p]
        L.po_clamp_count.restype = C.c_uint64
        L.po_clamp_count.argtypes = [C.c_void_p, C.c_int]
        L.po_norms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.c_int]
        L.po_reduce.restype = C.c_double
        L.po_reduce.argtypes = [C.POINTER(C.c_double), C.c_size_t]
        L.po_density.restype = C.c_int
        L.po_density.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.c_uint64, C.POINTER(C.c_double), C.c_char_p]
        _oracle = L
    return _oracle


def _rlib():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_LIB)
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_create.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32,
                                       C.c_char_p]
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_n_params.argtypes = [C.c_void_p]
        L.ref_param_variable.argtypes = [C.c_void_p, C.c_int32]
        L.ref_eval.restype = C.c_int
        L.ref_eval.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_int,
                               C.POINTER(C.c_double), C.c_char_p]
        L.ref_floor_count.restype = C.c_uint64
        L.ref_floor_count.argtypes = [C.c_void_p]
        L.ref_n_nodes.argtypes = [C.c_void_p]
        L.ref_norms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int32), C.c_int32]
        L.ref_clamp_count.restype = C.c_uint64
        L.ref_clamp_count.argtypes = [C.c_void_p, C.c_int32]
        L.ref_fit.restype = C.c_int
        L.ref_fit.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.c_char_p]
        L.ref_reduce.restype = C.c_double
        L.ref_reduce.argtypes = [C.POINTER(C.c_double), C.c_size_t]
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_uint64,
                                   C.c_uint64, C.c_uint32, C.POINTER(C.c_double), C.c_char_p]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    def __init__(self, msg):
        super().__init__(msg)
        self.code = msg.split(":", 1)[0]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _describe(pdf, data):
    """pf_graph / pf_data for a parfit-style pdf and data set (same marshalling
    as the product front-end, so all three consume identical bytes)"""
    from paper_1311_1753_b200 import parfit as pf, _abi
    desc = pf.GraphDesc(pdf, data.observables())
    values = np.ascontiguousarray(pf.to_event_table(data), dtype=np.float64)
    binned = isinstance(data, pf.BinnedDataSet)
    n = values.shape[1]
    obs = (C.c_int32 * max(len(data.observables()), 1))(
        *[desc.var_index(o) for o in data.observables()])
    total = data.total_content() if binned else 0.0
    cdata = _abi.pf_data(1 if binned else 0, len(data.observables()), obs, n, _dp(values), total)
    bins = (C.c_uint64 * max(len(data.observables()), 1))(*(data.bins() if binned else [0]))
    return desc, cdata, (values, obs, bins)


class Oracle:
    """The C restatement (pf_oracle.c) bound to a pdf and a data set."""

    def __init__(self, pdf, data, grid=1024):
        self.L = _olib()
        self.desc, self.cdata, self._keep = _describe(pdf, data)
        err = C.create_string_buffer(512)
        self.h = self.L.po_create(C.byref(self.desc.c_graph), C.byref(self.cdata), grid, err)
        if not self.h:
            raise OracleError(err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.po_destroy(self.h)
            self.h = None

    def param_names(self):
        return [self.desc.vars[self.L.po_param_variable(self.h, i)].name
                for i in range(self.L.po_n_params(self.h))]

    def eval(self, params, metric=0, threads=1):
        """threads > 1: the event loop on that many POSIX threads (bit-identical)"""
        p = np.ascontiguousarray(params, dtype=np.float64)
        out = C.c_double()
        err = C.create_string_buffer(512)
        if self.L.po_eval_mt(self.h, _dp(p), p.size, metric, int(threads), C.byref(out), err):
            raise OracleError(err.value.decode())
        return out.value

    def norms(self):
        n = self.L.po_n_nodes(self.h)
        a, b, v = (C.c_double * n)(), (C.c_double * n)(), (C.c_int * n)()
        self.L.po_norms(self.h, a, b, v, n)
        return list(a), list(b), list(v)

    def floor_count(self):
        return int(self.L.po_floor_count(self.h))

    def clamp_count(self, node):
        return int(self.L.po_clamp_count(self.h, node))

    def density(self, params, points):
        p = np.ascontiguousarray(params, dtype=np.float64)
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, np.shape(points)[-1])
        out = np.empty(pts.shape[1])
        err = C.create_string_buffer(512)
        if self.L.po_density(self.h, _dp(p), _dp(pts), pts.shape[1], _dp(out), err):
            raise OracleError(err.value.decode())
        return out


def reduce(terms):
    t = np.ascontiguousarray(terms, dtype=np.float64)
    return _olib().po_reduce(_dp(t), t.size)


class Reference:
    """The reference's own BoundModel / fit (oracle/_ref/libparfit_ref.so)."""

    @staticmethod
    def available():
        return os.path.exists(REF_LIB)

    def __init__(self, pdf, data, grid=1024):
        self.L = _rlib()
        self.desc, self.cdata, self._keep = _describe(pdf, data)
        err = C.create_string_buffer(512)
        self.h = self.L.ref_model_create(C.byref(self.desc.c_graph), C.byref(self.cdata),
                                         self._keep[2], grid, err)
        if not self.h:
            raise OracleError(err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_model_destroy(self.h)
            self.h = None

    def param_names(self):
        return [self.desc.vars[self.L.ref_param_variable(self.h, i)].name
                for i in range(self.L.ref_n_params(self.h))]

    def eval(self, params, metric=0, threads=0):
        p = np.ascontiguousarray(params, dtype=np.float64)
        out = C.c_double()
        err = C.create_string_buffer(512)
        if self.L.ref_eval(self.h, _dp(p), p.size, metric, threads, C.byref(out), err):
            raise OracleError(err.value.decode())
        return out.value

    def norms(self):
        n = self.L.ref_n_nodes(self.h)
        a, b, v = (C.c_double * n)(), (C.c_double * n)(), (C.c_int32 * n)()
        self.L.ref_norms(self.h, a, b, v, n)
        return list(a), list(b), list(v)

    def floor_count(self):
        return int(self.L.ref_floor_count(self.h))

    def clamp_count(self, node):
        return int(self.L.ref_clamp_count(self.h, node))

    def fit(self, metric=0, threads=0, minimizer=0):
        n = self.L.ref_n_params(self.h)
        p, u = np.zeros(n), np.zeros(n)
        mv, gm, wall = C.c_double(), C.c_double(), C.c_double()
        calls = C.c_uint64()
        st, ua = C.c_int32(), C.c_int32()
        err = C.create_string_buffer(512)
        if self.L.ref_fit(self.h, metric, threads, minimizer, _dp(p), _dp(u), C.byref(mv),
                          C.byref(calls), C.byref(st), C.byref(ua), C.byref(gm), C.byref(wall), err):
            raise OracleError(err.value.decode())
        return dict(params=p, uncertainties=u, metric_value=mv.value, calls=calls.value,
                    status=st.value, uncertainties_available=bool(ua.value),
                    grad_max_norm=gm.value, wall_time_s=wall.value)


def ref_generate(pdf, observables, n, seed, grid=1024):
    """reference generate_events (generate.hpp:33-86) -> (n_obs, n) array"""
    from paper_1311_1753_b200 import parfit as pf
    L = _rlib()
    desc = pf.GraphDesc(pdf, observables)
    idx = (C.c_int32 * len(observables))(*[desc.var_index(o) for o in observables])
    out = np.empty((len(observables), n))
    err = C.create_string_buffer(512)
    if L.ref_generate(C.byref(desc.c_graph), idx, len(observables), n, seed, grid, _dp(out), err):
        raise OracleError(err.value.decode())
    return out


def mt64_uniform(seed, n):
    """n draws of (mt19937_64(seed)() >> 11) * 2^-53 — the reference tests'
    uniform01 / ToyRng::uniform bit recipe (generate.hpp:19-27)"""
    L = _olib()
    L.po_mt64_uniform.restype = None
    L.po_mt64_uniform.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
    out = np.empty(int(n))
    L.po_mt64_uniform(seed, int(n), _dp(out))
    return out
