"""ctypes binding of include/pfb200.h (the C ABI of libpfb200.so).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the shared object is missing, importing the package fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpfb200.so")

PF_EXPONENTIAL, PF_GAUSSIAN, PF_BREIT_WIGNER, PF_POLYNOMIAL = 0, 1, 2, 3
PF_PRODUCT, PF_SUM, PF_COMPOSITE, PF_MAPPED, PF_CONVOLUTION, PF_ARGUS = 4, 5, 6, 7, 8, 9
PF_DALITZ = 10
PF_TDDP = 11
PF_NLL, PF_CHISQ = 0, 1
PF_FX_DIGITS = 6
PF_OBSERVABLE, PF_PARAMETER = 0, 1


class pf_variable(C.Structure):
    _fields_ = [("name", C.c_char_p), ("value", C.c_double), ("lower", C.c_double),
                ("upper", C.c_double), ("step", C.c_double), ("fixed", C.c_int32),
                ("role", C.c_int32)]


class pf_node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("name", C.c_char_p),
                ("n_children", C.c_int32), ("children", C.POINTER(C.c_int32)),
                ("n_params", C.c_int32), ("params", C.POINTER(C.c_int32)),
                ("n_obs", C.c_int32), ("obs", C.POINTER(C.c_int32)),
                ("n_reals", C.c_int32), ("reals", C.POINTER(C.c_double)),
                ("quadrature_points", C.c_int64)]


class pf_graph(C.Structure):
    _fields_ = [("n_variables", C.c_int32), ("variables", C.POINTER(pf_variable)),
                ("n_nodes", C.c_int32), ("nodes", C.POINTER(pf_node)), ("root", C.c_int32)]


class pf_data(C.Structure):
    _fields_ = [("binned", C.c_int32), ("n_obs", C.c_int32), ("obs", C.POINTER(C.c_int32)),
                ("n_events", C.c_uint64), ("values", C.POINTER(C.c_double)),
                ("total_content", C.c_double)]


class pf_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_devices", C.c_int32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("verbose", C.c_int32), ("oversubscribe", C.c_int32),
                ("reserved", C.c_int32 * 2)]


class pf_status(C.Structure):
    _fields_ = [("code", C.c_int32), ("message", C.c_char * 512)]


class pf_eval_info(C.Structure):
    _fields_ = [("log_floor_delta", C.c_uint64), ("penalty", C.c_int32),
                ("norms_recomputed", C.c_int32)]


class pf_fit_config(C.Structure):
    _fields_ = [("minimizer", C.c_int32), ("batch_probes", C.c_int32),
                ("max_iterations", C.c_uint64), ("gradient_tolerance", C.c_double),
                ("simplex_tolerance", C.c_double)]


class pf_fit_result(C.Structure):
    _fields_ = [("status", C.c_int32), ("uncertainties_available", C.c_int32),
                ("metric_value", C.c_double), ("n_metric_calls", C.c_uint64),
                ("wall_time_s", C.c_double), ("grad_max_norm", C.c_double),
                ("params", C.POINTER(C.c_double)), ("uncertainties", C.POINTER(C.c_double))]


class pf_bench_result(C.Structure):
    _fields_ = [("step_ms_mean", C.c_double), ("step_ms_min", C.c_double),
                ("event_kernel_ms_mean", C.c_double), ("event_kernel_ms_min", C.c_double),
                ("metric", C.c_double), ("kernels_per_step", C.c_uint64),
                ("h2d_bytes_per_step", C.c_uint64), ("d2h_bytes_per_step", C.c_uint64)]


# every symbol include/pfb200.h declares, with its signature
_SIGNATURES = {
    "pf_graph_finalize": (C.c_int, [C.POINTER(pf_graph), C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                    C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_uint32), C.c_int32, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.POINTER(pf_status)]),
    "pf_graph_codegen": (C.c_int, [C.POINTER(pf_graph), C.POINTER(pf_data), C.c_uint32, C.c_char_p,
                                   C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(pf_status)]),
    "pf_graph_compile_check": (C.c_int, [C.POINTER(pf_graph), C.POINTER(pf_data), C.c_uint32,
                                         C.POINTER(C.c_size_t), C.POINTER(pf_status)]),
    "pf_model_create": (C.c_int, [C.POINTER(pf_graph), C.POINTER(pf_data), C.c_uint32,
                                  C.POINTER(pf_options), C.POINTER(C.c_void_p), C.POINTER(pf_status)]),
    "pf_model_destroy": (None, [C.c_void_p]),
    "pf_model_n_events": (C.c_uint64, [C.c_void_p]),
    "pf_model_n_params": (C.c_int32, [C.c_void_p]),
    "pf_model_param_variable": (C.c_int32, [C.c_void_p, C.c_int32]),
    "pf_model_n_nodes": (C.c_int32, [C.c_void_p]),
    "pf_model_binned": (C.c_int32, [C.c_void_p]),
    "pf_eval_metric": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int32,
                                 C.POINTER(C.c_double), C.POINTER(pf_eval_info), C.POINTER(pf_status)]),
    "pf_eval_metric_batch": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_size_t,
                                       C.c_int32, C.POINTER(C.c_double), C.POINTER(pf_status)]),
    "pf_eval_partial": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int32,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(pf_status)]),
    "pf_combine_partials": (C.c_double, [C.POINTER(C.c_int64), C.c_int32]),
    "pf_node_norms": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int32), C.c_int32]),
    "pf_log_floor_count": (C.c_uint64, [C.c_void_p]),
    "pf_clamp_count": (C.c_uint64, [C.c_void_p, C.c_int32]),
    "pf_fit": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(pf_fit_config), C.POINTER(C.c_double),
                         C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_double),
                         C.POINTER(C.c_double), C.POINTER(pf_fit_result), C.POINTER(pf_status)]),
    "pf_bench": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_int32, C.c_int32,
                           C.c_int32, C.POINTER(pf_bench_result), C.POINTER(pf_status)]),
    "pf_shard_events": (None, [C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]),
    "pf_model_chunk": (C.c_uint64, [C.c_void_p]),
    "pf_model_fused": (C.c_int32, [C.c_void_p]),
    "pf_abi_version": (C.c_int32, []),
    "pf_device_count": (C.c_int32, []),
    "pf_kernel_launches": (C.c_uint64, []),
    "pf_debug_trace": (C.c_int64, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]),
    "pf_generate_events": (C.c_int, [C.POINTER(pf_graph), C.POINTER(C.c_int32), C.c_int32, C.c_uint64,
                                     C.c_uint64, C.c_uint32, C.POINTER(pf_options), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(pf_status)]),
    "pf_eval_launch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.POINTER(C.c_int32),
                                 C.POINTER(pf_status)]),
    "pf_model_stream": (C.c_uint64, [C.c_void_p]),
    "pf_model_partial_device": (C.c_uint64, [C.c_void_p]),
    "pf_group_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(pf_status)]),
    "pf_group_join": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(pf_status)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """libpfb200.so, dlopened on the first native call (not at import): the
    pure-Python model and data description types (pdf trees, data sets,
    GraphDesc) stay usable without mapping the product library, so the
    reference arm of bench.py and the oracle never load it.  A missing
    library still fails loudly, at the first call that needs it."""

    _lib = None

    def _get(self):
        if _LazyLib._lib is None:
            _LazyLib._lib = _load()
        return _LazyLib._lib

    def __getattr__(self, name):
        return getattr(self._get(), name)

    def __getitem__(self, name):
        return self._get()[name]


def loaded() -> bool:
    """True once libpfb200.so has been dlopened by this process"""
    return _LazyLib._lib is not None


lib = _LazyLib()
