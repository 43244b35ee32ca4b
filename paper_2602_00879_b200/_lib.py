"""ctypes binding of the C ABI (include/desmoe.h) -> libdesmoe.so.

The library is built in-tree (``make -C paper_2602_00879_b200``, or
``__graft_entry__.build()``). There is deliberately no fallback: if the shared
object is missing or fails to load, every public entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdesmoe.so")

OK, EINVAL, ECUDA, ENCCL = 0, 1, 2, 3
SOFTMAX, SIGMOID, IDENTITY = 0, 1, 2
VANILLA, SEQ, VOTE = -1, 0, 1
VOTE_ACTIVATED, VOTE_RAW_LOGITS = 0, 1
FFN_SWIGLU, FFN_LINEAR = 0, 1
EP_HANDLE_BYTES = 128


class RouteCfg(C.Structure):
    _fields_ = [("experts", C.c_int), ("top_k", C.c_int), ("activation", C.c_int),
                ("strategy", C.c_int), ("seq_k", C.c_int), ("vote_beta", C.c_double),
                ("vote_source", C.c_int)]


class RouteOut(C.Structure):
    _fields_ = [("route_idx_dev", C.c_void_p), ("route_gate_dev", C.c_void_p),
                ("route_cnt_dev", C.c_void_p), ("coreset_dev", C.c_void_p),
                ("coreset_size_dev", C.c_void_p), ("votes_dev", C.c_void_p),
                ("probs_dev", C.c_void_p)]


class BaselineCfg(C.Structure):  # desmoe_baseline_cfg = BaselineParams (baselines.hpp:17-24)
    _fields_ = [("method", C.c_int), ("k_reduced", C.c_int), ("naee_beta", C.c_double),
                ("mcmoe_beta", C.c_double), ("mcmoe_important_fraction", C.c_double),
                ("mcmoe_score", C.c_int)]


BASE_TOPK_REDUCE, BASE_NAEE, BASE_MCMOE = 0, 1, 2
SCORE_MAX_GATE, SCORE_NEG_ENTROPY = 0, 1

class MoetHeader(C.Structure):  # desmoe_moet_header = TraceHeader (trace.hpp:29-39)
    _fields_ = [("experts", C.c_int), ("top_k", C.c_int), ("layers", C.c_int),
                ("block_size", C.c_int), ("steps", C.c_int), ("model", C.c_int),
                ("rho", C.c_double), ("temperature", C.c_double), ("seed", C.c_uint64)]


MOET_BINARY, MOET_JSONL = 0, 1

# name -> (restype, argtypes)
_P, _I, _D = C.c_void_p, C.c_int, C.c_double
_SIGS = {
    "desmoe_create": (_I, [C.POINTER(C.c_void_p), _I, _I, _I, _I, _I]),
    "desmoe_destroy": (None, [_P]),
    "desmoe_last_error": (C.c_char_p, []),
    "desmoe_check": (_I, [_P, _P]),
    "desmoe_version": (_I, []),
    "desmoe_validate_pool": (_I, [_I, _I, C.c_uint64, _I]),
    "desmoe_vote_budget": (_I, [_D, _I]),
    "desmoe_validate_params": (_I, [C.POINTER(RouteCfg)]),
    "desmoe_select_top": (_I, [_P, _P, _I, _I, _P, _I, _P, _P]),
    "desmoe_renormalize": (_I, [_P, _P, _P, _I, _P, _P]),
    "desmoe_moe_forward_f64": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "desmoe_activate": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "desmoe_route": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(RouteOut), _P]),
    "desmoe_route_f32": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(RouteOut), _P]),
    "desmoe_moet_decode": (_I, [_P, C.c_size_t, C.POINTER(MoetHeader), _P,
                                C.POINTER(C.c_int)]),
    "desmoe_moet_encode": (_I, [C.POINTER(MoetHeader), _P, _I, _P, C.POINTER(C.c_size_t),
                                C.POINTER(C.c_int)]),
    "desmoe_baseline_route": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(BaselineCfg),
                                   C.POINTER(RouteOut), _P]),
    "desmoe_baseline_route_f32": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(BaselineCfg),
                                       C.POINTER(RouteOut), _P]),
    "desmoe_coreset": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(RouteOut), _P]),
    "desmoe_constrained_route": (_I, [_P, _P, _I, C.POINTER(RouteCfg), C.POINTER(C.c_int), _I,
                                      C.POINTER(RouteOut), _P]),
    "desmoe_permute": (_I, [_P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "desmoe_experts_create": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, C.POINTER(C.c_void_p)]),
    "desmoe_experts_destroy": (None, [_P]),
    "desmoe_experts_create_ep": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P,
                                      C.POINTER(C.c_void_p)]),
    "desmoe_ep_local_buffers": (_I, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "desmoe_ep_connect": (_I, [_P, _I, _I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "desmoe_ep_export": (_I, [_P, _P]),
    "desmoe_ep_import": (_I, [_P, _I, _I, _P]),
    "desmoe_expert_ffn": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _P, _P]),
    "desmoe_router_logits": (_I, [_P, _P, _P, _I, _I, _I, _P, _P]),
    "desmoe_layer_forward": (_I, [_P, _P, _P, _P, _I, C.POINTER(RouteCfg), _P, _P, _P]),
    "desmoe_layer_forward_host": (_I, [_P, _P, _P, _P, _I, C.POINTER(RouteCfg), _P, _P, _P]),
    "desmoe_layer_logits": (_I, [_P, _P, _I, _I, _P]),
    "desmoe_layer_route": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P]),
    "desmoe_stack_forward": (_I, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _I, _P, _I,
                                  C.POINTER(RouteCfg), _P, _P, _I, _P]),
    "desmoe_set_profiling": (_I, [_P, _I]),
    "desmoe_set_graphs": (_I, [_P, _I]),
    "desmoe_get_phase_ms": (_I, [_P, C.POINTER(C.c_float), _I]),
    "desmoe_last_launch_count": (_I, [_P]),
    "desmoe_set_trace": (_I, [_P, _P, _I]),
}

_lib = None
_lock = threading.Lock()


class DesmoeError(RuntimeError):
    pass


def lib():
    """Loads libdesmoe.so once; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DesmoeError(
                    f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                    "(or __graft_entry__.build()); there is no CPU fallback")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc: int):
    """Maps a C-ABI status to the reference's exception types."""
    if rc == OK:
        return
    msg = lib().desmoe_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise DesmoeError(msg)
