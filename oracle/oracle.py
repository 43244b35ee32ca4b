"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the two CPU checkers.

* ``Ref``   — the UNMODIFIED reference library (dessim) compiled from
  /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/, called
  through oracle/ref_shim.cpp.
* ``Port``  — the C restatement oracle/desmoe_oracle.c (liboracle.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
arm import this module; the product path (paper_2602_00879_b200) never does.
Both classes expose the same method names so tests can run one suite against
either. Errors raise ``ValueError`` (std::invalid_argument) with the reference's
message, or ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdessim_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


@dataclass
class Route:
    """Flattened RoutingAssignment: idx/gate [n x k] padded with -1 / 0."""

    idx: np.ndarray
    gate: np.ndarray
    cnt: np.ndarray

    def experts(self, t):
        return self.idx[t, : self.cnt[t]].tolist()

    def gates(self, t):
        return self.gate[t, : self.cnt[t]].tolist()


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class TraceDecodeError(Exception):
    """A MOET decode failure: TraceError::Code (trace.hpp:58-66) + message."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code
        self.message = message


class _Base:
    prefix = ""

    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._err().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


class Ref(_Base):
    """The reference library itself (oracle/_ref/libdessim_ref.so)."""

    prefix = "dsref_"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self._err = self._fn("last_error", [], C.c_char_p)

    def activate(self, logits, act=0, k=1):
        x = _f64(logits)
        n, m = x.shape
        p = np.empty_like(x)
        self._check(self._fn("activate", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, _f64p])(
            x, n, m, k, act, p))
        return p

    def _route_out(self, n, k):
        return (np.empty((n, k), np.int32), np.empty((n, k), np.float64), np.empty(n, np.int32))

    def topk_route(self, logits, k, act=0):
        x = _f64(logits)
        n, m = x.shape
        idx, gate, cnt = self._route_out(n, k)
        self._check(self._fn("topk_route", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                            _f64p, _i32p])(x, n, m, k, act, idx, gate, cnt))
        return Route(idx, gate, cnt)

    def baseline_route(self, logits, k, method, act=0, k_reduced=1, naee_beta=0.5,
                       mcmoe_beta=0.5, fraction=0.5, score=0):
        """baseline_route (baselines.cpp:125-137); method 0/1/2 = topk_reduce /
        naee / mcmoe, score 0/1 = max gate / -entropy."""
        x = _f64(logits)
        n, m = x.shape
        idx, gate, cnt = (np.empty((n, k), np.int32), np.empty((n, k), np.float64),
                          np.empty(n, np.int32))
        self._check(self._fn("baseline_route",
                             [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_double, C.c_double, C.c_double, C.c_int, _i32p, _f64p,
                              _i32p])(x, n, m, k, act, method, k_reduced, naee_beta,
                                      mcmoe_beta, fraction, score, idx, gate, cnt))
        return Route(idx, gate, cnt)

    def seq_coreset(self, logits, k, local_k, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        nm = C.c_int()
        self._check(self._fn("des_seq_coreset", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 C.c_int, _i32p, C.POINTER(C.c_int)])(
            x, n, m, k, act, local_k, mem, C.byref(nm)))
        return mem[: nm.value].copy()

    def vote_coreset(self, logits, k, beta, act=0, raw=False):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        votes = np.empty(m, np.float64)
        nm = C.c_int()
        self._check(self._fn("des_vote_coreset", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                  C.c_double, C.c_int, _i32p,
                                                  C.POINTER(C.c_int), _f64p])(
            x, n, m, k, act, beta, int(raw), mem, C.byref(nm), votes))
        return mem[: nm.value].copy(), votes

    def fused_vote(self, logits, k, beta, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        votes = np.empty(m, np.float64)
        nm = C.c_int()
        self._check(self._fn("fused_vote_pipeline", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                     C.c_double, _i32p, C.POINTER(C.c_int),
                                                     _f64p])(
            x, n, m, k, act, beta, mem, C.byref(nm), votes))
        return mem[: nm.value].copy(), votes

    def constrained_route(self, logits, k, members, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = _i32(members)
        idx, gate, cnt = self._route_out(n, k)
        self._check(self._fn("constrained_route", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                   _i32p, C.c_int, _i32p, _f64p, _i32p])(
            x, n, m, k, act, mem, len(mem), idx, gate, cnt))
        return Route(idx, gate, cnt)

    def des_run(self, logits, k, strategy, seq_k=1, beta=1.0, act=0):
        """strategy: 'seq' | 'vote' (des.hpp:16)."""
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        nm = C.c_int()
        idx, gate, cnt = self._route_out(n, k)
        self._check(self._fn("des_run", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_double, _i32p, C.POINTER(C.c_int),
                                         _i32p, _f64p, _i32p])(
            x, n, m, k, act, 0 if strategy == "seq" else 1, seq_k, beta, mem, C.byref(nm),
            idx, gate, cnt))
        return mem[: nm.value].copy(), Route(idx, gate, cnt)

    def vote_budget(self, beta, m):
        return self._fn("vote_budget", [C.c_double, C.c_int])(beta, m)

    def validate_config(self, m, k, act=0, bytes_per_expert=1, dim=1):
        self._check(self._fn("validate_config", [C.c_int, C.c_int, C.c_int, C.c_ulonglong,
                                                 C.c_int])(m, k, act, bytes_per_expert, dim))

    def make_expert_bank(self, m, dim, n, seed, k=1):
        w = np.empty((m, dim, dim), np.float64)
        x = np.empty((n, dim), np.float64)
        self._check(self._fn("make_expert_bank", [C.c_int, C.c_int, C.c_int, C.c_int,
                                                  C.c_ulonglong, _f64p, _f64p])(
            m, k, dim, n, seed, w, x))
        return w, x

    def moe_forward(self, route: Route, weights, inputs):
        w = _f64(weights)
        x = _f64(inputs)
        m, dim, _ = w.shape
        n, k = route.idx.shape
        out = np.empty((n, dim), np.float64)
        self._check(self._fn("moe_forward", [C.c_int, C.c_int, _i32p, _f64p, _i32p, C.c_int,
                                             C.c_int, _f64p, _f64p, _f64p])(
            n, k, _i32(route.idx), _f64(route.gate), _i32(route.cnt), m, dim, w, x, out))
        return out

    def moe_latency(self, route: Route, m):
        n, k = route.idx.shape
        per = np.empty(m, np.int32)
        u, tot = C.c_int(), C.c_int()
        self._check(self._fn("moe_latency", [C.c_int, C.c_int, _i32p, _i32p, C.c_int,
                                             C.POINTER(C.c_int), C.POINTER(C.c_int), _i32p])(
            n, k, _i32(route.idx), _i32(route.cnt), m, C.byref(u), C.byref(tot), per))
        return u.value, tot.value, per

    def expected_unique_experts(self, m, k, n):
        return self._fn("expected_unique_experts", [C.c_int, C.c_int, C.c_int], C.c_double)(
            m, k, n)

    def gen_trace(self, m, k, n, seed, rho=0.0, tau=1.0, model="shared_bias", layers=1,
                  steps=1):
        mid = {"iid_gaussian": 0, "dirichlet": 1, "shared_bias": 2}[model]
        out = np.empty((steps * layers, n, m), np.float64)
        self._check(self._fn("gen_trace", [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_int, C.c_int, C.c_int, C.c_ulonglong, _f64p])(
            m, k, mid, rho, tau, layers, steps, n, seed, out))
        return out

    def trace_bytes(self, m, k, n, seed, rho=0.0, tau=1.0, model="shared_bias", layers=1,
                    steps=1, fmt="binary"):
        """gen_trace + encode_trace: the reference's own MOET bytes."""
        mid = {"iid_gaussian": 0, "dirichlet": 1, "shared_bias": 2}[model]
        f = self._fn("trace_bytes", [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                     C.c_int, C.c_int, C.c_ulonglong, C.c_int, C.c_char_p,
                                     C.POINTER(C.c_size_t)])
        n_ = C.c_size_t(0)
        args = (m, k, mid, rho, tau, layers, steps, n, seed, 0 if fmt == "binary" else 1)
        self._check(f(*args, None, C.byref(n_)))
        buf = C.create_string_buffer(n_.value)
        self._check(f(*args, buf, C.byref(n_)))
        return buf.raw[: n_.value]

    def trace_decode(self, data: bytes):
        """decode_trace -> (header dict, logits [blocks, n, m]) or raises
        TraceDecodeError(code, message)."""
        hdr = (C.c_int * 6)()
        hd = (C.c_double * 2)()
        seed = C.c_ulonglong()
        code = C.c_int()
        f = self._fn("trace_decode", [C.c_char_p, C.c_size_t, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_double),
                                      C.POINTER(C.c_ulonglong), C.c_void_p])
        if f(data, len(data), C.byref(code), hdr, hd, C.byref(seed), None):
            raise TraceDecodeError(code.value, self._err().decode())
        m, k, layers, n, steps, model = list(hdr)
        x = np.empty((steps * layers, n, m), np.float64)
        f(data, len(data), C.byref(code), hdr, hd, C.byref(seed), x.ctypes.data)
        return dict(experts=m, top_k=k, layers=layers, block_size=n, steps=steps, model=model,
                    rho=hd[0], temperature=hd[1], seed=seed.value), x

    def rng_u64(self, seed, count):
        out = np.empty(count, np.uint64)
        self._fn("rng_u64", [C.c_ulonglong, C.c_int, _u64p], None)(seed, count, out)
        return out

    def rng_normal(self, seed, count):
        out = np.empty(count, np.float64)
        self._fn("rng_normal", [C.c_ulonglong, C.c_int, _f64p], None)(seed, count, out)
        return out

    def rng_mix(self, seed, stream):
        return self._fn("rng_mix", [C.c_ulonglong, C.c_ulonglong], C.c_ulonglong)(seed, stream)

    def time_routing(self, logits, k, strategy, seq_k=1, beta=1.0, reps=10, threads=1):
        """Blocks/s of the reference routing; strategy 'vanilla' | 'seq' | 'vote'."""
        x = _f64(logits)
        n, m = x.shape
        s = {"vanilla": -1, "seq": 0, "vote": 1}[strategy]
        return self._fn("time_routing", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_double, C.c_int, C.c_int], C.c_double)(
            x, n, m, k, s, seq_k, beta, reps, threads)


def _ref_time_layer(self, logits, k, strategy, seq_k=1, beta=1.0, dim=2048, reps=1, threads=1,
                    seed=7, ffn_tokens=0):
    """Estimated seconds per block of the reference layer (routing on the whole
    block + moe_forward with linear experts on `ffn_tokens` tokens, scaled);
    returns (seconds_per_block, unique_experts)."""
    x = _f64(logits)
    n, m = x.shape
    s = {"vanilla": -1, "seq": 0, "vote": 1}[strategy]
    u = C.c_int()
    f = self._fn("time_layer", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                C.c_int, C.c_int, C.c_int, C.c_ulonglong, C.c_int,
                                C.POINTER(C.c_int)], C.c_double)
    sec = f(x, n, m, k, s, seq_k, beta, dim, reps, threads, seed, ffn_tokens, C.byref(u))
    return sec, u.value


Ref.time_layer = _ref_time_layer


class Port(_Base):
    """The C restatement (oracle/liboracle.so)."""

    prefix = "or_"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self._err = self._fn("last_error", [], C.c_char_p)

    def activate(self, logits, act=0, k=1):
        x = _f64(logits)
        n, m = x.shape
        p = np.empty_like(x)
        self._check(self._fn("activate", [_f64p, C.c_int, C.c_int, C.c_int, _f64p])(
            x, n, m, act, p))
        return p

    def topk_route(self, logits, k, act=0):
        x = _f64(logits)
        n, m = x.shape
        idx, gate, cnt = (np.empty((n, k), np.int32), np.empty((n, k), np.float64),
                          np.empty(n, np.int32))
        self._check(self._fn("topk_route", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                            _f64p, _i32p])(x, n, m, k, act, idx, gate, cnt))
        return Route(idx, gate, cnt)

    def baseline_route(self, logits, k, method, act=0, k_reduced=1, naee_beta=0.5,
                       mcmoe_beta=0.5, fraction=0.5, score=0):
        """baseline_route (baselines.cpp:125-137); method 0/1/2 = topk_reduce /
        naee / mcmoe, score 0/1 = max gate / -entropy."""
        x = _f64(logits)
        n, m = x.shape
        idx, gate, cnt = (np.empty((n, k), np.int32), np.empty((n, k), np.float64),
                          np.empty(n, np.int32))
        self._check(self._fn("baseline_route",
                             [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_double, C.c_double, C.c_double, C.c_int, _i32p, _f64p,
                              _i32p])(x, n, m, k, act, method, k_reduced, naee_beta,
                                      mcmoe_beta, fraction, score, idx, gate, cnt))
        return Route(idx, gate, cnt)

    def seq_coreset(self, logits, k, local_k, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        nm = C.c_int()
        self._check(self._fn("seq_coreset", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             _i32p, C.POINTER(C.c_int)])(
            x, n, m, k, act, local_k, mem, C.byref(nm)))
        return mem[: nm.value].copy()

    def vote_coreset(self, logits, k, beta, act=0, raw=False):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        votes = np.empty(m, np.float64)
        nm = C.c_int()
        self._check(self._fn("vote_coreset", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_double, C.c_int, _i32p, C.POINTER(C.c_int),
                                              _f64p])(
            x, n, m, k, act, beta, int(raw), mem, C.byref(nm), votes))
        return mem[: nm.value].copy(), votes

    def constrained_route(self, logits, k, members, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = _i32(members)
        idx, gate, cnt = (np.empty((n, k), np.int32), np.empty((n, k), np.float64),
                          np.empty(n, np.int32))
        self._check(self._fn("constrained_route", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                   _i32p, C.c_int, _i32p, _f64p, _i32p])(
            x, n, m, k, act, mem, len(mem), idx, gate, cnt))
        return Route(idx, gate, cnt)

    def des_run(self, logits, k, strategy, seq_k=1, beta=1.0, act=0):
        x = _f64(logits)
        n, m = x.shape
        mem = np.empty(m, np.int32)
        nm = C.c_int()
        idx, gate, cnt = (np.empty((n, k), np.int32), np.empty((n, k), np.float64),
                          np.empty(n, np.int32))
        self._check(self._fn("des_run", [_f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_double, _i32p, C.POINTER(C.c_int), _i32p,
                                         _f64p, _i32p])(
            x, n, m, k, act, 0 if strategy == "seq" else 1, seq_k, beta, mem, C.byref(nm), idx,
            gate, cnt))
        return mem[: nm.value].copy(), Route(idx, gate, cnt)

    def vote_budget(self, beta, m):
        return self._fn("vote_budget", [C.c_double, C.c_int])(beta, m)

    def permute(self, route: Route, m):
        n, k = route.idx.shape
        count = np.empty(m, np.int32)
        offset = np.empty(m, np.int32)
        slot_of = np.empty((n, k), np.int32)
        slot_token = np.full(max(int(route.cnt.sum()), 1), -1, np.int32)
        active = np.empty(m, np.int32)
        na = C.c_int()
        self._check(self._fn("permute", [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i32p, _i32p,
                                         _i32p, _i32p, _i32p, C.POINTER(C.c_int)])(
            n, k, _i32(route.idx), _i32(route.cnt), m, count, offset, slot_of, slot_token,
            active, C.byref(na)))
        return dict(count=count, offset=offset, slot_of=slot_of,
                    slot_token=slot_token[: int(route.cnt.sum())], active=active[: na.value])

    def moe_ffn(self, route: Route, x, wg, wu=None, wd=None, mode="swiglu", threads=1):
        """x [n x d] f32 (bf16-valued); swiglu: wg/wu [m x f x d], wd [m x d x f];
        linear: wg = W [m x d x d]. Returns y [n x d] f32."""
        n, k = route.idx.shape
        x = np.ascontiguousarray(x, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        d = x.shape[1]
        m = wg.shape[0]
        if mode == "swiglu":
            f = wg.shape[1]
            wu = np.ascontiguousarray(wu, np.float32)
            wd = np.ascontiguousarray(wd, np.float32)
        else:
            f = d
            wu = wd = np.zeros(1, np.float32)
        y = np.empty((n, d), np.float32)
        self._check(self._fn("moe_ffn", [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _i32p, _f32p, _i32p, _f32p, _f32p, _f32p, _f32p, _f32p,
                                         C.c_int])(
            0 if mode == "swiglu" else 1, n, k, d, f, m, _i32(route.idx),
            np.ascontiguousarray(route.gate, np.float32), _i32(route.cnt), x, wg, wu, wd, y,
            threads))
        return y

    def router_logits(self, x, w):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        n, d = x.shape
        m = w.shape[0]
        out = np.empty((n, m), np.float64)
        self._fn("router_logits", [C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f64p], None)(
            n, m, d, x, w, out)
        return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 (finite inputs)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
