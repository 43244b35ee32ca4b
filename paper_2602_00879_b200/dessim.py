"""Python mirror of the reference's C++ operator API (namespace ``dessim``,
/root/reference/proj/core/include/dessim/{core,gating,des,analysis}.hpp),
backed by the sm_100a kernels through the C ABI (include/desmoe.h).

Same names, same argument meaning, same error behaviour (``ValueError`` where
the reference throws ``std::invalid_argument``, with the reference's
message), so the parity tests read like the reference's own tests. Inputs may
be lists, numpy arrays or torch tensors; they are staged to the current CUDA
device, routed by the GPU and copied back into the reference's value types.
There is no CPU path: without libdesmoe.so or a GPU every call raises.

Numerics: gating, votes and renormalisation are fp64 in the reference's order
(selections/coresets are the reference's; gates agree to ~1e-15, the last-bit
freedom of CUDA's fp64 exp). Expert FFNs run on tcgen05 tensor cores in bf16
with fp32 accumulation, so ``moe_forward`` agrees with the fp64 reference to
bf16 tolerance.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import RouteCfg, RouteOut, check, lib
from . import synth


class GateActivation(enum.IntEnum):  # core.hpp:11
    softmax = 0
    sigmoid = 1


class DesStrategy(enum.IntEnum):  # des.hpp:16
    seq = 0
    vote = 1


class VoteSource(enum.IntEnum):  # des.hpp:20
    activated = 0
    raw_logits = 1


@dataclass
class PoolConfig:  # core.hpp:13-19
    experts_total: int = 0
    top_k: int = 0
    gate_activation: GateActivation = GateActivation.softmax
    bytes_per_expert: int = 1
    hidden_dim: int = 1


def validate_config(cfg: PoolConfig) -> PoolConfig:  # core.cpp:11-28
    check(lib().desmoe_validate_pool(cfg.experts_total, cfg.top_k, cfg.bytes_per_expert,
                                     cfg.hidden_dim))
    return cfg


@dataclass
class RouterBlock:  # core.hpp:32-44
    block_size: int
    experts: int
    logits: np.ndarray  # [block_size x experts] fp64

    def at(self, token, expert):
        return float(self.logits[token, expert])

    def row(self, token):
        return self.logits[token]


def make_router_block(block_size: int, experts: int, logits) -> RouterBlock:  # core.cpp:63-79
    if block_size < 1:
        raise ValueError("block_size < 1")
    if experts < 1:
        raise ValueError("experts < 1")
    arr = np.asarray(_to_numpy(logits), dtype=np.float64).reshape(-1)
    if arr.size != block_size * experts:
        raise ValueError("logits size does not match block_size x experts")
    if not np.all(np.isfinite(arr)):
        raise ValueError("non-finite logit")
    return RouterBlock(block_size, experts, arr.reshape(block_size, experts).copy())


@dataclass
class GateMatrix:  # gating.hpp:11-23
    rows: int
    cols: int
    probs: np.ndarray

    def at(self, token, expert):
        return float(self.probs[token, expert])

    def row(self, token):
        return self.probs[token]


@dataclass
class Coreset:  # core.hpp:53-61
    members: List[int] = field(default_factory=list)

    def size(self):
        return len(self.members)

    def contains(self, expert):
        i = int(np.searchsorted(self.members, expert))
        return i < len(self.members) and self.members[i] == expert

    @staticmethod
    def of(indices) -> "Coreset":  # core.cpp:102-109
        v = sorted(set(int(i) for i in indices))
        if v and v[0] < 0:
            raise ValueError("negative expert index")
        return Coreset(v)


@dataclass
class TokenRoute:  # core.hpp:63-68
    experts: List[int] = field(default_factory=list)
    gates: List[float] = field(default_factory=list)


@dataclass
class RoutingAssignment:  # core.hpp:70-73
    tokens: List[TokenRoute] = field(default_factory=list)

    def block_size(self):
        return len(self.tokens)


@dataclass
class VoteVector:  # des.hpp:10-13
    votes: List[float] = field(default_factory=list)


@dataclass
class DesParams:  # des.hpp:20-24
    strategy: DesStrategy = DesStrategy.vote
    seq_k: int = 1
    vote_beta: float = 1.0


@dataclass
class VoteResult:  # des.hpp:35-38
    coreset: Coreset
    votes: VoteVector


@dataclass
class DesResult:  # des.hpp:52-55
    coreset: Coreset
    assignment: RoutingAssignment


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

def _to_numpy(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x)


class _Ctx:
    """One C-ABI context per (device, thread); grows on demand."""

    _local = threading.local()

    def __init__(self, device, n, m, k, d):
        import torch
        self.device = device
        self.caps = (n, m, k, d)
        h = C.c_void_p()
        with torch.cuda.device(device):
            check(lib().desmoe_create(C.byref(h), device, n, m, k, d))
        self.h = h

    def __del__(self):
        try:
            lib().desmoe_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def get(cls, n=1, m=1, k=1, d=128):
        import torch
        if not torch.cuda.is_available():
            raise _lib.DesmoeError("no CUDA device: the DES MoE path has no CPU fallback")
        dev = torch.cuda.current_device()
        cache = getattr(cls._local, "ctx", None)
        if cache is None:
            cache = cls._local.ctx = {}
        ctx = cache.get(dev)
        need = (max(n, 256), max(m, 256), max(k, 32), max(d, 4096))
        if ctx is None or any(a < b for a, b in zip(ctx.caps, (n, m, k, d))):
            if ctx is not None:
                need = tuple(max(a, b) for a, b in zip(ctx.caps, need))
            ctx = cache[dev] = _Ctx(dev, min(need[0], 1024), min(need[1], 1024), need[2],
                                    need[3])
        return ctx


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev_f64(x):
    import torch
    if isinstance(x, torch.Tensor):
        return x.detach().to(device="cuda", dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _cfg(cfg: PoolConfig, strategy=_lib.VANILLA, seq_k=1, beta=1.0, source=0, activation=None):
    return RouteCfg(cfg.experts_total, cfg.top_k,
                    int(cfg.gate_activation if activation is None else activation), strategy,
                    seq_k, float(beta), int(source))


def _finish(ctx):
    check(lib().desmoe_check(ctx.h, _stream()))


def _check_block(block: RouterBlock, cfg: PoolConfig):
    """validate_block (core.cpp:81-96); finiteness is also re-checked on device."""
    if block.experts != cfg.experts_total:
        raise ValueError("block column count does not match experts_total")
    if block.block_size < 1:
        raise ValueError("block_size < 1")
    if block.logits.size != block.block_size * block.experts:
        raise ValueError("logits size does not match block shape")


class _RouteBufs:
    def __init__(self, n, m, k):
        import torch
        d = "cuda"
        self.idx = torch.empty((n, k), dtype=torch.int32, device=d)
        self.gate = torch.empty((n, k), dtype=torch.float64, device=d)
        self.cnt = torch.empty((n,), dtype=torch.int32, device=d)
        self.core = torch.empty((m,), dtype=torch.int32, device=d)
        self.core_n = torch.empty((1,), dtype=torch.int32, device=d)
        self.votes = torch.empty((m,), dtype=torch.float64, device=d)
        self.probs = torch.empty((n, m), dtype=torch.float64, device=d)

    def out(self, probs=False):
        return RouteOut(self.idx.data_ptr(), self.gate.data_ptr(), self.cnt.data_ptr(),
                        self.core.data_ptr(), self.core_n.data_ptr(), self.votes.data_ptr(),
                        self.probs.data_ptr() if probs else None)

    def assignment(self) -> RoutingAssignment:
        idx = self.idx.cpu().numpy()
        gate = self.gate.cpu().numpy()
        cnt = self.cnt.cpu().numpy()
        return RoutingAssignment([TokenRoute(idx[t, : cnt[t]].tolist(), gate[t, : cnt[t]].tolist())
                                  for t in range(idx.shape[0])])

    def coreset(self) -> Coreset:
        n = int(self.core_n.item())
        return Coreset(self.core[:n].cpu().numpy().tolist())


# ---------------------------------------------------------------------------
# gating.hpp
# ---------------------------------------------------------------------------

def activate(block: RouterBlock, cfg: PoolConfig) -> GateMatrix:  # gating.cpp:10-40
    _check_block(block, cfg)
    import torch
    n, m = block.block_size, block.experts
    ctx = _Ctx.get(n, m)
    x = _dev_f64(block.logits)
    p = torch.empty((n, m), dtype=torch.float64, device="cuda")
    check(lib().desmoe_activate(ctx.h, _ptr(x), n, m, int(cfg.gate_activation), _ptr(p),
                                _stream()))
    _finish(ctx)
    return GateMatrix(n, m, p.cpu().numpy())


def _route_gates(probs: np.ndarray, top_k: int, members=None) -> RoutingAssignment:
    """Selection + renormalisation on gate values (IDENTITY activation)."""
    probs = np.atleast_2d(np.asarray(probs, np.float64))
    n, m = probs.shape
    ctx = _Ctx.get(n, m, top_k)
    bufs = _RouteBufs(n, m, top_k)
    x = _dev_f64(probs)
    pc = PoolConfig(m, top_k)
    if members is None:
        if top_k < 1 or top_k > m:
            raise ValueError("top_k out of range")
        cfg = _cfg(pc, _lib.VANILLA, activation=_lib.IDENTITY)
        check(lib().desmoe_route(ctx.h, _ptr(x), n, C.byref(cfg), C.byref(bufs.out()), _stream()))
    else:
        mem = (C.c_int * max(len(members), 1))(*members)
        cfg = _cfg(pc, _lib.VANILLA, activation=_lib.IDENTITY)
        check(lib().desmoe_constrained_route(ctx.h, _ptr(x), n, C.byref(cfg), mem, len(members),
                                             C.byref(bufs.out()), _stream()))
    _finish(ctx)
    return bufs.assignment()


def select_top_gates(gates: Sequence[float], k: int, candidates=None) -> List[int]:
    """gating.cpp:42-71: k largest by (value desc, index asc), ascending."""
    g = np.asarray(_to_numpy(gates), np.float64).reshape(1, -1)
    if candidates is None:
        if k > g.shape[1]:
            raise ValueError("selection count exceeds gate count")
        return _route_gates(g, k).tokens[0].experts
    cand = sorted(int(c) for c in candidates)
    if k > len(cand):
        raise ValueError("selection count exceeds candidate count")
    return _route_gates(g, k, cand).tokens[0].experts[:k] if k < len(cand) else cand


def renormalize_over(gates: Sequence[float], selected: Sequence[int]) -> List[float]:
    """gating.cpp:73-82 (sum over `selected` in ascending index)."""
    g = np.asarray(_to_numpy(gates), np.float64).reshape(1, -1)
    sel = sorted(int(s) for s in selected)
    return _route_gates(g, len(sel), sel).tokens[0].gates


def topk_route(gates: GateMatrix, top_k: int) -> RoutingAssignment:  # gating.cpp:84-97
    if top_k < 1 or top_k > gates.cols:
        raise ValueError("top_k out of range")
    return _route_gates(gates.probs, top_k)


def unique_experts(assign: RoutingAssignment) -> Coreset:  # gating.cpp:159-165
    import torch
    n = assign.block_size()
    k = max([len(t.experts) for t in assign.tokens] + [1])
    m = max([max(t.experts) for t in assign.tokens if t.experts] + [0]) + 1
    idx = np.full((n, k), -1, np.int32)
    cnt = np.zeros(n, np.int32)
    for i, t in enumerate(assign.tokens):
        idx[i, : len(t.experts)] = t.experts
        cnt[i] = len(t.experts)
    ctx = _Ctx.get(n, m, k)
    di = torch.as_tensor(idx, device="cuda")
    dc = torch.as_tensor(cnt, device="cuda")
    count = torch.empty(m, dtype=torch.int32, device="cuda")
    offset = torch.empty(m, dtype=torch.int32, device="cuda")
    active = torch.empty(m, dtype=torch.int32, device="cuda")
    na = torch.empty(1, dtype=torch.int32, device="cuda")
    check(lib().desmoe_permute(ctx.h, _ptr(di), _ptr(dc), n, k, m, _ptr(count), _ptr(offset),
                               None, None, _ptr(active), _ptr(na), _stream()))
    return Coreset(active[: int(na.item())].cpu().numpy().tolist())


# ---------------------------------------------------------------------------
# des.hpp
# ---------------------------------------------------------------------------

def vote_budget(beta: float, experts_total: int) -> int:  # des.cpp:29-31
    return lib().desmoe_vote_budget(float(beta), int(experts_total))


def validate_params(params: DesParams, cfg: PoolConfig):  # des.cpp:10-27
    validate_config(cfg)
    if params.strategy == DesStrategy.seq:
        if params.seq_k < 1:
            raise ValueError("seq_k < 1")
        if params.seq_k > cfg.top_k:
            raise ValueError("seq_k > top_k")
    else:
        if not (params.vote_beta > 0.0) or params.vote_beta > 1.0:
            raise ValueError("vote_beta outside (0, 1]")
        if vote_budget(params.vote_beta, cfg.experts_total) < 1:
            raise ValueError("vote budget floor(beta*M) < 1")


def _coreset(block, cfg, strategy, seq_k=1, beta=1.0, source=0):
    _check_block(block, cfg)
    n, m, k = block.block_size, block.experts, cfg.top_k
    ctx = _Ctx.get(n, m, k)
    bufs = _RouteBufs(n, m, max(k, 1))
    x = _dev_f64(block.logits)
    rc = _cfg(cfg, strategy, seq_k, beta, source)
    check(lib().desmoe_coreset(ctx.h, _ptr(x), n, C.byref(rc), C.byref(bufs.out()), _stream()))
    _finish(ctx)
    return bufs


def des_seq_coreset(block: RouterBlock, cfg: PoolConfig, local_k: int) -> Coreset:  # des.cpp:33
    return _coreset(block, cfg, _lib.SEQ, seq_k=local_k).coreset()


def des_vote_coreset(block: RouterBlock, cfg: PoolConfig, beta: float,
                     source: VoteSource = VoteSource.activated) -> VoteResult:  # des.cpp:65
    bufs = _coreset(block, cfg, _lib.VOTE, beta=beta, source=int(source))
    return VoteResult(bufs.coreset(), VoteVector(bufs.votes.cpu().numpy().tolist()))


def fused_vote_pipeline(block: RouterBlock, cfg: PoolConfig, beta: float) -> VoteResult:
    """des.cpp:166-224. On the GPU the composed and fused paths are the same
    kernels (one pass per token, fixed-order vote reduction), so the contract
    "same coreset, votes within 1e-9" holds with equality."""
    return des_vote_coreset(block, cfg, beta)


def constrained_route(block: RouterBlock, cfg: PoolConfig,
                      coreset: Coreset) -> RoutingAssignment:  # des.cpp:97-118
    _check_block(block, cfg)
    n, m, k = block.block_size, block.experts, cfg.top_k
    if not coreset.members:
        raise ValueError("empty coreset")
    if coreset.members[-1] >= cfg.experts_total:
        raise ValueError("coreset member out of range")
    ctx = _Ctx.get(n, m, k)
    bufs = _RouteBufs(n, m, k)
    x = _dev_f64(block.logits)
    rc = _cfg(cfg)
    mem = (C.c_int * len(coreset.members))(*coreset.members)
    check(lib().desmoe_constrained_route(ctx.h, _ptr(x), n, C.byref(rc), mem,
                                         len(coreset.members), C.byref(bufs.out()), _stream()))
    _finish(ctx)
    return bufs.assignment()


def des_run(block: RouterBlock, cfg: PoolConfig, params: DesParams) -> DesResult:  # des.cpp:120
    validate_params(params, cfg)
    _check_block(block, cfg)
    n, m, k = block.block_size, block.experts, cfg.top_k
    ctx = _Ctx.get(n, m, k)
    bufs = _RouteBufs(n, m, k)
    x = _dev_f64(block.logits)
    rc = _cfg(cfg, int(params.strategy), params.seq_k, params.vote_beta)
    check(lib().desmoe_route(ctx.h, _ptr(x), n, C.byref(rc), C.byref(bufs.out()), _stream()))
    _finish(ctx)
    return DesResult(bufs.coreset(), bufs.assignment())


# ---------------------------------------------------------------------------
# baselines.hpp: comparison expert-skipping policies (csrc/baselines.cu)
# ---------------------------------------------------------------------------

class BaselineMethod(enum.IntEnum):  # baselines.hpp:8
    topk_reduce = 0
    naee = 1
    mcmoe = 2


class ImportanceScore(enum.IntEnum):  # baselines.hpp:13
    max_gate = 0
    neg_entropy = 1


@dataclass
class BaselineParams:  # baselines.hpp:17-24
    method: BaselineMethod = BaselineMethod.topk_reduce
    k_reduced: int = 1
    naee_beta: float = 0.5
    mcmoe_beta: float = 0.5
    mcmoe_important_fraction: float = 0.5
    mcmoe_score: ImportanceScore = ImportanceScore.max_gate


def _baseline(block: RouterBlock, cfg: PoolConfig, b) -> RoutingAssignment:
    _check_block(block, cfg)
    n, m, k = block.block_size, block.experts, cfg.top_k
    ctx = _Ctx.get(n, m, k)
    bufs = _RouteBufs(n, m, k)
    x = _dev_f64(block.logits)
    rc = _cfg(cfg, _lib.VANILLA)
    check(lib().desmoe_baseline_route(ctx.h, _ptr(x), n, C.byref(rc), C.byref(b),
                                      C.byref(bufs.out()), _stream()))
    _finish(ctx)
    return bufs.assignment()


def topk_reduce_route(block: RouterBlock, cfg: PoolConfig, k_reduced: int) -> RoutingAssignment:
    """baselines.cpp:10-16: vanilla routing with K -> k_reduced."""
    if k_reduced < 1 or k_reduced > cfg.top_k:
        raise ValueError("k_reduced outside [1, top_k]")
    return _baseline(block, cfg, _lib.BaselineCfg(_lib.BASE_TOPK_REDUCE, k_reduced, 0.5, 0.5,
                                                  0.5, 0))


def naee_route(block: RouterBlock, cfg: PoolConfig, beta: float) -> RoutingAssignment:
    """baselines.cpp:64-76: drop the selected gates' cumulative tail below beta."""
    if not (beta > 0.0) or not (beta < 1.0):
        raise ValueError("naee beta outside (0, 1)")
    return _baseline(block, cfg, _lib.BaselineCfg(_lib.BASE_NAEE, 1, beta, 0.5, 0.5, 0))


def mcmoe_route(block: RouterBlock, cfg: PoolConfig, beta: float, important_fraction: float,
                score: ImportanceScore = ImportanceScore.max_gate) -> RoutingAssignment:
    """baselines.cpp:78-123: important tokens keep top-K, the rest get NAEE."""
    if not (beta > 0.0) or not (beta < 1.0):
        raise ValueError("mcmoe beta outside (0, 1)")
    if important_fraction < 0.0 or important_fraction > 1.0:
        raise ValueError("important_fraction outside [0, 1]")
    return _baseline(block, cfg, _lib.BaselineCfg(_lib.BASE_MCMOE, 1, 0.5, beta,
                                                  important_fraction, int(score)))


def baseline_route(block: RouterBlock, cfg: PoolConfig,
                   params: BaselineParams) -> RoutingAssignment:  # baselines.cpp:125-137
    if params.method == BaselineMethod.topk_reduce:
        return topk_reduce_route(block, cfg, params.k_reduced)
    if params.method == BaselineMethod.naee:
        return naee_route(block, cfg, params.naee_beta)
    if params.method == BaselineMethod.mcmoe:
        return mcmoe_route(block, cfg, params.mcmoe_beta, params.mcmoe_important_fraction,
                           params.mcmoe_score)
    raise ValueError("unknown baseline method")


# ---------------------------------------------------------------------------
# ExpertBank / moe_forward (gating.hpp:48-72) on the tcgen05 expert kernels
# ---------------------------------------------------------------------------

@dataclass
class ExpertBank:
    experts: int
    dim: int
    block_size: int
    expert_weights: np.ndarray  # [experts x dim x dim] fp64, [out][in]
    token_inputs: np.ndarray    # [block_size x dim] fp64

    def expert_matrix(self, expert):
        return self.expert_weights[expert]

    def token_input(self, token):
        return self.token_inputs[token]


def make_expert_bank(cfg: PoolConfig, block_size: int, seed: int) -> ExpertBank:
    validate_config(cfg)
    if block_size < 1:
        raise ValueError("block_size < 1")
    w, x = synth.make_expert_bank(cfg.experts_total, cfg.hidden_dim, block_size, seed)
    return ExpertBank(cfg.experts_total, cfg.hidden_dim, block_size, w, x)


def moe_forward(assign: RoutingAssignment, bank: ExpertBank) -> np.ndarray:
    """gating.cpp:136-157 on the GPU's linear-expert path: weights and inputs
    in bf16, fp32 accumulation and combine (ascending expert order). dim is
    zero-padded to a multiple of 128 for the tensor-core tiles."""
    import torch
    if assign.block_size() != bank.block_size:
        raise ValueError("assignment and bank block sizes differ")
    n, m, dim = bank.block_size, bank.experts, bank.dim
    for t in assign.tokens:
        for e in t.experts:
            if e < 0 or e >= m:
                raise ValueError("expert index out of range for bank")
    dp = max(128, -(-dim // 128) * 128)
    k = max([len(t.experts) for t in assign.tokens] + [1])
    w = torch.zeros((m, dp, dp), dtype=torch.bfloat16, device="cuda")
    w[:, :dim, :dim] = torch.as_tensor(bank.expert_weights, device="cuda").to(torch.bfloat16)
    x = torch.zeros((n, dp), dtype=torch.bfloat16, device="cuda")
    x[:, :dim] = torch.as_tensor(bank.token_inputs, device="cuda").to(torch.bfloat16)
    idx = np.full((n, k), -1, np.int32)
    gate = np.zeros((n, k), np.float64)
    cnt = np.zeros(n, np.int32)
    for i, t in enumerate(assign.tokens):
        idx[i, : len(t.experts)] = t.experts
        gate[i, : len(t.gates)] = t.gates
        cnt[i] = len(t.experts)
    y = expert_ffn(ExpertWeights.linear(w), x, idx, gate, cnt)
    return y[:, :dim].double().cpu().numpy()


class ExpertWeights:
    """Registered device-resident bf16 experts (desmoe_experts_create)."""

    def __init__(self, kind, experts, hidden, ffn, tensors, expert_range=None, ctx=None):
        """experts = pool size M; expert_range = (lo, hi) owned experts whose
        weights `tensors` hold (expert parallelism), default all M."""
        self.kind, self.experts, self.hidden, self.ffn = kind, experts, hidden, ffn
        self.lo, self.hi = expert_range if expert_range is not None else (0, experts)
        # the caller's tensors are only read while registering (the context
        # keeps its own tile-packed copy), so they are not retained here
        self.ctx = ctx if ctx is not None else _Ctx.get(256, experts, 32, hidden)
        h = C.c_void_p()
        ptrs = [_ptr(t) if t is not None else None for t in tensors]
        ptrs += [None] * (3 - len(ptrs))
        check(lib().desmoe_experts_create_ep(self.ctx.h, kind, experts, self.lo, self.hi, hidden,
                                             ffn, *ptrs, C.byref(h)))
        self.h = h

    @classmethod
    def swiglu(cls, w_gate, w_up, w_down, experts=None, expert_range=None, ctx=None):
        import torch
        if w_gate.dim() != 3:
            raise ValueError("w_gate must be [experts x ffn x hidden]")
        m, f, d = w_gate.shape
        for name, t, shape in (("w_gate", w_gate, (m, f, d)), ("w_up", w_up, (m, f, d)),
                               ("w_down", w_down, (m, d, f))):
            if tuple(t.shape) != shape:
                raise ValueError(f"{name} shape {tuple(t.shape)} != {shape}")
            if t.dtype != torch.bfloat16 or not t.is_cuda:
                raise ValueError(f"{name} must be a bf16 CUDA tensor")
        return cls(_lib.FFN_SWIGLU, experts or m, d, f,
                   (w_gate.contiguous(), w_up.contiguous(), w_down.contiguous()),
                   expert_range, ctx)

    @classmethod
    def linear(cls, w):
        import torch
        if w.dim() != 3 or w.shape[1] != w.shape[2]:
            raise ValueError("w must be [experts x hidden x hidden]")
        if w.dtype != torch.bfloat16 or not w.is_cuda:
            raise ValueError("w must be a bf16 CUDA tensor")
        m, d, _ = w.shape
        return cls(_lib.FFN_LINEAR, m, d, d, (w.contiguous(),))

    def __del__(self):
        try:
            lib().desmoe_experts_destroy(self.h)
        except Exception:
            pass


def expert_ffn(ex: ExpertWeights, x, route_idx, route_gate, route_cnt):
    """y [n x hidden] fp32 = sum_j gate * expert_j(x) in ascending expert order."""
    import torch
    n = x.shape[0]
    k = route_idx.shape[1]
    di = torch.as_tensor(np.ascontiguousarray(route_idx, np.int32), device="cuda")
    dg = torch.as_tensor(np.ascontiguousarray(route_gate, np.float64), device="cuda")
    dc = torch.as_tensor(np.ascontiguousarray(route_cnt, np.int32), device="cuda")
    y = torch.empty((n, ex.hidden), dtype=torch.float32, device="cuda")
    ctx = ex.ctx
    check(lib().desmoe_expert_ffn(ctx.h, ex.h, _ptr(x.contiguous()), n, k, _ptr(di), _ptr(dg),
                                  _ptr(dc), _ptr(y), _stream()))
    _finish(ctx)
    return y
