"""The DES MoE layer (router -> DES coreset -> constrained re-route ->
permutation -> grouped SwiGLU expert FFN + combine) on one B200, through the
C ABI's desmoe_layer_forward / desmoe_layer_forward_host.

Weights live in HBM as bf16: router [M x d], experts w_gate/w_up [M x F x d],
w_down [M x d x F] (the 2-D row-major views the TMA descriptors stream).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from ._lib import RouteCfg, check, lib
from .dessim import ExpertWeights, _Ctx, _ptr, _stream

STRATEGIES = {"vanilla": _lib.VANILLA, "seq": _lib.SEQ, "vote": _lib.VOTE}


@dataclass
class LayerConfig:
    experts: int
    top_k: int
    hidden: int
    ffn: int
    strategy: str = "vote"   # vanilla | seq | vote
    seq_k: int = 3
    vote_beta: float = 0.4
    activation: int = _lib.SOFTMAX

    def route_cfg(self, strategy=None):
        s = STRATEGIES[strategy or self.strategy]
        return RouteCfg(self.experts, self.top_k, self.activation, s, self.seq_k,
                        float(self.vote_beta), _lib.VOTE_ACTIVATED)


def _check_act(name, t, n_max, hidden, dtype, device_only=True):
    """A [n x hidden] activation tensor the C ABI reads / writes as packed
    `dtype` rows: reject anything else before its pointer crosses the ABI."""
    import torch
    if t.dim() != 2 or t.shape[1] != hidden or not (1 <= t.shape[0] <= n_max):
        raise ValueError(f"{name} must be [n x {hidden}] with 1 <= n <= {n_max}, "
                         f"got {tuple(t.shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device_only and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


class DesMoeLayer:
    """One DES MoE layer. With expert_range=(lo, hi), w_gate/w_up/w_down hold
    only the owned experts of an expert-parallel rank (see ep.py); connect the
    ranks with ep.connect_distributed / ep.connect_local before forward()."""

    def __init__(self, cfg: LayerConfig, w_router, w_gate, w_up, w_down, max_tokens=256,
                 expert_range=None, own_context=False):
        import torch
        self.cfg = cfg
        if tuple(w_router.shape) != (cfg.experts, cfg.hidden) or w_router.dtype != torch.bfloat16:
            raise ValueError(f"w_router must be bf16 [{cfg.experts} x {cfg.hidden}]")
        self.w_router = w_router.contiguous()
        self.max_tokens = max_tokens
        ctx = None
        if own_context:  # a private C-ABI context (several simulated ranks per thread)
            ctx = _Ctx(torch.cuda.current_device(), max_tokens, max(cfg.experts, 256), 32,
                       max(cfg.hidden, 4096))
        self.experts = ExpertWeights.swiglu(w_gate, w_up, w_down, experts=cfg.experts,
                                            expert_range=expert_range, ctx=ctx)
        self.ctx = self.experts.ctx
        self.stats = torch.zeros(4, dtype=torch.int32, device="cuda")
        self._rc = {}  # strategy -> RouteCfg (built once: the per-call path stays thin)

    def forward(self, x, y=None, strategy=None, stream=None):
        """x [n x d] bf16 on the device -> y [n x d] fp32 (stream-ordered)."""
        import torch
        _check_act("x", x, self.max_tokens, self.cfg.hidden, torch.bfloat16)
        n = x.shape[0]
        if y is None:
            y = torch.empty((n, self.cfg.hidden), dtype=torch.float32, device=x.device)
        _check_act("y", y, self.max_tokens, self.cfg.hidden, torch.float32)
        if y.shape[0] != n:
            raise ValueError("y must have as many rows as x")
        rc = self._route_cfg(strategy)
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(lib().desmoe_layer_forward(self.ctx.h, self.experts.h, self.w_router.data_ptr(),
                                         x.data_ptr(), n, C.byref(rc), y.data_ptr(),
                                         self.stats.data_ptr(), st))
        return y

    def _route_cfg(self, strategy):
        c = self.cfg  # LayerConfig is mutable (e.g. seq_k): key on every routed field
        key = (strategy, c.experts, c.top_k, c.activation, c.strategy, c.seq_k, c.vote_beta)
        rc = self._rc.get(key)
        if rc is None:
            rc = self._rc[key] = c.route_cfg(strategy)
        return rc

    def forward_host(self, x_host, y_host, stats_host=None, strategy=None):
        """Host (pinned) bf16 x -> host fp32 y through desmoe_layer_forward_host
        (H2D copy, layer, D2H copy, synchronise)."""
        import torch
        _check_act("x_host", x_host, self.max_tokens, self.cfg.hidden, torch.bfloat16, False)
        _check_act("y_host", y_host, self.max_tokens, self.cfg.hidden, torch.float32, False)
        if x_host.is_cuda or y_host.is_cuda or y_host.shape[0] != x_host.shape[0]:
            raise ValueError("x_host / y_host must be host tensors with the same row count")
        if stats_host is not None and (stats_host.is_cuda or stats_host.dtype != torch.int32
                                       or stats_host.numel() < 4):
            raise ValueError("stats_host must be a host int32 tensor of >= 4 entries")
        check(lib().desmoe_layer_forward_host(
            self.ctx.h, self.experts.h, self.w_router.data_ptr(), x_host.data_ptr(),
            x_host.shape[0], C.byref(self._route_cfg(strategy)), y_host.data_ptr(),
            stats_host.data_ptr() if stats_host is not None else None,
            torch.cuda.current_stream().cuda_stream))
        return y_host

    def last_logits(self, n):
        """fp32 router logits [n x M] the last forward() routed with."""
        import torch
        out = torch.empty((n, self.cfg.experts), dtype=torch.float32, device="cuda")
        check(lib().desmoe_layer_logits(self.ctx.h, _ptr(out), n, self.cfg.experts, _stream()))
        return out

    def last_route(self, n):
        """(idx [n x K] int32, gate [n x K] f64, cnt [n] int32, coreset members
        list) of the last forward() (numpy)."""
        import torch
        k, m = self.cfg.top_k, self.cfg.experts
        idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
        gate = torch.empty((n, k), dtype=torch.float64, device="cuda")
        cnt = torch.empty(n, dtype=torch.int32, device="cuda")
        mem = torch.empty(m, dtype=torch.int32, device="cuda")
        nm = torch.empty(1, dtype=torch.int32, device="cuda")
        check(lib().desmoe_layer_route(self.ctx.h, _ptr(idx), _ptr(gate), _ptr(cnt), _ptr(mem),
                                       _ptr(nm), n, k, m, _stream()))
        torch.cuda.synchronize()
        return (idx.cpu().numpy(), gate.cpu().numpy(), cnt.cpu().numpy(),
                mem[: int(nm.item())].cpu().numpy().tolist())

    def check(self):
        check(lib().desmoe_check(self.ctx.h, _stream()))


class DesMoeStack:
    """A stack of DES MoE layers (the MoE layers of one diffusion denoising
    step) run by desmoe_stack_forward as ONE CUDA graph: layer l's output
    feeds layer l+1 as bf16. `layers` = list of (w_router, w_gate, w_up,
    w_down) tuples; all layers share one C-ABI context."""

    def __init__(self, cfg: LayerConfig, layers, max_tokens=256, expert_range=None):
        import torch
        self.cfg = cfg
        self.max_tokens = max_tokens
        self.ctx = _Ctx(torch.cuda.current_device(), max_tokens, max(cfg.experts, 256), 32,
                        max(cfg.hidden, 4096))
        self.routers, self.experts = [], []
        for wr, wg, wu, wd in layers:
            self.routers.append(wr.contiguous())
            self.experts.append(ExpertWeights.swiglu(wg, wu, wd, experts=cfg.experts,
                                                     expert_range=expert_range, ctx=self.ctx))
        n = len(self.experts)
        self._ex = (C.c_void_p * n)(*[e.h.value for e in self.experts])
        self._wr = (C.c_void_p * n)(*[w.data_ptr() for w in self.routers])
        self.stats = torch.zeros((n, 4), dtype=torch.int32, device="cuda")

    def __len__(self):
        return len(self.experts)

    def forward(self, x, y=None, strategy=None, stream=None, residual=False):
        """x [n x d] bf16 -> y [n x d] fp32 after all layers (stream-ordered);
        residual=True: every layer outputs h + MoE(h)."""
        import torch
        _check_act("x", x, self.max_tokens, self.cfg.hidden, torch.bfloat16)
        n = x.shape[0]
        if y is None:
            y = torch.empty((n, self.cfg.hidden), dtype=torch.float32, device=x.device)
        _check_act("y", y, self.max_tokens, self.cfg.hidden, torch.float32)
        if y.shape[0] != n:
            raise ValueError("y must have as many rows as x")
        rc = self.cfg.route_cfg(strategy)
        st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream()
        check(lib().desmoe_stack_forward(self.ctx.h, self._ex, self._wr, len(self.experts),
                                         _ptr(x), n, C.byref(rc), _ptr(y), _ptr(self.stats),
                                         1 if residual else 0, st))
        return y
