"""Controlled-logit harness for the LAYER path (test helper, not a test file).

The layer computes its router logits itself (bf16 X . bf16 W_r^T on tensor
cores, fp32 accumulation), so routing edge cases (exact ties, near-ties
below the front kernel's 24-bit selection key, softmax underflow, saturated
sigmoids, tied DES-Vote votes) cannot be reached with random hidden states.
This helper injects ANY fp32 logit matrix L [n x m] into the layer's own GEMM:

  * every fp32 value v splits exactly into three bf16 pieces
        v = a + b * 2^-8 + c * 2^-16
    (a = v truncated to bf16, b = the next 8 significant bits scaled up,
    c = the rest); every partial sum of the pieces is representable in fp32;
  * hidden states X [n x d]: X[t, t] = 1, X[t, o1 + t] = 2^-8,
    X[t, o2 + t] = 2^-16 (o1 = n, o2 = 2n), zero elsewhere;
  * router weights W_r [m x d]: W_r[e, t] = a[t, e], W_r[e, o1 + t] = b[t, e],
    W_r[e, o2 + t] = c[t, e].

Each logit is then a dot product with exactly three non-zero exact products
(powers of two times bf16 values), accumulated in ascending K order (split-K
partials are summed in ascending CTA order = ascending K), so the layer's fp32
logits equal L bit for bit — which the tests assert through
desmoe_layer_logits before comparing the routing with the reference library
fed the same values.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

P8 = np.float32(2.0 ** -8)
P16 = np.float32(2.0 ** -16)


def bf16_trunc(v: np.ndarray) -> np.ndarray:
    """fp32 values truncated (toward zero) to bf16 precision, as fp32."""
    u = np.ascontiguousarray(v, np.float32).view(np.uint32) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


def split3(logits) -> tuple:
    """fp32 [n x m] -> (a, b, c), each bf16-exact, with a + b*2^-8 + c*2^-16 == v
    in fp32 arithmetic (asserted)."""
    v = np.ascontiguousarray(logits, np.float32)
    a = bf16_trunc(v)
    r1 = (v - a).astype(np.float32)                       # exact: the low 16 bits
    b = bf16_trunc((r1 * np.float32(256.0)).astype(np.float32))
    r2 = (r1 - b * P8).astype(np.float32)                 # exact: the low 8 bits
    c = (r2 * np.float32(65536.0)).astype(np.float32)
    if not (bf16_trunc(c) == c).all():
        raise ValueError("logit not representable as three bf16 pieces")
    rec = ((a + b * P8).astype(np.float32) + c * P16).astype(np.float32)
    if not np.array_equal(rec.view(np.uint32), v.view(np.uint32)):
        raise ValueError("three-piece split does not reconstruct the logits")
    return a, b, c


def hidden_for(n: int) -> int:
    """Hidden size that holds the three identity blocks (front kernel envelope:
    a multiple of 512)."""
    return 512 if 3 * n <= 512 else 1024


def exact_inputs(logits, d: int):
    """(X [n x d], W_r [m x d]) bf16 CUDA tensors whose router GEMM is `logits`."""
    import torch
    a, b, c = split3(logits)
    n, m = a.shape
    if 3 * n > d:
        raise ValueError("hidden too small for three identity blocks")
    x = np.zeros((n, d), np.float32)
    w = np.zeros((m, d), np.float32)
    t = np.arange(n)
    for off, piece, scale in ((0, a, 1.0), (n, b, 2.0 ** -8), (2 * n, c, 2.0 ** -16)):
        x[t, off + t] = scale
        w[:, off:off + n] = piece.T
    X = torch.from_numpy(x).to(torch.bfloat16)
    W = torch.from_numpy(w).to(torch.bfloat16)
    # the conversion must be exact (every value is bf16-representable)
    assert torch.equal(X.float(), torch.from_numpy(x)) and torch.equal(W.float(), torch.from_numpy(w))
    return X.cuda(), W.cuda()


class LayerProbe:
    """Runs desmoe_layer_forward on injected logits and returns what the layer
    routed with: its fp32 logits, route (idx, gate, cnt) and coreset.

    One context and one zero-weight expert bank per pool size (the FFN's
    output is irrelevant to routing parity); graphs off by default so every
    call launches its kernels eagerly (different shapes per call)."""

    def __init__(self, max_n=256, max_m=256, max_k=16, d=1024, f=128, graphs=False):
        import torch
        from paper_2602_00879_b200 import dessim as ds
        from paper_2602_00879_b200._lib import check, lib
        self.torch, self.ds, self.check, self.lib = torch, ds, check, lib()
        self.d, self.f, self.max_k = d, f, max_k
        self.ctx = ds._Ctx(torch.cuda.current_device(), max_n, max_m, max_k, d)
        if not graphs:
            check(self.lib.desmoe_set_graphs(self.ctx.h, 0))
        self.wg = torch.zeros((max_m, f, d), dtype=torch.bfloat16, device="cuda")
        self.wd = torch.zeros((max_m, d, f), dtype=torch.bfloat16, device="cuda")
        self._bank = (None, None)

    def bank(self, m):
        if self._bank[0] != m:
            self._bank = (None, None)  # release the previous registration first
            ex = self.ds.ExpertWeights.swiglu(self.wg[:m], self.wg[:m], self.wd[:m], experts=m,
                                              ctx=self.ctx)
            self._bank = (m, ex)
        return self._bank[1]

    def run(self, logits, k, strategy="vote", seq_k=1, beta=1.0, act=0, raw=False):
        from paper_2602_00879_b200 import _lib
        torch, ds = self.torch, self.ds
        L32 = np.ascontiguousarray(logits, np.float32)
        n, m = L32.shape
        X, W = exact_inputs(L32, self.d)
        strat = {"vanilla": _lib.VANILLA, "seq": _lib.SEQ, "vote": _lib.VOTE}[strategy]
        rc = _lib.RouteCfg(m, k, act, strat, seq_k, float(beta),
                           _lib.VOTE_RAW_LOGITS if raw else _lib.VOTE_ACTIVATED)
        y = torch.empty((n, self.d), dtype=torch.float32, device="cuda")
        stats = torch.zeros(4, dtype=torch.int32, device="cuda")
        ex = self.bank(m)
        self.check(self.lib.desmoe_layer_forward(self.ctx.h, ex.h, ds._ptr(W), ds._ptr(X), n,
                                                 C.byref(rc), ds._ptr(y), ds._ptr(stats),
                                                 ds._stream()))
        self.check(self.lib.desmoe_check(self.ctx.h, ds._stream()))
        lg = torch.empty((n, m), dtype=torch.float32, device="cuda")
        self.check(self.lib.desmoe_layer_logits(self.ctx.h, ds._ptr(lg), n, m, ds._stream()))
        idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
        gate = torch.empty((n, k), dtype=torch.float64, device="cuda")
        cnt = torch.empty(n, dtype=torch.int32, device="cuda")
        mem = torch.empty(m, dtype=torch.int32, device="cuda")
        nm = torch.empty(1, dtype=torch.int32, device="cuda")
        self.check(self.lib.desmoe_layer_route(self.ctx.h, ds._ptr(idx), ds._ptr(gate),
                                               ds._ptr(cnt), ds._ptr(mem), ds._ptr(nm), n, k, m,
                                               ds._stream()))
        torch.cuda.synchronize()
        return {"logits": lg.cpu().numpy(), "idx": idx.cpu().numpy(), "gate": gate.cpu().numpy(),
                "cnt": cnt.cpu().numpy(), "members": mem[: int(nm.item())].cpu().numpy().tolist(),
                "stats": stats.cpu().numpy(), "y": y}


def assert_same_route(got, want, gate_atol=0.0):
    """Exact ids and counts; gates bit-identical by default (the GPU's exp is
    glibc's, restated: paper_2602_00879_b200/csrc/libm_exp.cuh)."""
    np.testing.assert_array_equal(got["cnt"], want.cnt)
    for t in range(len(want.cnt)):
        c = int(want.cnt[t])
        np.testing.assert_array_equal(got["idx"][t, :c], want.idx[t, :c], err_msg=f"token {t}")
        np.testing.assert_allclose(got["gate"][t, :c], want.gate[t, :c], rtol=0, atol=gate_atol,
                                   err_msg=f"token {t}")
