"""Latency probes of the routing kernels through the C ABI (CUDA events,
median of repeats): fused single-CTA routing (desmoe_route) and the
activation-only kernel (desmoe_activate) at several block sizes."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_00879_b200 import _lib, synth  # noqa: E402
from paper_2602_00879_b200.dessim import _Ctx, _ptr, _stream  # noqa: E402


def med_us(fn, reps=50):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


L = _lib.lib()
out = {}
for m in (64, 256):
    for n in (1, 8, 32, 64):
        ctx = _Ctx.get(n, m, 8)
        x = torch.as_tensor(synth.gen_trace_block(m, n, 42, rho=0.3), device="cuda")
        idx = torch.empty((n, 8), dtype=torch.int32, device="cuda")
        gate = torch.empty((n, 8), dtype=torch.float64, device="cuda")
        cnt = torch.empty(n, dtype=torch.int32, device="cuda")
        probs = torch.empty((n, m), dtype=torch.float64, device="cuda")
        ro = _lib.RouteOut(idx.data_ptr(), gate.data_ptr(), cnt.data_ptr(), None, None, None, None)
        for strat, name in ((_lib.VANILLA, "vanilla"), (_lib.VOTE, "vote")):
            cfg = _lib.RouteCfg(m, 8, 0, strat, 3, 0.4 if m == 64 else 0.15, 0)
            out[f"route_{name}_m{m}_n{n}"] = med_us(lambda: L.desmoe_route(
                ctx.h, _ptr(x), n, C.byref(cfg), C.byref(ro), _stream()))
        out[f"activate_m{m}_n{n}"] = med_us(lambda: L.desmoe_activate(
            ctx.h, _ptr(x), n, m, 0, _ptr(probs), _stream()))
out["empty_kernel_like"] = med_us(lambda: torch.cuda._sleep(0))
print(json.dumps({k: round(v, 2) for k, v in out.items()}, indent=0))
