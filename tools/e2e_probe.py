"""Where the host-buffer entry's time goes (C2 DES-Vote layer): device-only
layer call vs + pinned H2D of x vs the full desmoe_layer_forward_host (H2D,
layer, y into pinned host memory, one synchronisation). GPU-event and host
wall-clock means per call.

    python tools/e2e_probe.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    cfg = CONFIGS["c2"]
    n, m, k, d, f = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000)
    wr = synth.router_weights(m, d, seed=2000)
    layer = DesMoeLayer(LayerConfig(m, k, d, f, strategy="vote", vote_beta=cfg["beta"]), wr, wg, wu, wd)
    x = synth.hidden_states(n, d, seed=7, rho=cfg["rho"])
    xh = x.cpu().pin_memory()
    xd = torch.empty_like(x)
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    sh = torch.empty(4, dtype=torch.int32).pin_memory()
    st = torch.cuda.current_stream()
    out = {}

    def timed(name, fn, reps=200):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        gpu, host = [], []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            host.append((time.perf_counter() - t0) * 1e6)
            gpu.append(e0.elapsed_time(e1) * 1e3)
        out[name] = {"gpu_us": round(float(np.median(gpu)), 2), "host_us": round(float(np.median(host)), 2)}

    timed("layer_device", lambda: layer.forward(x))
    timed("h2d_then_layer", lambda: (xd.copy_(xh, non_blocking=True), layer.forward(xd)))
    timed("h2d_only", lambda: xd.copy_(xh, non_blocking=True))
    timed("forward_host", lambda: layer.forward_host(xh, yh, sh, strategy="vote"))
    print(out)


if __name__ == "__main__":
    main()
