"""Where the host-buffer entry's time goes (C2 DES-Vote layer). Host
wall-clock and GPU-event medians per call for: the device-resident layer
(Python wrapper and a direct ctypes call), the host-buffer entry
desmoe_layer_forward_host (wrapper and direct), and its parts (pinned H2D of
x, an idle-stream synchronisation). Consecutive calls rotate over several
layers (>= 1 GiB of experts) as in bench.py, so weights stream from HBM.

    python tools/e2e_probe.py
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import _lib, synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    cfg = CONFIGS["c2"]
    n, m, k, d, f = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
    lc = LayerConfig(m, k, d, f, strategy="vote", vote_beta=cfg["beta"])
    layers = []
    for li in range(4):
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000 + li)
        layers.append(DesMoeLayer(lc, synth.router_weights(m, d, seed=2000 + li), wg, wu, wd,
                                  own_context=True))
    L = _lib.lib()
    x = synth.hidden_states(n, d, seed=7, rho=cfg["rho"])
    xh = x.cpu().pin_memory()
    xd = x.clone()
    y = torch.empty((n, d), dtype=torch.float32, device="cuda")
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    sh = torch.empty(4, dtype=torch.int32).pin_memory()
    st = torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)
    rc = lc.route_cfg()
    out = {}
    it = [0]

    def nxt():
        it[0] += 1
        return layers[it[0] % len(layers)]

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

    def direct_dev():
        l = nxt()
        L.desmoe_layer_forward(l.ctx.h, l.experts.h, l.w_router.data_ptr(), xd.data_ptr(), n,
                               C.byref(rc), y.data_ptr(), l.stats.data_ptr(), sp)

    def direct_host():
        l = nxt()
        L.desmoe_layer_forward_host(l.ctx.h, l.experts.h, l.w_router.data_ptr(), xh.data_ptr(), n,
                                    C.byref(rc), yh.data_ptr(), sh.data_ptr(), sp)

    def direct_dev_mapped_y():  # y written into pinned host memory by the combine
        l = nxt()
        L.desmoe_layer_forward(l.ctx.h, l.experts.h, l.w_router.data_ptr(), xd.data_ptr(), n,
                               C.byref(rc), yh.data_ptr(), l.stats.data_ptr(), sp)

    def h2d_then_dev():
        xd.copy_(xh, non_blocking=True)
        direct_dev()

    timed("layer_device_wrapper", lambda: nxt().forward(xd, y))
    timed("layer_device_direct", direct_dev)
    timed("layer_device_mapped_y", direct_dev_mapped_y)
    timed("h2d_then_layer_device", h2d_then_dev)
    timed("h2d_only", lambda: xd.copy_(xh, non_blocking=True))
    timed("forward_host_wrapper", lambda: nxt().forward_host(xh, yh, sh, strategy="vote"))
    timed("forward_host_direct", direct_host)
    xrot = [synth.hidden_states(n, d, seed=100 + i, rho=cfg["rho"]).cpu().pin_memory()
            for i in range(64)]
    r = [0]

    def direct_host_rot():  # a different pinned x buffer every call (as bench.py)
        l = nxt()
        r[0] += 1
        L.desmoe_layer_forward_host(l.ctx.h, l.experts.h, l.w_router.data_ptr(),
                                    xrot[r[0] % len(xrot)].data_ptr(), n, C.byref(rc),
                                    yh.data_ptr(), sh.data_ptr(), sp)

    timed("forward_host_direct_rotating_x", direct_host_rot)
    import json
    print(json.dumps({"variant": os.environ.get("DESMOE_INGRESS", "") + os.environ.get("DESMOE_HOST_MEMCPY", ""), **out}))


if __name__ == "__main__":
    main()
