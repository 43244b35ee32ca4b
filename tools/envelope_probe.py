"""Layer timing inside vs outside the front kernel's envelope (N, M <= 256,
d a multiple of 512): outside, the router runs as the split-K tile GEMM and
the routing as the single-CTA logits-in kernels. L2 flushed
before every block, CUDA events, median; one B200.

    python tools/envelope_probe.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # m, d, f, n, beta
    (256, 2048, 512, 32, 0.15),   # C3, in the envelope (router kernel + front)
    (512, 2048, 512, 32, 0.075),  # M = 512: router kernel + logits-in front
    (512, 2048, 512, 64, 0.075),
    (256, 1536, 512, 32, 0.15),   # d = 3 x 512: in the envelope
    (256, 1280, 512, 32, 0.15),   # d not a multiple of 512: split path
]


def main():
    import torch
    from paper_2602_00879_b200 import synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for m, d, f, n, beta in CASES:
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1)
        wr = synth.router_weights(m, d, seed=2)
        row = {"m": m, "d": d, "f": f, "n": n, "beta": beta,
               "front_envelope": bool(m <= 512 and n <= 256 and d % 512 == 0)}
        for strat in ("vanilla", "vote"):
            layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy=strat, vote_beta=beta), wr, wg, wu, wd)
            xs = [synth.hidden_states(n, d, seed=100 + i, rho=0.3) for i in range(23)]
            ts, us = [], []
            for i, x in enumerate(xs):
                flush.fill_(i & 0xFF)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(50_000)
                e0.record(st)
                layer.forward(x)
                e1.record(st)
                e1.synchronize()
                if i >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e3)
                    us.append(int(layer.stats[0].item()))
            layer.check()
            u = float(np.mean(us))
            row[strat] = {"us_per_block": round(float(np.median(ts)), 2), "unique_experts": round(u, 2),
                          "layer_frac_vs_weights": round(u * 3 * d * f * 2 / (np.median(ts) * 1e-6) / 1e9 / 6539, 3)}
            del layer
        print(json.dumps(row), flush=True)
        del wg, wu, wd
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
