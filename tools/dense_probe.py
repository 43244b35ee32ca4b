"""Dense vs routed FFN mode for a DES block (experiment): the dense mode
(every published expert x every token, no route / permutation) is allowed
when M x N rows fit the context's slot buffer (max_n x max_k); a context
with max_top_k = 64 lets C3 N = 64 (M = 256) run dense. L2 flushed,
CUDA events, median.

    python tools/dense_probe.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2602_00879_b200 import synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for (m, d, f, n, beta) in [(256, 2048, 512, 64, 0.15), (128, 2048, 768, 64, 0.3)]:
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1)
        wr = synth.router_weights(m, d, seed=2)
        for mk in (32, 64):  # max_tokens = 8 mk: slot capacity 256 x 32 or 512 x 32
            layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy="vote", vote_beta=beta), wr, wg, wu, wd,
                                own_context=True, max_tokens=8 * mk)
            x_in = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
            y = torch.empty((n, d), dtype=torch.float32, device="cuda")
            for fl in (True, False):
                ts = []
                for i in range(25):
                    x_in.copy_(synth.hidden_states(n, d, seed=100 + i, rho=0.3))
                    if fl:
                        flush.fill_(i & 0xFF)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    torch.cuda._sleep(50_000)
                    e0.record(st)
                    layer.forward(x_in, y)
                    e1.record(st)
                    e1.synchronize()
                    if i >= 5:
                        ts.append(e0.elapsed_time(e1) * 1e3)
                print(f"m={m} n={n} max_top_k={mk} ({'dense' if m * n <= 8 * mk * 32 else 'routed'}) "
                      f"{'flushed' if fl else 'warm'}: {np.median(ts):.2f} us, U={int(layer.stats[0])}",
                      flush=True)
            del layer
        del wg, wu, wd
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
