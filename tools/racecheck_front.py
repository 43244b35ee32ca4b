"""A few layer calls (vote / seq / vanilla; in-front GEMM and logits-in
modes) for compute-sanitizer --tool racecheck / synccheck (GPU box):

    compute-sanitizer --tool racecheck python tools/racecheck_front.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2602_00879_b200 import synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    for (m, d, f, n) in [(64, 512, 256, 32), (256, 512, 256, 64)]:
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1)
        wr = synth.router_weights(m, d, seed=2)
        for strat in ("vote", "seq", "vanilla"):
            layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy=strat, seq_k=3, vote_beta=0.3),
                                wr, wg, wu, wd, own_context=True)
            x = synth.hidden_states(n, d, seed=3, rho=0.3)
            layer.forward(x)
            torch.cuda.synchronize()
            layer.check()
            print(m, n, strat, layer.stats.cpu().tolist(), flush=True)


if __name__ == "__main__":
    main()
