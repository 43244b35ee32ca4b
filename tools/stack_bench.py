"""One diffusion denoising step through a stack of DES MoE layers (BASELINE
config 5: the 24 MoE layers of a LLaDA2.0-mini-shaped model, N=64, DES-Vote)
on one B200: desmoe_stack_forward runs all layers as ONE CUDA graph, layer l's
output feeding layer l+1 as bf16 on a residual stream (h + MoE(h)). Random-init weights (24 x 1.6 GB of
experts: every layer's experts come from HBM); device time per step with CUDA
events; vanilla top-K vs DES-Vote (and DES-Seq k=3).

    python tools/stack_bench.py [--config c3] [--layers 24] [--block 64] [--steps 20]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--block", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import synth
    from paper_2602_00879_b200.layer import DesMoeStack, LayerConfig

    cfg = CONFIGS[args.config]
    m, k, d, f, n = cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"], args.block
    lc = LayerConfig(m, k, d, f, strategy="vote", seq_k=3, vote_beta=cfg["beta"])
    params = []
    for l in range(args.layers):
        params.append((synth.router_weights(m, d, seed=7000 + l),
                       *synth.swiglu_weights(m, d, f, seed=8000 + 17 * l)))
    stack = DesMoeStack(lc, params, max_tokens=max(n, 256))
    del params
    torch.cuda.empty_cache()
    xs = [synth.hidden_states(n, d, seed=900 + i, rho=cfg["rho"])
          for i in range(args.warmup + args.steps)]
    x_in = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((n, d), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    out = {"workload": f"{args.layers}-layer MoE stack, {cfg['desc']}: M={m} top-{k} d={d} "
                       f"SwiGLU F={f}, block N={n}, one denoising step per measurement",
           "weights_GB": round(args.layers * m * 3 * d * f * 2 / 1e9, 1), "strategies": {}}
    for strat in ("vanilla", "seq", "vote"):
        times, us, streamed = [], [], []
        for i, x in enumerate(xs):
            x_in.copy_(x)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(50_000)  # keeps the host launch gap outside the events
            e0.record(st)
            stack.forward(x_in, y, strategy=strat, residual=True)
            e1.record(st)
            e1.synchronize()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1) * 1e3)
                us.append(stack.stats[:, 0].float().mean().item())
                streamed.append(stack.stats[:, 3].float().mean().item())
        out["strategies"][strat] = {"us_per_step": round(float(np.median(times)), 1),
                                    "us_per_layer": round(float(np.median(times)) / args.layers, 2),
                                    "unique_experts_per_layer": round(float(np.mean(us)), 2),
                                    "experts_streamed_per_layer": round(float(np.mean(streamed)), 2)}
    v, van = out["strategies"]["vote"], out["strategies"]["vanilla"]
    out["vote_step_reduction"] = round(1 - v["us_per_step"] / van["us_per_step"], 4)
    print(json.dumps(out))
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
