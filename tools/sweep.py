"""Block-size sweep of the DES MoE layer on one B200 (BASELINE.json configs
1-3): for each config and N in {8..256}, device µs/block (CUDA events, L2
flushed by a 256 MiB write before every block, median of the timed blocks),
unique experts loaded U and the front (router + routing) / expert-FFN phase
times, for vanilla top-K, DES-Seq k=3/k=2 and DES-Vote.

    python tools/sweep.py [--configs c2,c3,c4] [--blocks 8,16,32,64,128,256]
                          [--steps 20] [--json profiles/sweep_r01.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4")
    ap.add_argument("--blocks", default="8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import _lib, synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

    L = _lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    ph = (C.c_float * 8)()
    out = {"method": "CUDA events per block on the layer's stream, L2 flushed before every "
                     "block, median over timed blocks; phases from a second pass with events "
                     "between kernels", "rows": []}
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        m, k, d, f = cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000)
        wr = synth.router_weights(m, d, seed=2000)
        lc = LayerConfig(m, k, d, f, strategy="vote", seq_k=3, vote_beta=cfg["beta"])
        layer = DesMoeLayer(lc, wr, wg, wu, wd)
        for n in [int(b) for b in args.blocks.split(",")]:
            xs = [synth.hidden_states(n, d, seed=10_000 + i, rho=cfg["rho"])
                  for i in range(args.warmup + args.steps)]
            y = torch.empty((n, d), dtype=torch.float32, device="cuda")
            x_in = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
            row = {"config": name, "experts": m, "top_k": k, "hidden": d, "ffn": f,
                   "block": n, "vote_beta": cfg["beta"], "rho": cfg["rho"]}
            for strat in ("vanilla", "seq3", "seq2", "vote"):
                lc.seq_k = 2 if strat == "seq2" else 3
                s = "seq" if strat.startswith("seq") else strat
                res = {}
                for prof in (0, 1):
                    L.desmoe_set_profiling(layer.ctx.h, prof)
                    t, us, phs = [], [], []
                    for i, x in enumerate(xs):
                        x_in.copy_(x)
                        flush.fill_(i & 0xFF)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        torch.cuda._sleep(50_000)  # keeps the host launch gap outside the events
                        e0.record(stream)
                        layer.forward(x_in, y, strategy=s)
                        e1.record(stream)
                        e1.synchronize()
                        if i < args.warmup:
                            continue
                        t.append(e0.elapsed_time(e1) * 1e3)
                        us.append(int(layer.stats[0].item()))
                        if prof:
                            cnt = L.desmoe_get_phase_ms(layer.ctx.h, ph, 8)
                            phs.append([ph[j] * 1e3 for j in range(cnt)])
                    if prof:
                        p = np.array(phs)
                        res["front_us"] = round(float(np.median(p[:, :-2].sum(axis=1))), 2)
                        res["ffn_us"] = round(float(np.median(p[:, -2])), 2)
                        res["combine_us"] = round(float(np.median(p[:, -1])), 2)
                    else:
                        res["us_per_block"] = round(float(np.median(t)), 2)
                        res["unique_experts"] = round(float(np.mean(us)), 2)
                u = res["unique_experts"]
                res["expert_weight_GBps"] = round(u * 3 * d * f * 2 / (res["ffn_us"] * 1e-6) / 1e9, 1)
                row[strat] = res
            row["vote_latency_reduction"] = round(
                1 - row["vote"]["us_per_block"] / row["vanilla"]["us_per_block"], 4)
            row["vote_unique_reduction"] = round(
                1 - row["vote"]["unique_experts"] / row["vanilla"]["unique_experts"], 4)
            out["rows"].append(row)
            print(json.dumps(row), flush=True)
        del layer
        torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
