"""Routes every block of a MOET router trace (the reference's trace file,
binary or JSONL) on the GPU — the logits-in use of the routing path that
`dessim run` makes on the CPU. Prints one JSON line with per-block unique
experts (U) and coreset sizes per strategy and the mean GPU time per block.

    python tools/route_trace.py TRACE.moet [--strategies vanilla,seq3,vote]
                                [--beta 0.4] [--top-k K]
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
    ap.add_argument("trace")
    ap.add_argument("--strategies", default="vanilla,seq3,vote")
    ap.add_argument("--beta", type=float, default=0.4)
    ap.add_argument("--top-k", type=int, default=0, help="override the header's top_k")
    args = ap.parse_args()
    import torch
    from paper_2602_00879_b200 import dessim as ds
    from paper_2602_00879_b200 import moet

    f = moet.read_trace(args.trace)
    h = f.header
    k = args.top_k or h.top_k
    cfg = ds.PoolConfig(h.experts, k)
    out = {"trace": os.path.basename(args.trace), "experts": h.experts, "top_k": k,
           "layers": h.layers, "steps": h.steps, "block_size": h.block_size, "strategies": {}}
    for s in args.strategies.split(","):
        us, cs = [], []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for b in f.blocks:
            if s == "vanilla":
                a = ds.topk_route(ds.activate(b, cfg), k)
                core = ds.unique_experts(a)
            else:
                p = (ds.DesParams(ds.DesStrategy.seq, int(s[3:]), 1.0) if s.startswith("seq")
                     else ds.DesParams(ds.DesStrategy.vote, 1, args.beta))
                r = ds.des_run(b, cfg, p)
                a, core = r.assignment, r.coreset
            us.append(len(ds.unique_experts(a).members))
            cs.append(core.size())
        ev1.record()
        torch.cuda.synchronize()
        out["strategies"][s] = {"U_mean": float(np.mean(us)), "U_per_block": us,
                                "coreset_mean": float(np.mean(cs)),
                                "ms_per_block_incl_host": ev0.elapsed_time(ev1) / len(f.blocks)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
