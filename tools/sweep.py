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
    ap.add_argument("--no-cpu", action="store_true", help="skip the reference CPU column")
    ap.add_argument("--cpu-ffn-tokens", type=int, default=1,
                    help="tokens the reference's moe_forward runs per sample (time scaled to N)")
    args = ap.parse_args()
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import _lib, synth
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

    L = _lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    ph = (C.c_float * 8)()
    from bench import measured_peaks
    peak, peak_kind = measured_peaks()
    threads = os.cpu_count() or 1
    cpu_model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu_model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ref = None
    if not args.no_cpu:
        from oracle.oracle import Ref
        ref = Ref()
    out = {"method": "CUDA events per block on the layer's stream, L2 flushed before every "
                     "block, median over timed blocks; phases from a second pass with events "
                     "between kernels",
           "roofline": {"peak_GBps": peak, "peak_kind": peak_kind,
                        "ffn_frac": "U*3*d*F*2 / t_ffn / peak",
                        "layer_frac": "(U*3*d*F*2 + M*d*2 + N*d*2 + N*d*4) / t_block / peak"},
           "cpu_reference": None if ref is None else {
               "kind": "reference (oracle/_ref: the reference's own des_run / topk_route + "
                       "moe_forward with its linear d x d fp64 experts)",
               "cores": threads, "cpu_model": cpu_model,
               "latency_1t": "one block on one thread (taskset-free, steady_clock); moe_forward "
                             f"on {args.cpu_ffn_tokens} tokens scaled to N",
               "throughput_all": f"{threads} threads x 1 block each, blocks/s"},
           "rows": []}
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
                res["ffn_frac"] = round(res["expert_weight_GBps"] / peak, 4)
                layer_bytes = u * 3 * d * f * 2 + m * d * 2 + n * d * 2 + n * d * 4
                res["layer_frac"] = round(layer_bytes / (res["us_per_block"] * 1e-6) / 1e9 / peak, 4)
                if ref is not None and strat in ("vanilla", "seq3", "vote"):
                    lg = synth.gen_trace_block(m, n, 42, rho=cfg["rho"])
                    rs = {"vanilla": ("vanilla", 1), "seq3": ("seq", 3), "vote": ("vote", 1)}[strat]
                    kw = dict(seq_k=rs[1], beta=cfg["beta"], dim=d, reps=1,
                              ffn_tokens=min(n, args.cpu_ffn_tokens))
                    t1, _ = ref.time_layer(lg, k, rs[0], threads=1, **kw)
                    ta, _ = ref.time_layer(lg, k, rs[0], threads=threads, **kw)
                    rt = ref.time_routing(lg, k, rs[0], seq_k=rs[1], beta=cfg["beta"], reps=5)
                    res["cpu_ref"] = {"layer_us_1t": round(t1 * 1e6, 1),
                                      "layer_blocks_per_s_all": round(1.0 / ta, 2),
                                      "routing_us_1t": round(1e6 / rt, 2)}
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
