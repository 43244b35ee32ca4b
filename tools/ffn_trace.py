"""Timeline of the persistent expert-FFN kernel (desmoe_set_trace) for one
DES MoE layer block: when each SM starts streaming, unit durations, the phase
A -> B transition, the tail. Usage (GPU box):

    python tools/ffn_trace.py [--config c2] [--strategy vote] [--json out.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


FB = 100  # front-kernel marks: trace events FB + i (front.cu front_dump_marks)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--strategy", default="vote")
    ap.add_argument("--json", default="")
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm before the traced call")
    ap.add_argument("--block", type=int, default=0, help="override the block size N")
    ap.add_argument("--ffn", type=int, default=0, help="override the expert width F")
    ap.add_argument("--raw", default="", help="also save the raw records (.npz) for offline analysis")
    args = ap.parse_args()
    import torch
    from bench import CONFIGS
    from paper_2602_00879_b200 import _lib, synth
    from paper_2602_00879_b200.dessim import _ptr
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

    cfg = dict(CONFIGS[args.config])
    if args.block:
        cfg["block"] = args.block
    if args.ffn:
        cfg["ffn"] = args.ffn
    n, m, k, d, f = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000)
    wr = synth.router_weights(m, d, seed=2000)
    layer = DesMoeLayer(LayerConfig(m, k, d, f, strategy=args.strategy, vote_beta=cfg["beta"]),
                        wr, wg, wu, wd)
    cap = 1 << 17
    buf = torch.zeros(2 + 2 * cap, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    x = synth.hidden_states(n, d, seed=7, rho=cfg["rho"])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        layer.forward(x)
    L.desmoe_set_trace(layer.ctx.h, _ptr(buf), cap)
    for _ in range(2):  # second call is the traced one (graph warm)
        buf.zero_()
        if not args.no_flush:
            flush.fill_(1)
        torch.cuda.synchronize()
        layer.forward(x)
        torch.cuda.synchronize()
    L.desmoe_set_trace(layer.ctx.h, None, 0)
    raw = buf.cpu().numpy().view(np.uint64)
    cnt = min(int(raw[0]), cap)
    rec = raw[2: 2 + 2 * cnt].reshape(cnt, 2)
    rec = rec[(rec[:, 0] & 0xFF) != 255]  # unused per-thread trace records
    ev = (rec[:, 0] & 0xFF).astype(int)
    cta = ((rec[:, 0] >> 8) & 0xFFFFFF).astype(int)
    unit = (rec[:, 0] >> 32).astype(np.int64)
    unit[unit >= 2 ** 31] -= 2 ** 32
    t = rec[:, 1].astype(np.int64)
    t0 = t[ev == FB].min() if (ev == FB).any() else t[ev == 0].min()
    t = (t - t0) / 1e3  # µs
    if args.raw:
        np.savez(args.raw, ev=ev, cta=cta, unit=unit, t=t, raw=rec)
    stats = layer.stats.cpu().numpy()
    U = int(stats[0])
    tilesA = f // 64
    nA = U * tilesA
    out = {"U": U, "units": int((ev == 2).sum()), "records": cnt}
    names = {10: "front_start", 11: "front_setup_done", 12: "front_router_done",
             13: "front_sync1", 14: "front_gating_done", 15: "front_sync2",
             16: "front_coreset_done", 17: "front_reroute_done", 0: "ffn_start",
             20: "front_V_gathered", 21: "front_V_votes", 22: "front_V_ranked",
             33: "L_tok0_start", 30: "L_tok0_loaded", 31: "L_tok0_activated",
             32: "L_tok0_selected"}
    fnames = ["start", "setup", "drained", "partials_synced", "logits", "rowmax", "activated",
              "sums_topk", "selected", "sync2", "v_zeroed", "v_gathered", "coreset", "rerouted",
              "exit", "votes", "ranked", "arrived", "mma_done", "drain_done", "copies_issued", "sums_done", "topk_done"]
    fnames += [None] * (41 - len(fnames)) + ["setup_synced", "mma_full0", "mma_full_last", "x_issued",
                                             "wr_issued", "tmem_alloced", "pdl_waited"]
    fnames += [None] * (41 - len(fnames)) + ["setup_synced", "mma_full0", "mma_full_last", "x_issued",
                                             "wr_issued", "tmem_alloced", "pdl_waited"]
    for i, nm in enumerate(["l4_enter", "l4_call", "l4_selected", "l4_risky"]):
        if (ev == FB + 34 + i).any():
            out["front_" + nm] = [round(float(t[ev == FB + 34 + i].min()), 2),
                                  round(float(t[ev == FB + 34 + i].max()), 2)]
    chunks = [round(float(t[ev == FB + 26 + c].max()), 2) for c in range(5) if (ev == FB + 26 + c).any()
              and float(t[ev == FB + 26 + c].max()) < 1e6 and float(t[ev == FB + 26 + c].max()) > 0]
    if chunks:
        out["front_chunk_ends"] = chunks
    if (ev == FB + 23).any():
        out["select_cycles"] = int(rec[ev == FB + 23][:, 1].max())
    if (ev == FB + 24).any() and (ev == FB + 25).any() and (ev == FB).any() and (ev == FB + 13).any():
        cyc = rec[ev == FB + 25][:, 1].astype(np.int64) - rec[ev == FB + 24][:, 1].astype(np.int64)
        ns = rec[ev == FB + 13][:, 1].astype(np.int64) - rec[ev == FB][:, 1].astype(np.int64)
        out["front_sm_mhz"] = [round(float(c) / float(t) * 1e3, 1) for c, t in zip(cyc, ns)]
    by_cta = {}
    for i, nm in enumerate(fnames):
        e_ = FB + i
        if nm and (ev == e_).any():
            out["front_" + nm] = [round(float(t[ev == e_].min()), 2), round(float(t[ev == e_].max()), 2)]
            sel_ = ev == e_
            by_cta[nm] = {int(c): round(float(x), 2) for c, x in zip(cta[sel_], t[sel_])}
    for e_, nm in ((FB + 38, "rr_max_cycles"), (FB + 39, "rr_uncovered_mask"), (FB + 40, "rr_exact_mask")):
        sel_ = ev == e_
        if sel_.any():
            by_cta[nm] = {int(c): int(x) for c, x in zip(cta[sel_], rec[sel_][:, 1])}
    out["front_by_cta"] = by_cta
    for e_, nm in names.items():
        if (ev == e_).any():
            out[nm] = [round(float(t[ev == e_].min()), 2), round(float(t[ev == e_].max()), 2)]
    for i, nm in enumerate(["pdl_released", "counted", "slotted", "gathered", "x_ready_added",
                            "list_count_seen", "list_loaded"]):
        sel = (ev == 90 + i) & (rec[:, 1] != 0)  # (0 = not reached in this mode)
        if sel.any():
            out["ffn_" + nm] = [round(float(t[sel].min()), 2), round(float(np.median(t[sel])), 2),
                                round(float(t[sel].max()), 2)]
    if (ev == 80).any():
        out["combine_start_us"] = round(float(t[ev == 80].max()), 2)
    if (ev == 81).any():
        out["combine_end_us"] = round(float(t[ev == 81].max()), 2)
    out["kernel_span_us"] = float(t[ev == 5].max())
    out["cta_start_spread_us"] = float(t[ev == 0].max())
    out["cta_start_pct"] = [round(float(x), 2) for x in np.percentile(t[ev == 0], [0, 50, 90, 95, 100])]
    out["gather_done_us"] = ([float(t[ev == 1].min()), float(t[ev == 1].max())]
                             if (ev == 1).any() else None)
    out["first_dequeue_us"] = float(t[ev == 2].min())
    out["x_ready_seen_us"] = [float(t[ev == 6].min()), float(t[ev == 6].max())] if (ev == 6).any() else None
    done = {int(u): float(tt) for u, tt, e in zip(unit, t, ev) if e == 3}
    deq = {int(u): float(tt) for u, tt, e in zip(unit, t, ev) if e == 2}
    durA = [done[u] - deq[u] for u in deq if u < nA and u in done]
    durB = [done[u] - deq[u] for u in deq if u >= nA and u in done]
    out["phaseA_last_done_us"] = max(done[u] for u in done if u < nA) if nA else None
    out["phaseB_first_dequeue_us"] = min(deq[u] for u in deq if u >= nA)
    out["last_unit_done_us"] = max(done.values())
    out["unit_dur_A_us"] = [float(np.min(durA)), float(np.median(durA)), float(np.max(durA))] if durA else None
    out["unit_dur_B_us"] = [float(np.min(durB)), float(np.median(durB)), float(np.max(durB))]
    exits = t[ev == 5]
    out["cta_exit_us"] = [float(exits.min()), float(np.median(exits)), float(exits.max())]
    hwait = [tt for tt, e in zip(t, ev) if e == 7]
    out["h_ready_waits"] = len(hwait)
    per_cta = np.bincount(cta[ev == 2], minlength=int(cta.max()) + 1)
    out["units_per_cta"] = [int(per_cta.min()), float(per_cta.mean()), int(per_cta.max())]
    # SM clock during the front kernel's gating (events 33 -> 32 carry clock64 >> 4)
    c33 = {int(c): (int(u), tt) for c, u, tt, e in zip(cta, unit, t, ev) if e == 33}
    c32 = {int(c): (int(u), tt) for c, u, tt, e in zip(cta, unit, t, ev) if e == 32}
    mhz = [((c32[c][0] - c33[c][0]) * 16) / ((c32[c][1] - c33[c][1]) * 1e3) * 1e3
           for c in c33 if c in c32 and c32[c][1] > c33[c][1]]
    if mhz:
        out["front_sm_mhz"] = [round(min(mhz), 1), round(max(mhz), 1)]
    print(json.dumps(out, indent=1))
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
