#!/usr/bin/env python
"""Benchmark of the DES MoE layer on B200 (BASELINE.json metric: MoE-layer
µs/block and expert-weight HBM GB/s vs vanilla top-k, unique experts loaded).

Workload (BASELINE.json configs[1]): LLaDA-MoE-7B-shaped layer, M=64 experts,
top-8, hidden d=2048, SwiGLU expert width F=1024 (not fixed by the reference;
stated), block N=32 tokens, softmax router, DES-Vote beta=0.4 (M_core=25).
Random-init bf16 weights; synthetic hidden states X = rho*b + (1-rho)*eps
(rho=0.3). One step = one block through the whole layer: router GEMM ->
activation/top-K -> DES coreset -> constrained re-route -> permutation ->
grouped SwiGLU expert FFN -> combine.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c3|c4] [--block N]

`value` = device-timed µs/block of the DES-Vote layer (inputs resident in HBM,
CUDA events on the layer's stream); consecutive blocks run through different
layers of a rotated set with distinct weights (>= 1 GiB of experts), as in a
real stack, so every expert weight a block streams comes from HBM;
`value_l2_flushed` repeats the measurement with a 256 MiB L2 flush before
every block. `e2e` = the same through the host-buffer C-ABI entry
(desmoe_layer_forward_host: the caller's pinned X copied in inside the layer
graph, layer, fp32 Y written into the caller's pinned memory, return once it
is visible), timed with the host's steady_clock around each C call
(tools/e2e/libe2etimer.so); `e2e.cuda_event_value` is the same call bracketed
by CUDA events on the stream.
`--impl reference` times the reference library's own CPU layer
(oracle/_ref: des_run + moe_forward with its linear dim x dim experts) on the
host cores.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: experts, top_k, hidden, ffn, block, beta, rho, description
    "c1": dict(experts=64, top_k=8, hidden=512, ffn=512, block=32, beta=0.4, rho=0.3,
               desc="tiny synthetic MoE layer (proj/tests shape)"),
    "c2": dict(experts=64, top_k=8, hidden=2048, ffn=1024, block=32, beta=0.4, rho=0.3,
               desc="LLaDA-MoE-7B-A1B-shaped layer"),
    "c3": dict(experts=256, top_k=8, hidden=2048, ffn=512, block=32, beta=0.15, rho=0.3,
               desc="LLaDA2.0-mini-shaped layer"),
    "c4": dict(experts=128, top_k=8, hidden=2048, ffn=768, block=32, beta=0.3, rho=0.3,
               desc="Qwen3-30B-A3B-shaped layer"),
}
METRIC = "DES MoE-layer µs/block and expert-weight HBM GB/s vs vanilla top-k"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


SPIN_CYCLES = 50_000  # ~25 µs at 1.9 GHz


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def spawn_ranks(gpus):
    """`bench.py --gpus N` without a launcher: run N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and return its exit status."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        raise SystemExit(rc)


def run_reference(args, cfg):
    """Reference arm: the reference's own CPU layer (oracle/_ref)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Ref
    from paper_2602_00879_b200 import synth
    import numpy as np
    ref = Ref()
    threads = os.cpu_count() or 1
    n, m, k, d = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"]
    vals = []
    u = 0
    for i in range(args.warmup + args.steps):
        x = synth.gen_trace_block(m, n, 42, rho=cfg["rho"], block_index=i)
        sec, u = ref.time_layer(x, k, "vote", beta=cfg["beta"], dim=d, reps=1, threads=threads,
                                ffn_tokens=args.ref_ffn_tokens)
        if i >= args.warmup:
            vals.append(sec * 1e6)
    v = float(np.mean(vals))
    sample = (f"per step: {threads} threads x 1 block each; des_run(vote beta={cfg['beta']}) on "
              f"all {n} tokens + moe_forward (reference linear {d}x{d} fp64 experts) on "
              f"{args.ref_ffn_tokens or n} tokens scaled to {n}; gen_trace shared_bias rho="
              f"{cfg['rho']} logits")
    line = {"metric": METRIC, "value": round(v, 3), "unit": "us/block", "n_gpus": max(ws, args.gpus),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v / 1e3, 6),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, "vote"),
            "cpu_baseline": {"value": round(v, 3), "unit": "us/block", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "us/block", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "unique_experts": u}
    print(json.dumps(line), flush=True)


def config_dict(cfg, strategy, ws=1):
    return {"workload": f"{cfg['desc']}: M={cfg['experts']} experts top-{cfg['top_k']}, "
                        f"d={cfg['hidden']}, SwiGLU F={cfg['ffn']}, block N={cfg['block']}, "
                        f"DES-Vote beta={cfg['beta']}",
            "experts": cfg["experts"], "top_k": cfg["top_k"], "hidden": cfg["hidden"],
            "ffn": cfg["ffn"], "block_size": cfg["block"], "strategy": strategy,
            "vote_beta": cfg["beta"], "activation": "softmax", "rho": cfg["rho"],
            "l2": "not flushed: each block runs the next of several layers with distinct "
                  "weights (>= 1 GiB of experts rotated; every streamed expert weight comes "
                  "from HBM); value_l2_flushed repeats vanilla/vote with a 256 MiB L2 flush "
                  "before every block",
            "parallelism": f"ep{ws}" + (" (experts sharded in contiguous ranges; router and "
                                        "routing replicated; slot rows pushed over NVLink "
                                        "peer memory)" if ws > 1 else "")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--block", type=int, default=0, help="override block size N")
    ap.add_argument("--ref-ffn-tokens", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layers", type=int, default=0,
                    help="distinct layers rotated per block (default: >= 1 GiB of experts)")
    ap.add_argument("--strategies", default="vanilla,seq3,seq2,vote",
                    help="comma list; vote and vanilla are always timed")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.block:
        cfg["block"] = args.block
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        # (the driver may also launch it that way itself)
        return spawn_ranks(args.gpus)
    ws = dist_env()[0]
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")

    import ctypes as C
    import numpy as np
    import torch
    from paper_2602_00879_b200 import _lib, ep, synth
    from paper_2602_00879_b200.dessim import _ptr
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

    ws, rank, local = dist_env()
    # DESMOE_EP_SAME_DEVICE=1: every rank on cuda:0 with a gloo group — a
    # functional check of the multi-process IPC path on a 1-GPU box (the
    # processes time-share the GPU, so its timings mean nothing)
    same_dev = os.environ.get("DESMOE_EP_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m, k, d, f = cfg["block"], cfg["experts"], cfg["top_k"], cfg["hidden"], cfg["ffn"]
    # expert parallelism: rank r owns a contiguous expert range; router and
    # routing are replicated, so every rank sees the same weights and tokens
    lo, hi = ep.partition(m, ws)[rank]
    lc = LayerConfig(m, k, d, f, strategy="vote", seq_k=3, vote_beta=cfg["beta"])
    # A block runs through the next of `nl` layers with distinct weights
    # (rotation as in a real stack): every expert weight it streams was last
    # touched nl-1 blocks (>= 0.9 GB of streaming) ago, so it comes from HBM
    # without flushing L2 between blocks. The flushed variant is timed too.
    bytes_per_expert = 3 * d * f * 2
    nl = max(4, min(16, -(-(1 << 30) // (m * bytes_per_expert))))
    if args.layers:
        nl = args.layers
    layers = []
    for li in range(nl):
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1000 + 17 * li, lo=lo, hi=hi)
        wr = synth.router_weights(m, d, seed=2000 + 17 * li)
        layers.append(DesMoeLayer(lc, wr, wg, wu, wd, expert_range=(lo, hi), own_context=True))
        del wg, wu, wd
        if ws > 1:
            ep.connect_distributed(layers[-1].experts)
    torch.cuda.empty_cache()
    if ws > 1:
        torch.distributed.barrier()
    L = _lib.lib()
    total = args.warmup + args.steps
    xs = [synth.hidden_states(n, d, seed=10_000 + i, rho=cfg["rho"])
          for i in range(total)]
    y = torch.empty((n, d), dtype=torch.float32, device="cuda")
    x_ins = [torch.empty((n, d), dtype=torch.bfloat16, device="cuda") for _ in layers]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    ph = (C.c_float * 8)()

    def set_prof(on):
        for lay in layers:
            L.desmoe_set_profiling(lay.ctx.h, on)

    def run(strategy, steps_list, record=True, phases=True, l2_flush=False):
        times, ph_list, us = [], [], []
        lc.seq_k = 3 if strategy != "seq2" else 2
        strat = "seq" if strategy.startswith("seq") else strategy
        for i, x in steps_list:
            layer = layers[i % nl]
            x_in = x_ins[i % nl]
            x_in.copy_(x)  # the layer's static input buffer (graph replay)
            if l2_flush:
                flush.fill_(i & 0xFF)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            # a ~25 µs spin kernel ahead of the start event keeps the stream
            # busy while the host enqueues the layer, so the events bracket
            # device work only (no host launch gap inside the timed interval)
            torch.cuda._sleep(SPIN_CYCLES)
            e0.record(stream)
            layer.forward(x_in, y, strategy=strat)
            e1.record(stream)
            e1.synchronize()
            if record:
                times.append(e0.elapsed_time(e1) * 1e3)
                if phases:
                    cnt = L.desmoe_get_phase_ms(layer.ctx.h, ph, 8)
                    if cnt < 0 or cnt > 8:
                        raise RuntimeError(L.desmoe_last_error().decode())
                    ph_list.append([ph[j] * 1e3 for j in range(cnt)])
                us.append(layer.stats.cpu().numpy().copy())
        return times, ph_list, us

    steps = list(enumerate(xs))
    warm, timed = steps[: args.warmup], steps[args.warmup:]
    results = {}
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
        wanted = [s for s in args.strategies.split(",") if s]
        order = [s for s in ("vanilla", "seq3", "seq2", "vote")
                 if s in wanted or s in ("vanilla", "vote")]
        for strategy in order:
            # timed pass: only the outer events (no event nodes between kernels,
            # so the programmatic launches overlap exactly as in production)
            set_prof(0)
            run(strategy, warm, record=False)
            if strategy == "vote":
                if ws > 1:
                    torch.distributed.barrier()
                torch.cuda.synchronize()
            t, _, s = run(strategy, timed, phases=False)
            torch.cuda.synchronize()
            # phase pass: CUDA events between the layer's kernels (roofline)
            set_prof(1)
            run(strategy, warm[:nl], record=False)
            _, p, _ = run(strategy, timed)
            results[strategy] = (np.array(t), np.array(p), np.array(s))
        # the same with L2 flushed by a 256 MiB write before every block
        set_prof(0)
        flushed = {}
        for strategy in ("vanilla", "vote"):
            run(strategy, warm, record=False, l2_flush=True)
            if ws > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            tf, _, _ = run(strategy, timed, phases=False, l2_flush=True)
            flushed[strategy] = float(np.mean(tf))
    clocks = clk.summary()
    set_prof(0)
    run("vote", warm[:1], record=False)
    launches = L.desmoe_last_launch_count(layers[0].ctx.h)

    # e2e: host buffers through the C ABI's desmoe_layer_forward_host — the
    # call a C/C++ caller of the drop-in makes (include/desmoe.h), here through
    # ctypes with its arguments built once. Every step: the caller's pinned x
    # crosses the bus (in-graph ingress kernel), the layer runs, y (fp32) and
    # the stats are written into pinned host memory, the call returns once the
    # layer's completion word says they are visible.
    xh = [x.cpu().pin_memory() for _, x in timed]
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    sh = torch.empty(4, dtype=torch.int32).pin_memory()
    rc_vote = lc.route_cfg("vote")
    sp = C.c_void_p(stream.cuda_stream)

    def host_call(layer, x):
        r = L.desmoe_layer_forward_host(layer.ctx.h, layer.experts.h, layer.w_router.data_ptr(),
                                        x.data_ptr(), n, C.byref(rc_vote), yh.data_ptr(),
                                        sh.data_ptr(), sp)
        if r:
            raise RuntimeError(L.desmoe_last_error().decode())

    xw = [x.cpu().pin_memory() for _, x in warm]
    for i, x in enumerate(xw):
        host_call(layers[i % nl], x)
    # (1) CUDA events on the stream around the call (the event after the call
    # is submitted only once the host holds the result, so it adds the
    # stream's submission latency)
    e2e_ev = []
    for i, x in enumerate(xh):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        host_call(layers[i % nl], x)
        e1.record(stream)
        e1.synchronize()
        e2e_ev.append(e0.elapsed_time(e1) * 1e3)
    # (2) the headline: host clock (steady_clock, in C) around each C-ABI call
    # (tools/e2e/libe2etimer.so), the latency a C/C++ caller of the drop-in sees
    e2e_kind = "host steady_clock around each desmoe_layer_forward_host call (C)"
    try:
        T = C.CDLL(os.path.join(ROOT, "tools", "e2e", "libe2etimer.so"))
    except OSError as exc:
        raise SystemExit(f"tools/e2e/libe2etimer.so missing ({exc}): run __graft_entry__.build()")
    ctx_arr = (C.c_void_p * nl)(*[lay.ctx.h.value for lay in layers])
    ex_arr = (C.c_void_p * nl)(*[lay.experts.h.value for lay in layers])
    wr_arr = (C.c_void_p * nl)(*[lay.w_router.data_ptr() for lay in layers])
    x_arr = (C.c_void_p * len(xh))(*[x.data_ptr() for x in xh])
    outs = (C.c_double * len(xh))()
    T.e2e_time_host_calls.restype = C.c_int
    for _ in range(2):  # the first pass warms the call path; the second is kept
        r = T.e2e_time_host_calls(ctx_arr, ex_arr, wr_arr, nl, x_arr, len(xh), n, C.byref(rc_vote),
                                  C.c_void_p(yh.data_ptr()), C.c_void_p(sh.data_ptr()), sp,
                                  len(xh), outs)
        if r:
            raise RuntimeError(L.desmoe_last_error().decode())
    e2e = [outs[i] for i in range(len(xh))]
    e2e_us = float(np.mean(e2e))
    e2e_event_us = float(np.mean(e2e_ev))

    # max over ranks (µs per block for the timed steps)
    t_vote, p_vote, s_vote = results["vote"]
    tot_us = float(t_vote.sum())
    if ws > 1:
        tt = torch.tensor([tot_us, e2e_us * len(e2e), flushed["vanilla"], flushed["vote"],
                           e2e_event_us],
                          dtype=torch.float64, device="cpu" if same_dev else "cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        tot_us, e2e_tot = float(tt[0]), float(tt[1])
        flushed = {"vanilla": float(tt[2]), "vote": float(tt[3])}
        e2e_event_us = float(tt[4])
        e2e_us = e2e_tot / len(e2e)
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    # every rank serves the same block (expert parallel, strong scaling):
    # µs/block = the slowest rank's time per step
    value = tot_us / args.steps
    peak, peak_kind = measured_peaks()
    wbytes_per_expert = 3 * d * f * 2

    def summarize(name):
        t, p, s = results[name]
        names = (["router_and_routing", "expert_ffn", "combine"] if p.shape[1] == 3
                 else ["router", "routing", "expert_ffn", "combine"])
        ffn = p[:, -2]
        u = s[:, 0].astype(float)
        u_own = s[:, 3].astype(float)  # experts streamed by this rank (= U on 1 GPU)
        gbps = (u_own * wbytes_per_expert) / (ffn * 1e-6) / 1e9
        return {"us_per_block": round(float(t.mean()), 3),
                "us_median": round(float(np.median(t)), 3),
                "unique_experts": round(float(u.mean()), 2),
                "experts_streamed_rank0": round(float(u_own.mean()), 2),
                "coreset": round(float(s[:, 1].mean()), 2),
                "expert_weight_GBps": round(float(gbps.mean()), 1),
                "phase_us": {nm: round(float(p[:, j].mean()), 2) for j, nm in enumerate(names)}}

    summ = {nm: summarize(nm) for nm in results}
    v, van = summ["vote"], summ["vanilla"]
    ffn_us = v["phase_us"]["expert_ffn"]
    achieved = v["experts_streamed_rank0"] * wbytes_per_expert / (ffn_us * 1e-6) / 1e9
    traffic, traffic_src = None, None
    if ws == 1 and not args.block:
        # DRAM bytes of this kernel on this workload from the ncu --set full
        # capture of the CURRENT profile tag (profiles/LATEST, written with the
        # captures by tools/ncu_capture.sh -> tools/ncu_summary.py); a missing
        # capture for that tag is reported, never silently replaced by an
        # older one
        try:
            tag = open(os.path.join(ROOT, "profiles", "LATEST")).read().split()[0]
        except OSError:
            tag = None
        cap = os.path.join(ROOT, "profiles", f"ncu_{args.config}_{tag}.json")
        if tag and os.path.exists(cap):
            traffic = json.load(open(cap)).get("ffn_dram_bytes_per_block")
            traffic_src = os.path.relpath(cap, ROOT)
        else:
            traffic_src = f"no capture for profile tag {tag!r} (profiles/LATEST)"
            print(f"bench.py: roofline.traffic unavailable: {traffic_src}", file=sys.stderr)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "us/block", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value / 1e3, 6),
        "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, rho-correlated hidden states)",
        "config": config_dict(cfg, "vote", ws),
        "latency_reduction_vs_vanilla": round(1.0 - v["us_per_block"] / van["us_per_block"], 4),
        "layers_rotated": nl,
        "value_l2_flushed": round(flushed["vote"], 3),
        "vanilla_l2_flushed": round(flushed["vanilla"], 3),
        "latency_reduction_vs_vanilla_l2_flushed": round(1.0 - flushed["vote"] / flushed["vanilla"], 4),
        "unique_expert_reduction_vs_vanilla": round(
            1.0 - v["unique_experts"] / van["unique_experts"], 4),
        "strategies": summ,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "ffn_persistent_kernel (permute + gather + gate/up + down), "
                               "CUDA events around its launch in the phase pass",
                     "algorithmic_bytes": "U*3*d*F*2 expert-weight bytes per block",
                     "peak_kind": peak_kind},
        "e2e": {"value": round(e2e_us, 3), "unit": "us/block",
                "h2d_bytes_per_step": n * d * 2, "d2h_bytes_per_step": n * d * 4 + 16,
                "timer": e2e_kind,
                "median": round(float(np.median(e2e)), 3),
                "cuda_event_value": round(e2e_event_us, 3),
                "entry": "desmoe_layer_forward_host (C ABI, include/desmoe.h): pinned x in, fp32 "
                         "y + stats out, returns when they are visible in host memory"},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and ws == 1:
        try:
            from oracle.oracle import Ref
            ref = Ref()
            threads = os.cpu_count() or 1
            x0 = synth.gen_trace_block(m, n, 42, rho=cfg["rho"])
            sec, _u = ref.time_layer(x0, k, "vote", beta=cfg["beta"], dim=d, reps=1,
                                     threads=threads)
            # single-block latency on one thread (the reference library is
            # single-threaded by design); moe_forward on 4 tokens, scaled to N
            sec1, _u = ref.time_layer(x0, k, "vote", beta=cfg["beta"], dim=d, reps=1,
                                      threads=1, ffn_tokens=min(4, n))
            line["cpu_baseline"] = {
                "value": round(sec * 1e6, 1), "unit": "us/block", "cores": threads,
                "kind": "reference",
                "latency_1t_us": round(sec1 * 1e6, 1),
                "sample": f"1 step: {threads} threads x 1 block; reference des_run(vote) + "
                          f"moe_forward with its linear {d}x{d} fp64 experts (the reference has "
                          f"no SwiGLU expert), gen_trace shared_bias logits"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "us/block", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
