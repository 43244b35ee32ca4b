"""Multi-process expert-parallel check (run under torchrun): every rank builds
its expert shard, wires the peers through the C ABI's IPC handle exchange
(ep.connect_distributed), runs several DES layer calls and compares its output
bit-for-bit with the full single-rank layer computed in the same process.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/ep_check.py
    (DESMOE_EP_SAME_DEVICE=1: all ranks on cuda:0 over gloo — IPC between
     processes on one GPU; they time-share it)
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_00879_b200 import ep, synth  # noqa: E402
from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig  # noqa: E402


def main():
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    same = os.environ.get("DESMOE_EP_SAME_DEVICE") == "1"
    dev = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    if same:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    # DESMOE_EP_SHAPE="m,d,f,n,beta" (default: 64 experts, d=512, F=512, N=32, 0.4)
    shape = os.environ.get("DESMOE_EP_SHAPE", "64,512,512,32,0.4").split(",")
    m, d, f, n = (int(v) for v in shape[:4])
    beta, k = float(shape[4]), 8
    res = {}
    for strategy in ("vote", "vanilla"):
        cfg = LayerConfig(m, k, d, f, strategy=strategy, vote_beta=beta)
        wr = synth.router_weights(m, d, seed=5)
        full = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=9), own_context=True)
        lo, hi = ep.partition(m, ws)[rank]
        mine = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=9, lo=lo, hi=hi),
                           expert_range=(lo, hi), own_context=True)
        ep.connect_distributed(mine.experts)
        dist.barrier()
        ok = True
        for call in range(3):
            x = synth.hidden_states(n, d, seed=100 + call, rho=0.3)
            y1 = full.forward(x).clone()
            y = mine.forward(x)
            torch.cuda.synchronize()
            mine.check()
            ok &= bool(torch.equal(y, y1))
        res[strategy] = ok
        dist.barrier()
    print(json.dumps({"rank": rank, "world": ws, "bit_identical": res}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(res.values()) else 1)


if __name__ == "__main__":
    main()
