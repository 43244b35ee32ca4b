"""Expert parallelism on one B200: G simulated ranks (each its own C-ABI
context, expert shard, slot buffer and arrival counter) wired by
ep.connect_local and run concurrently on G streams. Every rank's output must
be bit-identical to the single-rank layer (the combine sums the same fp32
slot rows in the same ascending-expert order), over several calls (the
two-epoch slot buffers alternate)."""
import pytest
import torch

from paper_2602_00879_b200 import ep, synth
from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy", ["vote", "vanilla"])
@pytest.mark.parametrize("m,d,f,n,beta", [
    (64, 512, 512, 32, 0.4),      # dense FFN mode (DES) / routed pairs (vanilla)
    (64, 512, 512, 128, 0.4),     # N > 64: routed mode for every strategy
    (128, 2048, 768, 32, 0.3),    # C4 (SDAR-30B / Qwen3-30B-A3B shape, BASELINE configs[3])
])
def test_ep_ranks_match_single_gpu(world, strategy, m, d, f, n, beta):
    k = 8
    cfg = LayerConfig(m, k, d, f, strategy=strategy, vote_beta=beta)
    wr = synth.router_weights(m, d, seed=5)
    full = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=9))
    ranks = []
    for lo, hi in ep.partition(m, world):
        shard = synth.swiglu_weights(m, d, f, seed=9, lo=lo, hi=hi)
        ranks.append(DesMoeLayer(cfg, wr, *shard, expert_range=(lo, hi), own_context=True))
    ep.connect_local([r.experts for r in ranks])
    streams = [torch.cuda.Stream() for _ in ranks]
    ys = [torch.empty((n, d), dtype=torch.float32, device="cuda") for _ in ranks]
    for call in range(4):
        x = synth.hidden_states(n, d, seed=100 + call, rho=0.3)
        y1 = full.forward(x)
        want_stats = full.stats.cpu().tolist()
        torch.cuda.synchronize()
        for r, layer in enumerate(ranks):
            streams[r].wait_stream(torch.cuda.current_stream())
            layer.forward(x, ys[r], stream=streams[r])
        torch.cuda.synchronize()
        owned = 0
        for r, layer in enumerate(ranks):
            layer.check()
            assert torch.equal(ys[r], y1), (call, r, (ys[r] - y1).abs().max().item())
            st = layer.stats.cpu().tolist()
            assert st[:3] == want_stats[:3]
            owned += st[3]
        assert owned == want_stats[0]  # every active expert streamed by exactly one rank


def test_ep_rank_without_work():
    """A rank whose experts receive no token still arrives (no hang)."""
    m, d, f, n, k = 64, 512, 512, 4, 2
    cfg = LayerConfig(m, k, d, f, strategy="vote", vote_beta=0.05)  # 3-expert coreset
    wr = synth.router_weights(m, d, seed=6)
    full = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=3))
    ranks = [DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=3, lo=lo, hi=hi),
                         expert_range=(lo, hi), own_context=True)
             for lo, hi in ep.partition(m, 8)]
    ep.connect_local([r.experts for r in ranks])
    x = synth.hidden_states(n, d, seed=1, rho=0.3)
    y1 = full.forward(x)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in ranks]
    ys = [torch.empty((n, d), dtype=torch.float32, device="cuda") for _ in ranks]
    for r, layer in enumerate(ranks):
        streams[r].wait_stream(torch.cuda.current_stream())
        layer.forward(x, ys[r], stream=streams[r])
    torch.cuda.synchronize()
    idle = 0
    for r, layer in enumerate(ranks):
        layer.check()
        assert torch.equal(ys[r], y1)
        idle += layer.stats.cpu().tolist()[3] == 0
    assert idle > 0


def test_ep_two_processes_ipc():
    """Two processes (torchrun) on the same GPU wired through the C ABI's IPC
    handle export/import — the multi-GPU code path with real cross-process
    peer mappings; outputs bit-identical to the full layer."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, DESMOE_EP_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={port}", os.path.join(root, "tools", "ep_check.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert r.stdout.count('"vote": true, "vanilla": true') == 2, r.stdout


def _run_ep_check(nproc, env_extra):
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = {key: v for key, v in os.environ.items() if key != "DESMOE_EP_SAME_DEVICE"}
    env.update(env_extra)
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
                           f"--master-port={port}", os.path.join(root, "tools", "ep_check.py")],
                          capture_output=True, text=True, timeout=900, env=env)


@pytest.mark.parametrize("shape", ["64,512,512,128,0.4", "128,2048,768,32,0.3"])
def test_ep_two_processes_routed_and_c4(shape):
    """The cross-process IPC path at N=128 (routed FFN mode, DES-Vote) and at
    the C4 shape (d=2048), two ranks time-sharing one GPU."""
    r = _run_ep_check(2, {"DESMOE_EP_SAME_DEVICE": "1", "DESMOE_EP_SHAPE": shape})
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert r.stdout.count('"vote": true, "vanilla": true') == 2, r.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs of one NVLink box")
@pytest.mark.parametrize("shape", ["64,512,512,32,0.4", "128,2048,768,32,0.3"])
def test_ep_across_devices(shape):
    """One rank per GPU (NCCL group for the handle all-gather, CUDA IPC peer
    mappings over NVLink): every rank's output bit-identical to the one-GPU
    layer."""
    world = min(torch.cuda.device_count(), 8)
    r = _run_ep_check(world, {"DESMOE_EP_SHAPE": shape})
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert r.stdout.count('"vote": true, "vanilla": true') == world, r.stdout


@pytest.mark.parametrize("strategy", ["vote", "vanilla"])
def test_ep_stack_matches_single_gpu(strategy):
    """desmoe_stack_forward with expert-parallel layers (SURVEY §8f row 1 +
    §8e): G = 2 simulated ranks, each a whole stack of expert shards (one
    graph per rank), every layer's shards wired across the ranks; each rank's
    residual-stream output equals the single-rank stack bit for bit."""
    from paper_2602_00879_b200.layer import DesMoeStack
    m, d, f, n, k, layers, world = 64, 512, 512, 32, 8, 3, 2
    cfg = LayerConfig(m, k, d, f, strategy=strategy, vote_beta=0.4)
    params = [(synth.router_weights(m, d, seed=70 + l), *synth.swiglu_weights(m, d, f, seed=80 + l))
              for l in range(layers)]
    full = DesMoeStack(cfg, params)
    stacks = []
    for lo, hi in ep.partition(m, world):
        shard = [(wr, *synth.swiglu_weights(m, d, f, seed=80 + l, lo=lo, hi=hi))
                 for l, (wr, *_rest) in enumerate(params)]
        stacks.append(DesMoeStack(cfg, shard, expert_range=(lo, hi)))
    for l in range(layers):
        ep.connect_local([s.experts[l] for s in stacks])
    streams = [torch.cuda.Stream() for _ in stacks]
    ys = [torch.empty((n, d), dtype=torch.float32, device="cuda") for _ in stacks]
    for call in range(3):
        x = synth.hidden_states(n, d, seed=300 + call, rho=0.3)
        want = full.forward(x, residual=True).clone()
        want_stats = full.stats.cpu()
        torch.cuda.synchronize()
        for r, s in enumerate(stacks):
            streams[r].wait_stream(torch.cuda.current_stream())
            s.forward(x, ys[r], stream=streams[r], residual=True)
        torch.cuda.synchronize()
        owned = torch.zeros(layers, dtype=torch.int64)
        for r, s in enumerate(stacks):
            assert torch.equal(ys[r], want), (call, r, (ys[r] - want).abs().max().item())
            st = s.stats.cpu()
            assert torch.equal(st[:, :3], want_stats[:, :3])
            owned += st[:, 3].long()
        assert torch.equal(owned, want_stats[:, 0].long())


def test_ep_peer_loss_reports_timeout_not_hang():
    """A rank whose peer never runs the call (a lost process): its arrival
    wait (ep_wait_kernel, 4 s bound) raises the exchange-timeout flag and the
    call fails with the C ABI's error instead of hanging the stream; the
    device stays usable for the next layer."""
    import time
    m, d, f, n, k = 64, 512, 512, 32, 8
    cfg = LayerConfig(m, k, d, f, strategy="vote", vote_beta=0.4)
    wr = synth.router_weights(m, d, seed=5)
    ranks = [DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=9, lo=lo, hi=hi),
                         expert_range=(lo, hi), own_context=True)
             for lo, hi in ep.partition(m, 2)]
    ep.connect_local([r.experts for r in ranks])
    x = synth.hidden_states(n, d, seed=7, rho=0.3)
    y = torch.empty((n, d), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t0 = time.monotonic()
    ranks[0].forward(x, y)  # rank 1 never issues this call
    with pytest.raises(RuntimeError, match="timed out"):
        ranks[0].check()
    waited = time.monotonic() - t0
    assert 3.5 < waited < 30, waited
    full = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=9))
    y1 = full.forward(x)
    full.check()
    assert torch.isfinite(y1).all()
