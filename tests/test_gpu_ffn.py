"""GPU parity of the permutation (K3), router GEMM (K1), expert FFN (K4) and
the whole layer through the C ABI.

Tolerances (stated per north_star "within a stated bf16/fp32 tolerance"):
  * permutation, unique experts, per-expert counts: exact;
  * router logits vs an fp64 GEMM of the same bf16 values: |err| <= 1e-4;
  * linear experts (the reference's ExpertBank map) vs the reference's
    moe_forward on the same bf16-rounded values: |err| <= 1e-4 * max|y|
    (fp32 tensor-core accumulation);
  * SwiGLU experts vs the C restatement (fp64 sums, H rounded to bf16):
    max |err| <= 4e-3 * max|y| and mean |err| <= 4e-4 * max|y| (H's bf16
    rounding may differ by one ulp where the GPU's fp32 accumulation order
    moves G or U across a rounding boundary; observed max 5e-4);
  * routing IDs computed from the GPU's own logits: identical to the
    reference library fed those logits.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Route, bf16_round
from paper_2602_00879_b200 import _lib
from paper_2602_00879_b200 import dessim as ds
from paper_2602_00879_b200 import synth
from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

pytestmark = pytest.mark.gpu


def bf16(a):
    return torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16).cuda()


def route_arrays(r: Route):
    return r.idx, r.gate, r.cnt


def test_permute_matches_oracle(ref, port):
    import ctypes as C
    for seed in range(20):
        m, n, k = [(64, 32, 8), (256, 64, 8), (128, 256, 8), (16, 5, 4)][seed % 4]
        x = synth.gen_trace_block(m, n, 42 + seed, rho=0.3)
        _, r = ref.des_run(x, k, "vote", beta=0.3)
        want = port.permute(r, m)
        ctx = ds._Ctx.get(n, m, k)
        di = torch.as_tensor(r.idx, device="cuda")
        dc = torch.as_tensor(r.cnt, device="cuda")
        count = torch.empty(m, dtype=torch.int32, device="cuda")
        offset = torch.empty(m, dtype=torch.int32, device="cuda")
        slot_of = torch.empty((n, k), dtype=torch.int32, device="cuda")
        slot_token = torch.full((n * k,), -1, dtype=torch.int32, device="cuda")
        active = torch.empty(m, dtype=torch.int32, device="cuda")
        na = torch.empty(1, dtype=torch.int32, device="cuda")
        _lib.check(_lib.lib().desmoe_permute(ctx.h, ds._ptr(di), ds._ptr(dc), n, k, m,
                                             ds._ptr(count), ds._ptr(offset), ds._ptr(slot_of),
                                             ds._ptr(slot_token), ds._ptr(active), ds._ptr(na),
                                             ds._stream()))
        torch.cuda.synchronize()
        assert np.array_equal(count.cpu().numpy(), want["count"])
        assert np.array_equal(offset.cpu().numpy(), want["offset"])
        assert np.array_equal(slot_of.cpu().numpy(), want["slot_of"])
        tot = int(r.cnt.sum())
        assert np.array_equal(slot_token.cpu().numpy()[:tot], want["slot_token"])
        assert np.array_equal(active[: int(na.item())].cpu().numpy(), want["active"])
        u, total, per = ref.moe_latency(r, m)
        assert int(na.item()) == u and np.array_equal(count.cpu().numpy(), per)


@pytest.mark.parametrize("m,dim,n,k", [(16, 128, 5, 8), (8, 256, 32, 4), (64, 512, 32, 8)])
def test_linear_experts_match_moe_forward(ref, m, dim, n, k):
    w, xin = ref.make_expert_bank(m, dim, n, 7)
    wb = bf16_round(w.astype(np.float32)).astype(np.float64)
    xb = bf16_round(xin.astype(np.float32)).astype(np.float64)
    r = ref.topk_route(synth.random_block(n, m, 7), k)
    want = ref.moe_forward(r, wb, xb)
    ex = ds.ExpertWeights.linear(bf16(wb))
    got = ds.expert_ffn(ex, bf16(xb), *route_arrays(r)).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max()


def test_moe_forward_facade(ref):
    """ds.moe_forward on the reference bank at the tests' tiny dims (padded)."""
    cfg = ds.PoolConfig(16, 8, hidden_dim=6)
    bank = ds.make_expert_bank(cfg, 5, 7)
    a = ds.topk_route(ds.activate(ds.make_router_block(5, 16, synth.random_block(5, 16, 7)), cfg), 8)
    y = ds.moe_forward(a, bank)
    w, xin = ref.make_expert_bank(16, 6, 5, 7)
    r = ref.topk_route(synth.random_block(5, 16, 7), 8)
    want = ref.moe_forward(r, w, xin)
    assert np.abs(y - want).max() <= 2e-2 * np.abs(want).max()  # bf16 weights/inputs


# BASELINE configs: C1 M=64 d=512; C2 M=64 d=2048 F=1024 N=32;
# C3 M=256 d=2048 F=512 N=8-256; C4 M=128 d=2048 F=768
BETA = {64: 0.4, 128: 0.3, 256: 0.15, 512: 0.075}


@pytest.mark.parametrize("m,d,f,n,strategy", [
    (16, 256, 256, 16, "vanilla"),
    (64, 512, 512, 32, "vote"),       # C1
    (64, 2048, 1024, 32, "vote"),     # C2 (the bench workload)
    (64, 2048, 1024, 32, "seq"),      # C2 DES-Seq
    (64, 2048, 1024, 32, "vanilla"),  # C2 vanilla: routed mode with pair units
    (256, 2048, 512, 32, "vote"),     # C3 N=32 (Table 1 LLaDA2.0-mini point)
    (256, 2048, 512, 8, "vote"),      # C3 N=8
    (256, 1024, 512, 64, "seq"),
    (128, 2048, 768, 32, "vote"),     # C4
    (128, 2048, 768, 32, "vanilla"),  # C4 vanilla
    (128, 512, 768, 256, "vote"),
    (256, 2048, 512, 256, "vote"),    # token-split router GEMM at the C3 shape
    # outside the front kernel's envelope (M > 256, d not a multiple of 512):
    # split-K router GEMM + single-CTA routing kernels
    (512, 1024, 256, 32, "vote"),
    (512, 1024, 256, 64, "vanilla"),
    (64, 640, 256, 32, "vote"),
    (64, 640, 256, 32, "seq"),
    (64, 640, 256, 32, "vanilla"),
    (256, 1280, 512, 32, "vanilla"),
])
def test_swiglu_layer_matches_oracle(ref, port, m, d, f, n, strategy):
    swiglu_case(ref, port, m, d, f, n, strategy)


def swiglu_case(ref, port, m, d, f, n, strategy, rho=0.3):
    """Layer output vs the C restatement; returns the reference route."""
    torch.manual_seed(0)
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=11)
    wr = synth.router_weights(m, d, seed=12)
    x = synth.hidden_states(n, d, seed=13, rho=rho)
    beta = BETA.get(m, 0.4)
    cfg = LayerConfig(m, 8, d, f, strategy=strategy, seq_k=3, vote_beta=beta)
    layer = DesMoeLayer(cfg, wr, wg, wu, wd)
    y = layer.forward(x)
    torch.cuda.synchronize()
    layer.check()
    # 1. router logits (the ones the layer routed with) vs fp64 GEMM of the same
    #    bf16 values; the standalone router entry point agrees to fp32 rounding
    lg = layer.last_logits(n).cpu().numpy().astype(np.float64)
    want_logits = x.float().cpu().numpy().astype(np.float64) @ wr.float().cpu().numpy().astype(np.float64).T
    assert np.abs(lg - want_logits).max() <= 1e-4
    logits = torch.empty((n, m), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().desmoe_router_logits(layer.ctx.h, ds._ptr(x), ds._ptr(wr), n, m, d,
                                               ds._ptr(logits), ds._stream()))
    torch.cuda.synchronize()
    assert np.abs(logits.cpu().numpy() - want_logits).max() <= 1e-4
    # 2. routing from the GPU's logits == reference fed the same logits
    if strategy == "vanilla":
        r = ref.topk_route(lg, 8)
        mem = np.unique(r.idx[r.idx >= 0])
    else:
        mem, r = ref.des_run(lg, 8, strategy, seq_k=3, beta=beta)
    stats = layer.stats.cpu().numpy()
    u, total, _ = ref.moe_latency(r, m)
    assert stats[0] == u and stats[2] == total
    if strategy != "vanilla":
        assert stats[1] == len(mem)
    # 3. layer output vs the restated SwiGLU FFN on the reference routing
    want = port.moe_ffn(r, x.float().cpu().numpy(), wg.float().cpu().numpy(),
                        wu.float().cpu().numpy(), wd.float().cpu().numpy(), threads=8)
    got = y.cpu().numpy()
    scale = np.abs(want).max()
    err_max = np.abs(got - want).max() / scale
    err_mean = np.abs(got - want).mean() / scale
    print(f"swiglu m={m} d={d} f={f} n={n} {strategy}: max|err|/max|y| = {err_max:.2e}, "
          f"mean = {err_mean:.2e}")
    assert err_max <= 4e-3, err_max
    assert err_mean <= 4e-4, err_mean
    return r


@pytest.mark.parametrize("m,d,f,n,strategy", [
    (64, 512, 512, 32, "vote"),       # dense mode
    (16, 256, 256, 16, "vanilla"),    # dense mode, vanilla
    (64, 512, 512, 48, "vanilla"),    # routed mode
])
def test_pair_units_without_split(ref, port, monkeypatch, m, d, f, n, strategy):
    """Every phase-A / phase-B unit a pair (no single-tile tail), at shapes
    where the default split would leave none."""
    monkeypatch.setenv("DESMOE_FFN_SPLIT", "0")
    monkeypatch.setenv("DESMOE_FFN_SPLITA", "0")
    swiglu_case(ref, port, m, d, f, n, strategy)


def test_routed_pairs_over_64_tokens_per_expert(ref, port, monkeypatch):
    """Routed-mode pair units (vanilla, 16 < N <= 128, every unit a pair) where
    some expert receives more than 64 tokens: the pair's second tile then
    spans TMEM columns 384-511 of accumulator buffer 1."""
    monkeypatch.setenv("DESMOE_FFN_SPLIT", "0")
    monkeypatch.setenv("DESMOE_FFN_SPLITA", "0")
    r = swiglu_case(ref, port, 64, 512, 512, 128, "vanilla", rho=0.97)
    _, _, per = ref.moe_latency(r, 64)
    assert per.max() > 64, per.max()


def test_rejected_call_leaves_no_stale_handoff(ref, port):
    """A block the expert FFN cannot plan (N=256 with K=12: its prologue
    tables exceed the plan) is rejected BEFORE the front kernel launches, so a
    following valid call (graphs off: eager launches) never consumes stale
    published words from the rejected one."""
    from paper_2602_00879_b200._lib import DesmoeError
    m, d, f = 64, 512, 512
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=61)
    wr = synth.router_weights(m, d, seed=62)
    layer = DesMoeLayer(LayerConfig(m, 12, d, f, strategy="vote", vote_beta=0.4), wr, wg, wu, wd,
                        own_context=True)
    _lib.check(_lib.lib().desmoe_set_graphs(layer.ctx.h, 0))
    bad = synth.hidden_states(256, d, seed=63, rho=0.3)
    with pytest.raises((ValueError, DesmoeError), match="expert FFN"):
        layer.forward(bad)
    for call in range(3):
        x = synth.hidden_states(32, d, seed=64 + call, rho=0.3)
        y = layer.forward(x)
        torch.cuda.synchronize()
        layer.check()
        lg = layer.last_logits(32).double().cpu().numpy()
        mem, r = ref.des_run(lg, 12, "vote", beta=0.4)
        idx, gate, cnt, members = layer.last_route(32)
        assert members == mem.tolist()
        np.testing.assert_array_equal(idx, r.idx)
        want = port.moe_ffn(r, x.float().cpu().numpy(), wg.float().cpu().numpy(),
                            wu.float().cpu().numpy(), wd.float().cpu().numpy(), threads=8)
        err = np.abs(y.cpu().numpy() - want).max() / np.abs(want).max()
        assert err <= 4e-3, (call, err)


def test_layer_host_entry_matches_device_entry():
    m, d, f, n = 64, 512, 512, 32
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=21)
    wr = synth.router_weights(m, d, seed=22)
    x = synth.hidden_states(n, d, seed=23)
    layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy="vote", vote_beta=0.4), wr, wg, wu, wd)
    y_dev = layer.forward(x)
    torch.cuda.synchronize()
    xh = x.cpu().pin_memory()
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    sh = torch.empty(4, dtype=torch.int32).pin_memory()
    layer.forward_host(xh, yh, sh)
    assert torch.equal(yh, y_dev.cpu())  # deterministic: bit-identical
    assert sh[0].item() <= 25
    # pageable buffers: the entry copies y back instead of writing it in place
    yp = torch.empty((n, d), dtype=torch.float32)
    sp = torch.empty(4, dtype=torch.int32)
    layer.forward_host(x.cpu(), yp, sp)
    assert torch.equal(yp, y_dev.cpu()) and torch.equal(sp, sh)
    # a non-finite input is reported through the host-mapped check word
    xb = x.cpu().clone()
    xb[3, 5] = float("nan")
    with pytest.raises(ValueError, match="non-finite logit"):
        layer.forward_host(xb.pin_memory(), yh, sh)
    layer.forward_host(xh, yh, sh)  # the flag was cleared
    assert torch.equal(yh, y_dev.cpu())


def test_host_entry_rotating_buffers(monkeypatch):
    """Pinned x buffers that change every call (the in-graph ingress reads
    the address from a host-mapped word: no re-capture), interleaved with
    device-entry calls on the same context, the memcpy ingress
    (DESMOE_HOST_MEMCPY) and the stream-synchronising return
    (DESMOE_HOST_SYNC): every output equals the device entry's."""
    m, d, f, n = 64, 512, 512, 32
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=71)
    layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy="vote", vote_beta=0.4),
                        synth.router_weights(m, d, seed=72), wg, wu, wd, own_context=True)
    xs = [synth.hidden_states(n, d, seed=80 + i, rho=0.3) for i in range(6)]
    want = []
    for x in xs:
        want.append(layer.forward(x).cpu())
        torch.cuda.synchronize()
    xh = [x.cpu().pin_memory() for x in xs]
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    sh = torch.empty(4, dtype=torch.int32).pin_memory()
    for mode in ("", "DESMOE_HOST_MEMCPY", "DESMOE_HOST_SYNC"):
        if mode:
            monkeypatch.setenv(mode, "1")
        for rep in range(2):
            for i in range(len(xs)):
                layer.forward_host(xh[i], yh, sh)
                assert torch.equal(yh, want[i]), (mode, rep, i)
                if i % 3 == 0:  # a device-entry call in between (another graph)
                    assert torch.equal(layer.forward(xs[i]).cpu(), want[i])
        if mode:
            monkeypatch.delenv(mode)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["vote", "vanilla"])
def test_stack_equals_chained_layers(strategy):
    """desmoe_stack_forward (one graph, bf16 hand-over between layers) equals
    running the layers one by one with the output cast to bf16 in between."""
    import torch
    from paper_2602_00879_b200.layer import DesMoeLayer, DesMoeStack, LayerConfig
    m, d, f, n, k, L = 64, 512, 512, 32, 8, 3
    cfg = LayerConfig(m, k, d, f, strategy=strategy, vote_beta=0.4)
    params = [(synth.router_weights(m, d, seed=40 + l), *synth.swiglu_weights(m, d, f, seed=50 + l))
              for l in range(L)]
    stack = DesMoeStack(cfg, params)
    x = synth.hidden_states(n, d, seed=3, rho=0.3)
    y_stack = stack.forward(x).clone()
    stats = stack.stats.cpu().numpy()
    y_res = stack.forward(x, residual=True).clone()
    xin = x
    for l, (wr, wg, wu, wd) in enumerate(params):
        layer = DesMoeLayer(cfg, wr, wg, wu, wd, own_context=True)
        y = layer.forward(xin)
        torch.cuda.synchronize()
        assert stats[l].tolist() == layer.stats.cpu().tolist()
        xin = y.to(torch.bfloat16)
    assert torch.equal(y_stack, y)
    # residual stream: h + MoE(h) carried in bf16 between layers
    xin = x
    for l, (wr, wg, wu, wd) in enumerate(params):
        layer = DesMoeLayer(cfg, wr, wg, wu, wd, own_context=True)
        y = layer.forward(xin) + xin.float()
        xin = y.to(torch.bfloat16)
    assert torch.equal(y_res, y)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["vote", "seq"])
def test_stack_matches_oracle_chain(ref, port, strategy):
    """The stack path (desmoe_stack_forward, residual stream) layer by layer
    against CPU checkers on a 3-layer C3 shape (M=256, d=2048, SwiGLU F=512,
    N=32). Every layer l sees the GPU stack's own bf16 hand-over h_l (the
    stack's output equals chaining the layers one by one, bit for bit); on
    that h_l the checkers run router logits = fp64 GEMM of the bf16 values
    (Port.router_logits), routing = the reference's own des_run (oracle/_ref)
    and experts = the C restatement's SwiGLU (Port.moe_ffn). Per layer: unique
    experts / coreset / selections equal the reference's and h_l + MoE(h_l)
    agrees within the bf16 tolerance (SURVEY §8c parity plan 3). (A chain fed
    with its OWN outputs drifts by bf16 ulps per layer, which moves logit
    near-ties: that tests the arithmetic's chaos, not the kernels.)"""
    from paper_2602_00879_b200.layer import DesMoeStack
    m, d, f, n, k, L, beta = 256, 2048, 512, 32, 8, 3, 0.15
    cfg = LayerConfig(m, k, d, f, strategy=strategy, seq_k=3, vote_beta=beta)
    params = [(synth.router_weights(m, d, seed=90 + l), *synth.swiglu_weights(m, d, f, seed=95 + l))
              for l in range(L)]
    stack = DesMoeStack(cfg, params)
    x = synth.hidden_states(n, d, seed=11, rho=0.3)
    y_stack = stack.forward(x, residual=True).clone()
    stats = stack.stats.cpu().numpy()
    h = x
    for l, (wr, wg, wu, wd) in enumerate(params):
        layer = DesMoeLayer(cfg, wr, wg, wu, wd, own_context=True)
        y = layer.forward(h) + h.float()
        torch.cuda.synchronize()
        assert layer.stats.cpu().tolist()[:3] == stats[l].tolist()[:3]
        hn = h.float().cpu().numpy()
        logits = port.router_logits(hn, wr.float().cpu().numpy())
        mem, route = ref.des_run(logits, k, strategy, seq_k=3, beta=beta)
        u, total, _ = ref.moe_latency(route, m)
        assert stats[l].tolist()[:3] == [u, len(mem), total], (l, stats[l], u, len(mem), total)
        moe = port.moe_ffn(route, hn, wg.float().cpu().numpy(), wu.float().cpu().numpy(),
                           wd.float().cpu().numpy(), threads=8)
        want = moe + hn
        got = y.cpu().numpy()
        err = float(np.abs(got - want).max() / np.abs(want).max())
        print(f"stack layer {l} ({strategy}) vs reference routing + C SwiGLU: max rel err {err:.2e}")
        assert err <= 4e-3, (l, err)
        h = y.to(torch.bfloat16)
    assert torch.equal(y_stack, y)


@pytest.mark.gpu
def test_layer_config_changes_take_effect():
    """LayerConfig is mutable (bench.py switches seq_k between DES-Seq k=3 and
    k=2 on one layer): every call must route with the current fields."""
    m, d, f, n = 64, 512, 512, 32
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=31)
    wr = synth.router_weights(m, d, seed=32)
    x = synth.hidden_states(n, d, seed=33, rho=0.3)
    cfg = LayerConfig(m, 8, d, f, strategy="seq", seq_k=3)
    layer = DesMoeLayer(cfg, wr, wg, wu, wd)
    layer.forward(x)
    torch.cuda.synchronize()
    core3 = int(layer.stats[1].item())
    cfg.seq_k = 1
    layer.forward(x)
    torch.cuda.synchronize()
    core1 = int(layer.stats[1].item())
    assert core1 < core3, (core1, core3)


@pytest.mark.gpu
def test_recreated_expert_bank_does_not_replay_stale_graph(ref):
    """Captured layer graphs are keyed on a per-handle id, not the handle's
    address: a bank destroyed and re-created (the allocator hands back the
    same address) with other shapes and another strategy must not replay the
    previous call's graph (seen as U = the previous coreset size)."""
    import gc
    for (m, d, f, strat) in [(256, 1536, 512, "vote"), (256, 1280, 512, "vanilla"),
                             (256, 1536, 512, "vanilla"), (256, 1280, 512, "vote")]:
        wg, wu, wd = synth.swiglu_weights(m, d, f, seed=1)
        wr = synth.router_weights(m, d, seed=2)
        layer = DesMoeLayer(LayerConfig(m, 8, d, f, strategy=strat, vote_beta=0.15), wr, wg, wu, wd)
        x = synth.hidden_states(32, d, seed=5, rho=0.3)
        for _ in range(2):
            layer.forward(x)
        torch.cuda.synchronize()
        lg = layer.last_logits(32).double().cpu().numpy()
        r = ref.topk_route(lg, 8) if strat == "vanilla" else ref.des_run(lg, 8, "vote", beta=0.15)[1]
        u, total, _ = ref.moe_latency(r, m)
        st = layer.stats.cpu().tolist()
        assert st[0] == u and st[2] == total, (m, d, strat, st, u, total)
        del layer, wg, wu, wd
        gc.collect()


@pytest.mark.gpu
@pytest.mark.parametrize("m,d,f,n,beta", [
    (64, 2048, 1024, 32, 0.4),    # C2
    (256, 2048, 512, 32, 0.15),   # C3 at N = 32 (dense)
    (128, 2048, 768, 16, 0.3),    # C4 shape, N = 16
])
def test_streamed_combine_matches_grid_wait(monkeypatch, m, d, f, n, beta):
    """The host-buffer entry's combine streams on per-(expert, d tile) tags
    the FFN releases after each phase-B unit's stores, instead of waiting for
    the FFN grid: over repeated calls with rotating inputs its y equals the
    device entry's (grid wait) bit for bit; forced on the device entry too
    (DESMOE_STREAM_COMBINE=1, a fresh context so the graph is re-captured)."""
    import torch
    from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig
    wg, wu, wd = synth.swiglu_weights(m, d, f, seed=5)
    wr = synth.router_weights(m, d, seed=6)
    cfg = LayerConfig(m, 8, d, f, strategy="vote", vote_beta=beta)
    layer = DesMoeLayer(cfg, wr, wg, wu, wd, own_context=True)
    xs = [synth.hidden_states(n, d, seed=90 + i, rho=0.3) for i in range(4)]
    want = []
    for x in xs:
        want.append(layer.forward(x).cpu())
        torch.cuda.synchronize()
    xh = [x.cpu().pin_memory() for x in xs]
    yh = torch.empty((n, d), dtype=torch.float32).pin_memory()
    for rep in range(5):
        for i in range(len(xs)):
            layer.forward_host(xh[i], yh)
            assert torch.equal(yh, want[i]), (rep, i)
    monkeypatch.setenv("DESMOE_STREAM_COMBINE", "1")
    forced = DesMoeLayer(cfg, wr, wg, wu, wd, own_context=True)
    for rep in range(3):
        for i, x in enumerate(xs):
            y = forced.forward(x)
            forced.check()
            assert torch.equal(y.cpu(), want[i]), (rep, i)
