"""The fused front kernel (router GEMM + DES routing in one 8-CTA cluster) on
the layer path, against the UNMODIFIED reference library fed the GPU's own
fp32 logits: selected expert ids, coreset membership and token->expert
assignments must match exactly, gates bit for bit. Covers the kernel's shape
envelope (single token, ragged N, M not a multiple of 32, token-chunked
GEMM, M=256) and every routing variant it implements (vanilla, DES-Seq
k=1..K, DES-Vote with the coreset smaller / larger than K, sigmoid gates,
raw-logit votes)."""
import numpy as np
import pytest
import torch

from oracle.oracle import Ref
from paper_2602_00879_b200 import _lib, synth
from paper_2602_00879_b200.layer import DesMoeLayer, LayerConfig

pytestmark = pytest.mark.gpu

REF = None


def ref():
    global REF
    if REF is None:
        REF = Ref()
    return REF


def run_layer(m, k, n, d, strategy, seq_k=3, beta=0.4, act=_lib.SOFTMAX, seed=1, raw=False):
    f = 128
    cfg = LayerConfig(m, k, d, f, strategy=strategy, seq_k=seq_k, vote_beta=beta, activation=act)
    wr = synth.router_weights(m, d, seed=seed)
    layer = DesMoeLayer(cfg, wr, *synth.swiglu_weights(m, d, f, seed=seed + 1), own_context=True)
    x = synth.hidden_states(n, d, seed=seed + 2, rho=0.3)
    if raw:
        rc = cfg.route_cfg()
        rc.vote_source = _lib.VOTE_RAW_LOGITS
        import ctypes as C
        from paper_2602_00879_b200._lib import check, lib
        from paper_2602_00879_b200.dessim import _ptr, _stream
        y = torch.empty((n, d), dtype=torch.float32, device="cuda")
        check(lib().desmoe_layer_forward(layer.ctx.h, layer.experts.h, _ptr(layer.w_router),
                                         _ptr(x), n, C.byref(rc), _ptr(y), _ptr(layer.stats),
                                         _stream()))
    else:
        layer.forward(x)
    torch.cuda.synchronize()
    layer.check()
    logits = layer.last_logits(n).double().cpu().numpy()
    return layer, logits


def assert_route(gpu, want_idx, want_gate, want_cnt):
    idx, gate, cnt = gpu
    np.testing.assert_array_equal(cnt, want_cnt)
    for t in range(len(cnt)):
        c = cnt[t]
        np.testing.assert_array_equal(idx[t, :c], want_idx[t, :c])
        np.testing.assert_array_equal(gate[t, :c], want_gate[t, :c])


SHAPES = [  # m, k, n, d
    (64, 8, 32, 512),
    (64, 8, 1, 512),
    (64, 8, 13, 512),
    (40, 6, 29, 512),
    (256, 8, 64, 512),
    (128, 8, 160, 1024),   # N > 64: routed FFN mode
    (256, 8, 256, 512),    # token-chunked GEMM
    (16, 4, 200, 512),
]


@pytest.mark.parametrize("m,k,n,d", SHAPES)
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
def test_front_routing_matches_reference(m, k, n, d, strategy):
    beta = 0.4 if m <= 64 else 0.15
    layer, logits = run_layer(m, k, n, d, strategy, seq_k=min(3, k), beta=beta)
    idx, gate, cnt, members = layer.last_route(n)
    if strategy == "vanilla":
        want = ref().topk_route(logits, k)
    else:
        mem, want = ref().des_run(logits, k, strategy, seq_k=min(3, k), beta=beta)
        assert members == mem.tolist()
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)
    st = layer.stats.cpu().numpy()
    u, total, _ = ref().moe_latency(want, m)
    assert st[0] == u and st[2] == total


@pytest.mark.parametrize("seq_k", [1, 2, 8])
def test_front_seq_depths(seq_k):
    layer, logits = run_layer(64, 8, 32, 512, "seq", seq_k=seq_k, seed=5)
    idx, gate, cnt, members = layer.last_route(32)
    mem, want = ref().des_run(logits, 8, "seq", seq_k=seq_k)
    assert members == mem.tolist()
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)


def test_front_vote_coreset_smaller_than_k():
    # floor(0.05 * 64) = 3 < K = 8: every token takes all coreset members
    layer, logits = run_layer(64, 8, 32, 512, "vote", beta=0.05, seed=7)
    idx, gate, cnt, members = layer.last_route(32)
    mem, want = ref().des_run(logits, 8, "vote", beta=0.05)
    assert members == mem.tolist() and len(members) == 3
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)
    assert (cnt == 3).all()


@pytest.mark.parametrize("strategy", ["vanilla", "vote", "seq"])
def test_front_sigmoid_gates(strategy):
    layer, logits = run_layer(64, 8, 32, 512, strategy, act=_lib.SIGMOID, seed=11)
    idx, gate, cnt, members = layer.last_route(32)
    if strategy == "vanilla":
        want = ref().topk_route(logits, 8, act=1)
    else:
        mem, want = ref().des_run(logits, 8, strategy, seq_k=3, beta=0.4, act=1)
        assert members == mem.tolist()
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)


def test_front_raw_logit_votes():
    layer, logits = run_layer(64, 8, 32, 512, "vote", raw=True, seed=13)
    idx, gate, cnt, members = layer.last_route(32)
    mem, _votes = ref().vote_coreset(logits, 8, 0.4, raw=True)
    assert members == mem.tolist()
    want = ref().constrained_route(logits, 8, mem)
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)


def test_front_deterministic():
    """Same inputs, same outputs, bit for bit (no float atomics anywhere)."""
    m, k, n, d, f = 64, 8, 32, 512, 128
    cfg = LayerConfig(m, k, d, f, strategy="vote", vote_beta=0.4)
    layer = DesMoeLayer(cfg, synth.router_weights(m, d, seed=3),
                        *synth.swiglu_weights(m, d, f, seed=4), own_context=True)
    x = synth.hidden_states(n, d, seed=5, rho=0.3)
    ys = [layer.forward(x).clone() for _ in range(5)]
    for y in ys[1:]:
        assert torch.equal(y, ys[0])


@pytest.mark.parametrize("variant", ["0", "1", "2"])  # split-K, token split + multicast, token split
@pytest.mark.parametrize("m,k,n,d", [(64, 8, 32, 512), (256, 8, 128, 512), (40, 6, 13, 512)])
def test_front_gemm_variants(monkeypatch, variant, m, k, n, d):
    """Every router-GEMM variant of the front kernel (DESMOE_FRONT_TSPLIT):
    routes equal the reference's on the kernel's own logits, and the logits
    agree with an fp64 GEMM of the same bf16 inputs."""
    monkeypatch.setenv("DESMOE_FRONT_TSPLIT", variant)
    layer, logits = run_layer(m, k, n, d, "vote", beta=0.4 if m <= 64 else 0.15, seed=11)
    idx, gate, cnt, members = layer.last_route(n)
    mem, want = ref().des_run(logits, k, "vote", beta=0.4 if m <= 64 else 0.15)
    assert members == mem.tolist()
    assert_route((idx, gate, cnt), want.idx, want.gate, want.cnt)
    x = synth.hidden_states(n, d, seed=13, rho=0.3).double().cpu().numpy()
    w = layer.w_router.double().cpu().numpy()
    np.testing.assert_allclose(logits, x @ w.T, rtol=1e-4, atol=1e-4)
