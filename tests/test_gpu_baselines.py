"""GPU parity of the comparison policies (csrc/baselines.cu through the C ABI
desmoe_baseline_route and the Python mirror) vs the reference library
(oracle/_ref -> dessim::baseline_route, baselines.cpp:125-137).

IDs and counts must equal the reference's exactly; gates within 1e-12 (fp64 in
the reference's operation order; CUDA's exp / log may differ from glibc's in
the last bit). The hand cases are proj/tests/test_baselines.cpp's golden
values; tests/golden/baselines_golden.npz holds reference outputs at the
BASELINE shapes.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2602_00879_b200 import _lib
from paper_2602_00879_b200 import dessim as ds

pytestmark = pytest.mark.gpu

GATE_TOL = 1e-12
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cfg(m, k, act=0):
    return ds.PoolConfig(m, k, ds.GateActivation(act))


def block(x):
    x = np.asarray(x, np.float64)
    return ds.make_router_block(x.shape[0], x.shape[1], x)


def run(x, k, method, act=0, k_reduced=1, naee_beta=0.5, mcmoe_beta=0.5, fraction=0.5, score=0):
    b, c = block(x), cfg(np.asarray(x).shape[1], k, act)
    if method == 0:
        return ds.topk_reduce_route(b, c, k_reduced)
    if method == 1:
        return ds.naee_route(b, c, naee_beta)
    return ds.mcmoe_route(b, c, mcmoe_beta, fraction, ds.ImportanceScore(score))


def assert_same(gpu, ref_route, tol=GATE_TOL):
    for t, tok in enumerate(gpu.tokens):
        assert tok.experts == ref_route.experts(t), t
        assert np.all(np.abs(np.array(tok.gates) - np.array(ref_route.gates(t))) <= tol), t


def test_hand_cases():
    x = np.log([[0.5, 0.3, 0.15, 0.05]])
    a = run(x, 4, 1, naee_beta=0.2)
    assert a.tokens[0].experts == [0, 1, 2]
    assert np.allclose(a.tokens[0].gates, [0.5 / 0.95, 0.3 / 0.95, 0.15 / 0.95], atol=1e-9)
    b = run(x, 4, 1, naee_beta=0.6)
    assert b.tokens[0].experts == [0] and b.tokens[0].gates == [1.0]
    x = np.log([[0.9, 0.05, 0.03, 0.02], [0.3, 0.28, 0.22, 0.2]])
    r = run(x, 4, 2, mcmoe_beta=0.6, fraction=0.5)
    assert r.tokens[0].experts == [0, 1, 2, 3] and r.tokens[1].experts == [0, 1]
    assert np.allclose(r.tokens[1].gates, [0.3 / 0.58, 0.28 / 0.58], atol=1e-9)


def test_limits_equal_vanilla_and_naee(ref):
    x = np.random.default_rng(26).normal(size=(6, 16))
    van = ds.topk_route(ds.activate(block(x), cfg(16, 4)), 4)
    for r in (run(x, 4, 0, k_reduced=4), run(x, 4, 1, naee_beta=1e-12),
              run(x, 4, 2, mcmoe_beta=0.6, fraction=1.0)):
        for t in range(6):
            assert r.tokens[t].experts == van.tokens[t].experts
            assert r.tokens[t].gates == van.tokens[t].gates
    naee = run(x, 4, 1, naee_beta=0.6)
    zero = run(x, 4, 2, mcmoe_beta=0.6, fraction=0.0)
    for t in range(6):
        assert naee.tokens[t].experts == zero.tokens[t].experts
        assert naee.tokens[t].gates == zero.tokens[t].gates


@pytest.mark.parametrize("method,kw,msg", [
    (0, dict(k_reduced=5), "k_reduced outside"),
    (1, dict(naee_beta=1.0), "naee beta outside"),
    (2, dict(mcmoe_beta=0.0), "mcmoe beta outside"),
    (2, dict(fraction=1.5), "important_fraction outside"),
])
def test_validation_messages(method, kw, msg):
    with pytest.raises(ValueError, match=msg):
        run(np.zeros((2, 8)), 4, method, **kw)


def test_non_finite_rejected():
    x = np.zeros((2, 8))
    x[1, 3] = np.nan
    with pytest.raises(ValueError, match="non-finite logit"):
        run(x, 4, 1, naee_beta=0.5)


def test_random_parity(ref):
    rng = np.random.default_rng(4242)
    for _ in range(120):
        n, m = int(rng.integers(1, 80)), int(rng.integers(2, 300))
        k = int(rng.integers(1, min(m, 16) + 1))
        x = rng.normal(size=(n, m)) * rng.uniform(0.3, 4.0)
        act, method = int(rng.integers(0, 2)), int(rng.integers(0, 3))
        kw = dict(k_reduced=int(rng.integers(1, k + 1)), naee_beta=float(rng.uniform(0.02, 0.98)),
                  mcmoe_beta=float(rng.uniform(0.02, 0.98)), fraction=float(rng.uniform(0, 1)),
                  score=int(rng.integers(0, 2)))
        assert_same(run(x, k, method, act, **kw), ref.baseline_route(x, k, method, act, **kw))


def test_large_block_parity(ref):
    x = np.random.default_rng(7).normal(size=(256, 256)) * 2.0
    for method, kw in [(0, dict(k_reduced=3)), (1, dict(naee_beta=0.35)),
                       (2, dict(mcmoe_beta=0.35, fraction=0.3, score=1))]:
        assert_same(run(x, 8, method, **kw), ref.baseline_route(x, 8, method, **kw))


def test_golden_fixtures():
    g = np.load(os.path.join(GOLDEN, "baselines_golden.npz"))
    for i in range(int(g["count"])):
        x, k, act = g[f"x{i}"], int(g[f"k{i}"]), int(g[f"act{i}"])
        for j, (meth, kr, nb, mb, fr, sc) in enumerate(g["params"]):
            r = run(x, k, int(meth), act, k_reduced=min(int(kr), k), naee_beta=nb,
                    mcmoe_beta=mb, fraction=fr, score=int(sc))
            idx, gate, cnt = g[f"idx{i}_{j}"], g[f"gate{i}_{j}"], g[f"cnt{i}_{j}"]
            for t, tok in enumerate(r.tokens):
                assert tok.experts == idx[t, : cnt[t]].tolist(), (i, j, t)
                assert np.all(np.abs(np.array(tok.gates) - gate[t, : cnt[t]]) <= GATE_TOL)


def test_f32_logits_entry(ref):
    """desmoe_baseline_route_f32 (router / MOET trace logits) == the fp64 entry
    on the same fp32-exact values."""
    import torch
    x32 = (np.random.default_rng(11).normal(size=(40, 64)) * 2).astype(np.float32)
    n, m, k = 40, 64, 8
    ctx = ds._Ctx.get(n, m, k)
    idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
    gate = torch.empty((n, k), dtype=torch.float64, device="cuda")
    cnt = torch.empty((n,), dtype=torch.int32, device="cuda")
    out = _lib.RouteOut(idx.data_ptr(), gate.data_ptr(), cnt.data_ptr(), None, None, None, None)
    rc = _lib.RouteCfg(m, k, 0, _lib.VANILLA, 1, 1.0, 0)
    b = _lib.BaselineCfg(_lib.BASE_MCMOE, 1, 0.5, 0.45, 0.5, _lib.SCORE_NEG_ENTROPY)
    xd = torch.from_numpy(x32).cuda()
    _lib.check(_lib.lib().desmoe_baseline_route_f32(ctx.h, xd.data_ptr(), n, C.byref(rc),
                                                    C.byref(b), C.byref(out), None))
    torch.cuda.synchronize()
    want = ref.baseline_route(x32.astype(np.float64), k, 2, mcmoe_beta=0.45, fraction=0.5,
                              score=1)
    assert np.array_equal(idx.cpu().numpy(), want.idx)
    assert np.array_equal(cnt.cpu().numpy(), want.cnt)
    assert np.all(np.abs(gate.cpu().numpy() - want.gate) <= GATE_TOL)
