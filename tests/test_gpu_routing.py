"""GPU parity of the routing stage (K2) through the C ABI vs the reference.

Selections (per-token experts), coresets and assignments must equal the
reference library's (oracle/_ref, the reference's own sources) exactly.
Gates and votes: bit-identical (fp64 in the reference's operation order;
the kernels' exp is glibc's, restated in csrc/libm_exp.cuh).
The hand cases are the reference tests' golden values
(proj/tests/test_gating.cpp, test_des.cpp) restated on the Python mirror.
"""
import math

import numpy as np
import pytest

from paper_2602_00879_b200 import dessim as ds
from paper_2602_00879_b200 import synth

pytestmark = pytest.mark.gpu

GATE_TOL = 0.0
MIRRORED = [3, 2, 1, 0, 0, 1, 2, 3]


def cfg(m, k, act=0):
    return ds.PoolConfig(m, k, ds.GateActivation(act))


def block(x):
    x = np.asarray(x, np.float64)
    return ds.make_router_block(x.shape[0], x.shape[1], x)


def rb(n, m, seed, scale=1.0):
    return block(synth.random_block(n, m, seed, scale))


def assert_route_equal(gpu, ref_route, tol=GATE_TOL):
    for t, tok in enumerate(gpu.tokens):
        assert tok.experts == ref_route.experts(t), t
        assert np.all(np.abs(np.array(tok.gates) - np.array(ref_route.gates(t))) <= tol), t


# ---- golden hand values (test_gating.cpp / test_des.cpp) ----------------------

def test_softmax_golden():
    g = ds.activate(block([[3, 2, 1, 0]]), cfg(4, 2))
    for i, w in enumerate([0.6439, 0.2369, 0.0871, 0.0321]):
        assert abs(g.at(0, i) - w) <= 1e-4
    g = ds.activate(block([[0, 0, 0, 0]]), cfg(4, 2))
    assert np.all(np.abs(g.probs - 0.25) <= 1e-12)
    assert ds.activate(block([[0.0]]), cfg(1, 1)).at(0, 0) == 1.0
    g = ds.activate(block([[1000.0, 999.0, 998.0]]), cfg(3, 1))
    assert abs(g.probs.sum() - 1.0) <= 1e-9


def test_sigmoid_golden():
    g = ds.activate(block([[-1.0, 0.0, 2.0]]), cfg(3, 1, 1))
    assert abs(g.at(0, 1) - 0.5) <= 1e-12
    assert abs(g.at(0, 2) - 1.0 / (1.0 + math.exp(-2.0))) <= 1e-12


def test_nan_rejected_on_device():
    b = ds.RouterBlock(1, 2, np.array([[0.0, float("nan")]]))
    with pytest.raises(ValueError, match="non-finite logit"):
        ds.activate(b, cfg(2, 1))


def test_topk_route_golden():
    a = ds.topk_route(ds.activate(block([[3, 2, 1, 0]]), cfg(4, 2)), 2)
    assert a.tokens[0].experts == [0, 1]
    assert abs(a.tokens[0].gates[0] - 0.7310) <= 1e-4
    assert ds.topk_route(ds.activate(block([[0, 0, 0, 0]]), cfg(4, 2)), 2).tokens[0].experts == [0, 1]
    with pytest.raises(ValueError):
        ds.topk_route(ds.activate(block([[1, 2, 3]]), cfg(3, 3)), 4)


def test_select_and_renormalize():
    assert ds.select_top_gates([0.1, 0.5, 0.5, 0.2], 2) == [1, 2]
    assert ds.select_top_gates([0.1, 0.5, 0.5, 0.2], 2, [0, 2, 3]) == [2, 3]
    g = ds.renormalize_over([0.2, 0.3, 0.5], [0, 2])
    assert abs(g[0] - 0.2 / 0.7) <= 1e-15 and abs(g[1] - 0.5 / 0.7) <= 1e-15
    with pytest.raises(ValueError):
        ds.select_top_gates([0.1, 0.2], 3)


def test_des_golden():
    c = cfg(4, 2)
    assert ds.des_seq_coreset(block([[1, 5, 2, 0]]), c, 1).members == [1]
    assert ds.des_seq_coreset(block(np.reshape(MIRRORED, (2, 4))), c, 1).members == [0, 3]
    r = ds.des_vote_coreset(block(np.reshape(MIRRORED, (2, 4))), c, 0.5)
    for got, want in zip(r.votes.votes, [0.6439, 0.2369, 0.2369, 0.6439]):
        assert abs(got - want) <= 1e-4
    assert r.coreset.members == [0, 3]
    raw = ds.des_vote_coreset(block(np.reshape(MIRRORED, (2, 4))), c, 0.5, ds.VoteSource.raw_logits)
    assert np.allclose(raw.votes.votes, [3, 2, 2, 3], atol=1e-12, rtol=0)
    a = ds.constrained_route(block([[3, 2, 1, 0]]), c, ds.Coreset.of([0, 3]))
    e3 = math.exp(3.0)
    assert a.tokens[0].experts == [0, 3]
    assert abs(a.tokens[0].gates[0] - e3 / (e3 + 1)) <= 1e-9
    with pytest.raises(ValueError, match="empty coreset"):
        ds.constrained_route(rb(2, 4, 3), c, ds.Coreset())
    with pytest.raises(ValueError, match="coreset member out of range"):
        ds.constrained_route(rb(2, 4, 3), c, ds.Coreset.of([0, 4]))
    for beta in (0.05, 0.0, 1.5):
        with pytest.raises(ValueError):
            ds.des_vote_coreset(rb(2, 8, 9), cfg(8, 2), beta)


def test_des_limits():
    c = cfg(24, 6)
    b = rb(8, 24, 404)
    van = ds.topk_route(ds.activate(b, c), 6)
    full = ds.des_run(b, c, ds.DesParams(ds.DesStrategy.vote, 1, 1.0))
    assert full.coreset.size() == 24
    for t in range(8):
        assert full.assignment.tokens[t].experts == van.tokens[t].experts
        assert full.assignment.tokens[t].gates == van.tokens[t].gates
    seq = ds.des_run(b, c, ds.DesParams(ds.DesStrategy.seq, 6, 1.0))
    assert seq.coreset.members == ds.unique_experts(van).members


# ---- random instances vs the reference library --------------------------------

def instances(ref, count, base):
    for i in range(count):
        r = ref.rng_u64(base + i, 6)
        m = 2 + int(r[0] % 511)
        n = 1 + int(r[1] % 64)
        k = 1 + int(r[2] % min(m, 16))
        act = 1 if r[3] % 4 == 0 else 0
        m_core = 1 + int(r[4] % m)
        yield m, n, k, act, min(1.0, (m_core + 0.5) / m), synth.random_block(n, m, base + 1000 + i, 1.5)


def test_random_instances_match_reference(ref):
    """acceptance.cpp criterion-6 shapes (M<=512, N<=64, K<=16, 25 % sigmoid)."""
    for m, n, k, act, beta, x in instances(ref, 150, 61000):
        b, c = block(x), cfg(m, k, act)
        van = ds.topk_route(ds.activate(b, c), k)
        assert_route_equal(van, ref.topk_route(x, k, act))
        got = ds.des_vote_coreset(b, c, beta)
        want_mem, want_votes = ref.vote_coreset(x, k, beta, act)
        assert got.coreset.members == want_mem.tolist()
        v = np.array(got.votes.votes)
        assert np.array_equal(v, want_votes)
        seq_k = max(1, k // 2)
        assert ds.des_seq_coreset(b, c, seq_k).members == ref.seq_coreset(x, k, seq_k, act).tolist()
        for strat, p in (("vote", ds.DesParams(ds.DesStrategy.vote, 1, beta)),
                         ("seq", ds.DesParams(ds.DesStrategy.seq, seq_k, 1.0))):
            res = ds.des_run(b, c, p)
            mem, route = ref.des_run(x, k, strat, seq_k=seq_k, beta=beta, act=act)
            assert res.coreset.members == mem.tolist()
            assert_route_equal(res.assignment, route)


def test_baseline_config_traces_match_reference(ref):
    """gen_trace shared_bias logits at the BASELINE shapes (M=64/128/256, K=8,
    N=8..256) — the inputs the benchmark uses."""
    for m, beta in ((64, 0.4), (64, 0.6), (128, 0.3), (256, 0.15), (256, 0.10)):
        for n in (8, 32, 64, 256):
            for rho in (0.0, 0.3, 0.5):
                x = synth.gen_trace_block(m, n, 42, rho=rho)
                b, c = block(x), cfg(m, 8)
                for strat, p in (("vote", ds.DesParams(ds.DesStrategy.vote, 1, beta)),
                                 ("seq", ds.DesParams(ds.DesStrategy.seq, 3, 1.0))):
                    res = ds.des_run(b, c, p)
                    mem, route = ref.des_run(x, 8, strat, seq_k=3, beta=beta)
                    assert res.coreset.members == mem.tolist()
                    assert_route_equal(res.assignment, route)


def test_golden_fixtures():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "des_golden.npz"))
    for i in range(int(g["count"])):
        x = g[f"x{i}"]
        k, act, beta, seq_k = int(g[f"k{i}"]), int(g[f"act{i}"]), float(g[f"beta{i}"]), int(g[f"seqk{i}"])
        b, c = block(x), cfg(x.shape[1], k, act)
        res = ds.des_run(b, c, ds.DesParams(ds.DesStrategy.vote, 1, beta))
        assert res.coreset.members == g[f"vote_mem{i}"].tolist()
        for t, tok in enumerate(res.assignment.tokens):
            cnt = len(tok.experts)
            assert tok.experts == g[f"vote_idx{i}"][t, :cnt].tolist()
            assert np.all(np.abs(np.array(tok.gates) - g[f"vote_gate{i}"][t, :cnt]) <= GATE_TOL)
        votes = np.array(ds.des_vote_coreset(b, c, beta).votes.votes)
        assert np.array_equal(votes, g[f"votes{i}"])
        res = ds.des_run(b, c, ds.DesParams(ds.DesStrategy.seq, seq_k, 1.0))
        assert res.coreset.members == g[f"seq_mem{i}"].tolist()


def test_shift_invariance_and_nesting():
    c = cfg(12, 4)
    b = rb(5, 12, 611)
    shifted = b.logits + 3.0 * (np.arange(5)[:, None] + 1)
    b2 = block(shifted)
    assert ds.des_seq_coreset(b2, c, 2).members == ds.des_seq_coreset(b, c, 2).members
    assert (ds.des_vote_coreset(b2, c, 0.5).coreset.members
            == ds.des_vote_coreset(b, c, 0.5).coreset.members)
    c = cfg(20, 5)
    b = rb(6, 20, 808)
    prev = []
    for mc in range(1, 21):
        cur = ds.des_vote_coreset(b, c, (mc + 0.5) / 20.0).coreset.members
        assert len(cur) == mc and set(prev) <= set(cur)
        prev = cur
