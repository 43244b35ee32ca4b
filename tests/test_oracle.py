"""Pins the CPU checkers before anything is compared against them.

1. Both the reference library (oracle/_ref, compiled from the reference's own
   sources) and the C restatement (oracle/liboracle.so) must reproduce the
   golden values of the reference's unit tests (proj/tests/test_gating.cpp,
   test_des.cpp, test_core.cpp) — the same hand-derived numbers, same tolerances.
2. The restatement must be bit-identical to the reference on seeded random
   instances (acceptance.cpp criterion-6 shapes: M <= 512, N <= 64, K <= 16,
   sigmoid 25 %).
3. Committed fixtures under tests/golden/ (made by tests/golden/make_golden.py
   from the reference itself) must still match the restatement, so the oracle
   stays pinned on machines without the reference build.
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import Port, Ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def random_block(ref, n, m, seed, scale=1.0):
    """test_helpers.hpp:28-36 — scaled N(0,1) logits from Rng(seed)."""
    return (scale * ref.rng_normal(seed, n * m)).reshape(n, m)


MIRRORED = np.array([[3, 2, 1, 0], [0, 1, 2, 3]], np.float64)  # test_des.cpp:19-21


@pytest.fixture(params=["ref", "port"])
def impl(request, ref, port):
    return ref if request.param == "ref" else port


# ---- splitmix64 known answers (test_core.cpp:60-72) ---------------------------

def test_rng_known_answers(ref):
    assert [int(v) for v in ref.rng_u64(0, 3)] == [
        0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [int(v) for v in ref.rng_u64(42, 3)] == [
        13679457532755275413, 2949826092126892291, 5139283748462763858]
    assert ref.rng_mix(7, 0) != ref.rng_mix(7, 1)
    assert ref.rng_mix(7, 3) == ref.rng_mix(7, 3)


def test_validate_config_messages(ref):
    with pytest.raises(ValueError, match="top_k > experts_total"):
        ref.validate_config(8, 9)
    with pytest.raises(ValueError, match="bytes_per_expert == 0"):
        ref.validate_config(8, 2, bytes_per_expert=0)
    with pytest.raises(ValueError, match="hidden_dim < 1"):
        ref.validate_config(8, 2, dim=0)


# ---- gating golden values (test_gating.cpp) -----------------------------------

def test_softmax_uniform(impl):
    p = impl.activate(np.zeros((1, 4)))
    assert np.all(np.abs(p - 0.25) <= 1e-12)


def test_softmax_ramp(impl):
    p = impl.activate(np.array([[3, 2, 1, 0]], np.float64))[0]
    for got, want in zip(p, [0.6439, 0.2369, 0.0871, 0.0321]):
        assert abs(got - want) <= 1e-4


def test_single_expert_is_one(impl):
    assert impl.activate(np.zeros((1, 1)))[0, 0] == 1.0


def test_softmax_stable_large(impl):
    p = impl.activate(np.array([[1000.0, 999.0, 998.0]]))[0]
    assert abs(p.sum() - 1.0) <= 1e-9 and math.isfinite(p[0])


def test_sigmoid(impl):
    p = impl.activate(np.array([[-1.0, 0.0, 2.0]]), act=1)[0]
    assert abs(p[1] - 0.5) <= 1e-12
    assert abs(p[2] - 1.0 / (1.0 + math.exp(-2.0))) <= 1e-12
    assert np.all((p > 0) & (p < 1))


def test_nan_rejected(impl):
    with pytest.raises(ValueError):
        impl.activate(np.array([[0.0, float("nan")]]))


def test_topk_route_hand(impl):
    r = impl.topk_route(np.array([[3, 2, 1, 0]], np.float64), 2)
    assert r.experts(0) == [0, 1]
    assert abs(r.gates(0)[0] - 0.7310) <= 1e-4 and abs(r.gates(0)[1] - 0.2690) <= 1e-4


def test_topk_route_k_equals_m(impl, ref):
    x = random_block(ref, 4, 6, 31)
    r = impl.topk_route(x, 6)
    p = impl.activate(x)
    for t in range(4):
        assert r.experts(t) == list(range(6))
        assert np.all(np.abs(np.array(r.gates(t)) - p[t]) <= 1e-12)


def test_topk_ties_lowest_index(impl):
    assert impl.topk_route(np.zeros((1, 4)), 2).experts(0) == [0, 1]


def test_topk_oversized_k(impl):
    with pytest.raises(ValueError):
        impl.topk_route(np.array([[1.0, 2.0, 3.0]]), 4)


def test_unique_experts_set_oracle(ref):
    """test_gating.cpp:188-198 at M=256, N=32, seed 3."""
    r = ref.topk_route(random_block(ref, 32, 256, 3), 8)
    union = sorted({e for t in range(32) for e in r.experts(t)})
    u, tot, per = ref.moe_latency(r, 256)
    assert u == len(union) and tot == 256 and int((per > 0).sum()) == u


# ---- DES golden values (test_des.cpp) -----------------------------------------

def test_vote_budget(impl):
    assert [impl.vote_budget(b, m) for b, m in
            [(0.15, 256), (0.10, 256), (0.6, 64), (0.4, 64), (1.0, 64)]] == [38, 25, 38, 25, 64]


def test_seq_hand(impl):
    assert impl.seq_coreset(np.array([[1, 5, 2, 0]], np.float64), 2, 1).tolist() == [1]
    assert impl.seq_coreset(MIRRORED, 2, 1).tolist() == [0, 3]
    same = np.tile([0.4, 0.1, 0.9, 0.2], (5, 1))
    assert [len(impl.seq_coreset(same, 2, k)) for k in (1, 2)] == [1, 2]
    for bad in (0, 3):
        with pytest.raises(ValueError):
            impl.seq_coreset(MIRRORED, 2, bad)


def test_vote_hand(impl):
    mem, v = impl.vote_coreset(MIRRORED, 2, 0.5)
    for got, want in zip(v, [0.6439, 0.2369, 0.2369, 0.6439]):
        assert abs(got - want) <= 1e-4
    assert mem.tolist() == [0, 3]


def test_vote_raw_logits(impl):
    mem, v = impl.vote_coreset(MIRRORED, 2, 0.5, raw=True)
    assert np.all(np.abs(v - [3, 2, 2, 3]) <= 1e-12) and mem.tolist() == [0, 3]


def test_vote_budget_exact(impl, ref):
    big = random_block(ref, 16, 256, 40)
    assert len(impl.vote_coreset(big, 8, 0.15)[0]) == 38
    assert len(impl.vote_coreset(big, 8, 0.10)[0]) == 25
    small = random_block(ref, 16, 64, 41)
    assert len(impl.vote_coreset(small, 8, 0.4)[0]) == 25
    assert len(impl.vote_coreset(small, 8, 0.6)[0]) == 38


def test_vote_degenerate(impl, ref):
    x = random_block(ref, 2, 8, 9)
    for beta in (0.05, 0.0, 1.5):
        with pytest.raises(ValueError):
            impl.vote_coreset(x, 2, beta)


def test_constrained_hand(impl):
    r = impl.constrained_route(np.array([[3, 2, 1, 0]], np.float64), 2, [0, 3])
    e3 = math.exp(3.0)
    assert r.experts(0) == [0, 3]
    assert abs(r.gates(0)[0] - e3 / (e3 + 1)) <= 1e-9
    assert abs(r.gates(0)[1] - 1 / (e3 + 1)) <= 1e-9


def test_constrained_full_pool_is_vanilla(impl, ref):
    x = random_block(ref, 6, 16, 77)
    v = impl.topk_route(x, 4)
    c = impl.constrained_route(x, 4, list(range(16)))
    assert np.array_equal(v.idx, c.idx) and np.array_equal(v.gate, c.gate)


def test_constrained_saturates(impl, ref):
    r = impl.constrained_route(random_block(ref, 3, 8, 12), 4, [2, 5])
    assert all(r.experts(t) == [2, 5] for t in range(3))


def test_constrained_errors(impl, ref):
    x = random_block(ref, 2, 4, 3)
    with pytest.raises(ValueError, match="empty coreset"):
        impl.constrained_route(x, 2, [])
    with pytest.raises(ValueError, match="coreset member out of range"):
        impl.constrained_route(x, 2, [0, 4])


def test_des_run_limits(impl, ref):
    x = random_block(ref, 8, 24, 404)
    v = impl.topk_route(x, 6)
    mem, r = impl.des_run(x, 6, "vote", beta=1.0)
    assert len(mem) == 24 and np.array_equal(r.idx, v.idx) and np.array_equal(r.gate, v.gate)
    x = random_block(ref, 8, 24, 405)
    v = impl.topk_route(x, 6)
    mem, r = impl.des_run(x, 6, "seq", seq_k=6)
    assert mem.tolist() == sorted(set(v.idx.ravel().tolist()))
    assert np.array_equal(r.idx, v.idx)


def test_des_run_validates(impl):
    with pytest.raises(ValueError):
        impl.des_run(MIRRORED, 2, "seq", seq_k=0)
    with pytest.raises(ValueError):
        impl.des_run(MIRRORED, 2, "vote", beta=0.0)


def test_fused_equals_composed(ref):
    """test_des.cpp:231-252 (reference vs itself) — the contract the GPU must keep."""
    for seed in range(50):
        rng = ref.rng_u64(9000 + seed, 8)
        m = 2 + int(rng[0] % 100)
        n = 1 + int(rng[1] % 16)
        k = 1 + int(rng[2] % min(m, 8))
        x = random_block(ref, n, m, 7000 + seed, 1.5)
        m_core = 1 + int(rng[3] % m)
        beta = (m_core + 0.5) / m
        a, va = ref.vote_coreset(x, k, beta)
        b, vb = ref.fused_vote(x, k, beta)
        assert np.array_equal(a, b) and np.all(np.abs(va - vb) <= 1e-9)


# ---- restatement == reference, bit for bit ------------------------------------

def _instances(ref, count, base):
    for i in range(count):
        r = ref.rng_u64(base + i, 6)
        m = 2 + int(r[0] % 511)
        n = 1 + int(r[1] % 64)
        k = 1 + int(r[2] % min(m, 16))
        act = 1 if r[3] % 4 == 0 else 0
        m_core = 1 + int(r[4] % m)
        yield m, n, k, act, (m_core + 0.5) / m, random_block(ref, n, m, base + 1000 + i, 1.5)


def test_port_bit_identical_to_reference(ref, port):
    for m, n, k, act, beta, x in _instances(ref, 120, 61000):
        assert np.array_equal(ref.activate(x, act), port.activate(x, act))
        a = ref.topk_route(x, k, act)
        b = port.topk_route(x, k, act)
        assert np.array_equal(a.idx, b.idx) and np.array_equal(a.gate, b.gate)
        ma, va = ref.vote_coreset(x, k, beta, act)
        mb, vb = port.vote_coreset(x, k, beta, act)
        assert np.array_equal(ma, mb) and np.array_equal(va, vb)
        seq_k = max(1, k // 2)
        assert np.array_equal(ref.seq_coreset(x, k, seq_k, act), port.seq_coreset(x, k, seq_k, act))
        for strat in ("vote", "seq"):
            b = min(beta, 1.0)
            ca, ra = ref.des_run(x, k, strat, seq_k=seq_k, beta=b, act=act)
            cb, rb = port.des_run(x, k, strat, seq_k=seq_k, beta=b, act=act)
            assert np.array_equal(ca, cb)
            assert np.array_equal(ra.idx, rb.idx) and np.array_equal(ra.gate, rb.gate)
            assert np.array_equal(ra.cnt, rb.cnt)


def test_port_permutation_matches_reference_counts(ref, port):
    for m, n, k, act, beta, x in _instances(ref, 40, 71000):
        _, r = ref.des_run(x, k, "vote", beta=min(beta, 1.0), act=act)
        u, tot, per = ref.moe_latency(r, m)
        p = port.permute(r, m)
        assert np.array_equal(p["count"], per) and len(p["active"]) == u
        assert int(p["count"].sum()) == tot
        # stable: inside each expert's segment tokens ascend
        for e in p["active"]:
            seg = p["slot_token"][p["offset"][e]: p["offset"][e] + p["count"][e]]
            assert np.all(np.diff(seg) > 0)


def test_port_linear_ffn_matches_moe_forward(ref, port):
    """moe_forward (gating.cpp:136-157) on the reference bank vs the port's
    fp32-combine linear mode on the same values."""
    m, k, dim, n = 16, 8, 6, 5
    w, xin = ref.make_expert_bank(m, dim, n, 7)
    r = ref.topk_route(random_block(ref, n, m, 7), k)
    want = ref.moe_forward(r, w, xin)
    got = port.moe_ffn(r, xin.astype(np.float32), w.astype(np.float32), mode="linear")
    assert np.allclose(got, want, rtol=1e-5, atol=1e-5)


def test_golden_fixtures(port):
    path = os.path.join(GOLDEN, "des_golden.npz")
    g = np.load(path)
    for i in range(int(g["count"])):
        x = g[f"x{i}"]
        k, act, beta, seq_k = (int(g[f"k{i}"]), int(g[f"act{i}"]), float(g[f"beta{i}"]),
                               int(g[f"seqk{i}"]))
        mem, r = port.des_run(x, k, "vote", beta=beta, act=act)
        assert np.array_equal(mem, g[f"vote_mem{i}"])
        assert np.array_equal(r.idx, g[f"vote_idx{i}"])
        assert np.array_equal(r.gate, g[f"vote_gate{i}"])
        _, v = port.vote_coreset(x, k, beta, act)
        assert np.array_equal(v, g[f"votes{i}"])
        mem, r = port.des_run(x, k, "seq", seq_k=seq_k, act=act)
        assert np.array_equal(mem, g[f"seq_mem{i}"])
        assert np.array_equal(r.idx, g[f"seq_idx{i}"])
        r = port.topk_route(x, k, act)
        assert np.array_equal(r.idx, g[f"van_idx{i}"])
        assert np.array_equal(r.gate, g[f"van_gate{i}"])


# ---- comparison policies (baselines.cpp; proj/tests/test_baselines.cpp) --------

def _probs_block(rows):
    """block_with_probs (test_baselines.cpp:18-27): logits = log(p)."""
    return np.log(np.asarray(rows, np.float64))


def test_baselines_hand(impl):
    x = _probs_block([[0.5, 0.3, 0.15, 0.05]])
    # tail(4) = 0.05 < 0.2, tail(3) = 0.20 is not: ranks 1..3 stay (:61-69)
    r = impl.baseline_route(x, 4, 1, naee_beta=0.2)
    assert r.experts(0) == [0, 1, 2]
    for g, w in zip(r.gates(0), [0.5 / 0.95, 0.3 / 0.95, 0.15 / 0.95]):
        assert abs(g - w) <= 1e-9
    r = impl.baseline_route(x, 4, 1, naee_beta=0.6)  # tail(2) = 0.5 < 0.6 (:71-74)
    assert r.experts(0) == [0] and r.gates(0) == [1.0]
    # MC-MoE: the confident token keeps its top-K, the diffuse one is skipped (:133-146)
    x = _probs_block([[0.9, 0.05, 0.03, 0.02], [0.3, 0.28, 0.22, 0.2]])
    r = impl.baseline_route(x, 4, 2, mcmoe_beta=0.6, fraction=0.5)
    assert r.experts(0) == [0, 1, 2, 3] and r.experts(1) == [0, 1]
    assert abs(r.gates(1)[0] - 0.3 / 0.58) <= 1e-9 and abs(r.gates(1)[1] - 0.28 / 0.58) <= 1e-9
    # top-k reduce with k = 1 is the per-token argmax with gate 1 (:46-58)
    x = random_block_np(5, 16, 22)
    r = impl.baseline_route(x, 4, 0, k_reduced=1)
    for t in range(5):
        assert r.experts(t) == [int(np.argmax(x[t]))] and r.gates(t) == [1.0]


def random_block_np(n, m, seed):
    return np.random.default_rng(seed).normal(size=(n, m))


@pytest.mark.parametrize("method,kw,msg", [
    (0, dict(k_reduced=5), "k_reduced outside [1, top_k]"),
    (0, dict(k_reduced=0), "k_reduced outside [1, top_k]"),
    (1, dict(naee_beta=0.0), "naee beta outside (0, 1)"),
    (1, dict(naee_beta=1.0), "naee beta outside (0, 1)"),
    (2, dict(mcmoe_beta=1.0), "mcmoe beta outside (0, 1)"),
    (2, dict(fraction=-0.1), "important_fraction outside [0, 1]"),
    (2, dict(fraction=1.1), "important_fraction outside [0, 1]"),
])
def test_baselines_validate(impl, method, kw, msg):
    with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")
                       .replace("[", r"\[").replace("]", r"\]")):
        impl.baseline_route(random_block_np(2, 8, 23), 4, method, **kw)


def test_port_baselines_bit_identical_to_reference(ref, port):
    rng = np.random.default_rng(90210)
    for _ in range(200):
        n, m = int(rng.integers(1, 48)), int(rng.integers(2, 160))
        k = int(rng.integers(1, min(m, 16) + 1))
        x = rng.normal(size=(n, m)) * rng.uniform(0.3, 4.0)
        act, method = int(rng.integers(0, 2)), int(rng.integers(0, 3))
        kw = dict(k_reduced=int(rng.integers(1, k + 1)), naee_beta=float(rng.uniform(0.02, 0.98)),
                  mcmoe_beta=float(rng.uniform(0.02, 0.98)), fraction=float(rng.uniform(0, 1)),
                  score=int(rng.integers(0, 2)))
        a = ref.baseline_route(x, k, method, act, **kw)
        b = port.baseline_route(x, k, method, act, **kw)
        assert np.array_equal(a.idx, b.idx) and np.array_equal(a.cnt, b.cnt)
        assert np.array_equal(a.gate, b.gate)


def test_baselines_golden_fixtures(port):
    g = np.load(os.path.join(GOLDEN, "baselines_golden.npz"))
    for i in range(int(g["count"])):
        x, k, act = g[f"x{i}"], int(g[f"k{i}"]), int(g[f"act{i}"])
        for j, (meth, kr, nb, mb, fr, sc) in enumerate(g["params"]):
            r = port.baseline_route(x, k, int(meth), act, k_reduced=min(int(kr), k),
                                    naee_beta=nb, mcmoe_beta=mb, fraction=fr, score=int(sc))
            assert np.array_equal(r.idx, g[f"idx{i}_{j}"]) and np.array_equal(r.cnt, g[f"cnt{i}_{j}"])
            assert np.array_equal(r.gate, g[f"gate{i}_{j}"])


def test_exact_logit_split_reconstructs_fp32():
    """The controlled-logit harness (tests/_exact_logits.py) splits any fp32
    logit into three bf16 pieces whose fp32 sum in ascending K order is the
    value itself (the layer-path parity tests rely on it)."""
    from _exact_logits import bf16_trunc, split3
    rng = np.random.default_rng(0)
    cases = [rng.normal(size=(64, 256)) * 1.5, rng.uniform(-1000, -705, size=(8, 64)),
             rng.uniform(38, 60, size=(8, 64)), np.zeros((4, 4)),
             (np.float32(1.5) + np.arange(256, dtype=np.float32) * np.float32(2 ** -23))[None, :]]
    for v in cases:
        v = np.asarray(v, np.float32)
        a, b, c = split3(v)
        for piece in (a, b, c):
            assert np.array_equal(bf16_trunc(piece), piece)
        # every prefix / subset sum the split-K GEMM may form is exact too
        assert np.array_equal((a + b * np.float32(2 ** -8)).astype(np.float32) + c * np.float32(2 ** -16), v)


def test_glibc_exp_restatement():
    """oracle/desmoe_oracle.c:or_glibc_exp (the same steps as the kernels'
    csrc/libm_exp.cuh) equals the host libm's exp bit for bit over every
    range the routing reaches: softmax arguments down to the subnormal band
    and full underflow, sigmoid arguments, tiny, special values."""
    import ctypes as C
    lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                              "liboracle.so"))
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    for name in ("or_glibc_exp", "or_libm_exp"):
        getattr(lib, name).argtypes = [f64p, f64p, C.c_long]
        getattr(lib, name).restype = None
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.uniform(-1100.0, 0.0, 1_000_000), rng.uniform(-745.2, -708.0, 1_000_000),
        rng.uniform(-40.0, 40.0, 1_000_000), rng.uniform(-1e-15, 1e-15, 10_000),
        rng.uniform(700.0, 712.0, 10_000),
        # fp32 logit differences, as the kernels feed them
        (rng.normal(size=500_000).astype(np.float32).astype(np.float64)
         - rng.normal(size=500_000).astype(np.float32).astype(np.float64)),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -1024.0, -1023.99, -512.0, -511.99,
                  709.78, 709.79, -745.13, -745.14, 5e-324, -708.3964, -708.3965])])
    a, b = np.empty_like(x), np.empty_like(x)
    lib.or_glibc_exp(x, a, len(x))
    lib.or_libm_exp(x, b, len(x))
    same = (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))
    assert same.all(), x[~same][:8]
