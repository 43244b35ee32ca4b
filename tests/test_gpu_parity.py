"""Routing parity of the PRODUCTION layer path (front_kernel: router GEMM +
activation + top-K + DES coreset + constrained re-route in one cluster, or the
split path beyond its envelope) on controlled logits, against the UNMODIFIED
reference library (oracle/_ref) fed the same values.

The logits are injected through the layer's own router GEMM (tests/_exact_logits.py)
and read back bit-exact, so the cases reach the kernel's tie-break and
fallback paths that random hidden states never hit:

  * exact logit ties at the top-K boundary (lowest index wins, gating.cpp:49-52;
    the reference's own tie case test_gating.cpp:90-94);
  * near-ties below the front kernel's 24-bit selection key (logit gaps of
    1 .. 255 fp32 ulps: the fast path cannot order them and must fall back to
    the exact fp64 comparator);
  * softmax underflow (gates exactly 0 or subnormal at the boundary);
  * saturated sigmoids (distinct logits, gate == 1.0 exactly);
  * exactly tied DES-Vote votes at the floor(beta*M) coreset boundary
    (duplicated router columns), activated and raw-logit votes;
  * acceptance criterion 6's instance generator (acceptance.cpp:207-230;
    1000 instances, M <= 256, N <= 64, K <= 16, 25 % sigmoid) through the
    layer instead of the logits-in entry points.

Pass bar: the layer's logits equal the injected fp32 values bit for bit;
selected expert ids, per-token counts and coreset membership equal the
reference's; gates bit-identical (atol = 0: the kernels' exp is glibc's,
restated in csrc/libm_exp.cuh, and every sum runs in the reference's order).
"""
import numpy as np
import pytest

from _exact_logits import LayerProbe, assert_same_route
from paper_2602_00879_b200 import synth

pytestmark = pytest.mark.gpu

_PROBE = {}


def probe(d):
    if d not in _PROBE:
        _PROBE[d] = LayerProbe(max_n=256, max_m=512, max_k=16, d=d)
    return _PROBE[d]


def check_case(ref, logits, k, strategy, seq_k=1, beta=1.0, act=0, raw=False, d=None):
    from _exact_logits import hidden_for
    L = np.ascontiguousarray(logits, np.float32)
    n, m = L.shape
    got = probe(d or hidden_for(n)).run(L, k, strategy, seq_k=seq_k, beta=beta, act=act, raw=raw)
    assert np.array_equal(got["logits"].view(np.uint32), L.view(np.uint32)), \
        "layer logits differ from the injected values"
    L64 = L.astype(np.float64)
    if strategy == "vanilla":
        want = ref.topk_route(L64, k, act=act)
    elif raw:
        mem, _ = ref.vote_coreset(L64, k, beta, act=act, raw=True)
        want = ref.constrained_route(L64, k, mem, act=act)
        assert got["members"] == mem.tolist()
    else:
        mem, want = ref.des_run(L64, k, strategy, seq_k=seq_k, beta=beta, act=act)
        assert got["members"] == mem.tolist()
    assert_same_route(got, want)
    u, total, _ = ref.moe_latency(want, m)
    assert got["stats"][0] == u and got["stats"][2] == total
    return got


# ---- logit generators -------------------------------------------------------------


def tied_levels(n, m, seed, levels=6):
    """Logits from a few discrete levels: exact ties everywhere, including at
    every top-K boundary."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, levels, size=(n, m)) * 0.25 - 0.5).astype(np.float32)


def near_ties(n, m, seed, spread=255):
    """Per token one base value in [1, 2) plus 0..spread fp32 ulps (2^-23): the
    logits differ only below the selection key's 24 bits, with some exact
    duplicates as well."""
    rng = np.random.default_rng(seed)
    base = rng.uniform(1.0, 2.0, size=(n, 1)).astype(np.float32)
    base = (base.view(np.uint32) & np.uint32(0xFFFFFF00)).view(np.float32)
    ulps = rng.integers(0, spread + 1, size=(n, m)).astype(np.uint32)
    return (base.view(np.uint32) + ulps).view(np.float32)


def underflow(n, m, seed, live=3):
    """`live` experts per token near 0, the others between -1000 and -705:
    their softmax numerators are 0 or subnormal in fp64, so the K-th gate
    ties at 0 (lowest index) or sits in the subnormal range."""
    rng = np.random.default_rng(seed)
    L = rng.uniform(-1000.0, -705.0, size=(n, m)).astype(np.float32)
    for t in range(n):
        L[t, rng.choice(m, live, replace=False)] = rng.normal(size=live)
    return L


def saturated_sigmoid(n, m, seed):
    """Sigmoid gates 1/(1+exp(-x)) == 1.0 exactly for x > ~37: distinct logits,
    tied gates."""
    rng = np.random.default_rng(seed)
    L = rng.normal(size=(n, m)).astype(np.float32)
    hot = rng.random(size=(n, m)) < 0.3
    L[hot] = rng.uniform(38.0, 60.0, size=hot.sum()).astype(np.float32)
    return L


def duplicated_columns(n, m, seed, dup=8, rho=0.5):
    """Shared-bias logits with `dup` experts copied into their neighbours:
    identical columns give exactly equal votes."""
    rng = np.random.default_rng(seed)
    L = synth.gen_trace_block(m, n, seed, rho=rho).astype(np.float32)
    for j in rng.choice(m - 1, dup, replace=False):
        L[:, j + 1] = L[:, j]
    return L


def vote_tie_at_boundary(ref, n, m, k, beta, seed):
    """Duplicated-column logits where the coreset boundary (rank floor(beta*M))
    falls between two experts with exactly equal votes: expert order by a
    descending bias, the pair straddling the boundary duplicated."""
    m_core = ref.vote_budget(beta, m)
    rng = np.random.default_rng(seed)
    bias = np.linspace(3.0, -3.0, m)
    L = (bias[None, :] + 0.3 * rng.normal(size=(n, m))).astype(np.float32)
    for _ in range(50):
        _, votes = ref.vote_coreset(L.astype(np.float64), k, beta)
        order = sorted(range(m), key=lambda e: (-votes[e], e))
        a, b = order[m_core - 1], order[m_core]
        L[:, max(a, b)] = L[:, min(a, b)]
        mem, votes = ref.vote_coreset(L.astype(np.float64), k, beta)
        order = sorted(range(m), key=lambda e: (-votes[e], e))
        if votes[order[m_core - 1]] == votes[order[m_core]]:
            return L
    return constructed_vote_tie(n, m, k, m_core, seed)


def constructed_vote_tie(n, m, k, m_core, seed):
    """Every token routes the same row (as at rho = 1): its value order is a
    random permutation of the experts, with the experts at vote ranks
    m_core - 1 and m_core given the same logit. For m_core < k both are in
    every token's top-K, so their votes are equal and non-zero; otherwise
    only k experts get votes and the boundary tie is between zero-vote
    experts (filled by lowest index, des.cpp:93)."""
    rng = np.random.default_rng(seed)
    vals = np.sort(rng.uniform(-2.0, 2.0, size=m))[::-1].astype(np.float32)
    vals[m_core] = vals[m_core - 1]
    perm = rng.permutation(m)
    row = np.empty(m, np.float32)
    row[perm] = vals
    return np.tile(row, (n, 1))


# ---- cases ------------------------------------------------------------------------

SHAPES = [(8, 64, 8), (32, 64, 8), (64, 128, 8), (32, 256, 8), (160, 128, 8), (256, 256, 8),
          (29, 40, 6), (32, 512, 8), (96, 384, 8)]


@pytest.mark.parametrize("n,m,k", SHAPES)
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
@pytest.mark.parametrize("act", [0, 1])
def test_exact_logit_ties(ref, n, m, k, strategy, act):
    for seed in range(3):
        L = tied_levels(n, m, seed + 10 * n + m)
        check_case(ref, L, k, strategy, seq_k=3, beta=0.4 if m <= 64 else 0.15, act=act)


@pytest.mark.parametrize("n,m,k", SHAPES)
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
def test_near_ties_below_selection_key(ref, n, m, k, strategy):
    for seed, spread in ((1, 255), (2, 16), (3, 1)):
        L = near_ties(n, m, seed + n, spread)
        check_case(ref, L, k, strategy, seq_k=2, beta=0.3)


@pytest.mark.parametrize("n,m,k", [(32, 64, 8), (64, 256, 8), (256, 128, 8)])
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
@pytest.mark.parametrize("live", [1, 3, 12])
def test_softmax_underflow_boundary(ref, n, m, k, strategy, live):
    L = underflow(n, m, 7 + live, live=live)
    check_case(ref, L, k, strategy, seq_k=3, beta=0.25)


@pytest.mark.parametrize("n,m,k", [(32, 64, 8), (64, 256, 8), (256, 128, 8)])
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
def test_saturated_sigmoid_ties(ref, n, m, k, strategy):
    L = saturated_sigmoid(n, m, 5 + n)
    check_case(ref, L, k, strategy, seq_k=3, beta=0.3, act=1)


@pytest.mark.parametrize("n,m,k", [(32, 64, 8), (64, 256, 8), (256, 128, 8), (13, 40, 6)])
@pytest.mark.parametrize("act", [0, 1])
def test_vote_ties_at_coreset_boundary(ref, n, m, k, act):
    beta = 0.4 if m <= 64 else 0.15
    L = vote_tie_at_boundary(ref, n, m, k, beta, seed=n + m)
    got = check_case(ref, L, k, "vote", beta=beta, act=act)
    assert len(got["members"]) == ref.vote_budget(beta, m)


@pytest.mark.parametrize("n,m,k,m_core", [(32, 64, 8, 5), (32, 64, 8, 25), (64, 256, 8, 7),
                                           (64, 256, 8, 38), (120, 128, 16, 12)])
@pytest.mark.parametrize("act", [0, 1])
def test_constructed_vote_ties(ref, n, m, k, m_core, act):
    """Exactly equal votes at the coreset boundary, non-zero (m_core < K) and
    zero (m_core > K: lowest-index fill)."""
    beta = (m_core + 0.5) / m
    L = constructed_vote_tie(n, m, k, m_core, seed=m_core)
    mem, votes = ref.vote_coreset(L.astype(np.float64), k, beta, act=act)
    order = sorted(range(m), key=lambda e: (-votes[e], e))
    assert votes[order[m_core - 1]] == votes[order[m_core]]  # the tie is at the boundary
    got = check_case(ref, L, k, "vote", beta=beta, act=act)
    assert len(got["members"]) == m_core


@pytest.mark.parametrize("n,m,k", [(32, 64, 8), (128, 256, 8)])
@pytest.mark.parametrize("raw", [False, True])
def test_duplicated_columns(ref, n, m, k, raw):
    for seed in range(4):
        L = duplicated_columns(n, m, 100 + seed)
        check_case(ref, L, k, "vote", beta=0.4 if m <= 64 else 0.15, raw=raw)
        if not raw:
            check_case(ref, L, k, "seq", seq_k=2)
            check_case(ref, L, k, "vanilla")


def test_reference_tie_golden(ref):
    """test_gating.cpp:90-94: equal logits -> the lowest indices {0, 1}."""
    got = check_case(ref, np.zeros((4, 4), np.float32), 2, "vanilla")
    assert got["idx"][:, :2].tolist() == [[0, 1]] * 4
    np.testing.assert_allclose(got["gate"][:, :2], 0.5, rtol=0, atol=0)
    # DES-Vote on the same block: every vote ties, the coreset is {0, 1}
    got = check_case(ref, np.zeros((4, 4), np.float32), 2, "vote", beta=0.5)
    assert got["members"] == [0, 1]


@pytest.mark.parametrize("variant", ["0", "1", "2"])
def test_ties_every_gemm_variant(ref, monkeypatch, variant):
    """Split-K and both token-split router GEMMs carry the injected logits
    exactly (DESMOE_FRONT_TSPLIT)."""
    monkeypatch.setenv("DESMOE_FRONT_TSPLIT", variant)
    for n, m in ((32, 64), (128, 256)):
        check_case(ref, tied_levels(n, m, 3), 8, "vote", beta=0.3)
        check_case(ref, near_ties(n, m, 4), 8, "seq", seq_k=3)


def criterion6_instances(ref, count=1000):
    """acceptance.cpp:207-230's generator, exactly (Rng(61000 + i) draws m in
    2..512, n, k, the activation and the budget; random_block(n, m, 62000 + i,
    1.5) logits, quantised to fp32). Pools above 256 run the router kernel +
    the front's logits-in mode."""
    for i in range(count):
        u = synth.u64_stream(61000 + i, 64)
        draws = iter(int(v) for v in u)

        def below(b):
            # Rng::next_below (core.cpp:139-150): reject x < 2^64 mod b, then x % b
            threshold = (1 << 64) % b
            while True:
                x = next(draws)
                if x >= threshold:
                    return x % b

        m = 2 + below(511)
        n = 1 + below(64)
        k = 1 + below(min(m, 16))
        act = 1 if below(4) == 0 else 0
        m_core = 1 + below(m)
        beta = min(1.0, (m_core + 0.5) / m)  # des_run's validate_params caps beta at 1
        L = synth.random_block(n, m, 62000 + i, 1.5).astype(np.float32)
        yield i, m, n, k, act, beta, L


def test_criterion6_through_layer(ref):
    """1000 criterion-6 instances through desmoe_layer_forward (DES-Vote, plus
    DES-Seq and vanilla on every third instance)."""
    from _exact_logits import hidden_for
    done = 0
    for i, m, n, k, act, beta, L in criterion6_instances(ref):
        check_case(ref, L, k, "vote", beta=beta, act=act, d=512)
        if i % 3 == 0:
            check_case(ref, L, k, "seq", seq_k=1 + i % k, act=act, d=512)
            check_case(ref, L, k, "vanilla", act=act, d=512)
        done += 1
    assert done == 1000


@pytest.mark.parametrize("d", [384, 640, 1664])
@pytest.mark.parametrize("strategy", ["vanilla", "seq", "vote"])
def test_ties_uneven_router_split(ref, d, strategy):
    """Hidden sizes that are not a multiple of 8 x 64: the router kernel splits
    the K blocks unevenly over its cluster (384: two CTAs get none) and the
    front reads the logits — injected exactly, routed exactly."""
    n, m = 64, 128
    check_case(ref, tied_levels(n, m, 11), 8, strategy, seq_k=2, beta=0.3, d=d)
    check_case(ref, near_ties(n, m, 12), 8, strategy, seq_k=3, beta=0.25, d=d)
