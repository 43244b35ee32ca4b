"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/desmoe.h declares, and its host-only validation
reproduces the reference's messages (core.cpp:11-28, des.cpp:29-31). No
kernel is launched here."""
import os
import re

import pytest

from paper_2602_00879_b200 import _lib
from paper_2602_00879_b200 import dessim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "desmoe.h")).read()
    return sorted(set(re.findall(r"\b(desmoe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 18
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(_lib.exported_symbols()) == decl


def test_validate_pool_messages():
    with pytest.raises(ValueError, match="top_k > experts_total"):
        dessim.validate_config(dessim.PoolConfig(8, 9))
    with pytest.raises(ValueError, match="bytes_per_expert == 0"):
        dessim.validate_config(dessim.PoolConfig(8, 2, bytes_per_expert=0))
    with pytest.raises(ValueError, match="hidden_dim < 1"):
        dessim.validate_config(dessim.PoolConfig(8, 2, hidden_dim=0))
    with pytest.raises(ValueError):
        dessim.validate_config(dessim.PoolConfig(0, 1))
    dessim.validate_config(dessim.PoolConfig(64, 8))
    dessim.validate_config(dessim.PoolConfig(1, 1))


def test_vote_budget_floor():
    assert [dessim.vote_budget(b, m) for b, m in
            [(0.15, 256), (0.10, 256), (0.6, 64), (0.4, 64), (1.0, 64)]] == [38, 25, 38, 25, 64]


def test_validate_params_messages():
    cfg = dessim.PoolConfig(4, 2)
    with pytest.raises(ValueError, match="seq_k < 1"):
        dessim.validate_params(dessim.DesParams(dessim.DesStrategy.seq, 0, 1.0), cfg)
    with pytest.raises(ValueError, match="seq_k > top_k"):
        dessim.validate_params(dessim.DesParams(dessim.DesStrategy.seq, 3, 1.0), cfg)
    with pytest.raises(ValueError, match=r"vote_beta outside \(0, 1\]"):
        dessim.validate_params(dessim.DesParams(dessim.DesStrategy.vote, 1, 0.0), cfg)
    with pytest.raises(ValueError, match=r"vote budget floor\(beta\*M\) < 1"):
        dessim.validate_params(dessim.DesParams(dessim.DesStrategy.vote, 1, 0.1), cfg)


def test_router_block_factory():
    with pytest.raises(ValueError, match="non-finite logit"):
        dessim.make_router_block(1, 2, [0.0, float("inf")])
    with pytest.raises(ValueError, match="logits size"):
        dessim.make_router_block(2, 2, [0.0, 1.0, 2.0])
    b = dessim.make_router_block(1, 3, [1, 2, 3])
    assert b.row(0).tolist() == [1.0, 2.0, 3.0]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    b = dessim.make_router_block(1, 4, [3, 2, 1, 0])
    with pytest.raises(_lib.DesmoeError, match="no CPU fallback"):
        dessim.activate(b, dessim.PoolConfig(4, 2))


def test_synthetic_generators_match_reference(ref):
    from paper_2602_00879_b200 import synth
    import numpy as np
    assert np.array_equal(synth.u64_stream(0, 3), ref.rng_u64(0, 3))
    for rho in (0.0, 0.3, 0.5):
        assert np.array_equal(synth.gen_trace_block(64, 32, 42, rho=rho),
                              ref.gen_trace(64, 8, 32, 42, rho=rho)[0])
    w, x = synth.make_expert_bank(3, 8, 4, 77)
    w2, x2 = ref.make_expert_bank(3, 8, 4, 77)
    # numpy's log/sin/cos may differ from glibc in the last bit
    assert np.abs(w - w2).max() <= 1e-15 and np.abs(x - x2).max() <= 1e-15
