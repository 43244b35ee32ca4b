"""Deterministic synthetic inputs, bit-compatible with the reference's generators.

* ``Rng`` — splitmix64 (core.cpp:111-158): output i of Rng(seed) is
  mix64(seed + (i+1)*0x9E3779B97F4A7C15), so whole streams vectorise in numpy.
  Normals use the reference's Box-Muller pairing (cos first, cached sin).
* ``gen_trace_block`` — one block of gen_trace's shared_bias / iid models
  (trace.cpp:42-111), quantised to fp32 like the MOET file format.
* ``make_expert_bank`` — ExpertBank of make_expert_bank (gating.cpp:99-120).

The north-star SwiGLU experts and router weights have no reference
generator; ``swiglu_weights`` / ``router_weights`` draw them on the device with
a seeded torch generator (N(0,1)/sqrt(fan_in), bf16).
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def u64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Rng(seed).next_u64() outputs start .. start+count-1."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        return _mix64(np.uint64(seed) + k * GAMMA)


def mix(seed: int, stream: int) -> int:
    """Rng::mix (core.cpp:153-158)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + GAMMA * np.uint64(stream + 1)
        return int(_mix64(np.array([z], dtype=np.uint64))[0])


def normal_stream(seed: int, count: int) -> np.ndarray:
    """First `count` Rng(seed).next_normal() values (fresh generator)."""
    pairs = (count + 1) // 2
    u = u64_stream(seed, 2 * pairs)
    u1 = ((u[0::2] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (u[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    theta = 2.0 * 3.14159265358979323846 * u2
    out = np.empty(2 * pairs, np.float64)
    out[0::2] = r * np.cos(theta)
    out[1::2] = r * np.sin(theta)
    return out[:count]


def gen_trace_block(experts: int, block_size: int, seed: int, rho: float = 0.0,
                    tau: float = 1.0, model: str = "shared_bias", block_index: int = 0
                    ) -> np.ndarray:
    """Logits [block_size x experts] of block `block_index` = step*layers+layer."""
    s = mix(seed, block_index)
    m, n = experts, block_size
    if model == "iid_gaussian":
        v = tau * normal_stream(s, n * m)
    elif model == "shared_bias":
        z = normal_stream(s, m + n * m)
        bias, noise = z[:m], z[m:].reshape(n, m)
        v = tau * (rho * bias[None, :] + (1.0 - rho) * noise)
    else:
        raise ValueError(f"unsupported synth model: {model}")
    return v.reshape(n, m).astype(np.float32).astype(np.float64)


def random_block(block_size: int, experts: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """The reference tests' random_block (test_helpers.hpp:28-36)."""
    return scale * normal_stream(seed, block_size * experts).reshape(block_size, experts)


def make_expert_bank(experts: int, dim: int, block_size: int, seed: int):
    """(weights [experts x dim x dim], inputs [block_size x dim]) fp64."""
    z = normal_stream(seed, experts * dim * dim + block_size * dim)
    w = z[: experts * dim * dim].reshape(experts, dim, dim) * (1.0 / math.sqrt(dim))
    x = z[experts * dim * dim:].reshape(block_size, dim)
    return w, x


def swiglu_weights(experts: int, hidden: int, ffn: int, seed: int, device="cuda",
                   lo: int = 0, hi=None):
    """Random-init bf16 SwiGLU expert weights of experts [lo, hi) of an
    `experts`-expert pool: w_gate/w_up [hi-lo x F x d] ~ N(0,1)/sqrt(d),
    w_down [hi-lo x d x F] ~ N(0,1)/sqrt(F). Each (expert, matrix) has its own
    seed mix(seed, 3e + j), so a rank's shard equals the same slice of the
    full bank (expert parallelism needs no full copy)."""
    import torch

    hi = experts if hi is None else hi
    g = torch.Generator(device=device)
    out = []
    for j, (shape, fan) in enumerate((((ffn, hidden), hidden), ((ffn, hidden), hidden),
                                      ((hidden, ffn), ffn))):
        t = torch.empty((hi - lo,) + shape, dtype=torch.bfloat16, device=device)
        for e in range(lo, hi):  # per expert keeps the fp32 scratch small
            g.manual_seed(mix(seed, 3 * e + j) & ((1 << 63) - 1))
            t[e - lo] = (torch.randn(shape, generator=g, device=device) / math.sqrt(fan)).to(
                torch.bfloat16)
        out.append(t)
    return tuple(out)


def router_weights(experts: int, hidden: int, seed: int, device="cuda"):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn((experts, hidden), generator=g, device=device) / math.sqrt(hidden)).to(
        torch.bfloat16)


def hidden_states(block_size: int, hidden: int, seed: int, rho: float = 0.0, device="cuda"):
    """X[n, c] = bf16(rho * b_c + (1 - rho) * eps_{n,c}), b, eps ~ N(0,1)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    b = torch.randn((1, hidden), generator=g, device=device)
    eps = torch.randn((block_size, hidden), generator=g, device=device)
    return (rho * b + (1.0 - rho) * eps).to(torch.bfloat16)
