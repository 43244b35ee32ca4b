"""Generates tests/golden/des_golden.npz from the REFERENCE library itself
(oracle/_ref/libdessim_ref.so, compiled from /root/reference/proj/core/src).

Instances: trace-generator logits (gen_trace shared_bias, trace.cpp:42-111)
at the BASELINE configs' shapes plus criterion-6-style random blocks, so the
fixtures pin vanilla / DES-Vote / DES-Seq IDs, gates and votes bit-for-bit.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref  # noqa: E402


def main():
    ref = Ref()
    cases = []
    # (m, k, n, rho, beta, seq_k, act) — BASELINE configs C1/C2 (M=64), C3 (M=256), C4 (M=128)
    for m, k, n, rho, beta, seq_k in [(64, 8, 32, 0.3, 0.4, 3), (64, 8, 32, 0.3, 0.6, 2),
                                      (256, 8, 32, 0.5, 0.15, 3), (256, 8, 8, 0.0, 0.10, 2),
                                      (128, 8, 32, 0.0, 0.3, 3), (256, 8, 64, 0.5, 0.15, 3)]:
        x = ref.gen_trace(m, k, n, seed=42, rho=rho)[0]
        cases.append((x, k, 0, beta, seq_k))
    for i in range(6):
        r = ref.rng_u64(5150 + i, 4)
        m = 2 + int(r[0] % 300)
        n = 1 + int(r[1] % 40)
        k = 1 + int(r[2] % min(m, 16))
        act = 1 if i % 3 == 0 else 0
        x = 1.5 * ref.rng_normal(6150 + i, n * m).reshape(n, m)
        cases.append((x, k, act, min(1.0, (1 + int(r[3] % m) + 0.5) / m), max(1, k // 2)))
    out = {"count": len(cases)}
    for i, (x, k, act, beta, seq_k) in enumerate(cases):
        mem, r = ref.des_run(x, k, "vote", beta=beta, act=act)
        _, votes = ref.vote_coreset(x, k, beta, act)
        smem, sr = ref.des_run(x, k, "seq", seq_k=seq_k, act=act)
        v = ref.topk_route(x, k, act)
        out.update({f"x{i}": x, f"k{i}": k, f"act{i}": act, f"beta{i}": beta,
                    f"seqk{i}": seq_k, f"vote_mem{i}": mem, f"vote_idx{i}": r.idx,
                    f"vote_gate{i}": r.gate, f"votes{i}": votes, f"seq_mem{i}": smem,
                    f"seq_idx{i}": sr.idx, f"seq_gate{i}": sr.gate, f"van_idx{i}": v.idx,
                    f"van_gate{i}": v.gate})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "des_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({len(cases)} instances)")


if __name__ == "__main__":
    main()
