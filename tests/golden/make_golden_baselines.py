"""Generates tests/golden/baselines_golden.npz from the REFERENCE library
itself (oracle/_ref/libdessim_ref.so -> dessim::baseline_route,
baselines.cpp:125-137): top-k reduce, NAEE and MC-MoE (both importance
scores) routes, IDs and gates bit-for-bit, on trace-generator logits at the
BASELINE shapes and on seeded random blocks.

    python tests/golden/make_golden_baselines.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref  # noqa: E402

# (method, k_reduced, naee_beta, mcmoe_beta, fraction, score)
PARAMS = [(0, 1, 0.5, 0.5, 0.5, 0), (0, 4, 0.5, 0.5, 0.5, 0), (1, 1, 0.3, 0.5, 0.5, 0),
          (1, 1, 0.7, 0.5, 0.5, 0), (2, 1, 0.5, 0.4, 0.5, 0), (2, 1, 0.5, 0.6, 0.25, 1)]


def main():
    ref = Ref()
    cases = []
    for m, k, n, rho in [(64, 8, 32, 0.3), (256, 8, 32, 0.5), (128, 8, 64, 0.0)]:
        cases.append((ref.gen_trace(m, k, n, seed=42, rho=rho)[0], k, 0))
    for i in range(4):
        r = ref.rng_u64(7150 + i, 3)
        m = 4 + int(r[0] % 200)
        n = 1 + int(r[1] % 48)
        k = 2 + int(r[2] % min(m - 1, 15))
        cases.append((1.5 * ref.rng_normal(8150 + i, n * m).reshape(n, m), k, 1 if i % 2 else 0))
    out = {"count": len(cases), "params": np.array(PARAMS, np.float64)}
    for i, (x, k, act) in enumerate(cases):
        out.update({f"x{i}": x, f"k{i}": k, f"act{i}": act})
        for j, (meth, kr, nb, mb, fr, sc) in enumerate(PARAMS):
            r = ref.baseline_route(x, k, meth, act, k_reduced=min(kr, k), naee_beta=nb,
                                   mcmoe_beta=mb, fraction=fr, score=sc)
            out.update({f"idx{i}_{j}": r.idx, f"gate{i}_{j}": r.gate, f"cnt{i}_{j}": r.cnt})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baselines_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({len(cases)} instances x {len(PARAMS)} policies)")


if __name__ == "__main__":
    main()
