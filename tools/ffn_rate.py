"""Weight-streaming rate of the expert FFN over time, from a raw timeline
(tools/ffn_trace.py --raw out.npz): every unit's weight bytes spread evenly
over [dequeue, epilogue done], summed in 1 us bins -> TB/s. The unit map is
rebuilt as the kernel builds it (phase-A / phase-B pairs at the head of the
queue, the last split_a / split_b pairs as single tiles; capi.cu ffn_impl).

    python tools/ffn_rate.py trace.npz --d 2048 --f 1024 --u 25 [--dense]
"""
import argparse

import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("npz")
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--f", type=int, default=1024)
    ap.add_argument("--u", type=int, required=True)
    ap.add_argument("--sms", type=int, default=148)
    ap.add_argument("--pairs", type=int, default=1, help="pair units enabled (dense / routed pairs)")
    args = ap.parse_args()
    z = np.load(args.npz)
    ev, unit, t = z["ev"], z["unit"], z["t"]
    d, f, U = args.d, args.f, args.u
    tilesA, tilesB = f // 64, d // 128
    pa = pw = 2 if args.pairs else 1
    nAs = min(args.sms, U * (tilesA // 2)) if pa == 2 else 0
    nAp = U * (tilesA // pa) - nAs
    nA = nAp + pa * nAs
    nBs = min(args.sms // 2, U * (tilesB // 2)) if pw == 2 else 0
    nBp = U * (tilesB // pw) - nBs
    a_tile = 2 * 64 * d * 2   # gate + up rows of one 64-wide F tile
    b_tile = 128 * f * 2      # one 128-row d tile of W_d

    def nbytes(u):
        if u < nA:
            return 2 * a_tile if u < nAp else a_tile
        b = u - nA
        return 2 * b_tile if b < nBp else b_tile

    deq = {int(u): float(x) for u, x, e in zip(unit, t, ev) if e == 2}
    done = {int(u): float(x) for u, x, e in zip(unit, t, ev) if e == 3}
    t1 = max(done.values())
    bins = np.zeros(int(np.ceil(t1)) + 1)
    total = 0
    for u, s in deq.items():
        if u not in done:
            continue
        e = done[u]
        b = nbytes(u)
        total += b
        lo, hi = s, max(e, s + 1e-3)
        for k in range(int(lo), int(np.ceil(hi))):
            ov = min(hi, k + 1) - max(lo, k)
            if ov > 0:
                bins[k] += b * ov / (hi - lo)
    rate = bins / 1e-6 / 1e12  # TB/s per 1 us bin
    print(f"units {len(deq)} (A {nA}: {nAp} pairs; B {nBp} pairs + {nBs * pw} singles), "
          f"weight bytes {total / 1e6:.1f} MB (algorithmic {U * (tilesA * a_tile + tilesB * b_tile) / 1e6:.1f})")
    for k in range(0, len(rate), 2):
        print(f"{k:4d}-{k + 2:<4d} us  {np.mean(rate[k:k + 2]):5.2f} TB/s")


if __name__ == "__main__":
    main()
