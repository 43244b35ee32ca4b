"""Stress test (GPU box): one acceptance-criterion-6 instance (default 897:
m=156, n=60, k=9, DES-Seq k=7) through the layer REPS times, each call
after a DES-Vote call on the same context, against the reference. It found a
barrier missing between the DES-Seq coreset flags' zeroing and setting
(front.cu V stage: ~1 wrong coreset / re-route in 1500 calls; 0 in 3000 after
the fix).

    REPS=3000 INST=897 python tools/c6_stress.py
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle.oracle import Ref
from test_gpu_parity import criterion6_instances, probe
ref = Ref()
target = int(os.environ.get("INST", "897"))
inst = None
for i, m, n, k, act, beta, L in criterion6_instances(ref):
    if i == target:
        inst = (i, m, n, k, act, beta, L)
        break
i, m, n, k, act, beta, L = inst
L64 = L.astype(np.float64)
seq_k = 1 + i % k
mem, want = ref.des_run(L64, k, "seq", seq_k=seq_k, act=act)
bad = 0
reps = int(os.environ.get("REPS", "500"))
for r in range(reps):
    if os.environ.get("PREV", "1") == "1":
        probe(512).run(L, k, "vote", beta=beta, act=act)
    got = probe(512).run(L, k, "seq", seq_k=seq_k, act=act)
    lg_ok = np.array_equal(got["logits"].view(np.uint32), L.view(np.uint32))
    ok = got["members"] == mem.tolist() and all(
        np.array_equal(got["idx"][t, :int(want.cnt[t])], want.idx[t, :int(want.cnt[t])]) for t in range(n))
    if not ok or not lg_ok:
        bad += 1
        if bad <= 3:
            bt = [t for t in range(n) if not np.array_equal(got["idx"][t, :int(want.cnt[t])], want.idx[t, :int(want.cnt[t])])]
            print("rep", r, "logits ok", lg_ok, "members ok", got["members"] == mem.tolist(), "bad tokens", bt, flush=True)
print(os.environ.get("TAG", ""), "bad", bad, "of", reps)
