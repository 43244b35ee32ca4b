"""HBM probes on the GPU box: torch copy / read-reduction bandwidth, to put the
expert-FFN stream rate in context."""
import json
import torch


def timeit(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.normal_()
out = {}
t = timeit(lambda: b.copy_(a))
out["copy_GBps"] = 2 * a.numel() * 2 / t / 1e9
t = timeit(lambda: a.sum(dtype=torch.float32))
out["read_sum_GBps"] = a.numel() * 2 / t / 1e9
c = a[: 300 << 19]  # 300 MiB
t = timeit(lambda: c.sum(dtype=torch.float32))
out["read_300MiB_GBps"] = c.numel() * 2 / t / 1e9
out["read_300MiB_us"] = t * 1e6
print(json.dumps(out))
