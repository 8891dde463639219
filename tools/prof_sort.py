"""Sort micro-benchmark: lbvh_sort_pairs (one-sweep LSD, 30 / 24-bit keys, iota
values) next to torch.sort(stable=True) (CUB) on the same 1e7 keys -- the
library figure is a yardstick for the pass cost, not a product path.

    python tools/prof_sort.py [n] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1908_11807_b200 import _device as dv, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
l = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(0)
src = torch.randint(0, 1 << 30, (n,), device="cuda", dtype=torch.int32, generator=g)
ws = torch.empty(l.lbvh_sort_workspace_bytes(n), dtype=torch.uint8, device="cuda")
keys = torch.empty_like(src)
vals = torch.empty_like(src)
iota = torch.arange(n, device="cuda", dtype=torch.int32)


def timed(fn):
    ts = []
    for _ in range(reps):
        keys.copy_(src)
        vals.copy_(iota)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for bits in (30, 24):
    ms = timed(lambda: _lib.check(l.lbvh_sort_pairs(dv.ptr(keys), dv.ptr(vals), n, bits,
                                                    dv.ptr(ws), ws.numel(), dv.stream())))
    print(f"lbvh_sort_pairs bits={bits} n={n} ms={ms:.4f} GB/s/pass="
          f"{16 * n / ((ms / ((bits + 7) // 8)) * 1e-3) / 1e9:.0f}")
ref = torch.sort(src.long() if False else src, stable=True)
ok = torch.equal(ref.indices.int(), (lambda: (keys.copy_(src), vals.copy_(iota), l.lbvh_sort_pairs(
    dv.ptr(keys), dv.ptr(vals), n, 30, dv.ptr(ws), ws.numel(), dv.stream()), vals)[-1])())
print("equal to torch.sort:", ok)
ms = timed(lambda: torch.sort(keys, stable=True))
print(f"torch.sort(stable) int32 n={n} ms={ms:.4f}")

if "--trace" in sys.argv:
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            keys.copy_(src)
            vals.copy_(iota)
            _lib.check(l.lbvh_sort_pairs(dv.ptr(keys), dv.ptr(vals), n, 30, dv.ptr(ws),
                                         ws.numel(), dv.stream()))
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs[-12:]:
        print(f"{(e.time_range.start - t0):9.1f} us  dur {e.time_range.elapsed_us():7.1f} us  {e.name[:60]}")
