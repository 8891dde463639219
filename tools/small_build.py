"""Host-path cost of small builds (C5 low end): CUDA-event time of
lb.build on device-resident points vs the summed kernel time of the same
call (torch.profiler / CUPTI), at n = 1e4 and 1e5.

    python tools/small_build.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["10000", "100000"])]:
    pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
    for _ in range(5):
        lb.build(pts)
    torch.cuda.synchronize()
    reps = 50
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        lb.build(pts)
    host = (time.perf_counter() - t0) / reps
    b.record()
    torch.cuda.synchronize()
    ev = a.elapsed_time(b) / reps
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            lb.build(pts)
        torch.cuda.synchronize()
    kern = sum(e.device_time_total for e in prof.key_averages()) / 10 / 1e3
    names = sorted(((e.device_time_total / 10, e.key) for e in prof.key_averages()), reverse=True)
    print(f"n={n}: event ms/build {ev:.4f}  host ms/build {host * 1e3:.4f}  "
          f"kernel ms/build {kern:.4f}")
    for t, k in names[:14]:
        print(f"    {t:8.1f} us  {k[:90]}")
