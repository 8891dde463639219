"""GPU timeline of one device-resident kNN step at C2 (torch.profiler / CUPTI):
kernel start offsets and durations relative to the step's first GPU activity,
to see launch gaps and host-side latency inside a bench step.

    python tools/trace_knn.py [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
dev = torch.device("cuda")
pts = lb.datasets.generate_device(lb.CloudSpec("cube", "filled", n, 0), dev)
qs = lb.datasets.generate_device(lb.CloudSpec("cube", "filled", n, 1), dev)
t = lb.build(pts)
for _ in range(3):
    lb.query_knn(t, (qs, 10))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        torch.cuda.synchronize()
        marker = torch.cuda.Event(enable_timing=True)
        marker.record()
        lb.query_knn(t, (qs, 10))
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
# the second step: events after the largest gap
gaps = [(evs[i + 1].time_range.start - evs[i].time_range.end, i) for i in range(len(evs) - 1)]
cut = max(gaps)[1] + 1
step = evs[cut:]
t0 = step[0].time_range.start
prev = t0
for e in step:
    print(f"{e.time_range.start - t0:9.1f} us  gap {e.time_range.start - prev:6.1f}  dur "
          f"{e.time_range.elapsed_us():8.1f}  {e.name[:60]}")
    prev = e.time_range.end
print(f"GPU span {step[-1].time_range.end - t0:.1f} us")
cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith("cuda")]
