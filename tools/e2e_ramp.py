"""A/B of the kNN host pipeline's chunk ramp (e2e at C2, pinned host queries)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200 import traversal  # noqa: E402

n = 10_000_000
pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
qs = lb.generate(lb.CloudSpec("cube", "filled", n, 1))
pin = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
pin.numpy()[:] = qs
host_q = pin.numpy()
tree = lb.build(pts)
ramps = [0, 2, 3, 4, 5]
res = {r: [] for r in ramps}
for rep in range(10):
    for r in ramps:
        traversal._PIPELINE_RAMP = r
        torch.cuda.synchronize()
        t = time.perf_counter()
        rs = lb.query_knn(tree, (host_q, 10))
        torch.cuda.synchronize()
        res[r].append((time.perf_counter() - t) * 1e3)
        del rs
r_rad = lb.default_radius(10)
rres = {r: [] for r in ramps}
for rep in range(10):
    for r in ramps:
        traversal._RADIUS_RAMP = r
        torch.cuda.synchronize()
        t = time.perf_counter()
        rs = lb.query_spatial_2p(tree, (host_q, r_rad))
        torch.cuda.synchronize()
        rres[r].append((time.perf_counter() - t) * 1e3)
        del rs
for r, v in rres.items():
    v = sorted(v[2:])
    print(f"radius ramp={r} median_ms={v[len(v) // 2]:.3f} min_ms={v[0]:.3f}")
for r, v in res.items():
    v = sorted(v[2:])
    print(f"knn ramp={r} median_ms={v[len(v) // 2]:.3f} min_ms={v[0]:.3f}")
# a 800 MB device -> pinned host copy alone (the pipeline's bound)
d = torch.empty(200_000_000, dtype=torch.float32, device="cuda")
h = torch.empty(200_000_000, dtype=torch.float32, pin_memory=True)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
print(f"d2h 800MB min_ms={min(ts):.3f} GB/s={800 / min(ts):.1f}")
