"""A/B of the host pipelines' chunk size (kNN and radius 2P e2e at C2)."""
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
r = lb.default_radius(10)
sizes = [1 << 19, 1 << 20, 1 << 21]
res = {(op, c): [] for op in ("knn", "radius") for c in sizes}
for rep in range(8):
    for c in sizes:
        traversal._PIPELINE_CHUNK = c
        for op in ("knn", "radius"):
            torch.cuda.synchronize()
            t = time.perf_counter()
            rs = lb.query_knn(tree, (host_q, 10)) if op == "knn" else lb.query_spatial_2p(tree, (host_q, r))
            torch.cuda.synchronize()
            res[(op, c)].append((time.perf_counter() - t) * 1e3)
            del rs
for (op, c), v in res.items():
    v = sorted(v[2:])
    print(f"{op} chunk={c} median_ms={v[len(v) // 2]:.3f} min_ms={v[0]:.3f}")
