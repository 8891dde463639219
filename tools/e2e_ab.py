"""A/B of the host kNN e2e path: median ms of query_knn(tree, (pinned host
centers, k)) at C2, alternating traversal switches in one process."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200 import traversal  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
qs = lb.generate(lb.CloudSpec("cube", "filled", n, 1))
pin = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
pin.numpy()[:] = qs
host_q = pin.numpy()
tree = lb.build(pts)
res = {0: [], 1: []}
for rep in range(12):
    for mode in (0, 1):
        traversal._HOST_OFFSETS = bool(mode)
        torch.cuda.synchronize()
        t = time.perf_counter()
        rs = lb.query_knn(tree, (host_q, 10))
        torch.cuda.synchronize()
        res[mode].append((time.perf_counter() - t) * 1e3)
        del rs
for mode in (0, 1):
    v = sorted(res[mode][2:])
    print(f"host_offsets={mode} median_ms={v[len(v) // 2]:.3f} min_ms={v[0]:.3f}")
