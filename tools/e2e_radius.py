"""Host radius e2e at C2: median ms of query_spatial_2p(tree, (pinned host
centers, default_radius(10))) with numpy results."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
qs = lb.generate(lb.CloudSpec("cube", "filled", n, 1))
pin = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
pin.numpy()[:] = qs
tree = lb.build(pts)
r = lb.default_radius(10)
ts = []
chk = None
for _ in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rs = lb.query_spatial_2p(tree, (pin.numpy(), r))
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
    chk = (int(rs.offsets[-1]), int(rs.offsets[n // 2]), int(rs.indices[::9973].astype(np.int64).sum()))
    del rs
ts = sorted(ts[2:])
print(f"radius2p host e2e median_ms={ts[len(ts) // 2]:.3f} min_ms={ts[0]:.3f} check={chk}")
