"""A/B of the 2P row width at two radii (C2 sizes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200 import traversal  # noqa: E402

n = 10_000_000
pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
t = lb.build(pts)
for kk in (10, 30):
    r = lb.default_radius(kk)
    for rows in (24, 32, 48, 64):
        traversal._ROW_HITS = rows
        ts = []
        for rep in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rs = lb.query_spatial_2p(t, (qs, r))
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts = sorted(ts[1:])
        print(f"hits~{kk} rows={rows} median_ms={ts[len(ts) // 2]:.3f} total={int(rs.offsets[-1])}")
