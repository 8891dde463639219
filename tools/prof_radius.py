"""Driver for ncu: build a 1e7 filled-cube tree, then run 2P radius queries
(1e7 queries, default radius for k=10) -- covers hierarchy, one-sweep and
spatial kernels in one short process."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
pts = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
for _ in range(2):
    t = lb.build(pts)
    rs = lb.query_spatial_2p(t, (qs, lb.default_radius(10)))
torch.cuda.synchronize()
print("hits", int(rs.offsets[-1]))
