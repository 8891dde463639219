"""Small end-to-end run of every kernel, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200.tree import Topology, refit_bounds  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
pts = lb.generate(lb.CloudSpec("cube", "filled", n, 0))
qs = lb.generate(lb.CloudSpec("sphere", "hollow", n // 2, 1))
t = lb.build(pts)
rows = np.concatenate([pts, pts + 0.5], axis=1)
tb = lb.build(rows)
r = lb.default_radius(10)
rs = lb.query_spatial_2p(t, (qs, r))
rs1, fb = lb.query_spatial_1p(t, (qs, r), 4)
rs2, fb2 = lb.query_spatial_1p(t, (qs, r), 64)
rk = lb.query_knn(t, (qs, 10))
rk2 = lb.query_knn(t, (qs, np.arange(1, qs.shape[0] + 1) % 40 + 1))
rk3 = lb.query_knn(tb, (qs, 50))
topo = lb.generate_topology(np.sort(lb.morton_codes(pts, t.scene_min, t.scene_max)))
mins, maxs = t.node_mins.copy(), t.node_maxs.copy()
refit_bounds(mins, maxs, topo)
user = lb.Bvh(t.node_mins, t.node_maxs, t.left, t.right, t.leaf_obj, t.scene_min, t.scene_max)
ru = lb.query_knn(user, (qs, 7))
order = lb.query_sort_order(qs, t.scene)
torch.cuda.synchronize()
print("sanitize smoke ok", int(rs.offsets[-1]), fb, fb2, rk.indices.shape, rk3.indices.shape)
