"""Per-query node-visit statistics of the kNN kernel (instrumentation builds
with -DLBVH_KNN_COUNT_VISITS: the nearest distance slot carries the query's
node-visit count; the warp-packet experiment wrote minus its per-warp count).

    LBVH_LIB=paper_1908_11807_b200/_lib/variants/visits.so python tools/knn_visits.py [n] [src]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
src = sys.argv[2] if len(sys.argv) > 2 else "sphere"
kind = "hollow" if src == "sphere" else "filled"
pts = torch.from_numpy(lb.generate(lb.CloudSpec(src, kind, n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
t = lb.build(pts)
rs = lb.query_knn(t, (qs, 10))
v = rs.distances.view(-1, 10)[:, 0].cpu().numpy()
pk = v < 0
v = np.abs(v)
order = lb.query_sort_order(qs.cpu().numpy(), (t.scene_min, t.scene_max))
print(f"n={n} src={src} packet_queries={pk.mean():.4f}")
for name, sel in (("thread", ~pk), ("packet(per warp)", pk)):
    if sel.any():
        x = v[sel]
        print(f"{name}: count={sel.sum()} mean={x.mean():.0f} p50={np.percentile(x, 50):.0f} "
              f"p90={np.percentile(x, 90):.0f} p99={np.percentile(x, 99):.0f} max={x.max():.0f} "
              f"sum={x.sum():.3e}")
# warp view of the per-thread path: warp cost = max lane visits
vv = v[order] if len(order) == len(v) else v
w = vv[: len(vv) // 32 * 32].reshape(-1, 32)
print(f"warp max-lane visits: mean={w.max(1).mean():.0f}  warp mean-lane: {w.mean(1).mean():.0f}")
