"""C3 radius cost split: time query_spatial_2p on all C3 queries, on the
light ones (hits <= the 48-hit row) and on the heavy ones, each batch in its
original order (device-resident, CUDA events, L2 flushed).

    python tools/c3_split.py [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
pts = torch.from_numpy(lb.generate(lb.CloudSpec("sphere", "hollow", n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
t = lb.build(pts)
r = lb.default_radius(10)
rs = lb.query_spatial_2p(t, (qs, r))
cnt = (rs.offsets[1:] - rs.offsets[:-1])
heavy = cnt > 48
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(q, reps=5):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lb.query_spatial_2p(t, (q, r))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


qa, ql, qh = qs, qs[~heavy].contiguous(), qs[heavy].contiguous()
from paper_1908_11807_b200 import traversal  # noqa: E402
print(f"heavy queries {int(heavy.sum())} ({float(heavy.float().mean()):.4f}), hits in heavy "
      f"{float(cnt[heavy].sum()) / float(cnt.sum()):.3f}")
print(f"all {timed(qa):.3f} ms  light {timed(ql):.3f} ms  heavy {timed(qh):.3f} ms")
traversal._SPILL_INTS = 1200  # heavy-only batches need ~1000 pool ints per query
print(f"heavy, pool sized for it: {timed(qh):.3f} ms")
