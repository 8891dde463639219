"""kNN at 5e7 points (leaf directory of 24 bits: block seed at level 8) against
the CPU oracle on a query sample.

    python tools/check_knn_large.py [n] [sample]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from oracle import oracle  # noqa: E402  (checker only)
from paper_1908_11807_b200 import _lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 50_000_000
sample = int(float(sys.argv[2])) if len(sys.argv) > 2 else 200_000
pts = lb.generate(lb.CloudSpec("cube", "filled", n, 0))
qs = lb.generate(lb.CloudSpec("cube", "filled", n, 1))
print("directory bits", _lib.lib().lbvh_leaf_directory_bits(n))
t = lb.build(torch.from_numpy(pts).cuda())
dq = torch.from_numpy(qs).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
rs = lb.query_knn(t, (dq, 10))
torch.cuda.synchronize()
print(f"kNN {n} queries: {(time.perf_counter() - t0) * 1e3:.1f} ms")
h_idx = rs.indices.view(n, 10)[:sample].cpu().numpy()
h_dist = rs.distances.view(n, 10)[:sample].cpu().numpy()
ref = oracle.build(pts)
ko, ki, kd = oracle.query_knn(ref, qs[:sample], 10)
assert np.array_equal(h_idx.reshape(-1), ki), "indices differ"
assert h_dist.reshape(-1).tobytes() == kd.tobytes(), "distances differ"
print(f"ok: {sample} queries identical to the oracle")
