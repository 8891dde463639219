"""compute-sanitizer target for the 2P radius path with heavy queries
(hollow-sphere sources: rows overflow, warp-cooperative heavy pass, spill
chunks, count-only and serial fallbacks at large radii); results compared
with the C oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_heavy.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from oracle import oracle  # noqa: E402

pts = lb.generate(lb.CloudSpec("sphere", "hollow", 60_000, 0))
qs = lb.generate(lb.CloudSpec("sphere", "filled", 3_000, 4))
t, ref = lb.build(pts), oracle.build(pts)
for scale in (1.0, 4.0, 12.0):
    r = lb.default_radius(10) * scale
    rs = lb.query_spatial_2p(t, (qs, r))
    off, idx = oracle.query_spatial_2p(ref, qs, r)
    cnt = np.diff(off)
    print(f"scale {scale}: max hits {cnt.max()}, queries > 48 hits {(cnt > 48).sum()}, "
          f"offsets {np.array_equal(rs.offsets, off)}, indices {np.array_equal(rs.indices, idx)}",
          flush=True)
