"""63-bit Morton option (north_star "30/63-bit"; not in the reference).

Parity is pinned by our own restatement: the oracle's orc_morton63_codes /
orc_build63 (checked here against an independent Python bit-by-bit encoder
and against the 30-bit reference codes, which are its top 30 bits), and the
GPU build is compared with that oracle byte for byte.  Query results do not
depend on the tree shape, so they must equal the reference's exactly.
"""

import numpy as np
import pytest

from oracle import oracle
from paper_1908_11807_b200 import datasets

from helpers import sorted_concat


def _py_code63(p, lo, hi):
    code = 0
    cells = []
    for a in range(3):
        ext = float(hi[a]) - float(lo[a])
        t = (float(p[a]) - float(lo[a])) / ext if ext > 0 else 0.0
        t = min(max(t, 0.0), 1.0)
        cells.append(min(int(t * 2097152.0), 2097151))
    for b in range(21):
        for a in range(3):
            code |= ((cells[a] >> b) & 1) << (3 * b + (2 - a))
    return code


def test_oracle_code63_matches_bitwise_encoder_and_30bit_prefix():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-5, 7, size=(500, 3)).astype(np.float32)
    lo, hi = pts.min(0), pts.max(0)
    c63 = oracle.morton63_codes(pts, lo, hi)
    assert [int(c) for c in c63[:50]] == [_py_code63(p, lo, hi) for p in pts[:50]]
    c30 = oracle.morton_codes(pts, lo, hi)
    assert np.array_equal((c63 >> np.uint64(33)).astype(np.uint32), c30)
    big = np.float32([[-3e38] * 3, [3e38] * 3, [0, 0, 0], [3e38, -3e38, 0]])
    e63 = oracle.morton63_codes(big, big.min(0), big.max(0))
    assert int(e63[0]) == 0 and int(e63[1]) == (1 << 63) - 1


def test_oracle_build63_invariants():
    pts = datasets.generate(datasets.CloudSpec("sphere", "hollow", 5000, 2))
    t = oracle.build63(pts)
    codes = oracle.morton63_codes(pts, t.scene_min, t.scene_max)
    assert np.array_equal(t.leaf_obj, np.lexsort((np.arange(5000), codes)).astype(np.int32))
    n = 5000
    indeg = np.bincount(np.concatenate([t.left, t.right]), minlength=2 * n - 1)
    assert indeg[0] == 0 and (indeg[1:] == 1).all()
    assert (t.node_mins[0] == pts.min(0)).all() and (t.node_maxs[0] == pts.max(0)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("shape,n", [("cube:filled", 200_000), ("sphere:hollow", 100_000),
                                     ("cube:filled", 3)])
def test_gpu_build63_equals_oracle_and_queries_unchanged(shape, n):
    import paper_1908_11807_b200 as lb

    pts = datasets.generate(datasets.CloudSpec.parse(shape, n, 5))
    t = lb.build(pts, morton_bits=63)
    ref = oracle.build63(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), f
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 20_000, 6))
    r = datasets.default_radius(10)
    t30 = oracle.build(pts)
    rs = lb.query_spatial_2p(t, (q, r))
    off, idx = oracle.query_spatial_2p(t30, q, r)
    assert np.array_equal(rs.offsets, off)
    assert np.array_equal(sorted_concat(rs.offsets, rs.indices), sorted_concat(off, idx))
    rk = lb.query_knn(t, (q, 10))
    ko, ki, kd = oracle.query_knn(t30, q, 10)
    assert np.array_equal(rk.indices, ki) and rk.distances.tobytes() == kd.tobytes()
