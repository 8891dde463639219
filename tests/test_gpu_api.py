"""The reference's own test strategy (pkg/tests/test_build.py,
test_traversal.py, test_acceptance.py, test_estimator.py) run against the
GPU package through its public API."""

import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import paper_1908_11807_b200 as lb
from oracle import oracle
from paper_1908_11807_b200 import Box, KnnQuery, Point, SpatialQuery

from helpers import in_order_leaves

pytestmark = pytest.mark.gpu

LINE4 = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]], dtype=np.float32)


@pytest.fixture(scope="module")
def line_tree():
    return lb.build(LINE4)


@pytest.fixture(scope="module")
def cloud():
    return np.random.default_rng(42).uniform(-5, 5, size=(1000, 3)).astype(np.float32)


@pytest.fixture(scope="module")
def cloud_tree(cloud):
    return lb.build(cloud)


def sorted_sets(rs):
    return [np.sort(rs.hits(q)).tolist() for q in range(rs.query_count)]


def assert_tree_invariants(tree):
    """pkg/tests/test_build.py:28-57"""
    n = tree.leaf_count
    assert tree.node_count == 2 * n - 1
    assert sorted(tree.leaf_obj.tolist()) == list(range(n))
    if n == 1:
        return
    indegree = np.bincount(np.concatenate([tree.left, tree.right]), minlength=2 * n - 1)
    assert indegree[0] == 0 and (indegree[1:] == 1).all()
    seen = np.zeros(2 * n - 1, dtype=bool)
    stack = [0]
    while stack:
        node = stack.pop()
        assert not seen[node]
        seen[node] = True
        if not tree.is_leaf(node):
            stack.extend(tree.children(node))
    assert seen.all()
    left, right = tree.left, tree.right
    assert (tree.node_mins[: n - 1] <= tree.node_mins[left]).all()
    assert (tree.node_mins[: n - 1] <= tree.node_mins[right]).all()
    assert (tree.node_maxs[: n - 1] >= tree.node_maxs[left]).all()
    assert (tree.node_maxs[: n - 1] >= tree.node_maxs[right]).all()
    assert (tree.node_mins[0] == tree.scene_min).all()
    assert (tree.node_maxs[0] == tree.scene_max).all()


# --------------------------------------------------------------- build


def test_single_box_and_small_trees():
    t = lb.build(np.float32([[0.5, 0.5, 0.5]]))
    assert t.leaf_count == 1 and t.internal_count == 0 and t.node_count == 1
    assert t.node_box(0) == Box.from_point(Point(0.5, 0.5, 0.5))
    t = lb.build(np.array([[0, 0, 0, 1, 1, 1], [2, 2, 2, 3, 3, 3]], dtype=np.float32))
    assert t.node_box(0) == Box(Point(0, 0, 0), Point(3, 3, 3))
    pts = [[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    t = lb.build(np.float32(pts))
    assert (t.leaf_count, t.internal_count, t.node_count) == (8, 7, 15)
    assert_tree_invariants(lb.build(np.float32([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]])))


def test_empty_and_invalid_inputs():
    with pytest.raises(ValueError, match="empty scene"):
        lb.build(np.empty((0, 3), dtype=np.float32))
    with pytest.raises(ValueError, match="finite"):
        lb.build(np.float32([[0, 0, 0], [np.inf, 0, 0]]))
    with pytest.raises(ValueError, match="min corner above"):
        lb.build(np.float32([[1, 0, 0, 0, 1, 1]]))


@pytest.mark.parametrize("pos", [0, 517, 998, 999])
def test_device_build_flags_nonfinite_points(pos):
    # device input skips the host validation: the scene-reduce kernel's checks
    # (vectorised 4-point steps and the scalar tail) must flag every position
    pts = np.random.default_rng(3).uniform(-1, 1, size=(1000, 3)).astype(np.float32)
    pts[pos, pos % 3] = np.nan if pos % 2 else np.inf
    with pytest.raises(ValueError, match="finite"):
        lb.build(torch.from_numpy(pts).cuda())


@pytest.mark.parametrize("pos", [0, 1234, 4999])
def test_device_knn_flags_nonfinite_centers(pos):
    # device centers: the fused prologue (value check + offsets + Morton codes)
    # of the one-call kNN batch must flag a bad center anywhere in the batch
    pts = np.random.default_rng(4).uniform(-1, 1, size=(2000, 3)).astype(np.float32)
    t = lb.build(pts)
    qs = np.random.default_rng(5).uniform(-1, 1, size=(5000, 3)).astype(np.float32)
    qs[pos, 2 - pos % 3] = np.inf if pos % 2 else np.nan
    with pytest.raises(ValueError, match="finite"):
        lb.query_knn(t, (torch.from_numpy(qs).cuda(), 7))
    good = torch.from_numpy(np.nan_to_num(qs, posinf=0.5, nan=0.25)).cuda()
    rs = lb.query_knn(t, (good, 7))
    assert torch.equal(rs.offsets.cpu(), torch.arange(5001, dtype=torch.int64) * 7)


@pytest.mark.parametrize("pos", [0, 2500, 4999])
def test_device_radius_flags_nonfinite_centers(pos):
    # scalar radius on device centers: the value check is fused into the
    # query Morton pass of the one-call count stage
    pts = np.random.default_rng(6).uniform(-1, 1, size=(2000, 3)).astype(np.float32)
    t = lb.build(pts)
    qs = np.random.default_rng(7).uniform(-1, 1, size=(5000, 3)).astype(np.float32)
    qs[pos, pos % 3] = -np.inf if pos % 2 else np.nan
    for run in (lambda q: lb.query_spatial_2p(t, (q, 0.1)),
                lambda q: lb.query_spatial_1p(t, (q, 0.1), 16)):
        with pytest.raises(ValueError, match="finite"):
            run(torch.from_numpy(qs).cuda())


def test_leaves_in_morton_sorted_order():
    pts = np.random.default_rng(11).uniform(-3, 3, size=(200, 3)).astype(np.float32)
    t = lb.build(pts)
    codes = lb.morton_codes(pts, t.scene_min, t.scene_max)
    assert in_order_leaves(t.left, t.right, t.leaf_obj) == np.argsort(codes, kind="stable").tolist()


def test_deterministic_rebuild_and_frozen_arrays():
    pts = np.random.default_rng(5).uniform(0, 1, size=(500, 3)).astype(np.float32)
    a, b = lb.build(pts), lb.build(pts, threads=2)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes()
    with pytest.raises(ValueError):
        a.node_mins[0, 0] = 5.0


def test_duplicates_extremes_and_box_sequences():
    assert_tree_invariants(lb.build(np.tile(np.float32([2.5, -1.0, 0.25]), (64, 1))))
    big = 3e38
    pts = np.float32([[-big, -big, -big], [big, big, big], [0, 0, 0], [big, -big, 0]])
    assert_tree_invariants(lb.build(pts))
    assert_tree_invariants(lb.build(np.float32([[3e38, 3e38, 3e38], [0, 0, 0]])))
    t = lb.build([Box(Point(0, 0, 0), Point(1, 1, 1)), Box(Point(2, 2, 2), Point(3, 3, 3))])
    assert t.node_box(0) == Box(Point(0, 0, 0), Point(3, 3, 3))


@settings(deadline=None, max_examples=40)
@given(st.lists(st.tuples(st.integers(-100, 100), st.integers(-100, 100),
                          st.integers(-100, 100)), min_size=1, max_size=120))
def test_invariants_and_oracle_identity_for_arbitrary_clouds(rows):
    pts = np.array(rows, dtype=np.float32)
    t = lb.build(pts)
    assert_tree_invariants(t)
    ref = oracle.build(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), f


# --------------------------------------------------------------- traversal


def test_single_query_paths(line_tree):
    hits = []
    assert lb.traverse_spatial_one(line_tree, SpatialQuery(Point(0, 0, 0), 1.5), hits.append) == 2
    assert sorted(hits) == [0, 1]
    assert lb.traverse_spatial_one(line_tree, SpatialQuery(Point(10, 10, 10), 0.1)) == 0
    hits = []
    assert lb.traverse_spatial_one(line_tree, SpatialQuery(Point(0, 0, 0), 0.0), hits.append) == 1
    assert hits == [0]
    got = lb.traverse_knn_one(line_tree, KnnQuery(Point(0.1, 0, 0), 2))
    assert [o for o, _ in got] == [0, 1]
    assert got[0][1] == pytest.approx(0.1, rel=1e-6) and got[1][1] == pytest.approx(0.9, rel=1e-6)
    assert lb.traverse_knn_one(line_tree, KnnQuery(Point(2, 0, 0), 1)) == [(2, 0.0)]
    assert [o for o, _ in lb.traverse_knn_one(line_tree, KnnQuery(Point(0, 0, 0), 10))] == [0, 1, 2, 3]
    t = lb.build(np.float32([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0]]))
    assert [o for o, _ in lb.traverse_knn_one(t, KnnQuery(Point(0, 0, 0), 2))] == [0, 1]
    t1 = lb.build(np.array([[1, 1, 1]], dtype=np.float32))
    assert lb.traverse_spatial_one(t1, SpatialQuery(Point(1, 1, 1), 0.0)) == 1
    assert lb.traverse_spatial_one(t1, SpatialQuery(Point(5, 1, 1), 1.0)) == 0


def test_spatial_2p_offsets_and_forms(line_tree):
    qs = [SpatialQuery(Point(0, 0, 0), 1.0), SpatialQuery(Point(9, 9, 9), 0.5),
          SpatialQuery(Point(1, 0, 0), 1.2)]
    rs = lb.query_spatial_2p(line_tree, qs)
    assert rs.offsets.tolist() == [0, 2, 2, 5]
    rs = lb.query_spatial_2p(line_tree, [])
    assert rs.offsets.tolist() == [0] and rs.indices.size == 0
    assert sorted_sets(lb.query_spatial_2p(line_tree, (LINE4, 0.5))) == [[0], [1], [2], [3]]
    rs = lb.query_spatial_2p(line_tree, (LINE4[:2], np.float32([0.5, 1.5])))
    assert sorted_sets(rs) == [[0], [0, 1, 2]]
    assert rs.distances is None
    with pytest.raises(ValueError, match="finite"):
        lb.query_spatial_2p(line_tree, (np.float32([[np.nan, 0, 0]]), 1.0))
    with pytest.raises(ValueError, match="non-negative"):
        lb.query_spatial_2p(line_tree, (LINE4[:2], np.float32([0.5, -1])))


def test_spatial_matches_brute_force(cloud_tree, cloud):
    centers = np.random.default_rng(0).uniform(-6, 6, size=(200, 3)).astype(np.float32)
    rs = lb.query_spatial_2p(cloud_tree, (centers, 1.5))
    expected = oracle.brute_radius_sets(cloud, centers, 1.5)
    for q in range(200):
        assert np.array_equal(np.sort(rs.hits(q)), expected[q])


def test_spatial_1p_semantics(cloud_tree, cloud, line_tree):
    rs1, fb = lb.query_spatial_1p(cloud_tree, (cloud[:200], 1.5), buffer_size=64)
    base = lb.query_spatial_2p(cloud_tree, (cloud[:200], 1.5))
    assert not fb and sorted_sets(rs1) == sorted_sets(base)
    rs, fb = lb.query_spatial_1p(line_tree, [SpatialQuery(Point(1.5, 0, 0), 2.0)], buffer_size=1)
    assert fb and sorted_sets(rs) == [[0, 1, 2, 3]]
    rs, fb = lb.query_spatial_1p(line_tree, (np.float32([[50, 50, 50], [60, 60, 60]]), 0.5), 8)
    assert not fb and rs.offsets.tolist() == [0, 0, 0]
    counts = lb.query_spatial_2p(cloud_tree, (cloud[:250], 1.5)).counts()
    for b in (1, 2, 4, 32, int(counts.max()), int(counts.max()) + 1):
        r, fb = lb.query_spatial_1p(cloud_tree, (cloud[:250], 1.5), b)
        assert fb == bool((counts > b).any())
        assert sorted_sets(r) == sorted_sets(lb.query_spatial_2p(cloud_tree, (cloud[:250], 1.5)))
    with pytest.raises(ValueError):
        lb.query_spatial_1p(line_tree, (LINE4, 1.0), buffer_size=0)


def test_knn_semantics(cloud_tree, cloud):
    rs = lb.query_knn(cloud_tree, (cloud, 1))
    assert rs.indices.tolist() == list(range(1000)) and (rs.distances == 0).all()
    t = lb.build(np.float32([[0, 0, 0], [1, 1, 1]]))
    assert lb.query_knn(t, (np.float32([[0, 0, 0], [5, 5, 5], [9, 9, 9]]), 3)).counts().tolist() == [2, 2, 2]
    rs = lb.query_knn(cloud_tree, (cloud[:100], 8))
    for q in range(100):
        assert (np.diff(rs.hit_distances(q)) >= 0).all()
    pts = np.tile(np.float32([1, 2, 3]), (50, 1))
    rs = lb.query_knn(lb.build(pts), (pts[:3], 7))
    assert rs.counts().tolist() == [7, 7, 7] and (rs.distances == 0).all()
    for q in range(3):
        assert rs.hits(q).tolist() == list(range(7))
    with pytest.raises(ValueError, match=">= 1"):
        lb.query_knn(cloud_tree, (cloud[:3], np.int64([1, 0, 2])))
    e = lb.query_knn(cloud_tree, [])
    assert e.offsets.tolist() == [0] and e.distances.size == 0


def test_knn_equals_brute_force(cloud_tree, cloud):
    centers = np.random.default_rng(9).uniform(-6, 6, size=(150, 3)).astype(np.float32)
    rs = lb.query_knn(cloud_tree, (centers, 10))
    wi, wd = oracle.brute_knn_batch(cloud, centers, 10)
    for q in range(150):
        assert np.array_equal(rs.hits(q), wi[q])
        assert np.allclose(rs.hit_distances(q), wd[q], rtol=1e-6, atol=0)


def test_query_ordering(cloud_tree, cloud):
    smin, smax = cloud_tree.scene_min, cloud_tree.scene_max
    t = np.linspace(0.05, 0.95, 7, dtype=np.float32)[:, None]
    assert lb.query_sort_order(smin + t * (smax - smin), (smin, smax)).tolist() == list(range(7))
    centers = np.stack([smax, smin])
    assert lb.query_sort_order(centers, (smin, smax)).tolist() == [1, 0]
    assert lb.query_sort_order(centers, cloud_tree.scene).tolist() == [1, 0]
    c = np.random.default_rng(13).uniform(-5, 5, size=(333, 3)).astype(np.float32)
    on = lb.query_spatial_2p(cloud_tree, (c, 1.1), sort_queries=True)
    off = lb.query_spatial_2p(cloud_tree, (c, 1.1), sort_queries=False)
    assert np.array_equal(on.offsets, off.offsets) and sorted_sets(on) == sorted_sets(off)
    on = lb.query_knn(cloud_tree, (c, 4), sort_queries=True)
    off = lb.query_knn(cloud_tree, (c, 4), sort_queries=False)
    assert np.array_equal(on.indices, off.indices) and np.array_equal(on.distances, off.distances)


def make_pathological_tree(n=80):
    """pkg/tests/test_traversal.py:288-302"""
    internal = n - 1
    left = np.arange(1, n, dtype=np.int32)
    right = np.arange(1, n, dtype=np.int32)
    left[-1] = internal
    right[-1] = internal + 1
    zeros = np.zeros((2 * n - 1, 3), dtype=np.float32)
    return lb.Bvh(zeros, zeros.copy(), left, right, np.arange(n, dtype=np.int32),
                  np.zeros(3, dtype=np.float32), np.zeros(3, dtype=np.float32))


def test_stack_guard():
    tree = make_pathological_tree()
    z = np.zeros((1, 3), dtype=np.float32)
    with pytest.raises(RuntimeError, match="traversal stack exhausted"):
        lb.query_spatial_2p(tree, (z, 1.0))
    with pytest.raises(RuntimeError, match="traversal stack exhausted"):
        lb.query_spatial_1p(tree, (z, 1.0), 8)
    with pytest.raises(RuntimeError, match="traversal stack exhausted"):
        lb.query_knn(tree, (z, 1))
    with pytest.raises(RuntimeError, match="traversal stack exhausted"):
        lb.traverse_spatial_one(tree, SpatialQuery(Point(0, 0, 0), 1.0))
    with pytest.raises(RuntimeError, match="traversal stack exhausted"):
        lb.traverse_knn_one(tree, KnnQuery(Point(0, 0, 0), 1))


def test_user_built_tree_matches_built_tree(cloud_tree, cloud):
    t = cloud_tree
    copy = lb.Bvh(t.node_mins, t.node_maxs, t.left, t.right, t.leaf_obj, t.scene_min, t.scene_max)
    c = cloud[:300]
    a = lb.query_knn(t, (c, 9))
    b = lb.query_knn(copy, (c, 9))
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.distances, b.distances)
    a = lb.query_spatial_2p(t, (c, 1.3))
    b = lb.query_spatial_2p(copy, (c, 1.3))
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)


def test_volumetric_knn_box_distances():
    tree = lb.build((np.float32([[0, 0, 0], [10, 0, 0]]), np.float32([[4, 4, 4], [11, 1, 1]])))
    rk = lb.query_knn(tree, (np.float32([[5, 0, 0]]), 2))
    assert rk.hits(0).tolist() == [0, 1]
    assert rk.hit_distances(0) == pytest.approx([1.0, 5.0])


def test_soak_ten_thousand_points():
    rng = np.random.default_rng(99)
    pts = rng.uniform(-10, 10, size=(10_000, 3)).astype(np.float32)
    centers = rng.uniform(-11, 11, size=(500, 3)).astype(np.float32)
    tree = lb.build(pts)
    for r in (0.5, 2.0, 6.0):
        rs = lb.query_spatial_2p(tree, (centers, r))
        expected = oracle.brute_radius_sets(pts, centers, r)
        for q in range(500):
            assert np.array_equal(np.sort(rs.hits(q)), expected[q])
    rk = lb.query_knn(tree, (centers, 10))
    wi, wd = oracle.brute_knn_batch(pts, centers, 10)
    for q in range(500):
        assert np.array_equal(rk.hits(q), wi[q])


@settings(deadline=None, max_examples=25)
@given(st.lists(st.tuples(st.integers(-40, 40), st.integers(-40, 40), st.integers(-40, 40)),
                min_size=1, max_size=80),
       st.lists(st.tuples(st.integers(-50, 50), st.integers(-50, 50), st.integers(-50, 50)),
                min_size=1, max_size=20),
       st.integers(0, 20), st.integers(1, 12))
def test_oracle_equivalence_property(src_rows, centers_rows, radius, k):
    pts = np.array(src_rows, dtype=np.float32)
    centers = np.array(centers_rows, dtype=np.float32)
    tree = lb.build(pts)
    rs = lb.query_spatial_2p(tree, (centers, float(radius)))
    expected = oracle.brute_radius_sets(pts, centers, float(radius))
    for q in range(len(centers)):
        assert np.array_equal(np.sort(rs.hits(q)), expected[q])
    rk = lb.query_knn(tree, (centers, k))
    wi, wd = oracle.brute_knn_batch(pts, centers, k)
    for q in range(len(centers)):
        assert np.allclose(rk.hit_distances(q), wd[q], rtol=1e-6, atol=0)
        assert np.array_equal(rk.hits(q), wi[q])


# --------------------------------------------------------------- acceptance

SHAPES = ["cube:filled", "cube:hollow", "sphere:filled", "sphere:hollow"]


def _cloud(spec, n, seed):
    return lb.generate(lb.CloudSpec.parse(spec, n, seed))


def test_criterion_1_structural():
    for spec in SHAPES:
        for n in (1, 2, 3, 10, 1000, 100_000):
            pts = _cloud(spec, n, 17)
            t = lb.build(pts)
            assert t.node_count == 2 * n - 1 and t.leaf_count == n
            assert (t.node_mins[0] == pts.min(axis=0)).all()
            assert (t.node_maxs[0] == pts.max(axis=0)).all()
            codes = lb.morton_codes(pts, t.scene_min, t.scene_max)
            if n <= 1000:
                assert in_order_leaves(t.left, t.right, t.leaf_obj) == \
                    np.argsort(codes, kind="stable").tolist()
            ref = oracle.build(pts)
            for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
                assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), (spec, n, f)


def test_criterion_3_5_7():
    src, tgt = _cloud("cube:filled", 10_000, 2), _cloud("sphere:filled", 10_000, 3)
    tree, r = lb.build(src), lb.default_radius(10)
    base = lb.query_spatial_2p(tree, (tgt, r))
    counts = base.counts()
    for b in (1, 4, 32):
        rs, fb = lb.query_spatial_1p(tree, (tgt, r), b)
        assert sorted_sets(rs) == sorted_sets(base) and fb == bool((counts > b).any())
    ft = lb.build(_cloud("cube:filled", 100_000, 6))
    mean = lb.query_spatial_2p(ft, (_cloud("sphere:filled", 100_000, 7), r)).counts().mean()
    assert 9.0 <= mean <= 11.0
    pts = np.tile(np.float32([0.5, -2.0, 3.25]), (10_000, 1))
    t = lb.build(pts)
    rs = lb.query_spatial_2p(t, (pts[:8], 0.0))
    assert (rs.counts() == 10_000).all()
    for q in range(8):
        assert np.array_equal(np.sort(rs.hits(q)), np.arange(10_000))
    rk = lb.query_knn(t, (pts[:8], 10))
    assert (rk.counts() == 10).all() and (rk.distances == 0.0).all()


def test_estimator_facade():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError

    cloud = np.random.default_rng(21).uniform(-4, 4, size=(600, 3)).astype(np.float32)
    est = lb.BvhNeighbors(n_neighbors=5)
    assert est.fit(cloud) is est and est.n_samples_fit_ == 600
    with pytest.raises(NotFittedError):
        lb.BvhNeighbors().kneighbors(cloud[:2])
    rs = est.kneighbors(cloud[:50])
    wi, _ = oracle.brute_knn_batch(cloud, cloud[:50], 5)
    for q in range(50):
        assert np.array_equal(rs.hits(q), wi[q])
    a = lb.BvhNeighbors(radius=1.0).fit(cloud).radius_neighbors(cloud[:80])
    b = lb.BvhNeighbors(radius=1.0, buffer_size=4).fit(cloud).radius_neighbors(cloud[:80])
    assert sorted_sets(a) == sorted_sets(b)
    assert (lb.BvhNeighbors(radius=0.0).fit(cloud).radius_neighbors(cloud[:5], radius=100.0)
            .counts() == 600).all()
    assert clone(est).get_params() == est.get_params()
    with pytest.raises(TypeError):
        est.query([SpatialQuery(Point(0, 0, 0), 1.0), KnnQuery(Point(0, 0, 0), 1)])


def test_brute_force_helpers_match_reference_semantics():
    """oracle.py KATs (pkg/tests/test_oracle.py) and numpy brute force."""
    assert lb.brute_radius(np.float32([[0, 0, 0], [3, 0, 0]]),
                           SpatialQuery(Point(0, 0, 0), 1.0)).tolist() == [0]
    assert lb.brute_radius(np.float32([[1, 1, 1], [2, 2, 2], [1, 1, 1]]),
                           SpatialQuery(Point(1, 1, 1), 0.0)).tolist() == [0, 2]
    idx, dist = lb.brute_knn(np.float32([[0, 0, 0], [2, 0, 0], [1, 0, 0]]),
                             KnnQuery(Point(0, 0, 0), 3))
    assert idx.tolist() == [0, 2, 1] and dist.tolist() == [0.0, 1.0, 2.0]
    idx, _ = lb.brute_knn(np.float32([[1, 0, 0], [-1, 0, 0], [0, 1, 0]]), KnnQuery(Point(0, 0, 0), 2))
    assert idx.tolist() == [0, 1]
    rng = np.random.default_rng(5)
    pts = rng.integers(-20, 21, size=(3000, 3)).astype(np.float32)
    cs = rng.integers(-25, 26, size=(200, 3)).astype(np.float32)
    for k in (1, 10, 33, 70):
        wi, wd = oracle.brute_knn_batch(pts, cs, k)
        gi, gd = lb.brute_knn_batch(pts, cs, k)
        assert np.array_equal(gi, wi) and gd.tobytes() == wd.tobytes(), k
    for r in (0.0, 2.0, 7.5):
        want = oracle.brute_radius_sets(pts, cs, r)
        got = lb.brute_radius_sets(pts, cs, r)
        assert all(np.array_equal(a, b) for a, b in zip(got, want)), r
