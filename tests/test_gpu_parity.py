"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the CPU oracle.  Integer/index results must be
bit-exact; kNN distances too (same fp32 recipe, correctly rounded sqrt)."""

import numpy as np
import pytest
import torch

import paper_1908_11807_b200 as lb
from oracle import oracle
from paper_1908_11807_b200 import datasets

from helpers import assert_same_tree, in_order_leaves, sha16, sorted_concat

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["line4", "cloud", "ext", "dup"])
def test_tree_bitwise_equals_reference(golden, case):
    tree = lb.build(golden[case + "_pts"])
    assert_same_tree(tree, golden, case + "_")


def test_volumetric_boxes(golden):
    tree = lb.build((golden["vol_mins"], golden["vol_maxs"]))
    assert_same_tree(tree, golden, "vol_")
    rs = lb.query_spatial_2p(tree, (golden["vol_centers"], np.float32(1.7)))
    assert np.array_equal(rs.offsets, golden["vol_sp_offsets"])
    assert np.array_equal(sorted_concat(rs.offsets, rs.indices), golden["vol_sp_sorted_indices"])
    rk = lb.query_knn(tree, (golden["vol_centers"], 7))
    assert np.array_equal(rk.indices, golden["vol_knn_indices"])
    assert rk.distances.tobytes() == golden["vol_knn_distances"].tobytes()


def test_boxes_as_n6_rows_equal_pair_form(golden):
    rows = np.concatenate([golden["vol_mins"], golden["vol_maxs"]], axis=1)
    assert_same_tree(lb.build(rows), golden, "vol_")


def test_morton_codes_bitwise(golden):
    pts = golden["morton_pts"]
    z, one = np.zeros(3, np.float32), np.ones(3, np.float32)
    assert np.array_equal(lb.morton_codes(pts, z, one), golden["morton_codes_unit"])
    assert np.array_equal(lb.morton_codes(pts, z, np.float32([1, 0, 1])),
                          golden["morton_codes_flat"])
    t = lb.build(golden["ext_pts"])
    codes = lb.morton_codes(golden["ext_pts"], t.scene_min, t.scene_max)
    assert codes.tolist() == [0, 1073741823, 939524096, 747784484]


@pytest.mark.parametrize("prefix", ["topo", "topod"])
def test_generate_topology_bitwise(golden, prefix):
    topo = lb.generate_topology(golden[prefix + "_codes"])
    assert np.array_equal(topo.left, golden[prefix + "_left"])
    assert np.array_equal(topo.right, golden[prefix + "_right"])
    assert np.array_equal(topo.parent, golden[prefix + "_parent"])


def test_refit_bounds_matches_reference(golden):
    """refit_bounds (tree.py:108-119) on the reference's own topology and leaf
    rows (the goldens, not a GPU build) must reproduce the reference's
    internal boxes byte for byte."""
    from paper_1908_11807_b200.tree import refit_bounds, Topology

    left, right = golden["cloud_left"], golden["cloud_right"]
    n = golden["cloud_leaf_obj"].shape[0]
    mins = golden["cloud_node_mins"].copy()
    maxs = golden["cloud_node_maxs"].copy()
    mins[: n - 1] = 0
    maxs[: n - 1] = 0
    parent = np.full(2 * n - 1, -1, np.int32)
    parent[left] = np.arange(n - 1)
    parent[right] = np.arange(n - 1)
    refit_bounds(mins, maxs, Topology(left, right, parent))
    assert mins.tobytes() == golden["cloud_node_mins"].tobytes()
    assert maxs.tobytes() == golden["cloud_node_maxs"].tobytes()


def test_cloud_queries_against_reference(golden):
    tree = lb.build(golden["cloud_pts"])
    c = golden["cloud_sp_centers"]
    rs = lb.query_spatial_2p(tree, (c, 1.5))
    assert rs.offsets.dtype == np.int64 and rs.indices.dtype == np.int32
    assert np.array_equal(rs.offsets, golden["cloud_sp_offsets"])
    assert np.array_equal(sorted_concat(rs.offsets, rs.indices), golden["cloud_sp_sorted_indices"])
    rs = lb.query_spatial_2p(tree, (c, golden["cloud_spr_radii"]))
    assert np.array_equal(sorted_concat(rs.offsets, rs.indices), golden["cloud_spr_sorted_indices"])
    for b in (1, 4, 32):
        r1, fb = lb.query_spatial_1p(tree, (c, 1.5), b)
        assert fb == bool(golden[f"cloud_1p{b}_fellback"])
        assert np.array_equal(sorted_concat(r1.offsets, r1.indices),
                              golden[f"cloud_1p{b}_sorted_indices"])
    kc = golden["cloud_knn_centers"]
    for tag, k, cs in (("cloud_knn_", 10, kc), ("cloud_knnk_", golden["cloud_knnk_ks"], kc),
                       ("cloud_knn100_", 100, kc[:40])):
        rk = lb.query_knn(tree, (cs, k))
        assert np.array_equal(rk.offsets, golden[tag + "offsets"]), tag
        assert np.array_equal(rk.indices, golden[tag + "indices"]), tag
        assert rk.distances.tobytes() == golden[tag + "distances"].tobytes(), tag
    assert np.array_equal(lb.query_sort_order(c, (tree.scene_min, tree.scene_max)),
                          golden["cloud_order"])


def test_integer_clouds_with_heavy_ties(golden):
    for i in range(int(golden["int_ncases"])):
        p = f"int{i}_"
        tree = lb.build(golden[p + "pts"])
        assert_same_tree(tree, golden, p)
        cs = golden[p + "centers"]
        rs = lb.query_spatial_2p(tree, (cs, golden[p + "r"]))
        assert np.array_equal(rs.offsets, golden[p + "sp_offsets"])
        assert np.array_equal(sorted_concat(rs.offsets, rs.indices), golden[p + "sp_sorted_indices"])
        rk = lb.query_knn(tree, (cs, int(golden[p + "k"])))
        assert np.array_equal(rk.indices, golden[p + "knn_indices"]), p
        assert rk.distances.tobytes() == golden[p + "knn_distances"].tobytes(), p


@pytest.mark.parametrize("name", ["c1_filled", "c3_hollow_sphere", "hollow_cube"])
def test_reference_digests_c1_scale(digests, name):
    d = digests[name]
    pts = datasets.generate(datasets.CloudSpec.parse(d["source"], d["m"], d["seed"]))
    q = datasets.generate(datasets.CloudSpec.parse(d["target"], d["m"], d["target_seed"]))
    t = lb.build(pts)
    assert t.scene_min.tolist() == d["scene_min"] and t.scene_max.tolist() == d["scene_max"]
    for f in ("leaf_obj", "left", "right", "node_mins", "node_maxs"):
        assert sha16(getattr(t, f)) == d[f], f
    assert sha16(lb.morton_codes(pts, t.scene_min, t.scene_max)) == d["codes"]
    rs = lb.query_spatial_2p(t, (q, d["radius"]))
    assert sha16(rs.offsets) == d["sp_offsets"] and int(rs.offsets[-1]) == d["sp_total"]
    assert sha16(sorted_concat(rs.offsets, rs.indices)) == d["sp_sorted_indices"]
    rk = lb.query_knn(t, (q, d["k"]))
    assert sha16(rk.indices) == d["knn_indices"] and sha16(rk.distances) == d["knn_distances"]
    assert sha16(lb.query_sort_order(q, (t.scene_min, t.scene_max))) == d["query_order"]


@pytest.mark.parametrize("shape", ["cube:filled", "sphere:hollow", "cube:hollow"])
def test_against_oracle_unsorted_hit_order(shape):
    """Traversal order is the reference's, so even the unsorted CRS equals
    the oracle's byte for byte."""
    pts = datasets.generate(datasets.CloudSpec.parse(shape, 200_000, 3))
    q = datasets.generate(datasets.CloudSpec.parse("sphere:filled", 50_000, 4))
    t, ref = lb.build(pts), oracle.build(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), f
    r = datasets.default_radius(10)
    rs = lb.query_spatial_2p(t, (q, r))
    off, idx = oracle.query_spatial_2p(ref, q, r)
    assert np.array_equal(rs.offsets, off) and np.array_equal(rs.indices, idx)
    for k in (1, 5, 10, 16, 31, 50):
        rk = lb.query_knn(t, (q[:20_000], k))
        ko, ki, kd = oracle.query_knn(ref, q[:20_000], k)
        assert np.array_equal(rk.indices, ki), k
        assert rk.distances.tobytes() == kd.tobytes(), k


def test_device_resident_inputs_and_outputs():
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 50_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 10_000, 1))
    th = lb.build(pts)
    td = lb.build(torch.from_numpy(pts).cuda())
    assert th.node_mins.tobytes() == td.node_mins.tobytes()
    qd = torch.from_numpy(q).cuda()
    rk = lb.query_knn(td, (qd, 10))
    assert rk.on_device and rk.indices.is_cuda
    hk = lb.query_knn(th, (q, 10))
    assert np.array_equal(rk.to_host().indices, hk.indices)
    rs = lb.query_spatial_2p(td, (qd, 2.0))
    assert np.array_equal(rs.to_host().offsets, lb.query_spatial_2p(th, (q, 2.0)).offsets)


@pytest.mark.parametrize("kind", ["cube:filled", "sphere:hollow", "clustered"])
def test_leaf_directory_is_lower_bound_of_bucket_starts(kind):
    """The kNN seed's leaf directory: entry p = lower_bound(p << (30 - bits))
    over the sorted leaf codes, including empty buckets; kNN with and
    without it returns identical results (equal to the oracle)."""
    if kind == "clustered":
        rng = np.random.default_rng(5)
        pts = np.concatenate([rng.normal(c, 0.01, size=(4000, 3)) for c in (-50, 0, 3, 70)])
        pts = pts.astype(np.float32)
    else:
        src, k = kind.split(":")
        pts = datasets.generate(datasets.CloudSpec(src, k, 30_000, 0))
    tree = lb.build(pts)
    d = tree.device_arrays()
    codes = d["leaf_codes"].cpu().numpy().view(np.uint32).astype(np.int64)
    ld = d["leaf_dir"].cpu().numpy().view(np.uint32).astype(np.int64)
    bits = (ld.shape[0] - 1).bit_length() - 1
    assert ld.shape[0] == (1 << bits) + 1
    targets = np.arange((1 << bits) + 1, dtype=np.int64) << (30 - bits)
    assert np.array_equal(ld, np.searchsorted(codes, targets, side="left"))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 5_000, 1)) * 0.5
    ko, ki, kd = oracle.query_knn(oracle.build(pts), q, 10)
    rk = lb.query_knn(tree, (q, 10))
    assert np.array_equal(rk.indices, ki) and rk.distances.tobytes() == kd.tobytes()
    del d["leaf_dir"]  # seed falls back to the full binary search
    rk2 = lb.query_knn(tree, (q, 10))
    assert np.array_equal(rk2.indices, ki) and rk2.distances.tobytes() == kd.tobytes()


@pytest.mark.parametrize("shape,variant,count,seed", [
    ("cube", "filled", 100_000, 0), ("cube", "filled", 100_000, 1), ("cube", "filled", 12_345, 7),
    ("cube", "hollow", 100_000, 0), ("cube", "hollow", 9_999, 3),
    ("sphere", "hollow", 100_000, 0), ("sphere", "hollow", 10_001, 5),
    ("sphere", "filled", 5_000, 2), ("cube", "filled", 1, 0)])
def test_device_generators_match_host(shape, variant, count, seed):
    spec = datasets.CloudSpec(shape, variant, count, seed)
    host = datasets.generate(spec)
    dev = datasets.generate_device(spec)
    assert dev.is_cuda and dev.cpu().numpy().tobytes() == host.tobytes()


@pytest.mark.parametrize("k", [11, 16, 17, 24, 32, 33, 64, 400, 401])
def test_knn_list_sizes_against_oracle(k):
    """Every kNN kernel size class (register lists, shared-memory heap up to
    k = 400, global-memory heap beyond) returns the reference's spans."""
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 20_000, 0))
    pts[100:110] = pts[5]  # exact distance ties across ordinals
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 3_000, 1))
    q[0] = pts[5]
    ko, ki, kd = oracle.query_knn(oracle.build(pts), q, k)
    rk = lb.query_knn(lb.build(pts), (q, k))
    assert np.array_equal(rk.offsets, ko)
    assert np.array_equal(rk.indices, ki)
    assert rk.distances.tobytes() == kd.tobytes()


@pytest.mark.parametrize("budget_rows", [0, 12])
def test_radius_2p_without_or_with_narrow_rows(monkeypatch, budget_rows):
    """2P without a row buffer (budget exhausted: count -> scan -> full fill,
    the reference's scheme) and with rows narrower than most spans must give
    the same CRS as the default path."""
    from paper_1908_11807_b200 import traversal

    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 50_000, 0))
    q = torch.from_numpy(datasets.generate(datasets.CloudSpec("cube", "filled", 20_000, 1))).cuda()
    t = lb.build(pts)
    r = lb.default_radius(20)
    ref = lb.query_spatial_2p(t, (q, r)).to_host()
    if budget_rows == 0:
        monkeypatch.setattr(traversal, "_ROW_BUDGET", 1)
    else:
        monkeypatch.setattr(traversal, "_ROW_HITS", budget_rows)
    got = lb.query_spatial_2p(t, (q, r)).to_host()
    assert np.array_equal(got.offsets, ref.offsets)
    assert np.array_equal(got.indices, ref.indices)


@pytest.mark.parametrize("radius", [0.0, 2.673, 4.5])
def test_pipelined_host_radius_equals_device_path(radius):
    """Large pinned host 2P batches run chunked (software-pipelined count /
    fill / D2H); the CRS must equal the one-shot device path byte for byte
    (4.5 gives ~38 hits per query: row overflows and host buffer growth)."""
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 300_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", (1 << 20) * 2 + 777, 1)) * 0.4
    t = lb.build(pts)
    pin = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
    pin.numpy()[:] = q
    host = lb.query_spatial_2p(t, (pin.numpy(), radius))
    dev = lb.query_spatial_2p(t, (torch.from_numpy(q).cuda(), radius)).to_host()
    assert isinstance(host.offsets, np.ndarray)
    assert np.array_equal(host.offsets, dev.offsets)
    assert np.array_equal(host.indices, dev.indices)
    ref = oracle.build(pts)
    so, si = oracle.query_spatial_2p(ref, q[-3000:], radius)
    base = int(host.offsets[-3001])
    assert np.array_equal(host.offsets[-3001:] - base, so)
    assert np.array_equal(host.indices[base:], si)
    unsorted = lb.query_spatial_2p(t, (pin.numpy(), radius), sort_queries=False)
    assert np.array_equal(unsorted.offsets, host.offsets)


def test_pipelined_host_knn_equals_device_path():
    """Large pinned host batches take the chunked H2D/compute/D2H pipeline;
    results must equal the one-shot device path and the oracle."""
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 400_000, 0))
    q = datasets.generate(datasets.CloudSpec("sphere", "filled", (1 << 20) + 12345, 1))
    t = lb.build(pts)
    pin = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
    pin.numpy()[:] = q
    from paper_1908_11807_b200 import _device
    assert _device.is_pinned(pin.numpy())
    for k in (1, 10):
        host = lb.query_knn(t, (pin.numpy(), k))
        dev = lb.query_knn(t, (torch.from_numpy(q).cuda(), k)).to_host()
        assert np.array_equal(host.offsets, dev.offsets)
        assert np.array_equal(host.indices, dev.indices)
        assert host.distances.tobytes() == dev.distances.tobytes()
    ref = oracle.build(pts)
    ko, ki, kd = oracle.query_knn(ref, q[-5000:], 10)
    assert np.array_equal(host.indices[-50000:], ki)
    unsorted = lb.query_knn(t, (pin.numpy(), 10), sort_queries=False)
    assert np.array_equal(unsorted.indices, host.indices)


@pytest.mark.parametrize("kmax", [8, 16, 40])
def test_per_query_k_device_tensors_against_oracle(kmax):
    """Per-query k as a CUDA tensor: spans of min(k_q, n), register lists or the
    shared-memory heap chosen by max(k), identical to the reference."""
    rng = np.random.default_rng(kmax)
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 30_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 4_000, 1))
    ks = rng.integers(1, kmax + 1, size=q.shape[0])
    ko, ki, kd = oracle.query_knn(oracle.build(pts), q, ks)
    rk = lb.query_knn(lb.build(pts), (torch.from_numpy(q).cuda(), torch.from_numpy(ks).cuda()))
    h = rk.to_host()
    assert np.array_equal(h.offsets, ko)
    assert np.array_equal(h.indices, ki)
    assert h.distances.tobytes() == kd.tobytes()


def test_per_query_radii_device_tensors_2p_and_1p():
    pts = datasets.generate(datasets.CloudSpec("sphere", "hollow", 30_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", 4_000, 1)) * 0.3
    radii = np.random.default_rng(3).uniform(0.0, 4.0, size=q.shape[0]).astype(np.float32)
    ref = oracle.build(pts)
    so, si = oracle.query_spatial_2p(ref, q, radii)
    t = lb.build(pts)
    qd, rd = torch.from_numpy(q).cuda(), torch.from_numpy(radii).cuda()
    rs = lb.query_spatial_2p(t, (qd, rd)).to_host()
    assert np.array_equal(rs.offsets, so) and np.array_equal(rs.indices, si)
    r1, fb = lb.query_spatial_1p(t, (qd, rd), 8)
    o1, i1, fb1 = oracle.query_spatial_1p(ref, q, radii, 8)
    r1 = r1.to_host()
    assert fb == fb1 and np.array_equal(r1.offsets, o1)
    assert np.array_equal(sorted_concat(r1.offsets, r1.indices), sorted_concat(o1, i1))


@pytest.mark.parametrize("k", [10, 20, 100])
def test_all_duplicate_points_tie_order(k):
    """10,000 copies of one point (test_acceptance.py:171): every distance ties,
    so spans are decided by ordinal alone -- in every kernel size class."""
    pts = np.tile(np.array([[0.5, -2.0, 3.25]], dtype=np.float32), (10_000, 1))
    q = np.array([[0.5, -2.0, 3.25], [10.0, 10.0, 10.0], [-3.0, 0.0, 1.0]], dtype=np.float32)
    ko, ki, kd = oracle.query_knn(oracle.build(pts), q, k)
    rk = lb.query_knn(lb.build(pts), (q, k))
    assert np.array_equal(rk.offsets, ko)
    assert np.array_equal(rk.indices, ki)
    assert rk.distances.tobytes() == kd.tobytes()
    assert np.array_equal(rk.indices[:k], np.arange(k, dtype=np.int32))


@pytest.mark.parametrize("k", [3, 10, 20])
def test_extreme_magnitudes_infinite_distances(k):
    """Coordinates near +-3e38 (test_build.py:220-233): squared distances
    overflow to +inf, so many candidates tie at inf and the ordinal decides --
    register lists and the shared-memory heap must agree with the reference."""
    rng = np.random.default_rng(11)
    pts = (rng.uniform(-1, 1, size=(200, 3)) * 3e38).astype(np.float32)
    pts[:4] = [[-3e38] * 3, [3e38] * 3, [0, 0, 0], [3e38, -3e38, 0]]
    q = (rng.uniform(-1, 1, size=(64, 3)) * 3e38).astype(np.float32)
    ref = oracle.build(pts)
    t = lb.build(pts)
    ko, ki, kd = oracle.query_knn(ref, q, k)
    rk = lb.query_knn(t, (q, k))
    assert np.array_equal(rk.offsets, ko)
    assert np.array_equal(rk.indices, ki)
    assert rk.distances.tobytes() == kd.tobytes()
    so, si = oracle.query_spatial_2p(ref, q, 1e38)
    rs = lb.query_spatial_2p(t, (q, 1e38))
    assert np.array_equal(rs.offsets, so) and np.array_equal(rs.indices, si)


@pytest.mark.parametrize("k", [5, 24])
def test_volumetric_boxes_knn_and_radius_device(k):
    """(n, 6) box leaves given as a CUDA tensor: point-to-box distances (0 inside
    a box, so heavy ties at 0) through the fused device calls."""
    rng = np.random.default_rng(21)
    lo = rng.uniform(-20, 20, size=(5_000, 3)).astype(np.float32)
    hi = lo + rng.uniform(0, 3, size=(5_000, 3)).astype(np.float32)
    rows = np.concatenate([lo, hi], axis=1)
    q = rng.uniform(-22, 22, size=(2_000, 3)).astype(np.float32)
    ref = oracle.build(rows)
    t = lb.build(torch.from_numpy(rows).cuda())
    ko, ki, kd = oracle.query_knn(ref, q, k)
    h = lb.query_knn(t, (torch.from_numpy(q).cuda(), k)).to_host()
    assert np.array_equal(h.offsets, ko) and np.array_equal(h.indices, ki)
    assert h.distances.tobytes() == kd.tobytes()
    so, si = oracle.query_spatial_2p(ref, q, 1.5)
    rs = lb.query_spatial_2p(t, (torch.from_numpy(q).cuda(), 1.5)).to_host()
    assert np.array_equal(rs.offsets, so) and np.array_equal(rs.indices, si)


@pytest.mark.parametrize("shape,radius_scale", [("sphere:hollow", 1.0), ("sphere:hollow", 4.0),
                                                ("cube:filled", 3.0)])
def test_heavy_queries_spill_pool(shape, radius_scale, monkeypatch):
    """Queries with more hits than the 2P row (48) keep the rest in the spill
    pool during the count pass (no second traversal); with the pool too small
    they fall back to the fill pass.  Counts, offsets and the UNSORTED hit
    order must be the reference's (oracle) either way, for scalar and
    per-query radii, device and host batches, and the 1P fallback."""
    pts = datasets.generate(datasets.CloudSpec.parse(shape, 200_000, 3))
    q = datasets.generate(datasets.CloudSpec.parse("cube:filled", 40_003, 4))
    t, ref = lb.build(pts), oracle.build(pts)
    r = np.float32(datasets.default_radius(10) * radius_scale)
    off, idx = oracle.query_spatial_2p(ref, q, r)
    assert int(np.diff(off).max()) > 48  # heavy queries exist
    rs = lb.query_spatial_2p(t, (q, r))
    assert np.array_equal(rs.offsets, off) and np.array_equal(rs.indices, idx)
    rd = lb.query_spatial_2p(t, (torch.from_numpy(q).cuda(), r))
    assert np.array_equal(rd.offsets.cpu().numpy(), off)
    assert np.array_equal(rd.indices.cpu().numpy(), idx)
    rr = np.random.default_rng(5).uniform(0, 2 * r, q.shape[0]).astype(np.float32)
    rr[::7] = 0.0
    off2, idx2 = oracle.query_spatial_2p(ref, q, rr)
    rs2 = lb.query_spatial_2p(t, (q, rr))
    assert np.array_equal(rs2.offsets, off2) and np.array_equal(rs2.indices, idx2)
    rs3, fb = lb.query_spatial_1p(t, (q, r), 16)
    assert fb and np.array_equal(rs3.offsets, off) and np.array_equal(rs3.indices, idx)
    rs4 = lb.query_spatial_2p(t, (q, r), sort_queries=False)
    assert np.array_equal(rs4.offsets, off) and np.array_equal(rs4.indices, idx)
    # a pool of 64 chunks runs dry: the queries that find it exhausted are refilled
    from paper_1908_11807_b200 import traversal

    monkeypatch.setattr(traversal, "_SPILL_INTS", 0)
    rs5 = lb.query_spatial_2p(t, (q, r))
    assert np.array_equal(rs5.offsets, off) and np.array_equal(rs5.indices, idx)


def test_heavy_queries_pipelined_host_batch():
    """A pinned host batch above the pipeline threshold (2^20 queries) with
    heavy queries: chunked count (+ spill pool) / compaction / spill copy /
    D2H."""
    pts = datasets.generate(datasets.CloudSpec("sphere", "hollow", 300_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", (1 << 20) + 4097, 1))
    t, ref = lb.build(pts), oracle.build(pts)
    r = np.float32(datasets.default_radius(10) * 2.0)
    pin = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
    pin.numpy()[:] = q
    rs = lb.query_spatial_2p(t, (pin.numpy(), r))
    off, idx = oracle.query_spatial_2p(ref, q, r)
    assert int(np.diff(off).max()) > 48
    assert np.array_equal(rs.offsets, off) and np.array_equal(rs.indices, idx)


@pytest.mark.parametrize("n", [262_144, 262_145, 300_001])
def test_frontier_stages_around_the_threshold(n):
    """Trees up to 4 * 2^16 leaves finish the frontier in one CTA (CTA-scope
    handshakes), larger ones climb at GPU scope first and defer nodes spanning
    2^16 leaves to it: byte-identical to the oracle on both sides, for uniform
    and for clustered codes (many equal Morton codes and long empty leaf-
    directory runs)."""
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", n, 7))
    rng = np.random.default_rng(n)
    clustered = (rng.normal(0.0, 1.0, size=(n, 3)) * rng.choice([0.01, 50.0], size=(n, 1)))
    for cloud in (pts, clustered.astype(np.float32)):
        t, ref = lb.build(cloud), oracle.build(cloud)
        for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
            assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), (n, f)


@pytest.mark.parametrize("nq", [1, 2, 4095, 4096, 4097, 12_289])
def test_query_order_sizes_with_implicit_positions(nq):
    """The query ordering sort takes its digit histograms from the query
    Morton pass and the positions as implicit values (1 pair and tile-edge
    batches included): results equal the oracle's, unsorted CRS included."""
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", 20_000, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", nq, 5))
    t, ref = lb.build(pts), oracle.build(pts)
    rk = lb.query_knn(t, (q, 10))
    ko, ki, kd = oracle.query_knn(ref, q, 10)
    assert np.array_equal(rk.indices, ki) and rk.distances.tobytes() == kd.tobytes()
    r = datasets.default_radius(10)
    rs = lb.query_spatial_2p(t, (q, r))
    off, idx = oracle.query_spatial_2p(ref, q, r)
    assert np.array_equal(rs.offsets, off) and np.array_equal(rs.indices, idx)
    qd = torch.from_numpy(q).cuda()
    rd = lb.query_knn(t, (qd, 10)).to_host()
    assert np.array_equal(rd.indices, ki)
