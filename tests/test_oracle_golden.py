"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference
implementation (tests/golden/make_golden.py).  These tests need no GPU.
"""

import numpy as np
import pytest

from oracle import oracle
from paper_1908_11807_b200 import datasets

from helpers import assert_same_tree, sha16, sorted_concat


@pytest.mark.parametrize("case", ["line4", "cloud", "ext", "dup"])
def test_oracle_tree_matches_reference(golden, case):
    tree = oracle.build(golden[case + "_pts"], threads=2)
    assert_same_tree(tree, golden, case + "_")


def test_oracle_volumetric_tree(golden):
    tree = oracle.build((golden["vol_mins"], golden["vol_maxs"]))
    assert_same_tree(tree, golden, "vol_")
    off, idx = oracle.query_spatial_2p(tree, golden["vol_centers"], np.float32(1.7))
    assert np.array_equal(off, golden["vol_sp_offsets"])
    assert np.array_equal(sorted_concat(off, idx), golden["vol_sp_sorted_indices"])
    ko, ki, kd = oracle.query_knn(tree, golden["vol_centers"], 7)
    assert np.array_equal(ki, golden["vol_knn_indices"])
    assert kd.tobytes() == golden["vol_knn_distances"].tobytes()


def test_oracle_extreme_codes(golden):
    t = oracle.build(golden["ext_pts"])
    codes = oracle.morton_codes(golden["ext_pts"], t.scene_min, t.scene_max)
    assert codes.tolist() == [0, 1073741823, 939524096, 747784484]
    assert np.array_equal(codes, golden["ext_codes"])


def test_oracle_morton_kat(golden):
    pts = golden["morton_pts"]
    z, one = np.zeros(3, np.float32), np.ones(3, np.float32)
    assert np.array_equal(oracle.morton_codes(pts, z, one), golden["morton_codes_unit"])
    flat = np.float32([1, 0, 1])
    assert np.array_equal(oracle.morton_codes(pts, z, flat), golden["morton_codes_flat"])


@pytest.mark.parametrize("prefix", ["topo", "topod"])
def test_oracle_topology(golden, prefix):
    left, right, parent = oracle.generate_topology(golden[prefix + "_codes"], threads=3)
    assert np.array_equal(left, golden[prefix + "_left"])
    assert np.array_equal(right, golden[prefix + "_right"])
    assert np.array_equal(parent, golden[prefix + "_parent"])


def test_oracle_cloud_queries(golden):
    tree = oracle.build(golden["cloud_pts"])
    c = golden["cloud_sp_centers"]
    off, idx = oracle.query_spatial_2p(tree, c, 1.5)
    assert np.array_equal(off, golden["cloud_sp_offsets"])
    assert np.array_equal(sorted_concat(off, idx), golden["cloud_sp_sorted_indices"])
    off, idx = oracle.query_spatial_2p(tree, c, golden["cloud_spr_radii"])
    assert np.array_equal(sorted_concat(off, idx), golden["cloud_spr_sorted_indices"])
    for b in (1, 4, 32):
        o1, i1, fb = oracle.query_spatial_1p(tree, c, 1.5, b)
        assert fb == bool(golden[f"cloud_1p{b}_fellback"])
        assert np.array_equal(sorted_concat(o1, i1), golden[f"cloud_1p{b}_sorted_indices"])
    kc = golden["cloud_knn_centers"]
    for tag, k, cs in (("cloud_knn_", 10, kc), ("cloud_knnk_", golden["cloud_knnk_ks"], kc),
                       ("cloud_knn100_", 100, kc[:40])):
        ko, ki, kd = oracle.query_knn(tree, cs, k)
        assert np.array_equal(ko, golden[tag + "offsets"])
        assert np.array_equal(ki, golden[tag + "indices"])
        assert kd.tobytes() == golden[tag + "distances"].tobytes()
    assert np.array_equal(oracle.query_sort_order(c, tree.scene_min, tree.scene_max),
                          golden["cloud_order"])


def test_oracle_integer_clouds_with_ties(golden):
    for i in range(int(golden["int_ncases"])):
        p = f"int{i}_"
        tree = oracle.build(golden[p + "pts"])
        assert_same_tree(tree, golden, p)
        off, idx = oracle.query_spatial_2p(tree, golden[p + "centers"], golden[p + "r"])
        assert np.array_equal(off, golden[p + "sp_offsets"])
        assert np.array_equal(sorted_concat(off, idx), golden[p + "sp_sorted_indices"])
        ko, ki, kd = oracle.query_knn(tree, golden[p + "centers"], int(golden[p + "k"]))
        assert np.array_equal(ki, golden[p + "knn_indices"])
        assert kd.tobytes() == golden[p + "knn_distances"].tobytes()


def test_oracle_brute_force_agrees(golden):
    pts = golden["cloud_pts"]
    tree = oracle.build(pts)
    c = golden["cloud_sp_centers"][:50]
    off, idx = oracle.query_spatial_2p(tree, c, 1.5)
    want = oracle.brute_radius_sets(pts, c, 1.5)
    for q in range(50):
        assert np.array_equal(np.sort(idx[off[q]:off[q + 1]]), want[q])
    ko, ki, kd = oracle.query_knn(tree, c, 10)
    wi, wd = oracle.brute_knn_batch(pts, c, 10)
    assert np.array_equal(ki.reshape(50, 10), wi)
    assert np.allclose(kd.reshape(50, 10), wd, rtol=1e-6, atol=0)


@pytest.mark.parametrize("name", ["c1_filled", "c3_hollow_sphere", "hollow_cube"])
def test_oracle_matches_reference_digests(digests, name):
    d = digests[name]
    pts = datasets.generate(datasets.CloudSpec.parse(d["source"], d["m"], d["seed"]))
    q = datasets.generate(datasets.CloudSpec.parse(d["target"], d["m"], d["target_seed"]))
    assert sha16(pts) == d["points"] and sha16(q) == d["queries"]
    t = oracle.build(pts)
    assert t.scene_min.tolist() == d["scene_min"] and t.scene_max.tolist() == d["scene_max"]
    assert sha16(oracle.morton_codes(pts, t.scene_min, t.scene_max)) == d["codes"]
    for f in ("leaf_obj", "left", "right", "node_mins", "node_maxs"):
        assert sha16(getattr(t, f)) == d[f], f
    off, idx = oracle.query_spatial_2p(t, q, d["radius"])
    assert sha16(off) == d["sp_offsets"] and int(off[-1]) == d["sp_total"]
    assert sha16(sorted_concat(off, idx)) == d["sp_sorted_indices"]
    ko, ki, kd = oracle.query_knn(t, q, d["k"])
    assert sha16(ki) == d["knn_indices"] and sha16(kd) == d["knn_distances"]
    assert sha16(oracle.query_sort_order(q, t.scene_min, t.scene_max)) == d["query_order"]


@pytest.fixture(scope="module")
def large_digests():
    import json
    import os

    from conftest import GOLDEN

    with open(os.path.join(GOLDEN, "digests_large.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["c2_filled", "c3_hollow_sphere"])
def test_oracle_at_baseline_scale(large_digests, name):
    """The oracle at full BASELINE size (1e7 points / 1e7 queries, C2 and C3)
    against the reference's digests (tests/golden/make_golden_large.py):
    tree arrays, radius CRS in fill order (and kNN for C2).  ~30 s here."""
    want = large_digests[name]
    src = want["source"].split(":")
    tgt = want["target"].split(":")
    pts = datasets.generate(datasets.CloudSpec(src[0], src[1], want["m"], want["seed"]))
    q = datasets.generate(datasets.CloudSpec(tgt[0], tgt[1], want["nq"], want["target_seed"]))
    assert sha16(pts) == want["points"] and sha16(q) == want["queries"]
    ref = oracle.build(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert sha16(getattr(ref, f)) == want[f], f
    off, idx = oracle.query_spatial_2p(ref, q, want["radius"])
    assert sha16(off) == want["sp_offsets"] and sha16(idx) == want["sp_indices_fill_order"]
    del off, idx
    if name == "c2_filled":
        ko, ki, kd = oracle.query_knn(ref, q, want["k"])
        assert sha16(ko) == want["knn_offsets"]
        assert sha16(ki) == want["knn_indices"] and sha16(kd) == want["knn_distances"]
