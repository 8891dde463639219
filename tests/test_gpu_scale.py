"""Parity at BASELINE scale: the CUDA path against the REFERENCE's own outputs
on the full C2 / C3 / C5 configurations (BASELINE.json ``configs``).

The reference (``lbvh`` 0.1.0, run in the build container by
``tests/golden/make_golden_large.py``) produced sha256 digests of every output
at these sizes (``tests/golden/digests_large.json``); the arrays are GBs, so
only the digests travel.  Here the same inputs are regenerated (device PCG64
generators, bit-identical to the reference's numpy streams), the GPU builds
and queries them, and every output is hashed:

* tree arrays ``node_mins``/``node_maxs``/``left``/``right``/``leaf_obj``
  byte for byte, the Morton codes and the query pre-sort permutation
  (reference ``tree.py:177-209``, ``morton.py:68-91``, ``traversal.py:146-159``);
* radius 2P CRS: offsets, the indices in the reference's fill order and
  per-query sorted (``traversal.py:184-211``);
* kNN k=10: offsets, indices and distance bits (``traversal.py:251-272``).

C2 is also checked query by query against the C oracle run on an
independently built oracle tree (no GPU array feeds the oracle).
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_1908_11807_b200 as lb
from oracle import oracle
from paper_1908_11807_b200 import datasets

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def sha16(a) -> str:
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def large():
    with open(os.path.join(GOLDEN, "digests_large.json")) as fh:
        return json.load(fh)


def per_query_sorted(offsets: torch.Tensor, indices: torch.Tensor) -> torch.Tensor:
    counts = offsets[1:] - offsets[:-1]
    qid = torch.repeat_interleave(torch.arange(counts.numel(), device=offsets.device), counts)
    key = (qid << 32) | indices.to(torch.int64)
    return (torch.sort(key).values & 0xFFFFFFFF).to(torch.int32)


def check_tree(t, pts_dev, want):
    assert sha16(pts_dev) == want["points"]
    assert t.scene_min.tolist() == want["scene_min"]
    assert t.scene_max.tolist() == want["scene_max"]
    for f in ("leaf_obj", "left", "right", "node_mins", "node_maxs"):
        assert sha16(getattr(t, f)) == want[f], f"tree.{f} differs from the reference"
    # unsorted Morton codes (morton.py:68-91) from the leaf-order codes
    d = t._device()
    codes = torch.empty_like(d["leaf_codes"])
    codes[d["leaf_obj"].long()] = d["leaf_codes"]
    assert sha16(codes) == want["codes"]


def gen(spec: str, n: int, seed: int) -> torch.Tensor:
    shape, variant = spec.split(":")
    return datasets.generate_device(datasets.CloudSpec(shape, variant, n, seed))


@pytest.mark.parametrize("name", ["c2_filled", "c3_hollow_sphere"])
def test_baseline_config_against_reference(large, name):
    want = large[name]
    pts = gen(want["source"], want["m"], want["seed"])
    q = gen(want["target"], want["nq"], want["target_seed"])
    assert sha16(q) == want["queries"]
    t = lb.build(pts)
    check_tree(t, pts, want)
    # query pre-sort permutation (exact f64 codes on the tree's scene box)
    order = lb.query_sort_order(q.cpu().numpy(), (t.scene_min, t.scene_max))
    assert sha16(order) == want["query_order"]
    # radius 2P, device-resident batch (one-shot path)
    rs = lb.query_spatial_2p(t, (q, np.float32(want["radius"])))
    assert sha16(rs.offsets) == want["sp_offsets"]
    assert int(rs.offsets[-1]) == want["sp_total"]
    assert sha16(rs.indices) == want["sp_indices_fill_order"]
    assert sha16(per_query_sorted(rs.offsets, rs.indices)) == want["sp_sorted_indices"]
    del rs
    if "knn_indices" in want:
        rk = lb.query_knn(t, (q, want["k"]))
        assert sha16(rk.offsets) == want["knn_offsets"]
        assert sha16(rk.indices) == want["knn_indices"]
        assert sha16(rk.distances) == want["knn_distances"]


def test_c2_host_api_against_reference(large):
    """The same C2 outputs through the reference-facing host API (numpy in,
    numpy ResultSet out: the chunked pinned pipelines)."""
    want = large["c2_filled"]
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", want["m"], 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", want["nq"], 1))
    t = lb.build(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert sha16(getattr(t, f)) == want[f], f
    rs = lb.query_spatial_2p(t, (q, want["radius"]))
    assert sha16(rs.offsets) == want["sp_offsets"]
    assert sha16(rs.indices) == want["sp_indices_fill_order"]
    rk = lb.query_knn(t, (q, want["k"]))
    assert sha16(rk.indices) == want["knn_indices"]
    assert sha16(rk.distances) == want["knn_distances"]
    assert float(rk.distances.astype(np.float64).sum()) == want["knn_dist_sum"]


@pytest.mark.parametrize("m", [10_000, 100_000, 1_000_000, 10_000_000, 100_000_000])
def test_c5_build_sweep_against_reference(large, m):
    want = large["c5_build_sweep"][str(m)]
    pts = gen("cube:filled", m, 0)
    t = lb.build(pts)
    check_tree(t, pts, want)


def test_c2_against_independent_oracle_tree():
    """Full C2 (1e7 points, 1e7 queries): the oracle builds its own tree from
    the host points (C restatement of tree.py:177-209) and answers every
    query on it; the GPU tree and every GPU result must equal it."""
    n = 10_000_000
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", n, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", n, 1))
    ref = oracle.build(pts)
    t = lb.build(pts)
    for f in ("node_mins", "node_maxs", "left", "right", "leaf_obj"):
        assert getattr(t, f).tobytes() == getattr(ref, f).tobytes(), f
    r = datasets.default_radius(10)
    off, idx = oracle.query_spatial_2p(ref, q, r)
    rs = lb.query_spatial_2p(t, (q, r))
    assert np.array_equal(rs.offsets, off) and np.array_equal(rs.indices, idx)
    del rs, off, idx
    ko, ki, kd = oracle.query_knn(ref, q, 10)
    rk = lb.query_knn(t, (q, 10))
    assert np.array_equal(rk.offsets, ko)
    assert np.array_equal(rk.indices, ki)
    assert rk.distances.tobytes() == kd.tobytes()


def test_knn_5e7_block_seed_level8_against_oracle():
    """5e7 points: the leaf directory reaches 24 bits (the block seed's
    level-8 cells); a 100k-query sample of the full 5e7-query device batch
    must equal the oracle on its own tree."""
    from paper_1908_11807_b200 import _lib

    n, sample = 50_000_000, 100_000
    assert _lib.lib().lbvh_leaf_directory_bits(n) == 24
    pts = datasets.generate(datasets.CloudSpec("cube", "filled", n, 0))
    q = datasets.generate(datasets.CloudSpec("cube", "filled", n, 1))
    t = lb.build(torch.from_numpy(pts).cuda())
    rs = lb.query_knn(t, (torch.from_numpy(q).cuda(), 10))
    idx = rs.indices.view(n, 10)[:sample].cpu().numpy().reshape(-1)
    dist = rs.distances.view(n, 10)[:sample].cpu().numpy().reshape(-1)
    del rs, t
    ref = oracle.build(pts)
    ko, ki, kd = oracle.query_knn(ref, q[:sample], 10)
    assert np.array_equal(idx, ki)
    assert dist.tobytes() == kd.tobytes()


@pytest.mark.parametrize("name", ["c2_filled", "c3_hollow_sphere"])
def test_large_tree_structure(large, name):
    """Size-independent properties on the full trees: every
    internal box equals the union of its children's (both corners, both
    children, the refit's left-first rule), every node but the root has
    exactly one parent, leaf codes are sorted with index tie-break, and the
    root box is the scene box."""
    want = large[name]
    pts = gen(want["source"], want["m"], want["seed"])
    t = lb.build(pts)
    n = t.leaf_count
    d = t.device_arrays()
    nm, nx = d["node_mins"], d["node_maxs"]
    left, right = d["left"].long(), d["right"].long()
    # union: min/max with the left operand kept on ties (bit-exact)
    assert torch.equal(nm[: n - 1], torch.where(nm[left] <= nm[right], nm[left], nm[right]))
    assert torch.equal(nx[: n - 1], torch.where(nx[left] >= nx[right], nx[left], nx[right]))
    assert bool((nm[: n - 1] <= nm[left]).all()) and bool((nm[: n - 1] <= nm[right]).all())
    assert bool((nx[: n - 1] >= nx[left]).all()) and bool((nx[: n - 1] >= nx[right]).all())
    indeg = torch.bincount(torch.cat([left, right]), minlength=2 * n - 1)
    assert int(indeg[0]) == 0 and bool((indeg[1:] == 1).all())
    codes = d["leaf_codes"].long()
    lo = d["leaf_obj"].long()
    assert bool((codes[1:] >= codes[:-1]).all())
    ties = codes[1:] == codes[:-1]
    assert bool((lo[1:][ties] > lo[:-1][ties]).all())
    assert torch.equal(nm[0], d["root_box"][:3]) and torch.equal(nx[0], d["root_box"][3:])
    # leaf rows are the input points in leaf order
    assert torch.equal(nm[n - 1:], pts[lo]) and torch.equal(nx[n - 1:], pts[lo])
