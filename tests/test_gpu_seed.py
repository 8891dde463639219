"""GPU parity of the kNN search-radius seeds (csrc/seed.cuh): the block seed
(2x2x2 leaf-directory cells around a query, lists of K >= 8) and its fallback
to the Morton window must never change results, only where pruning starts.
Clouds here stress the cases where the block is sparse, empty, clamped at the
grid edge or degenerate; every result is compared with the CPU oracle
(bit-exact indices and distances)."""

import numpy as np
import pytest
import torch

import paper_1908_11807_b200 as lb
from oracle import oracle
from paper_1908_11807_b200 import _lib

pytestmark = pytest.mark.gpu


def _clouds():
    rng = np.random.default_rng(7)
    # Gaussian blobs: most cells empty, a few dense (block runs of 0 or ~100 leaves)
    centres = rng.uniform(-50, 50, size=(12, 3))
    blobs = (centres[rng.integers(0, 12, 60_000)] +
             rng.normal(0, 0.4, size=(60_000, 3))).astype(np.float32)
    # flat z axis: every leaf in cell z = 0 (scale 0 on that axis)
    flat = rng.uniform(-1, 1, size=(40_000, 3)).astype(np.float32)
    flat[:, 2] = 3.0
    # a line: two flat axes
    line = np.zeros((20_000, 3), np.float32)
    line[:, 0] = rng.uniform(0, 100, 20_000)
    # duplicates: 500 distinct points, 40 copies each (distance ties everywhere)
    dup = np.repeat(rng.uniform(-5, 5, size=(500, 3)).astype(np.float32), 40, axis=0)
    # few leaves: directory of 3 or 6 bits
    few = rng.uniform(-1, 1, size=(37, 3)).astype(np.float32)
    return {"blobs": blobs, "flat": flat, "line": line, "dup": dup, "few": few}


CLOUDS = _clouds()


def _queries(pts, n=6_000, seed=3):
    rng = np.random.default_rng(seed)
    lo, hi = pts.min(0), pts.max(0)
    ext = np.maximum(hi - lo, 1.0)
    near = pts[rng.integers(0, len(pts), n // 2)] + rng.normal(0, 0.01, (n // 2, 3)) * ext
    # uniform over a box 1.5x the scene: queries outside the tree's grid too
    far = rng.uniform(lo - 0.25 * ext, hi + 0.25 * ext, size=(n - n // 2, 3))
    return np.concatenate([near, far]).astype(np.float32)


@pytest.mark.parametrize("name", sorted(CLOUDS))
@pytest.mark.parametrize("k", [1, 5, 8, 10, 12, 16])
def test_seeded_knn_against_oracle(name, k):
    pts = CLOUDS[name]
    q = _queries(pts)
    ref = oracle.build(pts)
    t = lb.build(torch.from_numpy(pts).cuda())
    ko, ki, kd = oracle.query_knn(ref, q, k)
    h = lb.query_knn(t, (torch.from_numpy(q).cuda(), k)).to_host()
    assert np.array_equal(h.offsets, ko)
    assert np.array_equal(h.indices, ki)
    assert h.distances.tobytes() == kd.tobytes()


def test_mixed_per_query_k_in_one_list_size():
    """Per-query k from 1 to 16 in one K = 16 batch: queries below the block
    seed's minimum k take the window inside the same kernel."""
    pts = CLOUDS["blobs"]
    q = _queries(pts, 4_000, 5)
    ks = np.random.default_rng(2).integers(1, 17, size=len(q)).astype(np.int64)
    ref = oracle.build(pts)
    t = lb.build(torch.from_numpy(pts).cuda())
    ko, ki, kd = oracle.query_knn(ref, q, ks)
    h = lb.query_knn(t, (torch.from_numpy(q).cuda(), torch.from_numpy(ks).cuda())).to_host()
    assert np.array_equal(h.offsets, ko)
    assert np.array_equal(h.indices, ki)
    assert h.distances.tobytes() == kd.tobytes()


@pytest.mark.parametrize("k", [8, 16])
def test_seeded_knn_volumetric_leaves(k):
    """Box leaves: the seed's leaf distances are point-to-box (0 inside)."""
    rng = np.random.default_rng(11)
    lo = rng.uniform(-10, 10, size=(30_000, 3)).astype(np.float32)
    hi = lo + rng.uniform(0, 0.5, size=(30_000, 3)).astype(np.float32)
    rows = np.concatenate([lo, hi], axis=1)
    q = rng.uniform(-12, 12, size=(5_000, 3)).astype(np.float32)
    ref = oracle.build(rows)
    t = lb.build(torch.from_numpy(rows).cuda())
    ko, ki, kd = oracle.query_knn(ref, q, k)
    h = lb.query_knn(t, (torch.from_numpy(q).cuda(), k)).to_host()
    assert np.array_equal(h.indices, ki)
    assert h.distances.tobytes() == kd.tobytes()


def test_directory_is_cubic_cells():
    """The build writes a directory of 3L bits (what the block seed needs)."""
    l = _lib.load_library()
    for n in (20, 37, 40_000, 1_000_000):
        assert l.lbvh_leaf_directory_bits(n) % 3 == 0
    t = lb.build(torch.from_numpy(CLOUDS["flat"]).cuda())
    d = t._device()
    bits = l.lbvh_leaf_directory_bits(40_000)
    assert d["leaf_dir"].numel() == (1 << bits) + 1
    dirv = d["leaf_dir"].cpu().numpy().view(np.uint32).astype(np.int64)
    codes = d["leaf_codes"].cpu().numpy().view(np.uint32).astype(np.int64)
    # entry b = first leaf whose top `bits` code bits are >= b
    buckets = np.arange((1 << bits) + 1)
    expect = np.searchsorted(codes >> (30 - bits), buckets, side="left")
    assert np.array_equal(dirv, expect)
