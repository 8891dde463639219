"""Brute-force search on the GPU -- drop-in for the reference's oracle.py.

The reference exports ``brute_radius`` / ``brute_knn`` (and the batch forms
used by its verify harness) from its package root; these run the same O(n)
per-query scan with the same fp32 recipe (oracle.py:18-21) in
``csrc/brute.cu``.  They are the library's verification helpers, not part of
the BVH path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .traversal import KnnQuery, SpatialQuery
from .validation import check_points

__all__ = ["brute_radius", "brute_knn", "brute_radius_sets", "brute_knn_batch"]


def _radius_batch(pts: np.ndarray, centers: np.ndarray, radii: np.ndarray):
    l = _lib.lib()
    st = dv.stream()
    n, nq = pts.shape[0], centers.shape[0]
    dp, dc, dr = dv.h2d(pts), dv.h2d(centers), dv.h2d(radii)
    counts = dv.empty(nq, torch.int32)
    _lib.check(l.lbvh_brute_radius(dv.ptr(dp), n, dv.ptr(dc), dv.ptr(dr), 0.0, nq,
                                   dv.ptr(counts), None, None, st))
    offsets = torch.zeros(nq + 1, dtype=torch.int64, device=dv.device())
    offsets[1:] = torch.cumsum(counts.to(torch.int64), 0)
    total = int(offsets[-1].item())
    out = dv.empty(max(total, 1), torch.int32)
    _lib.check(l.lbvh_brute_radius(dv.ptr(dp), n, dv.ptr(dc), dv.ptr(dr), 0.0, nq, None,
                                   dv.ptr(offsets), dv.ptr(out), st))
    off, idx = dv.d2h_many(offsets, out[:total])
    return off, idx


def brute_radius(points, q: SpatialQuery) -> np.ndarray:
    """Ascending ordinals of all points within q.radius of q.center (oracle.py:26-32)."""
    pts = check_points(points, "points")
    c = np.array([[q.center.x, q.center.y, q.center.z]], dtype=np.float32)
    off, idx = _radius_batch(pts, c, np.array([q.radius], dtype=np.float32))
    return idx.astype(np.int64)


def brute_radius_sets(points, centers, radii) -> list[np.ndarray]:
    """Per-query ascending hit ordinals for a batch (oracle.py:48-59)."""
    pts = check_points(points, "points")
    cs = check_points(centers, "centers")
    r = np.asarray(radii, dtype=np.float32)
    if r.ndim == 0:
        r = np.full(cs.shape[0], r, dtype=np.float32)
    off, idx = _radius_batch(pts, cs, np.ascontiguousarray(r))
    idx = idx.astype(np.int64)
    return [idx[off[i]:off[i + 1]] for i in range(cs.shape[0])]


def _knn_batch(pts: np.ndarray, centers: np.ndarray, k: int):
    l = _lib.lib()
    n, nq = pts.shape[0], centers.shape[0]
    kk = min(int(k), n)
    idx = dv.empty((nq, kk), torch.int32)
    dist = dv.empty((nq, kk), torch.float32)
    dp, dc = dv.h2d(pts), dv.h2d(centers)
    _lib.check(l.lbvh_brute_knn(dv.ptr(dp), n, dv.ptr(dc), nq, int(k), dv.ptr(idx),
                                dv.ptr(dist), dv.stream()))
    hi, hd = dv.d2h_many(idx, dist)
    return hi.astype(np.int64), hd.copy()


def brute_knn(points, q: KnnQuery) -> tuple[np.ndarray, np.ndarray]:
    """The min(k, n) nearest ordinals and distances, sorted by (distance,
    ordinal) (oracle.py:35-45)."""
    pts = check_points(points, "points")
    c = np.array([[q.center.x, q.center.y, q.center.z]], dtype=np.float32)
    idx, dist = _knn_batch(pts, c, q.k)
    return idx[0], dist[0]


def brute_knn_batch(points, centers, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Batched k-nearest: (nq, min(k, n)) index and distance arrays (oracle.py:62-70)."""
    pts = check_points(points, "points")
    cs = check_points(centers, "centers")
    return _knn_batch(pts, cs, k)
