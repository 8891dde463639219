"""Batched radius and k-nearest queries on the GPU -- drop-in for reference traversal.py.

Every batch runs as a short sequence of kernels on the current stream
(csrc/traverse.cu, csrc/scan.cu, csrc/build.cu):

  query_spatial_2p   check -> Morton order -> count -> scan -> [sync: total]
                     -> fill                                  (traversal.py:184-211)
  query_spatial_1p   check -> order -> buffered pass -> scan -> [sync]
                     -> compact, or the 2P path on overflow   (traversal.py:214-248)
  query_knn          check -> spans/scan -> order -> kNN      (traversal.py:251-272)

Results are CRS like the reference's: ``offsets`` int64 (nq+1), ``indices``
int32, ``distances`` float32 for kNN.  Host (numpy) inputs give a host
ResultSet backed by pinned memory; CUDA-tensor inputs give a ResultSet of
CUDA tensors (no D2H), the device-resident entry used by the benchmark.
Errors carry the reference's exception types and messages.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .geometry import Box, Point
from .tree import Bvh
from .validation import check_neighbor_counts, check_points, check_radii

__all__ = ["SpatialQuery", "KnnQuery", "ResultSet", "STACK_CAPACITY", "traverse_spatial_one",
           "traverse_knn_one", "query_spatial_2p", "query_spatial_1p", "query_knn",
           "query_sort_order"]

STACK_CAPACITY = _lib.STACK_CAPACITY

# Host batches at least this large, from pinned memory, run as a chunked
# pipeline: H2D of chunk i+1, compute of chunk i and D2H of chunk i-1
# overlap on three streams (copy engines both ways + SMs).
_PIPELINE_MIN = 1 << 20
_PIPELINE_CHUNK = 1 << 20
_PIPELINE_RAMP = 2  # kNN pipeline: first chunk = chunk >> 2, doubling up to chunk
_RADIUS_RAMP = 0  # radius 2P pipeline: no ramp (11.34 ms vs 11.41 from a quarter chunk: its per-chunk host sync)

# Traversal order = stable sort by the top 24 of the 30 Morton bits (3 radix
# passes instead of 4); ~0.6 queries share a 24-bit cell at 1e7, so warps
# stay as coherent, and the order never changes results.
_ORDER_BITS = 24

# Benchmark hook: when set to an object with ``wrap(name, call)``, the main
# traversal launches are bracketed by CUDA events on the launching stream.
KERNEL_TIMER = None


def _launch(name: str, call) -> int:
    t = KERNEL_TIMER
    return call() if t is None else t.wrap(name, call)


def _kernel_events(name: str):
    """(before, after) raw cudaEvent_t handles for a kernel timed inside a
    fused C call, or (None, None) when no timer is installed."""
    t = KERNEL_TIMER
    pair = t.pair(name) if t is not None and hasattr(t, "pair") else None
    if pair is None:
        return None, None
    return pair[0].cuda_event, pair[1].cuda_event


@dataclass(frozen=True)
class SpatialQuery:
    """All objects within ``radius`` of ``center``, inclusive (traversal.py:46-55)."""

    center: Point
    radius: float

    def __post_init__(self):
        if not math.isfinite(self.radius) or self.radius < 0:
            raise ValueError(f"radius must be finite and non-negative, got {self.radius}")


@dataclass(frozen=True)
class KnnQuery:
    """The ``k`` objects nearest to ``center`` (traversal.py:58-67)."""

    center: Point
    k: int

    def __post_init__(self):
        if self.k < 1:
            raise ValueError(f"k must be >= 1, got {self.k}")


class ResultSet:
    """CSR batch output (traversal.py:70-106).

    ``offsets`` (nq+1) non-decreasing from 0, hits of query q at
    ``indices[offsets[q]:offsets[q+1]]``; ``distances`` only for kNN.  The
    arrays are numpy for host queries or CUDA tensors for device queries.
    """

    __slots__ = ("offsets", "indices", "distances")

    def __init__(self, offsets, indices, distances=None):
        offsets = np.asarray(offsets) if not isinstance(offsets, torch.Tensor) else offsets
        if offsets.ndim != 1 or offsets.shape[0] < 1 or offsets[0] != 0:
            raise ValueError("offsets must be 1-D and start at 0")
        diff = offsets[1:] - offsets[:-1]
        if (diff < 0).any():
            raise ValueError("offsets must be non-decreasing")
        if int(offsets[-1]) != indices.shape[0]:
            raise ValueError("offsets total must equal indices length")
        if distances is not None and tuple(distances.shape) != tuple(indices.shape):
            raise ValueError("distances must align with indices")
        self.offsets, self.indices, self.distances = offsets, indices, distances

    @classmethod
    def _trusted(cls, offsets, indices, distances=None) -> "ResultSet":
        # CRS built by the device scan is well-formed by construction.
        rs = object.__new__(cls)
        rs.offsets, rs.indices, rs.distances = offsets, indices, distances
        return rs

    @property
    def query_count(self) -> int:
        return self.offsets.shape[0] - 1

    @property
    def on_device(self) -> bool:
        return isinstance(self.indices, torch.Tensor)

    def counts(self):
        return self.offsets[1:] - self.offsets[:-1]

    def hits(self, q: int):
        return self.indices[int(self.offsets[q]):int(self.offsets[q + 1])]

    def hit_distances(self, q: int):
        if self.distances is None:
            raise ValueError("result set carries no distances")
        return self.distances[int(self.offsets[q]):int(self.offsets[q + 1])]

    def to_host(self) -> "ResultSet":
        if not self.on_device:
            return self
        o, i, d = dv.d2h_many(self.offsets, self.indices, self.distances)
        return ResultSet._trusted(o, i, d)

    def __repr__(self) -> str:
        kind = "knn" if self.distances is not None else "spatial"
        where = "cuda" if self.on_device else "host"
        return f"ResultSet({kind}, queries={self.query_count}, hits={self.indices.shape[0]}, {where})"


# ---------------------------------------------------------------------------
# Input normalisation (traversal.py:114-143)
# ---------------------------------------------------------------------------


class _Batch:
    """Query batch staged on the device."""

    __slots__ = ("centers", "radii", "radius", "ks", "k", "nq", "host", "host_centers")

    def __init__(self):
        self.radii = self.ks = self.centers = self.host_centers = None
        self.radius = 0.0
        self.k = 0


def _device_centers(c) -> torch.Tensor:
    t = c.to(torch.float32)
    if t.ndim == 1 and t.shape[0] == 3:
        t = t.reshape(1, 3)
    if t.ndim != 2 or t.shape[1] != 3:
        raise ValueError(f"query centers must have shape (n, 3), got {tuple(t.shape)}")
    return t.contiguous()


def _spatial_batch(queries) -> _Batch:
    b = _Batch()
    if isinstance(queries, tuple) and len(queries) == 2:
        c, r = queries
        if dv.is_cuda_tensor(c):
            b.host = False
            b.centers = _device_centers(c)
            b.nq = int(b.centers.shape[0])
            if dv.is_cuda_tensor(r):
                b.radii = r.to(torch.float32).reshape(-1).contiguous()
                if b.radii.shape[0] != b.nq:
                    raise ValueError(f"radius must be a scalar or shape ({b.nq},), "
                                     f"got {tuple(r.shape)}")
            else:
                ra = check_radii(r, b.nq, device_checks=True)
                if ra.ndim == 0:
                    b.radius = float(ra)
                else:
                    b.radii = dv.h2d(ra)
            return b
        centers = check_points(c, "query centers", device_checks=True)
        ra = check_radii(r, centers.shape[0], device_checks=True)
    else:
        qs = list(queries)
        if not all(isinstance(q, SpatialQuery) for q in qs):
            raise TypeError("expected SpatialQuery items or a (centers, radii) pair")
        centers = np.array([[q.center.x, q.center.y, q.center.z] for q in qs],
                           dtype=np.float32).reshape(-1, 3)
        ra = np.array([q.radius for q in qs], dtype=np.float32)
    b.host = True
    b.nq = int(centers.shape[0])
    if b.nq:
        if ra.ndim == 0:
            b.radius = float(ra)
            if b.nq >= _PIPELINE_MIN and dv.is_pinned(centers):
                # large pinned batch: 2P runs as a chunked H2D/compute/D2H pipeline
                b.host_centers = centers
                return b
        else:
            b.radii = dv.h2d(ra)
        b.centers = dv.h2d(centers)
    return b


def _staged(b: _Batch) -> _Batch:
    """Upload a batch kept on the host for the pipelined paths."""
    if b.centers is None and b.host_centers is not None:
        b.centers = dv.h2d(b.host_centers)
        b.host_centers = None
    return b


def _knn_batch(queries) -> _Batch:
    b = _Batch()
    if isinstance(queries, tuple) and len(queries) == 2:
        c, k = queries
        if dv.is_cuda_tensor(c):
            b.host = False
            b.centers = _device_centers(c)
            b.nq = int(b.centers.shape[0])
            if dv.is_cuda_tensor(k):
                b.ks = k.to(torch.int64).reshape(-1).contiguous()
                if b.ks.shape[0] != b.nq:
                    raise ValueError(f"k must be a scalar or shape ({b.nq},), got {tuple(k.shape)}")
            else:
                ka = check_neighbor_counts(k, b.nq, device_checks=True)
                if ka.ndim == 0:
                    b.k = int(ka)
                else:
                    b.ks = dv.h2d(ka)
            return b
        centers = check_points(c, "query centers", device_checks=True)
        ka = check_neighbor_counts(k, centers.shape[0], device_checks=True)
    else:
        qs = list(queries)
        if not all(isinstance(q, KnnQuery) for q in qs):
            raise TypeError("expected KnnQuery items or a (centers, k) pair")
        centers = np.array([[q.center.x, q.center.y, q.center.z] for q in qs],
                           dtype=np.float32).reshape(-1, 3)
        ka = np.array([q.k for q in qs], dtype=np.int64)
    b.host = True
    b.nq = int(centers.shape[0])
    if b.nq:
        if ka.ndim == 0:
            b.k = int(ka)
            if b.nq >= _PIPELINE_MIN and dv.is_pinned(centers):
                # large pinned batch: H2D is chunked inside the pipelined path
                b.host_centers = centers
                return b
        else:
            b.ks = dv.h2d(ka)
        b.centers = dv.h2d(centers)
    return b


def _raise_flags(flags: int) -> None:
    """Reference exception for a device status word (validation first)."""
    if flags & _lib.FLAG_NONFINITE:
        raise ValueError("query centers must contain only finite values")
    if flags & _lib.FLAG_BAD_RADIUS:
        raise ValueError("radius must be finite and non-negative")
    if flags & _lib.FLAG_BAD_K:
        raise ValueError("k must be >= 1")
    if flags & _lib.FLAG_STACK_EXHAUSTED:
        raise RuntimeError("traversal stack exhausted")


def _empty_result(host: bool, knn: bool) -> ResultSet:
    if host:
        return ResultSet._trusted(np.zeros(1, dtype=np.int64), np.empty(0, dtype=np.int32),
                                  np.empty(0, dtype=np.float32) if knn else None)
    dev = dv.device()
    return ResultSet._trusted(torch.zeros(1, dtype=torch.int64, device=dev),
                              torch.empty(0, dtype=torch.int32, device=dev),
                              torch.empty(0, dtype=torch.float32, device=dev) if knn else None)


def _order(tree: Bvh, b: _Batch, sort_queries: bool, with_codes: bool = False):
    """Device Morton order of the batch on the tree's scene grid (or None);
    with ``with_codes`` also the sorted query codes (kNN radius seed)."""
    if not sort_queries or b.nq <= 1:
        return (None, None) if with_codes else None
    l = _lib.lib()
    order = dv.empty(b.nq, torch.int32)
    codes = dv.empty(b.nq, torch.int32) if with_codes else None
    ws = dv.workspace(l.lbvh_query_workspace_bytes(b.nq))
    _lib.check(l.lbvh_query_order(dv.ptr(b.centers), b.nq,
                                  dv.ptr(tree._device()["root_box"]), _ORDER_BITS,
                                  dv.ptr(order), dv.ptr(codes), dv.ptr(ws), ws.numel(),
                                  dv.stream()))
    return (order, codes) if with_codes else order


def _finish(host: bool, status: dv.Status, *arrays):
    """Read status (+ results when host) in one sync; raise on flags."""
    if host:
        res = dv.d2h_many(status.dev, *arrays)
        _raise_flags(int(res[0][0]) & 0xFFFFFFFF)
        return res[1:]
    _raise_flags(status.read())
    return list(arrays)


# ---------------------------------------------------------------------------
# Batched queries
# ---------------------------------------------------------------------------


# Two-pass radius queries keep the first _ROW_HITS hits of every query from
# the count pass (in traversal order, so bytes are the reference's fill
# order); the fill pass then revisits only queries with more hits.  The row
# buffer is skipped when it would exceed _ROW_BUDGET bytes.
_ROW_HITS = 48
_ROW_BUDGET = 8 << 30
# Hits beyond the row are kept by the count pass in a pool of LBVH_SPILL_CHUNK-int chunks
# (lbvh_spatial_count_batch's spill pool), so heavy queries are traversed
# once; sized at _SPILL_INTS ints per query (C3 needs ~8.2), a query that
# finds it exhausted falls back to the fill pass.
_SPILL_INTS = 16


def _spill_args(sp):
    if sp is None:
        return (None, None, 0, None, None)
    return (dv.ptr(sp["heads"]), dv.ptr(sp["pool"]), sp["chunks"], dv.ptr(sp["list"]),
            dv.ptr(sp["n"]))


def _spill_arrays(nq: int):
    chunks = min(max(64, nq * _SPILL_INTS // _lib.SPILL_CHUNK), _ROW_BUDGET // (4 * _lib.SPILL_CHUNK))
    return dict(heads=dv.empty(nq, torch.int32),
                pool=dv.empty((chunks + 1) * _lib.SPILL_CHUNK, torch.int32), chunks=chunks + 1,
                list=dv.empty(nq, torch.int32), n=dv.empty(1, torch.int32))


def _spatial_2p_fused(tree: Bvh, b: _Batch, sort_queries: bool, status: dv.Status):
    """query_spatial_2p on a staged batch: the count stage (checks, order,
    count with row buffer, scan, overflow list) in one C call, one sync for
    the total, then compaction and the overflow fill."""
    l = _lib.lib()
    ct = tree.ctree()
    st = dv.stream()
    nq = b.nq
    rows = next((r for r in (_ROW_HITS, _ROW_HITS // 2) if r and nq * r * 4 <= _ROW_BUDGET), 0)
    counts = dv.empty(nq, torch.int32)
    buf = dv.empty((nq, rows), torch.int32) if rows else None
    offsets = dv.empty(nq + 1, torch.int64)
    order = dv.empty(nq, torch.int32)
    over_list = dv.empty(nq, torch.int32) if rows else None
    over_n = dv.empty(1, torch.int32)
    sp = _spill_arrays(nq) if rows else None
    ws = dv.workspace(l.lbvh_spatial_count_batch_workspace_bytes(nq))
    evs = _kernel_events("spatial_count")
    _lib.check(l.lbvh_spatial_count_batch(
        ct, dv.ptr(b.centers), dv.ptr(b.radii), b.radius, nq, _ORDER_BITS if sort_queries else 0,
        rows, dv.ptr(order), dv.ptr(counts), dv.ptr(buf), dv.ptr(offsets), dv.ptr(over_list),
        dv.ptr(over_n), *(_spill_args(sp)), dv.ptr(ws), ws.numel(), status.ptr, evs[0], evs[1],
        st))
    flags, total, n_over, n_spill = dv.d2h_many(status.dev, offsets[nq:], over_n,
                                                sp["n"] if sp else over_n)
    _raise_flags(int(flags[0]) & 0xFFFFFFFF)
    total, n_over, n_spill = int(total[0]), int(n_over[0]), int(n_spill[0]) if sp else 0
    out = dv.empty(total, torch.int32)
    if total:
        if rows:
            _lib.check(l.lbvh_compact(dv.ptr(buf), rows, dv.ptr(counts), dv.ptr(offsets), nq,
                                      dv.ptr(out), st))
            if n_spill:
                _lib.check(l.lbvh_spill_copy(
                    dv.ptr(buf), rows, dv.ptr(counts), dv.ptr(offsets), dv.ptr(sp["heads"]),
                    dv.ptr(sp["pool"]), dv.ptr(sp["list"]), dv.ptr(sp["n"]), n_spill,
                    dv.ptr(out), st))
            if n_over:
                _lib.check(_launch("spatial_fill", lambda: l.lbvh_spatial_fill_list(
                    ct, dv.ptr(b.centers), dv.ptr(b.radii), b.radius, dv.ptr(over_list),
                    dv.ptr(over_n), n_over, dv.ptr(offsets), dv.ptr(out), status.ptr, st)))
        else:
            _lib.check(_launch("spatial_fill", lambda: l.lbvh_spatial_fill(
                ct, dv.ptr(b.centers), dv.ptr(b.radii), b.radius,
                dv.ptr(order) if sort_queries and nq > 1 else None, nq, dv.ptr(offsets),
                dv.ptr(out), None, 0, status.ptr, st)))
    return offsets, out


def _check_batch(b: _Batch, status: dv.Status, radii: bool) -> None:
    l = _lib.lib()
    _lib.check(l.lbvh_check_queries(dv.ptr(b.centers), b.nq, dv.ptr(b.radii) if radii else None,
                                    status.ptr, dv.stream()))


def query_spatial_2p(tree: Bvh, queries, sort_queries: bool = True,
                     threads: int = 1) -> ResultSet:
    """Within-radius batch, count-then-fill (traversal.py:184-211)."""
    b = _spatial_batch(queries)
    if b.nq == 0:
        return _empty_result(b.host, knn=False)
    if b.host_centers is not None:
        return _spatial_2p_pipelined(tree, b, sort_queries)
    status = dv.Status()
    offsets, out = _spatial_2p_fused(tree, b, sort_queries, status)
    offsets, out = _finish(b.host, status, offsets, out)
    return ResultSet._trusted(offsets, out)


def _spatial_2p_pipelined(tree: Bvh, b: _Batch, sort_queries: bool) -> ResultSet:
    """Host 2P batch (scalar radius, pinned centers) as a chunked pipeline:
    while chunk i is counted on the device, chunk i-1's rows are compacted
    (its total is read from a pinned scalar, not a stream sync) and its
    offsets and hits stream to the host, and chunk i+1 is uploaded.  Every
    query's hits are computed exactly as in the one-shot path; chunk offsets
    are shifted by the running total, so the CRS equals the one-shot one."""
    l = _lib.lib()
    dev = dv.device()
    nq = b.nq
    C = _PIPELINE_CHUNK
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    status = dv.Status()
    host_c = dv.as_tensor(b.host_centers)
    dev_c = torch.empty((nq, 3), dtype=torch.float32, device=dev)
    ct = tree.ctree()
    rows = _ROW_HITS
    bounds = list(_ramp_chunks(nq, C, _RADIUS_RAMP))
    nch = len(bounds)
    ws = dv.workspace(l.lbvh_spatial_count_batch_workspace_bytes(C))
    slots = [dict(counts=dv.empty(C, torch.int32), buf=dv.empty((C, rows), torch.int32),
                  offs=dv.empty(C + 1, torch.int64), over=dv.empty(C, torch.int32),
                  over_n=dv.empty(1, torch.int32), order=dv.empty(C, torch.int32),
                  tot_h=dv.pinned(1, torch.int64), over_h=dv.pinned(1, torch.int32),
                  spill=_spill_arrays(C), ev=torch.cuda.Event()) for _ in range(2)]
    h_off = dv.pinned(nq + 1, torch.int64)
    h_off[0] = 0
    cap = max(nq * 16, 1 << 20)
    h_idx = dv.pinned(cap, torch.int32)
    base = 0
    c_ptr = dv.ptr(dev_c)

    def span(i):
        return bounds[i]

    def stage_count(i, sl):
        c0, c1 = span(i)
        m = c1 - c0
        e_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            dev_c[c0:c1].copy_(host_c[c0:c1], non_blocking=True)
            e_in.record(s_in)
        comp.wait_event(e_in)
        cc = c_ptr + 12 * c0
        st = comp.cuda_stream
        # value check, query order, count (+ warp-packet pass for heavy
        # queries), scan and overflow list in one call
        _lib.check(_launch("spatial_count", lambda: l.lbvh_spatial_count_batch(
            ct, cc, None, b.radius, m, _ORDER_BITS if sort_queries else 0, rows,
            dv.ptr(sl["order"]), dv.ptr(sl["counts"]), dv.ptr(sl["buf"]), dv.ptr(sl["offs"]),
            dv.ptr(sl["over"]), dv.ptr(sl["over_n"]), *(_spill_args(sl["spill"])), dv.ptr(ws),
            ws.numel(), status.ptr, None, None, st)))
        sl["tot_h"].copy_(sl["offs"][m:m + 1], non_blocking=True)
        sl["over_h"].copy_(sl["over_n"], non_blocking=True)
        sl["ev"].record(comp)

    def stage_fill(i, sl):
        nonlocal base, cap, h_idx
        c0, c1 = span(i)
        m = c1 - c0
        sl["ev"].synchronize()
        total, n_over = int(sl["tot_h"][0]), int(sl["over_h"][0])
        st = comp.cuda_stream
        out = dv.empty(max(total, 1), torch.int32)
        if total:
            _lib.check(l.lbvh_compact(dv.ptr(sl["buf"]), rows, dv.ptr(sl["counts"]),
                                      dv.ptr(sl["offs"]), m, dv.ptr(out), st))
            sp = sl["spill"]
            _lib.check(l.lbvh_spill_copy(dv.ptr(sl["buf"]), rows, dv.ptr(sl["counts"]),
                                         dv.ptr(sl["offs"]), dv.ptr(sp["heads"]),
                                         dv.ptr(sp["pool"]), dv.ptr(sp["list"]),
                                         dv.ptr(sp["n"]), m, dv.ptr(out), st))
            if n_over:
                _lib.check(_launch("spatial_fill", lambda: l.lbvh_spatial_fill_list(
                    ct, c_ptr + 12 * c0, None, b.radius, dv.ptr(sl["over"]),
                    dv.ptr(sl["over_n"]), n_over, dv.ptr(sl["offs"]), dv.ptr(out), status.ptr,
                    st)))
        goff = sl["offs"][1:m + 1] + base
        if base + total > cap:  # grow the host hit buffer (rare)
            s_out.synchronize()
            cap = max(2 * cap, base + total)
            bigger = dv.pinned(cap, torch.int32)
            bigger[:base].copy_(h_idx[:base])
            h_idx = bigger
        e = torch.cuda.Event()
        e.record(comp)
        s_out.wait_event(e)
        with torch.cuda.stream(s_out):
            h_off[c0 + 1:c1 + 1].copy_(goff, non_blocking=True)
            if total:
                h_idx[base:base + total].copy_(out[:total], non_blocking=True)
            goff.record_stream(s_out)
            out.record_stream(s_out)
        base += total

    for i in range(nch + 1):
        if i < nch:
            stage_count(i, slots[i % 2])
        if i >= 1:
            stage_fill(i - 1, slots[(i - 1) % 2])
    comp.wait_stream(s_out)
    comp.wait_stream(s_in)
    _raise_flags(status.read())  # synchronises the current stream
    return ResultSet._trusted(h_off.numpy(), h_idx.numpy()[:base])


def query_spatial_1p(tree: Bvh, queries, buffer_size: int, sort_queries: bool = True,
                     threads: int = 1) -> tuple[ResultSet, bool]:
    """Within-radius batch with ``buffer_size`` slots per query; falls back to
    the two-pass path for the whole batch if any query overflows
    (traversal.py:214-248).  Returns ``(result, fell_back)``."""
    buffer_size = int(buffer_size)
    if buffer_size < 1:
        raise ValueError(f"buffer_size must be >= 1, got {buffer_size}")
    b = _staged(_spatial_batch(queries))
    if b.nq == 0:
        return _empty_result(b.host, knn=False), False
    l = _lib.lib()
    st = dv.stream()
    nq = b.nq
    status = dv.Status()
    _check_batch(b, status, radii=True)
    order = _order(tree, b, sort_queries)
    ct = tree.ctree()
    buf = dv.empty((nq, buffer_size), torch.int32)
    counts = dv.empty(nq, torch.int32)
    _lib.check(_launch("spatial_1p", lambda: l.lbvh_spatial_1p(
        ct, dv.ptr(b.centers), dv.ptr(b.radii), b.radius, dv.ptr(order), nq, dv.ptr(buf),
        buffer_size, dv.ptr(counts), status.ptr, st)))
    offsets = dv.empty(nq + 1, torch.int64)
    ws = dv.workspace(l.lbvh_scan_workspace_bytes(nq))
    _lib.check(l.lbvh_exclusive_scan(dv.ptr(counts), nq, dv.ptr(offsets), dv.ptr(ws),
                                     ws.numel(), st))
    flags, total = dv.d2h_many(status.dev, offsets[nq:])
    flags = int(flags[0]) & 0xFFFFFFFF
    _raise_flags(flags)
    if flags & _lib.FLAG_BUFFER_OVERFLOW:
        del buf
        status = dv.Status()
        offsets, out = _spatial_2p_fused(tree, b, sort_queries, status)
        offsets, out = _finish(b.host, status, offsets, out)
        return ResultSet._trusted(offsets, out), True
    total = int(total[0])
    out = dv.empty(total, torch.int32)
    if total:
        _lib.check(l.lbvh_compact(dv.ptr(buf), buffer_size, dv.ptr(counts), dv.ptr(offsets), nq,
                                  dv.ptr(out), st))
    offsets, out = _finish(b.host, status, offsets, out)
    return ResultSet._trusted(offsets, out), False


def query_knn(tree: Bvh, queries, sort_queries: bool = True, threads: int = 1) -> ResultSet:
    """k-nearest batch (traversal.py:251-272): spans of min(k, n) sorted by
    (distance, ordinal) with true distances."""
    return _query_knn(tree, queries, sort_queries, squared=False)


def query_knn_squared(tree: Bvh, queries, sort_queries: bool = True) -> ResultSet:
    """As :func:`query_knn` but ``distances`` holds the exact squared fp32
    distances (no sqrt); the distributed merge orders by these."""
    return _query_knn(tree, queries, sort_queries, squared=True)


def _query_knn(tree: Bvh, queries, sort_queries: bool, squared: bool) -> ResultSet:
    flags = _lib.KNN_SQUARED if squared else 0
    b = _knn_batch(queries)
    if b.nq == 0:
        return _empty_result(b.host, knn=True)
    if b.host_centers is not None:
        return _knn_pipelined(tree, b, sort_queries, flags)
    l = _lib.lib()
    st = dv.stream()
    nq, n = b.nq, tree.leaf_count
    status = dv.Status()
    offsets = dv.empty(nq + 1, torch.int64)
    if b.ks is None:
        # uniform k: checks, offsets, query order and search in one C call
        span = min(b.k, n)
        out_idx = dv.empty(span * nq, torch.int32)
        out_dist = dv.empty(span * nq, torch.float32)
        ws = dv.workspace(l.lbvh_knn_batch_workspace_bytes(nq))
        evs = _kernel_events("knn")
        _lib.check(l.lbvh_knn_batch(
            tree.ctree(), dv.ptr(b.centers), nq, b.k, _ORDER_BITS if sort_queries else 0,
            dv.ptr(offsets), dv.ptr(out_idx), dv.ptr(out_dist), flags, dv.ptr(ws), ws.numel(),
            status.ptr, None, evs[0], evs[1], st))
        offsets, out_idx, out_dist = _finish(b.host, status, offsets, out_idx, out_dist)
        return ResultSet._trusted(offsets, out_idx, out_dist)
    _check_batch(b, status, radii=False)
    ws = dv.workspace(l.lbvh_scan_workspace_bytes(nq))
    if b.ks is None:
        # uniform k: spans, total and the kernel variant are known on the host
        span = min(b.k, n)
        max_span, total = span, span * nq
        _lib.check(l.lbvh_knn_offsets(None, b.k, n, nq, dv.ptr(offsets), None, status.ptr,
                                      dv.ptr(ws), ws.numel(), st))
    else:
        mx = dv.empty(1, torch.int32)
        _lib.check(l.lbvh_knn_offsets(dv.ptr(b.ks), 0, n, nq, dv.ptr(offsets), dv.ptr(mx),
                                      status.ptr, dv.ptr(ws), ws.numel(), st))
        st_word, mxh, tot = dv.d2h_many(status.dev, mx, offsets[nq:])
        _raise_flags(int(st_word[0]) & 0xFFFFFFFF)
        max_span, total = int(mxh[0]), int(tot[0])
    order, qcodes = _order(tree, b, sort_queries, with_codes=True)
    out_idx = dv.empty(total, torch.int32)
    out_dist = dv.empty(total, torch.float32)
    ct = tree.ctree()
    kws = dv.workspace(l.lbvh_knn_workspace_bytes(nq))
    _lib.check(_launch("knn", lambda: l.lbvh_knn(
        ct, dv.ptr(b.centers), dv.ptr(order), dv.ptr(qcodes), nq, dv.ptr(offsets), max_span,
        dv.ptr(out_idx), dv.ptr(out_dist), flags, dv.ptr(kws), kws.numel(), status.ptr, st)))
    offsets, out_idx, out_dist = _finish(b.host, status, offsets, out_idx, out_dist)
    return ResultSet._trusted(offsets, out_idx, out_dist)


_HOST_POOL = None
# 1 (measured 16.07 vs 16.63 ms e2e at C2): host threads write the uniform
# offsets instead of copying them from the device
_HOST_OFFSETS = True


def _host_arange_into(out: np.ndarray, step: int, parts: int = 8):
    """out[i] = i * step, filled by ``parts`` pool threads (numpy releases the
    GIL); returns the futures."""
    global _HOST_POOL
    if _HOST_POOL is None:
        import concurrent.futures as cf

        _HOST_POOL = cf.ThreadPoolExecutor(max_workers=parts, thread_name_prefix="lbvh-host")
    n = out.shape[0]
    per = -(-n // parts)

    def fill(c0, c1):
        np.multiply(np.arange(c0, c1, dtype=np.int64), step, out=out[c0:c1])

    return [_HOST_POOL.submit(fill, c0, min(n, c0 + per)) for c0 in range(0, n, per)]


def knn_with_kth(tree: Bvh, centers: torch.Tensor, k: int):
    """Device kNN (k <= 32) returning ``(ordinals i32 (m, kk), distances f32
    (m, kk), kth_d2 f32 (m,))``: the final sqrt'ed lists plus each query's
    exact squared k-th distance (the sharded search's forwarding bound), in
    one C call."""
    b = _knn_batch((centers, k))
    l = _lib.lib()
    st = dv.stream()
    nq, n = b.nq, tree.leaf_count
    span = min(b.k, n)
    out_idx = dv.empty(nq * span, torch.int32)
    out_dist = dv.empty(nq * span, torch.float32)
    kth = dv.empty(nq, torch.float32)
    if nq == 0:
        return out_idx.reshape(0, span), out_dist.reshape(0, span), kth
    status = dv.Status()
    offsets = dv.empty(nq + 1, torch.int64)
    ws = dv.workspace(l.lbvh_knn_batch_workspace_bytes(nq))
    evs = _kernel_events("knn")
    _lib.check(l.lbvh_knn_batch(
        tree.ctree(), dv.ptr(b.centers), nq, b.k, _ORDER_BITS, dv.ptr(offsets), dv.ptr(out_idx),
        dv.ptr(out_dist), 0, dv.ptr(ws), ws.numel(), status.ptr, dv.ptr(kth), evs[0], evs[1],
        st))
    _raise_flags(status.read())
    return out_idx.reshape(nq, span), out_dist.reshape(nq, span), kth


def _ramp_chunks(nq: int, chunk: int, ramp: int = None):
    """Chunk bounds of a host pipeline: the first chunks grow from chunk/4 so
    the first D2H (the pipeline's bound) starts after a short H2D + compute
    head instead of a full chunk's."""
    c0, size = 0, max(1, chunk >> (_PIPELINE_RAMP if ramp is None else ramp))
    while c0 < nq:
        c1 = min(nq, c0 + size)
        yield c0, c1
        c0, size = c1, min(chunk, size * 2)


def _knn_pipelined(tree: Bvh, b: _Batch, sort_queries: bool, flags: int = 0) -> ResultSet:
    """Host kNN batch as an H2D / compute / D2H pipeline over query chunks.

    Chunk results are identical to the one-shot path: every query's span is
    independent and sits at its global offset; only the Morton pre-sort is
    per chunk, and query order never changes results (traversal.py:146-165).
    """
    l = _lib.lib()
    dev = dv.device()
    nq, n = b.nq, tree.leaf_count
    span = min(b.k, n)
    total = span * nq
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    status = dv.Status()
    host_c = dv.as_tensor(b.host_centers)
    dev_c = torch.empty((nq, 3), dtype=torch.float32, device=dev)
    offsets = dv.empty(nq + 1, torch.int64)
    out_idx = dv.empty(total, torch.int32)
    out_dist = dv.empty(total, torch.float32)
    h_off = dv.pinned(nq + 1, torch.int64)
    h_idx = dv.pinned(total, torch.int32)
    h_dist = dv.pinned(total, torch.float32)
    chunk = _PIPELINE_CHUNK
    order = dv.empty(chunk, torch.int32) if sort_queries else None
    qcodes = dv.empty(chunk, torch.int32) if sort_queries else None
    ws = dv.workspace(max(l.lbvh_query_workspace_bytes(chunk), l.lbvh_scan_workspace_bytes(nq)))
    kws = dv.workspace(l.lbvh_knn_workspace_bytes(chunk))
    _lib.check(l.lbvh_knn_offsets(None, b.k, n, nq, dv.ptr(offsets), None, status.ptr,
                                  dv.ptr(ws), ws.numel(), comp.cuda_stream))
    # Uniform spans: the host offsets are arange(nq + 1) * span, written by
    # host threads while the copy engines stream the results (saves 8 B per
    # query of D2H, the pipeline's bound).
    if _HOST_OFFSETS:
        off_jobs = _host_arange_into(h_off.numpy(), span)
    else:
        off_jobs = []
        ev = torch.cuda.Event()
        ev.record(comp)
        s_out.wait_event(ev)
        with torch.cuda.stream(s_out):
            h_off.copy_(offsets, non_blocking=True)
    ct = tree.ctree()
    root_box = dv.ptr(tree._device()["root_box"])
    c_ptr, o_ptr = dv.ptr(dev_c), dv.ptr(offsets)
    for c0, c1 in _ramp_chunks(nq, chunk):
        m = c1 - c0
        e_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            dev_c[c0:c1].copy_(host_c[c0:c1], non_blocking=True)
            e_in.record(s_in)
        comp.wait_event(e_in)
        cc = c_ptr + 12 * c0
        _lib.check(l.lbvh_check_queries(cc, m, None, status.ptr, comp.cuda_stream))
        srt = sort_queries and m > 1
        if srt:
            _lib.check(l.lbvh_query_order(cc, m, root_box, _ORDER_BITS, dv.ptr(order),
                                          dv.ptr(qcodes), dv.ptr(ws), ws.numel(),
                                          comp.cuda_stream))
        _lib.check(_launch("knn", lambda: l.lbvh_knn(
            ct, cc, dv.ptr(order) if srt else None, dv.ptr(qcodes) if srt else None, m,
            o_ptr + 8 * c0, span, dv.ptr(out_idx), dv.ptr(out_dist), flags, dv.ptr(kws),
            kws.numel(), status.ptr, comp.cuda_stream)))
        e_c = torch.cuda.Event()
        e_c.record(comp)
        s_out.wait_event(e_c)
        with torch.cuda.stream(s_out):
            h_idx[c0 * span:c1 * span].copy_(out_idx[c0 * span:c1 * span], non_blocking=True)
            h_dist[c0 * span:c1 * span].copy_(out_dist[c0 * span:c1 * span], non_blocking=True)
    comp.wait_stream(s_out)
    comp.wait_stream(s_in)
    for j in off_jobs:
        j.result()
    _raise_flags(status.read())  # synchronises the current stream
    return ResultSet._trusted(h_off.numpy(), h_idx.numpy(), h_dist.numpy())


def query_sort_order(centers, scene: Box | tuple) -> np.ndarray:
    """Morton permutation of query centers with ordinal tie-break
    (traversal.py:146-159), computed on the GPU (f64 codes + radix sort)."""
    centers = check_points(centers, "query centers")
    if isinstance(scene, Box):
        smin = np.array([scene.min.x, scene.min.y, scene.min.z], dtype=np.float32)
        smax = np.array([scene.max.x, scene.max.y, scene.max.z], dtype=np.float32)
    else:
        smin, smax = scene
    lo = np.ascontiguousarray(smin, dtype=np.float64).reshape(3)
    hi = np.ascontiguousarray(smax, dtype=np.float64).reshape(3)
    nq = centers.shape[0]
    if nq == 0:
        return np.empty(0, dtype=np.int64)
    l = _lib.lib()
    st = dv.stream()
    pts = dv.h2d(centers.astype(np.float64))
    codes = dv.empty(nq, torch.int32)
    _lib.check(l.lbvh_morton_codes(dv.ptr(pts), nq, lo.ctypes.data, hi.ctypes.data,
                                   dv.ptr(codes), st))
    perm = torch.arange(nq, dtype=torch.int32, device=dv.device())
    ws = dv.workspace(l.lbvh_sort_workspace_bytes(nq))
    _lib.check(l.lbvh_sort_pairs(dv.ptr(codes), dv.ptr(perm), nq, 30, dv.ptr(ws), ws.numel(),
                                 st))
    return dv.d2h(perm).astype(np.int64)


# ---------------------------------------------------------------------------
# Single-query entry points (traversal.py:295-378): one-query GPU batches
# ---------------------------------------------------------------------------


def traverse_spatial_one(tree: Bvh, query: SpatialQuery,
                         sink: Callable[[int], None] | None = None) -> int:
    """One within-radius query; feeds each hit ordinal to ``sink`` (in the
    reference's traversal order) and returns the hit count."""
    rs = query_spatial_2p(tree, [query], sort_queries=False)
    hits = rs.hits(0)
    if sink is not None:
        for h in hits.tolist():
            sink(int(h))
    return int(hits.shape[0])


def traverse_knn_one(tree: Bvh, query: KnnQuery) -> list[tuple[int, float]]:
    """One k-nearest query: min(k, n) (ordinal, distance) pairs sorted by
    (distance, ordinal)."""
    rs = query_knn(tree, [query], sort_queries=False)
    return [(int(i), float(d)) for i, d in zip(rs.hits(0).tolist(),
                                               rs.hit_distances(0).tolist())]
