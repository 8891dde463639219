"""Linear BVH construction on the GPU -- drop-in for reference tree.py.

``build`` runs the whole pipeline on the device in one stream (scene
reduction, f64 Morton codes, one-sweep radix sort, fused Apetrei
hierarchy + atomic-flag refit + packed-node write; csrc/build.cu) and returns
a :class:`Bvh` whose arrays stay resident in HBM.  The reference-layout numpy
fields (``node_mins`` ... ``scene_max``) are materialised lazily, read-only,
on first access.

Node numbering is the reference's (tree.py:8-12): internal nodes 0..n-2 with
root 0, the leaf at Morton-sorted position p is node (n-1)+p.
"""

from __future__ import annotations

from typing import NamedTuple


import numpy as np
import torch

from . import _device as dv
from . import _lib
from .geometry import Box
from .validation import check_boxes

__all__ = ["Bvh", "Topology", "build", "common_prefix", "find_split", "node_range",
           "generate_topology", "refit_bounds"]


# Benchmark hook (see traversal.KERNEL_TIMER).
KERNEL_TIMER = None


def _launch(name: str, call) -> int:
    t = KERNEL_TIMER
    return call() if t is None else t.wrap(name, call)


def _readonly(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


class Bvh:
    """Immutable linear BVH (reference tree.py:122-174).

    Constructed either by :func:`build` (device-resident) or directly from
    reference-layout numpy arrays ``Bvh(node_mins, node_maxs, left, right,
    leaf_obj, scene_min, scene_max)`` -- e.g. a hand-made or modified tree --
    in which case the arrays are uploaded and packed on first query.
    """

    __slots__ = ("_host", "_dev", "_n", "_ct")

    _FIELDS = ("node_mins", "node_maxs", "left", "right", "leaf_obj", "scene_min", "scene_max")

    def __init__(self, node_mins, node_maxs, left, right, leaf_obj, scene_min, scene_max):
        host = {
            "node_mins": np.asarray(node_mins, dtype=np.float32),
            "node_maxs": np.asarray(node_maxs, dtype=np.float32),
            "left": np.asarray(left, dtype=np.int32),
            "right": np.asarray(right, dtype=np.int32),
            "leaf_obj": np.asarray(leaf_obj, dtype=np.int32),
            "scene_min": np.asarray(scene_min, dtype=np.float32),
            "scene_max": np.asarray(scene_max, dtype=np.float32),
        }
        object.__setattr__(self, "_host", host)
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_n", int(host["leaf_obj"].shape[0]))

    @classmethod
    def _from_device(cls, dev: dict, n: int) -> "Bvh":
        self = object.__new__(cls)
        object.__setattr__(self, "_host", {})
        object.__setattr__(self, "_dev", dev)
        object.__setattr__(self, "_n", n)
        return self

    def __setattr__(self, name, value):
        raise AttributeError("Bvh is immutable")

    # -- reference-layout host views (lazy D2H) ---------------------------
    def _field(self, name: str) -> np.ndarray:
        h = self._host
        if name not in h:
            d = self._dev
            if name in ("scene_min", "scene_max"):
                box = dv.d2h(d["root_box"])
                h["scene_min"] = _readonly(box[:3].copy())
                h["scene_max"] = _readonly(box[3:].copy())
            else:
                if name in ("node_mins", "node_maxs"):
                    self._finish_rows()
                h[name] = _readonly(dv.d2h(d[name]))
        return h[name]

    node_mins = property(lambda self: self._field("node_mins"))
    node_maxs = property(lambda self: self._field("node_maxs"))
    left = property(lambda self: self._field("left"))
    right = property(lambda self: self._field("right"))
    leaf_obj = property(lambda self: self._field("leaf_obj"))
    scene_min = property(lambda self: self._field("scene_min"))
    scene_max = property(lambda self: self._field("scene_max"))

    # -- device view -------------------------------------------------------
    def device_arrays(self) -> dict:
        """Device tensors: node_mins, node_maxs, left, right, leaf_obj,
        nodes (packed (n-1) x 64 B), root_box (6 f32).  Uploads and packs a
        host-constructed tree on first use; writes the reference-layout rows a
        build deferred (LBVH_BUILD_DEFER_ROWS) on first access."""
        d = self._device()
        self._finish_rows()
        return d

    def _device(self) -> dict:
        """Device tensors as they are: the deferred reference rows (internal
        node_mins/node_maxs rows, node_maxs leaf rows of a point tree) may
        still be unwritten -- no query reads them."""
        if self._dev is None:
            self._upload()
        return self._dev

    def _finish_rows(self) -> None:
        d = self._dev
        if d is not None and d.get("rows_pending"):
            _lib.check(_lib.lib().lbvh_finish_rows(self.ctree(), dv.ptr(d["node_mins"]),
                                                   dv.ptr(d["node_maxs"]), dv.stream()))
            d["rows_pending"] = False

    def _upload(self) -> None:
        h = self._host
        n = self._n
        if n < 1:
            raise ValueError("empty scene")
        l = _lib.lib()
        d = {k: dv.h2d(np.ascontiguousarray(h[k])) for k in
             ("node_mins", "node_maxs", "left", "right", "leaf_obj")}
        d["nodes"] = dv.empty(max(n - 1, 1) * _lib.NODE_BYTES, torch.uint8)
        d["root_box"] = dv.empty(6, torch.float32)
        status = dv.Status()
        ct = _ctree(d, n)
        _lib.check(l.lbvh_pack(ct, dv.ptr(d["nodes"]), dv.ptr(d["root_box"]), status.ptr,
                               dv.stream()))
        if status.read() & _lib.FLAG_BAD_TREE:
            raise ValueError("tree links or leaf ordinals out of range")
        object.__setattr__(self, "_dev", d)

    def ctree(self) -> _lib.CTree:
        """The C-ABI tree struct (cached: device buffers never move once built)."""
        d = self._device()
        ct = getattr(self, "_ct", None)
        if ct is None or ct[0] is not d:
            ct = (d, _ctree(d, self._n))
            object.__setattr__(self, "_ct", ct)
        return ct[1]

    # -- reference API -----------------------------------------------------
    @property
    def leaf_count(self) -> int:
        return self._n

    @property
    def internal_count(self) -> int:
        return self._n - 1

    @property
    def node_count(self) -> int:
        return 2 * self._n - 1

    @property
    def scene(self) -> Box:
        return Box.from_arrays(self.scene_min, self.scene_max)

    def is_leaf(self, node: int) -> bool:
        return node >= self.internal_count

    def leaf_ordinal(self, node: int) -> int:
        if not self.is_leaf(node):
            raise ValueError(f"node {node} is internal")
        return int(self.leaf_obj[node - self.internal_count])

    def children(self, node: int) -> tuple[int, int]:
        if self.is_leaf(node):
            raise ValueError(f"node {node} is a leaf")
        return int(self.left[node]), int(self.right[node])

    def node_box(self, node: int) -> Box:
        return Box.from_arrays(self.node_mins[node], self.node_maxs[node])

    def __repr__(self) -> str:
        return f"Bvh(leaves={self.leaf_count}, nodes={self.node_count})"


def _ctree(d: dict, n: int) -> _lib.CTree:
    ld = d.get("leaf_dir")
    bits = (int(ld.numel()) - 1).bit_length() - 1 if ld is not None else 0
    return _lib.CTree(n, dv.ptr(d["node_mins"]), dv.ptr(d["node_maxs"]),
                      dv.ptr(d.get("left")), dv.ptr(d.get("right")), dv.ptr(d["leaf_obj"]),
                      dv.ptr(d["nodes"]), dv.ptr(d["root_box"]), dv.ptr(d.get("leaf_codes")),
                      dv.ptr(ld), bits, int(d.get("flags", 0)))


def _device_boxes(boxes):
    """CUDA tensor input: (n,3) points or (n,6) rows -> (mins, maxs) views."""
    t = boxes.to(torch.float32)
    if t.ndim != 2 or t.shape[1] not in (3, 6):
        raise ValueError(f"X must have shape (n, 3) or (n, 6), got {tuple(t.shape)}")
    if t.shape[1] == 3:
        t = t.contiguous()
        return t, t
    return t[:, :3].contiguous(), t[:, 3:].contiguous()


def build_device(mins: torch.Tensor, maxs: torch.Tensor, check: bool = True,
                 morton_bits: int = 30, leaf_ids: torch.Tensor | None = None) -> Bvh:
    """Build from device-resident (n, 3) f32 ``mins``/``maxs`` (``maxs`` may
    be ``mins`` for point input).  The device-resident entry of :func:`build`.
    ``leaf_ids`` (optional, n i32 on the device): the ordinals the leaves
    report instead of their input index (a shard's global ordinals)."""
    n = int(mins.shape[0])
    if n == 0:
        raise ValueError("empty scene")
    if n > _lib.MAX_ITEMS:
        raise ValueError(f"at most {_lib.MAX_ITEMS} primitives per tree")
    if morton_bits not in (30, 63):
        raise ValueError(f"morton_bits must be 30 or 63, got {morton_bits}")
    l = _lib.lib()
    f32, i32 = torch.float32, torch.int32
    d = {
        "node_mins": dv.empty((2 * n - 1, 3), f32),
        "node_maxs": dv.empty((2 * n - 1, 3), f32),
        "left": dv.empty(max(n - 1, 0), i32),
        "right": dv.empty(max(n - 1, 0), i32),
        "leaf_obj": dv.empty(n, i32),
        "root_box": dv.empty(6, f32),
        "nodes": dv.empty(max(n - 1, 1) * _lib.NODE_BYTES, torch.uint8),
        "leaf_codes": dv.empty(n, i32),  # Morton codes in leaf order (kNN seed)
    }
    # kNN seed index over the sorted leaf codes (2^bits + 1 bucket starts),
    # written by the build's hierarchy pass
    bits = l.lbvh_leaf_directory_bits(n)
    d["leaf_dir"] = dv.empty((1 << bits) + 1, i32)
    ws = dv.workspace(l.lbvh_build_workspace_bytes(n))
    status = dv.Status()
    # the reference-layout rows no query reads are written on first access
    # (Bvh._finish_rows: host fields, device_arrays())
    _lib.check(_launch("build", lambda: l.lbvh_build(
                            dv.ptr(mins), dv.ptr(maxs), n, morton_bits, dv.ptr(ws), ws.numel(),
                            dv.ptr(d["node_mins"]), dv.ptr(d["node_maxs"]), dv.ptr(d["left"]),
                            dv.ptr(d["right"]), dv.ptr(d["leaf_obj"]), dv.ptr(d["root_box"]),
                            dv.ptr(d["nodes"]), dv.ptr(d["leaf_codes"]), dv.ptr(d["leaf_dir"]),
                            bits, _lib.BUILD_DEFER_ROWS,
                            dv.ptr(leaf_ids) if leaf_ids is not None else None, status.ptr,
                            dv.stream())))
    d["rows_pending"] = True
    d["flags"] = ((_lib.TREE_POINT_LEAVES if maxs is mins else 0)
                  | (_lib.TREE_CODES30 if morton_bits == 30 else 0) | _lib.TREE_BUILT)
    if check:
        flags = status.read()
        if flags & _lib.FLAG_NONFINITE:
            raise ValueError("X must contain only finite values")
        if flags & _lib.FLAG_INVERTED_BOX:
            raise ValueError("X contains boxes with min corner above max corner")
    return Bvh._from_device(d, n)


def build(boxes, threads: int = 1, morton_bits: int = 30) -> Bvh:
    """Build a linear BVH over a non-empty collection of boxes (tree.py:177-209).

    Accepts (n, 3) points, (n, 6) corner rows, a ``(mins, maxs)`` pair,
    Box/Point sequences -- or a CUDA tensor of shape (n, 3)/(n, 6), which
    skips the host round trip.  ``threads`` is accepted and ignored.
    Deterministic: identical input gives bit-identical arrays.

    ``morton_bits=63`` (an extension; the reference is 30-bit only) orders the
    leaves by 63-bit codes, 21 bits per axis, for very large clouds.  Queries
    on such a tree return exactly the same results (they are independent of
    the tree shape); only the tree arrays differ from the reference's.
    """
    if dv.is_cuda_tensor(boxes):
        mins, maxs = _device_boxes(boxes)
        return build_device(mins, maxs, morton_bits=morton_bits)
    # Large ndarray inputs are value-checked on the device; pairs and
    # sequences on the host (exact reference messages either way).
    device_checks = isinstance(boxes, np.ndarray)
    mins, maxs = check_boxes(boxes, device_checks=device_checks)
    if mins.shape[0] == 0:
        raise ValueError("empty scene")
    dmins = dv.h2d(mins)
    dmaxs = dmins if maxs is mins else dv.h2d(maxs)
    return build_device(dmins, dmaxs, morton_bits=morton_bits)


# ---------------------------------------------------------------------------
# Topology helpers (reference tree.py:40-119)
# ---------------------------------------------------------------------------


def common_prefix(codes, i: int, j: int) -> int:
    """Common-prefix length of augmented keys i and j (-1 if j out of range).

    Scalar diagnostic helper (tree.py:47-58); the device kernels compute the
    same quantity with ``__clz`` on the fly.
    """
    codes = np.asarray(codes, dtype=np.int64)
    n = codes.shape[0]
    if j < 0 or j >= n:
        return -1
    x = (int(codes[i]) << 32 | i) ^ (int(codes[j]) << 32 | j)
    return 64 - x.bit_length()


def find_split(codes, first: int, last: int) -> int:
    """Karras split of [first, last] (tree.py:61-65); scalar helper."""
    n = len(codes)
    if not 0 <= first < last < n:
        raise ValueError(f"need 0 <= first < last < {n}, got ({first}, {last})")
    common = common_prefix(codes, first, last)
    split, step = first, last - first
    while True:
        step = (step + 1) >> 1
        cand = split + step
        if cand < last and common_prefix(codes, first, cand) > common:
            split = cand
        if step <= 1:
            return split


def node_range(codes, i: int) -> tuple[int, int]:
    """Leaf range of internal node i (tree.py:68-74); scalar helper."""
    n = len(codes)
    if not 0 <= i < n - 1:
        raise ValueError(f"internal ordinal must be in [0, {n - 1}), got {i}")
    d = 1 if common_prefix(codes, i, i + 1) > common_prefix(codes, i, i - 1) else -1
    floor = common_prefix(codes, i, i - d)
    hi = 2
    while common_prefix(codes, i, i + hi * d) > floor:
        hi <<= 1
    span, t = 0, hi >> 1
    while t >= 1:
        if common_prefix(codes, i, i + (span + t) * d) > floor:
            span += t
        t >>= 1
    j = i + span * d
    return (i, j) if i < j else (j, i)


class Topology(NamedTuple):
    """Child links of the n-1 internal nodes plus the parent array."""

    left: np.ndarray
    right: np.ndarray
    parent: np.ndarray


def generate_topology(sorted_codes, threads: int = 1) -> Topology:
    """Radix-tree topology over sorted codes (tree.py:85-105), on the GPU.

    Uses the bottom-up kernel of :func:`build` (topology-only variant); the
    result equals the reference's top-down Karras construction exactly.
    """
    codes = np.ascontiguousarray(sorted_codes, dtype=np.uint32)
    n = codes.shape[0]
    if n < 1:
        raise ValueError("empty scene")
    l = _lib.lib()
    dc = dv.h2d(codes.view(np.int32))
    left = dv.empty(max(n - 1, 0), torch.int32)
    right = dv.empty(max(n - 1, 0), torch.int32)
    parent = dv.empty(2 * n - 1, torch.int32)
    ws = dv.workspace(l.lbvh_topology_workspace_bytes(n))
    _lib.check(l.lbvh_generate_topology(dv.ptr(dc), n, dv.ptr(left), dv.ptr(right),
                                        dv.ptr(parent), dv.ptr(ws), ws.numel(), dv.stream()))
    le, ri, pa = dv.d2h_many(left, right, parent)
    return Topology(le.copy(), ri.copy(), pa.copy())


def refit_bounds(node_mins, node_maxs, topology: Topology) -> None:
    """Fill internal boxes bottom-up in place (tree.py:108-119), on the GPU."""
    n = (node_mins.shape[0] + 1) // 2
    if n <= 1:
        return
    l = _lib.lib()
    dmin = dv.h2d(np.ascontiguousarray(node_mins, dtype=np.float32))
    dmax = dv.h2d(np.ascontiguousarray(node_maxs, dtype=np.float32))
    dl = dv.h2d(np.ascontiguousarray(topology.left, dtype=np.int32))
    dr = dv.h2d(np.ascontiguousarray(topology.right, dtype=np.int32))
    dp = dv.h2d(np.ascontiguousarray(topology.parent, dtype=np.int32))
    ws = dv.workspace(l.lbvh_topology_workspace_bytes(n))
    _lib.check(l.lbvh_refit(dv.ptr(dmin), dv.ptr(dmax), dv.ptr(dl), dv.ptr(dr), dv.ptr(dp), n,
                            dv.ptr(ws), ws.numel(), dv.stream()))
    hmin, hmax = dv.d2h_many(dmin, dmax)
    node_mins[...] = hmin
    node_maxs[...] = hmax
