"""Sharded multi-GPU search: local BVHs under a top tree of rank boxes.

SURVEY.md §8(e).  One process per GPU (``torch.distributed``, NCCL over
NVLink/NVSwitch).  The reference has no distributed path (PAPER.md:1127-1137,
SPEC.md:14); results here are defined as the single-process reference result
on the concatenated cloud with **global** ordinals, and every step below keeps
that exact:

build
  1. global scene box: all-reduce min / max of the local primitives;
  2. 30-bit Morton codes on that grid (the reference recipe, f64) and keys
     ``code << 32 | global ordinal``;
  3. splitters from an all-gathered key sample cut the key space into P
     contiguous Morton ranges; primitives move to their range's rank with one
     variable all-to-all (counts first, then payload);
  4. each rank builds a local BVH on its range (device kernels) and keeps
     the global ordinal of every local primitive;
  5. the top tree is the all-gathered array of P rank boxes.

kNN
  1. every query goes to its *home* rank (the Morton range holding its
     code); the home runs a local kNN (squared distances) and takes its k-th
     distance^2 R (inf if the home has fewer than k primitives);
  2. the query is forwarded to every other rank whose box distance^2 <= R
     (non-strict, so ordinal ties survive); those run a local kNN;
  3. candidates return to the home, which keeps the k smallest by the
     reference's lexicographic (d^2, global ordinal) order
     (_kernels.py:293-296) and takes sqrt;
  4. results return to the query's origin rank, in its query order.
  Any point of the global top-k lies on a rank whose box distance is <= its
  distance <= R, so nothing is lost; the merge order is exact.

radius
  a query goes to every rank whose box distance^2 <= r*r (fp32, as the
  kernels); hits come back as global ordinals, sorted per query.

The local search and the few dense helpers go through an ``Engine``: the
default :class:`GpuEngine` uses this package's CUDA kernels; tests may plug a
CPU engine (the oracle) to exercise the routing on ``gloo``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["GpuEngine", "DistributedBvh", "build_distributed", "query_knn_distributed",
           "query_knn_distributed_host", "query_spatial_distributed"]


# ---------------------------------------------------------------------------
# engines
# ---------------------------------------------------------------------------


class GpuEngine:
    """Local search on this rank's GPU through the C ABI (no CPU path)."""

    def __init__(self, device: torch.device | None = None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def morton(self, pts: torch.Tensor, lo: np.ndarray, hi: np.ndarray) -> torch.Tensor:
        from . import _device as dv
        from . import _lib

        n = int(pts.shape[0])
        codes = torch.empty(n, dtype=torch.int32, device=self.device)
        if n:
            p64 = pts.to(torch.float64).contiguous()
            lo = np.ascontiguousarray(lo, dtype=np.float64)
            hi = np.ascontiguousarray(hi, dtype=np.float64)
            _lib.check(_lib.lib().lbvh_morton_codes(dv.ptr(p64), n, lo.ctypes.data,
                                                    hi.ctypes.data, dv.ptr(codes), dv.stream()))
        return codes.to(torch.int64)

    def morton32(self, pts: torch.Tensor, box: torch.Tensor) -> torch.Tensor:
        """i32 codes of f32 points on a device (6,) f32 scene box -- the same
        codes as :meth:`morton` without the f64 staging copy."""
        from . import _device as dv
        from . import _lib

        n = int(pts.shape[0])
        codes = torch.empty(n, dtype=torch.int32, device=self.device)
        if n:
            _lib.check(_lib.lib().lbvh_morton_codes_f32(dv.ptr(pts.contiguous()), n,
                                                        dv.ptr(box), dv.ptr(codes),
                                                        dv.stream()))
        return codes

    def build(self, pts: torch.Tensor, gids: torch.Tensor | None = None):
        """Local BVH; with ``gids`` its leaves report those (global) ordinals."""
        from .tree import build, build_device

        if gids is None:
            return build(pts.contiguous())
        p = pts.contiguous()
        return build_device(p, p, leaf_ids=gids.to(torch.int32).contiguous())

    def box(self, tree) -> torch.Tensor:
        return tree._device()["root_box"].clone()

    def knn_sq(self, tree, centers: torch.Tensor, k: int):
        from .traversal import query_knn_squared

        m = int(centers.shape[0])
        kk = min(k, tree.leaf_count)
        rs = query_knn_squared(tree, (centers.contiguous(), k))
        return (rs.indices.to(torch.int64).reshape(m, kk), rs.distances.reshape(m, kk))

    def knn_final(self, tree, centers: torch.Tensor, k: int):
        """Final lists in one kernel: (ordinals i32 (m, kk), sqrt distances
        f32 (m, kk), exact k-th d^2 (m,)); k <= 32."""
        from .traversal import knn_with_kth

        return knn_with_kth(tree, centers.contiguous(), k)

    def knn_sq_raw(self, tree, centers: torch.Tensor, k: int):
        """(m, min(k, n)) local ordinals (i32) and exact fp32 d^2, on device."""
        from .traversal import query_knn_squared

        m = int(centers.shape[0])
        kk = min(k, tree.leaf_count)
        rs = query_knn_squared(tree, (centers.contiguous(), k))
        return rs.indices.reshape(m, kk), rs.distances.reshape(m, kk)

    def globalize(self, tree, gids: torch.Tensor) -> None:
        """Renumber the local tree's leaves with global ordinals (< 2^31): its
        queries then report them and break distance ties by them."""
        from . import _device as dv
        from . import _lib

        d = tree._device()
        g = gids.to(torch.int64).contiguous()
        _lib.check(_lib.lib().lbvh_remap_leaves(tree.ctree(), dv.ptr(d["leaf_obj"]),
                                                dv.ptr(d["nodes"]), dv.ptr(g), dv.stream()))
        tree._host.clear()  # host views are re-read on access

    def radius(self, tree, centers: torch.Tensor, radii: torch.Tensor):
        from .traversal import query_spatial_2p

        rs = query_spatial_2p(tree, (centers.contiguous(), radii.contiguous()))
        return rs.offsets, rs.indices.to(torch.int64)

    def unpack_keys(self, keys: torch.Tensor):
        """(d^2 bits << 32 | ordinal) keys -> (ordinals, __fsqrt_rn(d^2))."""
        from . import _device as dv
        from . import _lib

        gid = torch.empty(keys.shape, dtype=torch.int64, device=self.device)
        dd = torch.empty(keys.shape, dtype=torch.float32, device=self.device)
        _lib.check(_lib.lib().lbvh_unpack_knn_keys(dv.ptr(keys), keys.numel(), dv.ptr(gid),
                                                   dv.ptr(dd), dv.stream()))
        return gid, dd


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------


_COMM = {}  # group -> device collectives run on (the data device unless overridden)
# Payload bytes this rank has sent to OTHER ranks through the all-to-alls
# (counts exchanges excluded); bench.py reads it for nvlink_frac.
STATS = {"a2a_bytes_sent": 0}


def _count_sent(splits, row_bytes: int, group) -> None:
    me = dist.get_rank(group)
    STATS["a2a_bytes_sent"] += (sum(splits) - splits[me]) * row_bytes


def _comm_device(group, data_dev):
    return _COMM.get(group, data_dev)


def _partition(dest: torch.Tensor, world: int):
    """Stable partition of row indices by destination rank -> (order, counts
    tensor).  On CUDA one radix pass of the library's sort over
    ceil(log2 world) key bits; elsewhere torch."""
    if dest.is_cuda and dest.numel() > 1:
        from . import _device as dv
        from . import _lib

        n = int(dest.numel())
        keys = dest.to(torch.int32).contiguous()
        order = torch.arange(n, dtype=torch.int32, device=dest.device)
        l = _lib.lib()
        ws = dv.workspace(l.lbvh_sort_workspace_bytes(n))
        bits = max(1, (world - 1).bit_length())
        _lib.check(l.lbvh_sort_pairs(dv.ptr(keys), dv.ptr(order), n, bits, dv.ptr(ws),
                                     ws.numel(), dv.stream()))
        edges = torch.searchsorted(keys, torch.arange(world + 1, dtype=torch.int32,
                                                      device=dest.device))
        return order.to(torch.int64), (edges[1:] - edges[:-1]).to(torch.int64)
    order = torch.argsort(dest, stable=True)
    return order, torch.bincount(dest, minlength=world).to(torch.int64)


def _query_flags(c: torch.Tensor, r: torch.Tensor | None = None) -> torch.Tensor:
    """This rank's batch value checks as LBVH_FLAG_* bits in a device int64
    scalar (no host sync): non-finite centers, non-finite or negative radii."""
    from . import _lib

    f = (~torch.isfinite(c)).any().to(torch.int64) * _lib.FLAG_NONFINITE
    if r is not None:
        bad_r = (~torch.isfinite(r)) | (r < 0)
        f = f | (bad_r.any().to(torch.int64) * _lib.FLAG_BAD_RADIUS)
    return f


def _raise_flags(flags: int) -> None:
    if flags:
        from .traversal import _raise_flags as raise_reference

        raise_reference(flags)


def _alltoallv(rows: torch.Tensor, dest: torch.Tensor, world: int, group=None,
               grouped_counts=None, flags: torch.Tensor | None = None):
    """Send row i of ``rows`` to rank ``dest[i]``; returns (received rows,
    per-source counts).  Counts are exchanged first, then the payload.
    ``grouped_counts`` (list): rows are already grouped by destination with
    these counts (``dest`` is then ignored).  ``flags`` (device int64
    scalar, :func:`_query_flags`): this rank's input checks travel with the
    counts, and EVERY rank raises the reference's ValueError before any
    payload moves if any rank's batch is invalid (a rank raising alone would
    leave the others blocked in the collective)."""
    if world == 1:
        if flags is not None:
            _raise_flags(int(flags))
        return rows, [int(rows.shape[0])]
    cdev = _comm_device(group, rows.device)
    if grouped_counts is not None:
        send = rows.contiguous().to(cdev)
        counts = torch.tensor(grouped_counts, dtype=torch.int64, device=cdev)
    else:
        order, counts = _partition(dest, world)
        send = rows[order].contiguous().to(cdev)
        counts = counts.to(cdev)
    if flags is not None:
        pair = torch.stack([counts, flags.to(cdev).expand(world)], dim=1).contiguous()
        recv_pair = torch.empty_like(pair)
        dist.all_to_all_single(recv_pair, pair, group=group)
        got = recv_pair.tolist()
        f = 0
        for _, x in got:
            f |= int(x)
        _raise_flags(f)
        sc, rc = counts.tolist(), [int(x) for x, _ in got]
    else:
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=group)
        sc, rc = counts.tolist(), recv_counts.tolist()
    _count_sent(sc, rows[:1].numel() * rows.element_size() if rows.shape[0] else 0, group)
    recv = torch.empty((sum(rc),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=cdev)
    dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=sc,
                           group=group)
    return recv.to(rows.device), rc


def _all_reduce(x: torch.Tensor, op, group):
    cdev = _comm_device(group, x.device)
    y = x.to(cdev)
    dist.all_reduce(y, op=op, group=group)
    return y.to(x.device)


def _all_gather(x: torch.Tensor, world: int, group):
    if world == 1:  # nothing to exchange
        return [x]
    cdev = _comm_device(group, x.device)
    y = x.to(cdev)
    out = [torch.empty_like(y) for _ in range(world)]
    dist.all_gather(out, y, group=group)
    return [o.to(x.device) for o in out]


def set_comm_device(device, group=None) -> None:
    """Run this group's collectives on ``device`` (e.g. CPU tensors for a
    gloo group whose ranks share one GPU in tests)."""
    _COMM[group] = torch.device(device)


def _source_ranks(counts, device) -> torch.Tensor:
    return torch.repeat_interleave(torch.arange(len(counts), device=device),
                                   torch.tensor(counts, device=device))


def _box_dist_sq(c: torch.Tensor, boxes: torch.Tensor) -> torch.Tensor:
    """(m,3) centers x (P,6) boxes -> (m,P) fp32 distance^2, the kernels'
    recipe: per-axis clamp gap, squared, summed x -> y -> z, unfused."""
    d = None
    for a in range(3):
        v = c[:, a:a + 1]
        lo, hi = boxes[None, :, a], boxes[None, :, 3 + a]
        g = torch.clamp(torch.maximum(lo - v, v - hi), min=0.0)
        g2 = g * g
        d = g2 if d is None else d + g2
    return d


# ---------------------------------------------------------------------------
# distributed tree
# ---------------------------------------------------------------------------


@dataclass
class DistributedBvh:
    engine: object
    tree: object | None          # local BVH (None when this rank got no primitives)
    gids: torch.Tensor           # global ordinal of each local primitive
    boxes: torch.Tensor          # (P, 6) rank boxes (+inf / -inf for empty ranks)
    counts: list                 # primitives per rank
    split_codes: torch.Tensor    # (P-1,) Morton codes cutting the ranges
    scene_lo: np.ndarray
    scene_hi: np.ndarray
    world: int
    rank: int
    group: object = None
    monotone: bool = True        # local ordinal order == global ordinal order
    global_leaves: bool = False  # the local tree's leaves carry global ordinals

    @property
    def total(self) -> int:
        return int(sum(self.counts))


def build_distributed(local_points, global_offset: int, engine=None, group=None,
                      samples_per_rank: int = 1024) -> DistributedBvh:
    """Collective: every rank passes its (n_r, 3) primitives whose global
    ordinals are ``global_offset .. global_offset + n_r - 1``."""
    engine = engine or GpuEngine()
    dev = engine.device
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts = torch.as_tensor(local_points, dtype=torch.float32).to(dev).reshape(-1, 3).contiguous()
    n = int(pts.shape[0])
    # every rank's ordinal range: the total, the payload width, and whether
    # received primitives arrive in global ordinal order
    ranges = _all_gather(torch.tensor([int(global_offset), n], dtype=torch.int64, device=dev),
                         world, group)
    ranges = ([(int(global_offset), n)] if world == 1 else
              [(int(r[0]), int(r[1])) for r in torch.stack(ranges).cpu()])
    total = sum(c for _, c in ranges)
    # GPU engine: the local build writes global ordinals straight into its
    # leaves (lbvh_build leaf_ids), so local searches report -- and break
    # distance ties by -- global ordinals
    global_ids = hasattr(engine, "globalize") and total < 2 ** 31
    gdt = torch.int32 if global_ids else torch.int64
    gids = torch.arange(int(global_offset), int(global_offset) + n, dtype=gdt, device=dev)
    scene_lo = scene_hi = None
    if world > 1:
        # 1. global scene box: one all-reduce (MAX) of (-min, max)
        if n:
            box = torch.cat([-pts.amin(dim=0), pts.amax(dim=0)])
        else:
            box = torch.full((6,), -math.inf, device=dev)
        box = _all_reduce(box, dist.ReduceOp.MAX, group)
        scene = torch.cat([-box[:3], box[3:]]).contiguous()
        scene_h = scene.cpu().numpy().astype(np.float64)
        scene_lo, scene_hi = scene_h[:3], scene_h[3:]
        # 2. keys on the global grid: (30-bit code << 32) | global ordinal
        if hasattr(engine, "morton32"):  # f32 points on a device box: no f64 staging
            codes = engine.morton32(pts, scene).to(torch.int64)
        else:
            codes = engine.morton(pts, scene_lo, scene_hi)
        keys = (codes << 32) | gids.to(torch.int64)
        # 3. splitters from a strided sample of the (unsorted) keys: exact
        #    results for any splitters, the sample only sets the balance
        s = samples_per_rank
        if n:
            pick = torch.linspace(0, n - 1, s, device=dev).round().to(torch.int64)
            sample = keys[pick]
        else:
            sample = torch.full((s,), torch.iinfo(torch.int64).max, dtype=torch.int64,
                                device=dev)
        gathered = _all_gather(sample, world, group)
        allsamp = torch.sort(torch.cat(gathered)).values
        cut = [allsamp[(i * allsamp.numel()) // world] for i in range(1, world)]
        splitters = torch.stack(cut)
        dest = torch.searchsorted(splitters, keys, right=True)
        # primitives travel as 32-bit words: f32 x, y, z and the global
        # ordinal (one word below 2^31, else two)
        wide = max(o + c for o, c in ranges) > 2 ** 31 - 1
        rows = torch.empty((n, 5 if wide else 4), dtype=torch.int32, device=dev)
        rows[:, :3] = pts.view(torch.int32)
        if wide:
            rows[:, 3:5] = gids.to(torch.int64).view(torch.int32).reshape(n, 2)
        else:
            rows[:, 3] = gids.to(torch.int32)
        recv, _ = _alltoallv(rows, dest, world, group)
        rpts = recv[:, :3].contiguous().view(torch.float32)
        rgids = (recv[:, 3:5].contiguous().view(torch.int64).reshape(-1) if wide
                 else recv[:, 3].to(gdt))
        # sources arrive in rank order, each in its own ordinal order (the
        # partition is stable): already sorted when the ranks' ordinal ranges
        # increase with the rank; otherwise sort (the local kNN breaks
        # distance ties by local ordinal, _kernels.py:293-296)
        live = [(o, c) for o, c in ranges if c]
        if any(live[i][0] + live[i][1] > live[i + 1][0] for i in range(len(live) - 1)):
            gorder = torch.argsort(rgids)
            rgids = rgids[gorder]
            rpts = rpts[gorder].contiguous()
    else:
        splitters = torch.empty(0, dtype=torch.int64, device=dev)
        rpts, rgids = pts, gids
    # 4. local build
    m = int(rpts.shape[0])
    if m:
        tree = engine.build(rpts, rgids) if global_ids else engine.build(rpts)
        box = engine.box(tree).to(dev)
    else:
        tree = None
        box = torch.tensor([math.inf] * 3 + [-math.inf] * 3, dtype=torch.float32, device=dev)
    # 5. top tree: rank boxes and primitive counts in one gather
    top = _all_gather(torch.cat([box.to(torch.float32),
                                 torch.tensor([m], dtype=torch.int32,
                                              device=dev).view(torch.float32)]), world, group)
    top = torch.stack(top)
    boxes = top[:, :6].contiguous()
    counts = [m] if world == 1 else top[:, 6].contiguous().view(torch.int32).tolist()
    if scene_lo is None:  # one rank: the scene box is the local tree's
        scene_h = boxes[0].cpu().numpy().astype(np.float64)
        scene_lo, scene_hi = scene_h[:3], scene_h[3:]
    return DistributedBvh(engine, tree, rgids, boxes, counts, splitters >> 32, scene_lo,
                          scene_hi, world, rank, group, True, global_ids)


def _local_knn(t: DistributedBvh, centers: torch.Tensor, k: int):
    """(m, k) global ordinals and d^2 (padded with -1 / inf) from this rank."""
    dev = t.engine.device
    m = int(centers.shape[0])
    gid = torch.full((m, k), -1, dtype=torch.int64, device=dev)
    d2 = torch.full((m, k), math.inf, dtype=torch.float32, device=dev)
    if m and t.tree is not None:
        idx, dd = t.engine.knn_sq(t.tree, centers, k)
        kk = idx.shape[1]
        gid[:, :kk] = idx if t.global_leaves else t.gids[idx]
        d2[:, :kk] = dd
    return gid, d2


def _merge_keys(gid: torch.Tensor, d2: torch.Tensor) -> torch.Tensor:
    """Lexicographic (d^2, ordinal) as one int64 key; padding sorts last."""
    bits = d2.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    key = (bits << 32) | (gid & 0xFFFFFFFF)
    return torch.where(gid < 0, torch.full_like(key, torch.iinfo(torch.int64).max), key)


def _merge_remote(own_keys_rows: torch.Tensor, brow: torch.Tensor, bq: torch.Tensor, k: int,
                  kk: int, nresp: torch.Tensor, rows: torch.Tensor, mh: int):
    """k smallest (d^2, global ordinal) keys of each listed row over its own
    candidates and every responder's (bq rows: [row, d^2 x k, ordinal x k])."""
    dev = own_keys_rows.device
    nr = rows.numel()
    pos = torch.full((mh,), -1, dtype=torch.int64, device=dev)
    pos[rows] = torch.arange(nr, device=dev)
    width = k * (1 + int(nresp[rows].max().item()))
    cand = torch.full((nr, width), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
    cand[:, :own_keys_rows.shape[1]] = own_keys_rows
    if brow.numel():
        o = torch.argsort(brow, stable=True)
        brow_s = brow[o]
        starts = torch.cumsum(nresp, 0) - nresp
        slot = torch.arange(brow_s.numel(), device=dev) - starts[brow_s]
        cols = (1 + slot)[:, None] * k + torch.arange(k, device=dev)[None, :]
        cand[pos[brow_s][:, None], cols] = _merge_keys(
            bq[o, 1 + k:1 + 2 * k].to(torch.int64),
            bq[o, 1:1 + k].contiguous().view(torch.float32))
    return torch.sort(cand, dim=1).values[:, :kk].contiguous(), pos


def _home_chunk(t: DistributedBvh, hc: torch.Tensor, k: int, kk: int):
    """Home-side kNN of received queries ``hc`` (collective: every rank calls
    it the same number of times): local kNN, forwarding to ranks within the
    bound, merge, and the return arrays (sqrt(d^2) f32, global ordinal i32),
    rows in ``hc`` order."""
    from . import _device as dv
    from . import _lib

    l = _lib.lib()
    dev, world, g = t.engine.device, t.world, t.group
    mh = int(hc.shape[0])
    nloc = t.counts[t.rank] if t.tree is not None else 0
    if (nloc and mh and k <= 32 and t.global_leaves and hasattr(t.engine, "knn_final")):
        return _home_chunk_fused(t, hc, k, kk)
    if nloc and mh:
        lidx, ld2 = t.engine.knn_sq_raw(t.tree, hc, k)
    else:
        kl = min(k, nloc)
        lidx = torch.empty((mh, kl), dtype=torch.int32, device=dev)
        ld2 = torch.empty((mh, kl), dtype=torch.float32, device=dev)
    if nloc >= k:
        bound = ld2[:, k - 1].contiguous()
    else:
        bound = torch.full((mh,), math.inf, dtype=torch.float32, device=dev)
    # forward to the other ranks within the bound
    cand_ranks = 0
    for r in range(world):
        if t.counts[r] > 0 and r != t.rank:
            cand_ranks |= 1 << r
    merged_pos = top = None
    if cand_ranks:
        mask = torch.zeros(mh, dtype=torch.int32, device=dev)
        boxes = t.boxes.to(torch.float32).contiguous()
        _lib.check(l.lbvh_rank_forward_mask(dv.ptr(hc), dv.ptr(bound), 0.0, mh, dv.ptr(boxes),
                                            world, cand_ranks, dv.ptr(mask), dv.stream()))
        sel = torch.nonzero(mask, as_tuple=True)[0]
        shifts = torch.arange(world, dtype=torch.int32, device=dev)[None, :]
        si, rr = torch.nonzero((mask[sel, None] >> shifts) & 1, as_tuple=True)
        qi = sel[si]
        frows = torch.empty((qi.numel(), 4), dtype=torch.float32, device=dev)
        frows[:, :3] = hc[qi]
        frows[:, 3] = qi.to(torch.int32).view(torch.float32)
        fq, fcounts = _alltoallv(frows, rr, world, g)
        f_gid, f_d2 = _local_knn(t, fq[:, :3].contiguous(), k)
        back = torch.cat([fq[:, 3:4].contiguous().view(torch.int32), f_d2.view(torch.int32),
                          f_gid.to(torch.int32)], dim=1)
        bq, _ = _alltoallv(back, None, world, g, grouped_counts=fcounts)
        # merge at home, only for queries that got remote candidates
        brow = bq[:, 0].to(torch.int64)
        nresp = torch.bincount(brow, minlength=mh) if brow.numel() else torch.zeros(
            mh, dtype=torch.int64, device=dev)
        if nloc < kk:  # the home alone cannot fill a span: every query merges
            mrows = torch.arange(mh, device=dev)
        else:
            mrows = torch.nonzero(nresp > 0, as_tuple=True)[0]
        if mrows.numel():
            if nloc:
                lm = lidx[mrows].to(torch.int64)
                own = _merge_keys(lm if t.global_leaves else t.gids[lm], ld2[mrows])
            else:
                own = torch.empty((mrows.numel(), 0), dtype=torch.int64, device=dev)
            top, merged_pos = _merge_remote(own, brow, bq, k, kk, nresp, mrows, mh)
    # return arrays (sqrt(d^2), global ordinal), rows in arrival order
    if nloc < kk:  # every row is merged; the local lists are not read
        lidx = torch.zeros((mh, kk), dtype=torch.int32, device=dev)
        ld2 = torch.zeros((mh, kk), dtype=torch.float32, device=dev)
    rd = torch.empty((mh, kk), dtype=torch.float32, device=dev)
    rg = torch.empty((mh, kk), dtype=torch.int32, device=dev)
    _lib.check(l.lbvh_knn_finalize(mh, kk, dv.ptr(lidx.contiguous()), dv.ptr(ld2.contiguous()),
                                   None if t.global_leaves else dv.ptr(t.gids),
                                   dv.ptr(merged_pos), dv.ptr(top), dv.ptr(rd), dv.ptr(rg),
                                   dv.stream()))
    return rd, rg


def _home_chunk_fused(t: DistributedBvh, hc: torch.Tensor, k: int, kk: int):
    """_home_chunk whose local kNN writes the final lists (sqrt distances,
    global ordinals) and the exact k-th d^2 bound in one kernel; only the
    queries that received remote candidates are searched again (squared) to
    merge, and their rows are overwritten."""
    from . import _device as dv
    from . import _lib

    l = _lib.lib()
    dev, world, g = t.engine.device, t.world, t.group
    mh = int(hc.shape[0])
    nloc = t.counts[t.rank]
    rg, rd, kth = t.engine.knn_final(t.tree, hc, k)
    bound = kth if nloc >= k else torch.full((mh,), math.inf, dtype=torch.float32, device=dev)
    if rg.shape[1] < kk:  # the home alone cannot fill a span: every row is merged below
        rg = torch.empty((mh, kk), dtype=torch.int32, device=dev)
        rd = torch.empty((mh, kk), dtype=torch.float32, device=dev)
    cand_ranks = 0
    for r in range(world):
        if t.counts[r] > 0 and r != t.rank:
            cand_ranks |= 1 << r
    if not cand_ranks:
        return rd, rg
    mask = torch.zeros(mh, dtype=torch.int32, device=dev)
    boxes = t.boxes.to(torch.float32).contiguous()
    _lib.check(l.lbvh_rank_forward_mask(dv.ptr(hc), dv.ptr(bound), 0.0, mh, dv.ptr(boxes),
                                        world, cand_ranks, dv.ptr(mask), dv.stream()))
    sel = torch.nonzero(mask, as_tuple=True)[0]
    shifts = torch.arange(world, dtype=torch.int32, device=dev)[None, :]
    si, rr = torch.nonzero((mask[sel, None] >> shifts) & 1, as_tuple=True)
    qi = sel[si]
    frows = torch.empty((qi.numel(), 4), dtype=torch.float32, device=dev)
    frows[:, :3] = hc[qi]
    frows[:, 3] = qi.to(torch.int32).view(torch.float32)
    fq, fcounts = _alltoallv(frows, rr, world, g)
    f_gid, f_d2 = _local_knn(t, fq[:, :3].contiguous(), k)
    back = torch.cat([fq[:, 3:4].contiguous().view(torch.int32), f_d2.view(torch.int32),
                      f_gid.to(torch.int32)], dim=1)
    bq, _ = _alltoallv(back, None, world, g, grouped_counts=fcounts)
    brow = bq[:, 0].to(torch.int64)
    nresp = torch.bincount(brow, minlength=mh) if brow.numel() else torch.zeros(
        mh, dtype=torch.int64, device=dev)
    if nloc < kk:
        mrows = torch.arange(mh, device=dev)
    else:
        mrows = torch.nonzero(nresp > 0, as_tuple=True)[0]
    if mrows.numel():
        lidx, ld2 = t.engine.knn_sq_raw(t.tree, hc[mrows].contiguous(), k)
        own = _merge_keys(lidx.to(torch.int64), ld2)
        top, _ = _merge_remote(own, brow, bq, k, kk, nresp, mrows, mh)
        gid, dd = t.engine.unpack_keys(top)
        rd[mrows] = dd
        rg[mrows] = gid.to(torch.int32)
    return rd, rg


# Home queries can be processed in chunks when world > 1 so that the
# all-to-all returning chunk j's results overlaps chunk j+1's search; each
# chunk adds host syncs (measured on one GPU, routed: 12.0 / 13.3 / 14.2 ms
# per 1e7-query step for 1 / 2 / 4 chunks), so the default is 1.
_SHARD_CHUNKS = 1
# measurement switch: take the routed (partition + exchange) path even on one rank
_FORCE_ROUTE = False


class _PendingReturn:
    """One chunk's result exchange in flight (split sizes already agreed)."""

    def __init__(self, rd, rg, splits, world, group):
        cdev = _comm_device(group, rd.device)
        counts = torch.tensor(splits, dtype=torch.int64, device=cdev)
        rcounts = torch.empty_like(counts)
        dist.all_to_all_single(rcounts, counts, group=group)
        self.rc = rcounts.tolist()
        self.dev = rd.device
        self.sends = (rd.contiguous().to(cdev), rg.contiguous().to(cdev))
        for x in self.sends:
            _count_sent(splits, x[:1].numel() * x.element_size() if x.shape[0] else 0, group)
        self.recvs = tuple(torch.empty((sum(self.rc),) + tuple(x.shape[1:]), dtype=x.dtype,
                                       device=cdev) for x in self.sends)
        self.works = [dist.all_to_all_single(r, x, output_split_sizes=self.rc,
                                             input_split_sizes=splits, group=group,
                                             async_op=True)
                      for r, x in zip(self.recvs, self.sends)]

    def finish(self, order, out_d, out_g, cursor):
        """Wait, then scatter each source's piece straight to its queries:
        piece rows are the next ``cnt`` entries of that source's slice of the
        origin's partition permutation ``order``."""
        from . import _device as dv
        from . import _lib

        for w in self.works:
            w.wait()
        rd, rg = (x.to(self.dev) for x in self.recvs)
        kk = out_d.shape[1]
        off = 0
        for src, cnt in enumerate(self.rc):
            if cnt:
                _lib.check(_lib.lib().lbvh_scatter_result_rows(
                    cnt, kk, dv.ptr(order[cursor[src]:cursor[src] + cnt]),
                    dv.ptr(rd[off:off + cnt]), dv.ptr(rg[off:off + cnt]), dv.ptr(out_d),
                    dv.ptr(out_g), dv.stream()))
                cursor[src] += cnt
                off += cnt


def _query_knn_gpu(t: DistributedBvh, c: torch.Tensor, k: int):
    """query_knn_distributed on CUDA.  Results come back in the order the
    queries were sent, so the origin scatters them with its own partition
    permutation; library kernels compute the forwarding masks and the return
    arrays, tensor ops touch only the forwarded minority (queries near a
    rank boundary).  With several ranks the home work runs in chunks and
    chunk j's results travel (asynchronous all-to-all) while chunk j+1 is
    searched."""
    from . import _device as dv
    from . import _lib

    dev, world, g = t.engine.device, t.world, t.group
    c = c.contiguous()
    nq = int(c.shape[0])
    kk = min(k, t.total)
    if world == 1 and not _FORCE_ROUTE:
        rd, rg = _home_chunk(t, c.contiguous(), k, kk)
        offsets = torch.arange(nq + 1, dtype=torch.int64, device=dev) * kk
        return offsets, rg.reshape(-1), rd.reshape(-1)
    # 1. to the home rank (its Morton range)
    box = torch.tensor(np.concatenate([t.scene_lo, t.scene_hi]).astype(np.float32), device=dev)
    codes = t.engine.morton32(c, box)
    home = torch.searchsorted(t.split_codes.to(torch.int32), codes, right=True)
    order, counts = _partition(home, world)
    sent = counts.tolist()
    send = torch.empty_like(c)
    _lib.check(_lib.lib().lbvh_gather_rows3(dv.ptr(c), dv.ptr(order), nq, dv.ptr(send),
                                             dv.stream()))
    hc, hcounts = _alltoallv(send, None, world, g, grouped_counts=sent, flags=_query_flags(c))
    hc = hc.contiguous()
    mh = int(hc.shape[0])
    # rows of origin o occupy [hstart[o], hstart[o + 1]) of hc
    hstart = [0]
    for x in hcounts:
        hstart.append(hstart[-1] + x)
    # results are scattered straight into query order: a piece from home h
    # covers the next rows of h's slice of this rank's send order
    rd_out = torch.empty((nq, kk), dtype=torch.float32, device=dev)
    rg_out = torch.empty((nq, kk), dtype=torch.int32, device=dev)
    cursor = [0]
    for x in sent[:-1]:
        cursor.append(cursor[-1] + x)
    chunks = max(1, _SHARD_CHUNKS)
    pending = None
    for j in range(chunks):
        r0, r1 = j * mh // chunks, (j + 1) * mh // chunks
        rd, rg = _home_chunk(t, hc[r0:r1], k, kk)
        splits = [max(0, min(r1, hstart[o + 1]) - max(r0, hstart[o])) for o in range(world)]
        nxt = _PendingReturn(rd, rg, splits, world, g)
        if pending is not None:
            pending.finish(order, rd_out, rg_out, cursor)
        pending = nxt
    pending.finish(order, rd_out, rg_out, cursor)
    offsets = torch.arange(nq + 1, dtype=torch.int64, device=dev) * kk
    return offsets, rg_out.reshape(-1), rd_out.reshape(-1)


def query_knn_distributed(t: DistributedBvh, centers, k: int):
    """Collective kNN over the sharded cloud.  Returns (offsets int64,
    global ordinals, distances f32) for this rank's queries, in order; spans
    are min(k, total) long, sorted by (distance, ordinal).  Ordinals are
    int32 on the CUDA path (clouds below 2^31 points), int64 otherwise."""
    if k < 1:
        raise ValueError("k must be >= 1")
    dev, world, g = t.engine.device, t.world, t.group
    c = torch.as_tensor(centers, dtype=torch.float32).to(dev).reshape(-1, 3)
    if c.is_cuda and isinstance(t.engine, GpuEngine) and world <= 32 and t.total < 2 ** 31:
        return _query_knn_gpu(t, c, k)
    nq = int(c.shape[0])
    kk = min(k, t.total)
    # Payload rows are 32-bit words: f32 coordinates / d^2 and i32 indices
    # (bit-cast), so every exchange moves 16 B per query and 4 B per candidate.
    # 1. to the home rank
    codes = t.engine.morton(c, t.scene_lo, t.scene_hi)
    home = torch.searchsorted(t.split_codes, codes, right=True)
    rows = torch.empty((nq, 4), dtype=torch.float32, device=dev)
    rows[:, :3] = c
    rows[:, 3] = torch.arange(nq, dtype=torch.int32, device=dev).view(torch.float32)
    hq, hcounts = _alltoallv(rows, home, world, g, flags=_query_flags(c))
    origin = _source_ranks(hcounts, dev)
    hc = hq[:, :3].contiguous()
    mh = int(hc.shape[0])
    own_gid, own_d2 = _local_knn(t, hc, k)
    if t.tree is not None and t.counts[t.rank] >= k:
        bound = own_d2[:, k - 1]
    else:
        bound = torch.full((mh,), math.inf, dtype=torch.float32, device=dev)
    # 2. forward to ranks within the bound
    bd = _box_dist_sq(hc, t.boxes)                                  # (mh, P)
    need = (bd <= bound[:, None]) & (torch.tensor(t.counts, device=dev) > 0)[None, :]
    need[:, t.rank] = False
    qi, rr = torch.nonzero(need, as_tuple=True)
    frows = torch.empty((qi.numel(), 4), dtype=torch.float32, device=dev)
    frows[:, :3] = hc[qi]
    frows[:, 3] = qi.to(torch.int32).view(torch.float32)
    fq, fcounts = _alltoallv(frows, rr, world, g)
    fsrc = _source_ranks(fcounts, dev)
    f_gid, f_d2 = _local_knn(t, fq[:, :3].contiguous(), k)
    back = torch.cat([fq[:, 3:4].contiguous().view(torch.int32), f_d2.view(torch.int32),
                      f_gid.to(torch.int32)], dim=1)
    bq, _ = _alltoallv(back, fsrc, world, g)
    # 3. merge at home: own candidates + every responder's
    brow = bq[:, 0].to(torch.int64)
    nresp = torch.bincount(brow, minlength=mh) if brow.numel() else torch.zeros(
        mh, dtype=torch.int64, device=dev)
    own_keys = _merge_keys(own_gid, own_d2)
    if t.monotone:
        # local ordinals map to global ones in increasing order, so an own
        # list (sorted by (d^2, local ordinal)) is already in merge order
        top = own_keys[:, :kk].clone()
        rows = torch.nonzero(nresp > 0, as_tuple=True)[0]
    else:
        top = torch.empty((mh, kk), dtype=torch.int64, device=dev)
        rows = torch.arange(mh, device=dev)
    if rows.numel():
        nr = rows.numel()
        pos = torch.full((mh,), -1, dtype=torch.int64, device=dev)
        pos[rows] = torch.arange(nr, device=dev)
        width = k * (1 + int(nresp[rows].max().item()))
        cand = torch.full((nr, width), torch.iinfo(torch.int64).max, dtype=torch.int64,
                          device=dev)
        cand[:, :k] = own_keys[rows]
        if brow.numel():
            o = torch.argsort(brow, stable=True)
            brow_s = brow[o]
            starts = torch.cumsum(nresp, 0) - nresp
            slot = torch.arange(brow_s.numel(), device=dev) - starts[brow_s]
            cols = (1 + slot)[:, None] * k + torch.arange(k, device=dev)[None, :]
            cand[pos[brow_s][:, None], cols] = _merge_keys(
                bq[o, 1 + k:1 + 2 * k].to(torch.int64),
                bq[o, 1:1 + k].contiguous().view(torch.float32))
        top[rows] = torch.sort(cand, dim=1).values[:, :kk]
    # ordinals and correctly rounded sqrt(d^2) (torch's CPU sqrt is not)
    res_gid, res_dist = t.engine.unpack_keys(top.contiguous())
    # 4. back to the origin rank, scattered straight into query order
    ret = torch.cat([hq[:, 3:4].contiguous().view(torch.int32), res_dist.view(torch.int32),
                     res_gid.to(torch.int32)], dim=1)
    got, _ = _alltoallv(ret, origin, world, g)
    qix = got[:, 0].to(torch.int64)
    dist_out = torch.empty((nq, kk), dtype=torch.float32, device=dev)
    gid_out = torch.empty((nq, kk), dtype=torch.int64, device=dev)
    dist_out[qix] = got[:, 1:1 + kk].contiguous().view(torch.float32)
    gid_out[qix] = got[:, 1 + kk:1 + 2 * kk].to(torch.int64)
    offsets = torch.arange(nq + 1, dtype=torch.int64, device=dev) * kk
    return offsets, gid_out.reshape(-1), dist_out.reshape(-1)


def query_knn_distributed_host(t: DistributedBvh, centers, k: int, chunk: int = 1 << 21,
                               out=None):
    """Collective kNN for host (pinned or pageable numpy / CPU tensor) queries,
    pipelined over chunks: the H2D copy of chunk i+1 and the D2H copy of
    chunk i-1 overlap the sharded search of chunk i.  Every rank must pass
    the same number of chunks (the chunk count is agreed with an all-reduce).
    Returns numpy (offsets int64, ordinals, distances f32) -- views of pinned
    buffers, or of ``out`` = (offsets, ordinals, distances) pinned tensors when
    given.  Results are identical to :func:`query_knn_distributed`."""
    dev, world, g = t.engine.device, t.world, t.group
    host = torch.as_tensor(centers, dtype=torch.float32).reshape(-1, 3)
    if not host.is_pinned():
        host = host.pin_memory()
    nq = int(host.shape[0])
    kk = min(k, t.total)
    nchunks = torch.tensor([max(1, -(-nq // chunk))], dtype=torch.int64, device=dev)
    if world > 1:
        nchunks = _all_reduce(nchunks, dist.ReduceOp.MAX, g)
    nchunks = int(nchunks.item())
    gid_dtype = torch.int32 if t.total < 2 ** 31 and dev.type == "cuda" else torch.int64
    if out is None:
        h_off = torch.empty(nq + 1, dtype=torch.int64, pin_memory=True)
        h_gid = torch.empty(nq * kk, dtype=gid_dtype, pin_memory=True)
        h_dd = torch.empty(nq * kk, dtype=torch.float32, pin_memory=True)
    else:
        h_off, h_gid, h_dd = out
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    dev_c = torch.empty((nq, 3), dtype=torch.float32, device=dev)
    from .traversal import _host_arange_into

    off_jobs = _host_arange_into(h_off.numpy(), kk)  # host threads, no D2H
    per = -(-nq // nchunks) if nq else 0
    for i in range(nchunks):
        c0, c1 = min(nq, i * per), min(nq, (i + 1) * per)
        e_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            dev_c[c0:c1].copy_(host[c0:c1], non_blocking=True)
            e_in.record(s_in)
        comp.wait_event(e_in)
        off, gid, dd = query_knn_distributed(t, dev_c[c0:c1], k)
        e_c = torch.cuda.Event()
        e_c.record(comp)
        s_out.wait_event(e_c)
        with torch.cuda.stream(s_out):
            h_gid[c0 * kk:c1 * kk].copy_(gid, non_blocking=True)
            h_dd[c0 * kk:c1 * kk].copy_(dd, non_blocking=True)
            gid.record_stream(s_out)
            dd.record_stream(s_out)
    s_out.synchronize()
    comp.wait_stream(s_out)
    for j in off_jobs:
        j.result()
    return h_off.numpy(), h_gid.numpy(), h_dd.numpy()


def query_spatial_distributed(t: DistributedBvh, centers, radius):
    """Collective radius search.  Returns (offsets int64, global ordinals
    int64) for this rank's queries, in order.  A query's hits are grouped by
    the rank that holds them (rank order), each rank's in its traversal
    (fill) order -- a deterministic order; as sets they equal the reference's
    on the concatenated cloud."""
    dev, world, g = t.engine.device, t.world, t.group
    c = torch.as_tensor(centers, dtype=torch.float32).to(dev).reshape(-1, 3).contiguous()
    nq = int(c.shape[0])
    r = torch.as_tensor(radius, dtype=torch.float32).to(dev)
    r = r.expand(nq).contiguous() if r.ndim == 0 else r.reshape(-1).contiguous()
    flags = _query_flags(c, r)
    if c.is_cuda and isinstance(t.engine, GpuEngine) and world <= 32:
        return _query_spatial_gpu(t, c, r, flags)
    r2 = r * r
    bd = _box_dist_sq(c, t.boxes)
    need = (bd <= r2[:, None]) & (torch.tensor(t.counts, device=dev) > 0)[None, :]
    qi, rr = torch.nonzero(need, as_tuple=True)
    rows = torch.empty((qi.numel(), 5), dtype=torch.float32, device=dev)
    rows[:, :3] = c[qi]
    rows[:, 3] = r[qi]
    rows[:, 4] = qi.to(torch.int32).view(torch.float32)
    rq, rcounts = _alltoallv(rows, rr, world, g, flags=flags)
    src = _source_ranks(rcounts, dev)
    m = int(rq.shape[0])
    if m and t.tree is not None:
        off, idx = t.engine.radius(t.tree, rq[:, :3].contiguous(), rq[:, 3].contiguous())
        cnt = off[1:] - off[:-1]
        owner = torch.repeat_interleave(torch.arange(m, device=dev), cnt)
        qcol = rq[:, 4].contiguous().view(torch.int32)
        hit = idx if t.global_leaves else t.gids[idx]
        hit_rows = torch.stack([qcol[owner], hit.to(torch.int32)], dim=1)
        hit_dest = src[owner]
    else:
        hit_rows = torch.empty((0, 2), dtype=torch.int32, device=dev)
        hit_dest = torch.empty(0, dtype=torch.int64, device=dev)
    got, _ = _alltoallv(hit_rows, hit_dest, world, g)
    # rows arrive grouped by source rank, each source's in its fill order: a
    # stable sort by query keeps exactly that order inside every query
    qix = got[:, 0].to(torch.int64)
    o = torch.argsort(qix, stable=True)
    counts = torch.bincount(qix, minlength=nq) if qix.numel() else torch.zeros(
        nq, dtype=torch.int64, device=dev)
    offsets = torch.zeros(nq + 1, dtype=torch.int64, device=dev)
    offsets[1:] = torch.cumsum(counts, 0)
    return offsets, got[:, 1].to(torch.int64)[o]


def _query_spatial_gpu(t: DistributedBvh, c: torch.Tensor, r: torch.Tensor, flags):
    """query_spatial_distributed on CUDA: forward mask, forwarded rows, the
    per-row hit counts and the hits travel back, and the origin appends each
    source's hits per query -- library kernels, no sort."""
    from . import _device as dv
    from . import _lib

    l = _lib.lib()
    st = dv.stream()
    dev, world, g = t.engine.device, t.world, t.group
    nq = int(c.shape[0])
    i64, i32 = torch.int64, torch.int32
    if world == 1 and not _FORCE_ROUTE:
        _raise_flags(int(flags))
        if t.tree is None or nq == 0:
            return torch.zeros(nq + 1, dtype=i64, device=dev), torch.empty(0, dtype=i64,
                                                                            device=dev)
        off, idx = t.engine.radius(t.tree, c, r)
        hit = idx if t.global_leaves else t.gids[idx]
        return off, hit.to(i64)
    # 1. forward every query to each non-empty rank within its radius
    cand = 0
    for rk in range(world):
        if t.counts[rk] > 0:
            cand |= 1 << rk
    mask = torch.zeros(nq, dtype=i32, device=dev)
    r2 = (r * r).contiguous()
    boxes = t.boxes.to(torch.float32).contiguous()
    if nq:
        _lib.check(l.lbvh_rank_forward_mask(dv.ptr(c), dv.ptr(r2), 0.0, nq, dv.ptr(boxes),
                                            world, cand, dv.ptr(mask), st))
    per_rank = torch.empty(world, dtype=i32, device=dev)
    _lib.check(l.lbvh_forward_rows(dv.ptr(c), dv.ptr(r), dv.ptr(mask), nq, world,
                                   dv.ptr(per_rank), None, None, None, 0, st))
    sent = per_rank.tolist()
    starts = [0]
    for x in sent:
        starts.append(starts[-1] + x)
    start_d = torch.tensor(starts[:-1], dtype=i64, device=dev)
    cursor = torch.empty(world, dtype=i32, device=dev)
    rows = torch.empty((starts[-1], 5), dtype=torch.float32, device=dev)
    _lib.check(l.lbvh_forward_rows(dv.ptr(c), dv.ptr(r), dv.ptr(mask), nq, world, None,
                                   dv.ptr(start_d), dv.ptr(cursor), dv.ptr(rows), 1, st))
    rq, rcounts = _alltoallv(rows, None, world, g, grouped_counts=sent, flags=flags)
    # 2. responder: local search of the received rows (fill order, global ordinals)
    m = int(rq.shape[0])
    if m and t.tree is not None:
        off, idx = t.engine.radius(t.tree, rq[:, :3].contiguous(), rq[:, 3].contiguous())
        hits = (idx if t.global_leaves else t.gids[idx]).to(i32)
        rec = (off[1:] - off[:-1]).to(i32)
        bnd = [0]
        for x in rcounts:
            bnd.append(bnd[-1] + x)
        edges = off[torch.tensor(bnd, dtype=i64, device=dev)].tolist()
        hit_split = [edges[i + 1] - edges[i] for i in range(world)]
    else:
        hits = torch.empty(0, dtype=i32, device=dev)
        rec = torch.zeros(m, dtype=i32, device=dev)
        hit_split = [0] * world
    got_rec, _ = _alltoallv(rec, None, world, g, grouped_counts=list(rcounts))
    got_hits, _ = _alltoallv(hits, None, world, g, grouped_counts=hit_split)
    got_rec = got_rec.contiguous()
    got_hits = got_hits.contiguous()
    # 3. origin: per-query totals, CRS offsets, then sources appended in rank order
    n_rec = int(got_rec.shape[0])
    acc = torch.zeros(nq, dtype=i32, device=dev)
    _lib.check(l.lbvh_merge_records(dv.ptr(rows), dv.ptr(got_rec), None, n_rec, None, world,
                                    None, None, dv.ptr(acc), None, 0, st))
    ws = dv.workspace(l.lbvh_scan_workspace_bytes(max(nq, n_rec, 1)))
    offsets = torch.empty(nq + 1, dtype=i64, device=dev)
    _lib.check(l.lbvh_exclusive_scan(dv.ptr(acc), nq, dv.ptr(offsets), dv.ptr(ws), ws.numel(),
                                     st))
    rec_off = torch.empty(n_rec + 1, dtype=i64, device=dev)
    _lib.check(l.lbvh_exclusive_scan(dv.ptr(got_rec), n_rec, dv.ptr(rec_off), dv.ptr(ws),
                                     ws.numel(), st))
    total = int(offsets[nq].item()) if nq else 0
    out = torch.empty(total, dtype=i64, device=dev)
    if total == 0:
        return offsets, out
    acc.zero_()
    src_starts = np.array(starts, dtype=np.int64)
    _lib.check(l.lbvh_merge_records(dv.ptr(rows), dv.ptr(got_rec), dv.ptr(rec_off), n_rec,
                                    src_starts.ctypes.data, world, dv.ptr(got_hits),
                                    dv.ptr(offsets), dv.ptr(acc), dv.ptr(out), 1, st))
    return offsets, out
