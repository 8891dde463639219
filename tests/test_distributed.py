"""Sharded distributed search on world-size-2 process groups.

CPU: the routing / exchange / merge host logic on ``gloo`` with the CPU
oracle as the local engine (test infrastructure).  GPU: the same protocol with
the CUDA engine (two ranks sharing cuda:0 over gloo with CPU collectives).
The distributed answer must equal the single-process reference answer on the
concatenated cloud with global ordinals, bit for bit.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """CPU local engine backed by oracle/ (tests only)."""

    device = torch.device("cpu")

    def __init__(self):
        from oracle import oracle

        self.o = oracle

    def morton(self, pts, lo, hi):
        return torch.from_numpy(self.o.morton_codes(pts.numpy(), lo, hi).astype(np.int64))

    def build(self, pts):
        t = self.o.build(pts.numpy(), threads=1)
        t._pts = pts.numpy()
        return t

    def box(self, tree):
        return torch.from_numpy(np.concatenate([tree.scene_min, tree.scene_max]))

    def knn_sq(self, tree, centers, k):
        c = centers.numpy()
        off, idx, _ = self.o.query_knn(tree, c, k, threads=1)
        kk = min(k, tree.leaf_count)
        idx = idx.reshape(-1, kk)
        p = tree._pts[idx]                                      # (m, kk, 3)
        g = np.maximum(np.maximum(p - c[:, None, :], c[:, None, :] - p), np.float32(0))
        d2 = g[..., 0] * g[..., 0]
        d2 = d2 + g[..., 1] * g[..., 1]
        d2 = d2 + g[..., 2] * g[..., 2]
        return torch.from_numpy(idx.astype(np.int64)), torch.from_numpy(d2.astype(np.float32))

    def unpack_keys(self, keys):
        k = keys.numpy()
        d2 = ((k >> 32) & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
        return torch.from_numpy(k & 0xFFFFFFFF), torch.from_numpy(np.sqrt(d2))

    def radius(self, tree, centers, radii):
        off, idx = self.o.query_spatial_2p(tree, centers.numpy(), radii.numpy(), threads=1)
        return torch.from_numpy(off), torch.from_numpy(idx.astype(np.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cloud(n_total, seed):
    from paper_1908_11807_b200 import datasets

    pts = datasets.generate(datasets.CloudSpec("cube", "filled", n_total, seed))
    # force ordinal ties across ranks: exact duplicates in both halves
    pts[n_total // 2 + 7] = pts[3]
    pts[n_total // 2 + 8] = pts[3]
    return pts


def _worker(rank, world, port, engine_kind, n_total, split, queue):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1908_11807_b200 import distributed as D
        from oracle import oracle

        if engine_kind == "gpu":
            torch.cuda.set_device(0)
            engine = D.GpuEngine()
            D.set_comm_device("cpu")
        else:
            engine = OracleEngine()
        pts = _cloud(n_total, 0)
        cut = int(n_total * split)
        lo, hi = (0, cut) if rank == 0 else (cut, n_total)
        if split < 0:  # ranks hold the halves in reverse ordinal order
            cut = n_total // 2
            lo, hi = (cut, n_total) if rank == 0 else (0, cut)
        t = D.build_distributed(pts[lo:hi], lo, engine=engine)
        assert t.total == n_total
        rng = np.random.default_rng(100 + rank)
        a = n_total ** (1 / 3)
        q = rng.uniform(-1.1 * a, 1.1 * a, size=(300, 3)).astype(np.float32)
        q[0] = pts[3]  # query on the duplicated point
        ref = oracle.build(pts, threads=1)
        for k in (1, 10, 37):
            off, gid, dd = D.query_knn_distributed(t, q, k)
            ko, ki, kd = oracle.query_knn(ref, q, k, threads=1)
            assert np.array_equal(off.cpu().numpy(), ko), k
            assert np.array_equal(gid.cpu().numpy(), ki.astype(np.int64)), k
            assert dd.cpu().numpy().tobytes() == kd.tobytes(), k
        for r in (0.0, 1.3, 4.0):
            off, gid = D.query_spatial_distributed(t, q, r)
            so, si = oracle.query_spatial_2p(ref, q, r, threads=1)
            assert np.array_equal(off.cpu().numpy(), so), r
            gh = gid.cpu().numpy()
            for i in range(q.shape[0]):
                assert np.array_equal(np.sort(gh[off[i]:off[i + 1]]),
                                      np.sort(si[so[i]:so[i + 1]])), (r, i)
        if engine_kind == "gpu":
            # pipelined host entry point: chunk counts differ per rank
            qh = q[:300 - 50 * rank]
            ho, hg, hd = D.query_knn_distributed_host(t, qh, 10, chunk=64)
            ko, ki, kd = oracle.query_knn(ref, qh, 10, threads=1)
            assert np.array_equal(ho, ko) and np.array_equal(hg, ki) and hd.tobytes() == kd.tobytes()
        # k beyond the whole cloud
        off, gid, dd = D.query_knn_distributed(t, q[:5], n_total + 3)
        assert int(off[-1]) == 5 * n_total
        # invalid input on ONE rank: every rank raises the reference's
        # ValueError before any payload moves (no rank left blocked)
        bad = q[:20].copy()
        if rank == 1:
            bad[5, 1] = np.nan
        rr = np.full(20, 1.0, np.float32)
        if rank == 0:
            rr[3] = -1.0
        for call, msg in ((lambda: D.query_knn_distributed(t, bad, 10), "finite"),
                          (lambda: D.query_spatial_distributed(t, bad, 1.0), "finite"),
                          (lambda: D.query_spatial_distributed(t, q[:20], rr), "non-negative")):
            try:
                call()
            except ValueError as exc:
                assert msg in str(exc), exc
            else:
                raise AssertionError("invalid input accepted")
        # the group is still usable afterwards
        off, gid, dd = D.query_knn_distributed(t, q[:7], 3)
        assert int(off[-1]) == 21
        dist.barrier()
        dist.destroy_process_group()
        queue.put((rank, "ok"))
    except Exception as exc:  # report to the parent
        import traceback

        queue.put((rank, traceback.format_exc()))
        raise


def _run(engine_kind, n_total, split):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, engine_kind, n_total, split, queue))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    msgs = dict(queue.get(timeout=5) for _ in range(2))
    for r in range(2):
        assert msgs.get(r) == "ok", msgs.get(r)


@pytest.mark.parametrize("split", [0.5, 0.97, -1])
def test_sharded_search_equals_single_process_gloo(split):
    _run("cpu", 2000, split)


@pytest.mark.gpu
@pytest.mark.parametrize("split", [0.5, 0.97, -1])
def test_sharded_search_gpu_engine(split):
    _run("gpu", 20000, split)


def _worker_tiny(rank, world, port, queue):
    """One primitive per rank and k=1: the home's forwarding bound is the
    k-th distance of a one-leaf local tree (traverse.cu n == 1 branch)."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1908_11807_b200 import distributed as D
        from oracle import oracle

        torch.cuda.set_device(0)
        D.set_comm_device("cpu")
        pts = np.array([[0.0, 0.0, 0.0], [10.0, 0.0, 0.0]], np.float32)
        t = D.build_distributed(pts[rank:rank + 1], rank)
        assert t.counts == [1, 1], t.counts
        q = np.random.default_rng(rank).uniform(-5, 15, size=(200, 3)).astype(np.float32)
        ref = oracle.build(pts, threads=1)
        for k in (1, 2):
            off, gid, dd = D.query_knn_distributed(t, torch.from_numpy(q).cuda(), k)
            ko, ki, kd = oracle.query_knn(ref, q, k, threads=1)
            assert np.array_equal(gid.cpu().numpy(), ki), k
            assert dd.cpu().numpy().tobytes() == kd.tobytes(), k
        dist.destroy_process_group()
        queue.put((rank, "ok"))
    except Exception:
        import traceback

        queue.put((rank, traceback.format_exc()))
        raise


@pytest.mark.gpu
def test_sharded_search_one_primitive_per_rank_gpu():
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tiny, args=(r, 2, port, queue)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    msgs = dict(queue.get(timeout=5) for _ in range(2))
    assert msgs == {0: "ok", 1: "ok"}, msgs


def _worker_single(port, queue):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=0, world_size=1)
        from paper_1908_11807_b200 import distributed as D
        from oracle import oracle

        torch.cuda.set_device(0)
        pts = _cloud(5000, 0)
        t = D.build_distributed(pts, 0)
        assert t.global_leaves and t.total == 5000
        q = np.random.default_rng(7).uniform(-20, 20, size=(400, 3)).astype(np.float32)
        ref = oracle.build(pts, threads=1)
        for k in (1, 10, 5003):
            off, gid, dd = D.query_knn_distributed(t, torch.from_numpy(q).cuda(), k)
            ko, ki, kd = oracle.query_knn(ref, q, k, threads=1)
            assert np.array_equal(off.cpu().numpy(), ko) and np.array_equal(gid.cpu().numpy(), ki)
            assert dd.cpu().numpy().tobytes() == kd.tobytes()
        ho, hg, hd = D.query_knn_distributed_host(t, q, 10, chunk=128)
        ko, ki, kd = oracle.query_knn(ref, q, 10, threads=1)
        assert np.array_equal(hg, ki) and hd.tobytes() == kd.tobytes()
        # radius through the full forward / return / merge kernels on one
        # rank: the merged order is then exactly the reference's fill order
        for route in (False, True):
            D._FORCE_ROUTE = route
            for r in (0.0, 1.7, 3.5):
                so, si = oracle.query_spatial_2p(ref, q, r, threads=1)
                off, gid = D.query_spatial_distributed(t, torch.from_numpy(q).cuda(), r)
                assert np.array_equal(off.cpu().numpy(), so), (route, r)
                assert np.array_equal(gid.cpu().numpy(), si.astype(np.int64)), (route, r)
        D._FORCE_ROUTE = False
        dist.destroy_process_group()
        queue.put("ok")
    except Exception:
        import traceback

        queue.put(traceback.format_exc())
        raise


@pytest.mark.gpu
def test_sharded_search_single_rank_gpu():
    """world_size 1: the sharded protocol without exchanges (BENCH_FORCE_SHARDED)."""
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    p = ctx.Process(target=_worker_single, args=(_free_port(), queue))
    p.start()
    p.join(timeout=600)
    assert queue.get(timeout=5) == "ok"
