"""Benchmark of the B200 LBVH hot path (BASELINE.json metric, config C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (``value``): kNN (k=10) queries/sec, 1e7 filled-box points indexed,
1e7 filled-box queries (cube:filled seed 0 / seed 1, the reference bench's
clouds), inputs resident in HBM, query Morton pre-sort included, timed with
CUDA events on the launching stream; L2 is flushed (256 MiB write) before
every timed step.  One step = one query batch of nq queries through
``query_knn`` (device-resident entry).  ``e2e`` is the same metric through
the public API with pinned host input and numpy (pinned) results.  Extra
metrics of the same run (build prims/s, radius 2P / 1P, hollow sphere C3)
are in ``extra``.

``--impl reference`` times the CPU restatement of the reference path
(oracle/, all host threads) on a bounded sample of the same workload.

Multi-GPU (torchrun): one process per GPU over NCCL; the step is the
sharded search of SURVEY §8(e) (``distributed.query_knn_distributed``:
Morton-range shards, rank-box top tree, all-to-all query forwarding, exact
merge); time is the max over ranks.  Default: weak scaling, the global cloud
is N*1e7 points and N*1e7 queries, rank r holds the r-th chunk of each.
``--global-points G`` (C4: G = 8e7): strong scaling, G points and G queries
in total, G/N per rank.  ``BENCH_BACKEND=gloo`` runs the same protocol with
CPU collectives (testing several ranks on one GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# This image sets NCCL_DEBUG=VERSION, which makes NCCL print "NCCL version ..."
# to stdout at communicator init; stdout must carry only the one JSON line, so
# that setting (and only that one) is dropped before torch loads NCCL.
if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
    del os.environ["NCCL_DEBUG"]

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")

# Algorithmic bytes; T = box tests per query of the
# reference algorithm on the reference tree (filled 1e7).
T_KNN_FILLED_1E7 = 157.8
T_RAD_FILLED_1E7 = 133.1
T_RAD_HOLLOW_1E7 = 43.7
BUILD_BYTES_PER_PRIM = 152


def knn_bytes_per_query(k: int, t: float = T_KNN_FILLED_1E7) -> float:
    return 12 + 8 + 8 * k + 28 * t


def radius_bytes_per_query(hits: float, t: float) -> float:
    return 12 + 4 + 8 + 4 * hits + 28 * t


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--points", dest="m", type=int, default=10_000_000, help="indexed points per GPU")
    p.add_argument("--queries", dest="nq", type=int, default=None, help="queries per GPU (default m)")
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--no-extra", action="store_true", help="headline metric only")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--cpu-sample", type=int, default=1_000_000,
                   help="queries in the CPU baseline sample")
    p.add_argument("--sweep-max", type=int, default=100_000_000,
                   help="largest n of the C5 construction sweep")
    p.add_argument("--profile", action="store_true",
                   help="short run for ncu: no clocks/cpu/e2e/extra legs")
    p.add_argument("--global-points", type=int, default=0,
                   help="strong scaling (C4): this many points and queries in total, "
                        "split over the ranks")
    return p.parse_args(argv)


def world_size(args) -> int:
    return int(os.environ.get("WORLD_SIZE", str(args.gpus if args.impl == "reference" else 1)))


def shape_of(args, world: int):
    """(points per rank, queries per rank, global points, global queries)."""
    if args.global_points:
        g = args.global_points
        return g // world, g // world, g // world * world, g // world * world
    m = args.m
    nq = args.nq or m
    return m, nq, world * m, world * nq


def workload(args, world: int) -> dict:
    """The ``config`` object both arms print (same workload, same keys)."""
    m, nq, gm, gq = shape_of(args, world)
    k = args.k
    if world == 1 and not args.global_points:
        wl = (f"C2 kNN: cube:filled m={m} seed 0 / cube:filled nq={nq} seed 1, k={k}, "
              "query Morton pre-sort on")
    else:
        tag = "C4 strong" if args.global_points else "weak"
        wl = (f"{tag} sharded kNN: global cube:filled {gm} points seed 0 / cube:filled {gq} "
              f"queries seed 1, rank r holds the r-th contiguous chunk of each, k={k}")
    return {"workload": wl, "m_per_gpu": m, "nq_per_gpu": nq, "k": k,
            "global_points": gm, "global_queries": gq,
            "l2": "flushed before every timed step (256 MiB device write)",
            "parallelism": (f"sharded x{world}: Morton-range shards, rank-box top tree, "
                            "NCCL all-to-all forwarding" if world > 1 else "single GPU")}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def load_peaks():
    try:
        with open(PEAKS_PATH) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    try:
        with open(NCU_SUMMARY) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during a timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        loaded = []
        for r in rows:
            for i, nm in enumerate(names):
                if "Active" in r[2 + i] and "Not" not in r[2 + i]:
                    reasons.add(nm)
            try:
                if float(r[6]) > 0:
                    loaded.append(float(r[0]))
            except ValueError:
                pass
        all_sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        sm = statistics.median(loaded or all_sm) if (loaded or all_sm) else None
        return {"sm_mhz": sm, "sm_max_mhz": float(rows[0][1]), "reasons": sorted(reasons),
                "samples": len(rows), "samples_under_load": len(loaded)}


class KernelTimer:
    """CUDA-event brackets around named launches (traversal.KERNEL_TIMER)."""

    def __init__(self):
        import torch

        self.torch = torch
        self.events = {}
        self.enabled = False

    def wrap(self, name, call):
        if not self.enabled:
            return call()
        t = self.torch
        s, e = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        s.record()
        rc = call()
        e.record()
        self.events.setdefault(name, []).append((s, e))
        return rc

    def pair(self, name):
        """Events for a kernel the library brackets itself (fused calls)."""
        if not self.enabled:
            return None
        t = self.torch
        s, e = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        s.record()  # materialise the handles; the library re-records them
        e.record()
        self.events.setdefault(name, []).append((s, e))
        return s, e

    def mean_ms(self, name):
        ev = self.events.get(name, [])
        if not ev:
            return None
        return sum(s.elapsed_time(e) for s, e in ev) / len(ev)

    def reset(self):
        self.events = {}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as tdist

    import paper_1908_11807_b200 as lb
    from paper_1908_11807_b200 import _lib, traversal, tree as tree_mod

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one GPU per rank; several ranks share a GPU only in BENCH_BACKEND=gloo tests
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # BENCH_FORCE_SHARDED=1 runs the sharded protocol (and its NCCL calls) even
    # at N=1, to exercise it on a one-GPU box
    dist_mode = world > 1 or os.environ.get("BENCH_FORCE_SHARDED") == "1"
    if dist_mode:
        backend = os.environ.get("BENCH_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
            from paper_1908_11807_b200 import distributed as _D

            _D.set_comm_device("cpu")

    def barrier():
        if dist_mode:
            tdist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist_mode:
            return x
        on_gpu = tdist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    m, nq, gm, gq = shape_of(args, world)
    k = args.k
    lib = _lib.lib()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush_l2():
        flush_buf.fill_(rank & 0xFF)

    # One global cloud of gm filled-box points (seed 0) and gq queries (seed
    # 1), the reference bench's clouds; rank r holds the r-th contiguous chunk
    # of each (N=1: exactly configuration C2; weak: gm = N*m; C4: gm fixed).
    if world == 1:
        pts = lb.generate(lb.CloudSpec("cube", "filled", m, 0))
        qs = lb.generate(lb.CloudSpec("cube", "filled", nq, 1))
    else:
        # the global clouds generated on each GPU (bit-identical to numpy's)
        # and sliced; the host copies feed the e2e leg and the CPU baseline
        pts_d = lb.datasets.generate_device(
            lb.CloudSpec("cube", "filled", gm, 0), dev)[rank * m:(rank + 1) * m].clone()
        qs_d = lb.datasets.generate_device(
            lb.CloudSpec("cube", "filled", gq, 1), dev)[rank * nq:(rank + 1) * nq].clone()
        torch.cuda.empty_cache()
        pts, qs = pts_d.cpu().numpy(), qs_d.cpu().numpy()
    if world == 1:
        pts_d = torch.from_numpy(pts).to(dev)
        qs_d = torch.from_numpy(qs).to(dev)
    r = lb.default_radius(k)

    timer = KernelTimer()
    traversal.KERNEL_TIMER = timer
    tree_mod.KERNEL_TIMER = timer

    def timed_loop(step_fn, steps, warmup, kernel=None):
        for _ in range(warmup):
            step_fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        timer.reset()
        timer.enabled = True
        launches0 = lib.lbvh_launch_count()
        total_ms = 0.0
        for _ in range(steps):
            flush_l2()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step_fn()
            e.record()
            e.synchronize()
            total_ms += s.elapsed_time(e)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        timer.enabled = False
        launches = lib.lbvh_launch_count() - launches0
        kms = timer.mean_ms(kernel) if kernel else None
        return max_over_ranks(total_ms), launches, kms

    # -- build the index once (its own timed leg below) ----------------------
    sharded = None
    if not dist_mode:
        tree = lb.build(pts_d)

        def knn_step():
            return lb.query_knn(tree, (qs_d, k))
    else:
        # sharded search: local BVHs under a rank-box top tree,
        # NCCL all-to-all query forwarding and exact kNN merge
        from paper_1908_11807_b200 import distributed as D

        tree = None
        sharded = {}

        def dbuild():
            sharded.pop("t", None)  # free the previous tree first (allocator reuse)
            sharded["t"] = D.build_distributed(pts_d, rank * m)

        bt, _, _ = timed_loop(dbuild, 3, 1)
        sharded["build_ms"] = bt / 3

        def knn_step():
            return D.query_knn_distributed(sharded["t"], qs_d, k)

    clocks = None
    if dist_mode:
        from paper_1908_11807_b200 import distributed as D
    sent0 = D.STATS["a2a_bytes_sent"] if dist_mode else 0
    if args.profile:
        tot, launches, knn_ms = timed_loop(knn_step, args.steps, args.warmup, "knn")
    else:
        with ClockSampler(local) as cs:
            tot, launches, knn_ms = timed_loop(knn_step, args.steps, args.warmup, "knn")
        clocks = cs.summary()
    if dist_mode:
        # bytes every rank sent to the others during warm-up + timed steps,
        # scaled to the timed steps; NVLink 5: 900 GB/s per direction per GPU
        sent = (D.STATS["a2a_bytes_sent"] - sent0) * args.steps / (args.steps + args.warmup)
        on_gpu = tdist.get_backend() == "nccl"
        st = torch.tensor([float(sent)], dtype=torch.float64, device=dev if on_gpu else "cpu")
        tdist.all_reduce(st)
        a2a_bytes = float(st.item())
    ms_per_step = tot / args.steps
    value = world * nq * args.steps / (tot / 1e3)

    peak_gbs, peak_src = load_peaks()
    bq = knn_bytes_per_query(k)
    achieved = nq * bq / (knn_ms / 1e3) / 1e9 if knn_ms else None
    traffic = load_traffic().get("knn_kernel_dram_bytes_per_launch")
    roofline = {
        "bound": "hbm", "kernel": "knn_kernel<10>",
        "achieved": round(achieved, 1) if achieved else None, "peak": peak_gbs, "unit": "GB/s",
        "frac": round(achieved / peak_gbs, 4) if achieved else None,
        "traffic": traffic,
        "kernel_ms": round(knn_ms, 4) if knn_ms else None,
        "kernel_share_of_step": round(knn_ms / ms_per_step, 3) if knn_ms else None,
        "algorithmic_bytes_per_query": bq,
        "bytes_model": "modeled, not a hardware ceiling: 12 center + 8 offset + 8k idx/dist "
                       f"+ 28 B x T box tests, T={T_KNN_FILLED_1E7} (SURVEY.md 6.3, filled 1e7), "
                       "every box test counted as an HBM read (no cache reuse); frac > 1 "
                       "because node records are L1/L2 hits and the seeded traversal makes "
                       "fewer box tests (2 x 71.7 node visits per query) than the reference "
                       "algorithm's T -- the bound is instruction issue, see 'hardware'",
        "peak_source": peak_src,
    }
    hw = load_traffic().get("knn_hardware")
    if hw:
        # the measured side (ncu --set full of the same kernel, profiles/):
        # DRAM bytes per launch over the live kernel time, and the issue /
        # SIMT figures that actually bound it
        hw = dict(hw)
        if knn_ms and traffic:
            hw["dram_gbs"] = round(traffic / (knn_ms / 1e3) / 1e9, 1)
            hw["dram_frac"] = round(traffic / (knn_ms / 1e3) / 1e9 / peak_gbs, 4)
        roofline["hardware"] = hw

    out = {
        "metric": f"knn_queries_per_sec (k={k}, {m:.0e} filled-box points, {nq:.0e} queries)",
        "value": round(value, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if args.global_points else "weak", "vs_baseline": None,
        "dtype": "f32",
        "dtype_note": "fp32 box distances (reference recipe, unfused); f64 Morton normalisation",
        "data": "synthetic: paper_1908_11807_b200.datasets PCG64 clouds (reference generators)",
        "config": workload(args, world),
        "roofline": roofline,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
    }
    if clocks is not None:
        out["clocks"] = clocks
    if dist_mode:
        out["nvlink"] = {"a2a_bytes_per_step": round(a2a_bytes / args.steps),
                         "nvlink_frac": round(a2a_bytes / args.steps / (ms_per_step / 1e3)
                                              / (900e9 * world), 6),
                         "peak": "900 GB/s per direction per GPU (NVLink 5)"}

    if not args.profile:
        # -- e2e through the public API with pinned host buffers --------------
        pin = torch.empty((nq, 3), dtype=torch.float32, pin_memory=True)
        pin.numpy()[:] = qs
        host_q = pin.numpy()
        if sharded is not None:
            span_s = min(k, world * m)
            h_off = torch.empty(nq + 1, dtype=torch.int64, pin_memory=True)
            gid_dtype = torch.int32 if world * m < 2 ** 31 else torch.int64
            h_gid = torch.empty(nq * span_s, dtype=gid_dtype, pin_memory=True)
            h_dd = torch.empty(nq * span_s, dtype=torch.float32, pin_memory=True)

        def e2e_step():
            if sharded is not None:
                # pinned host queries in, pinned host results out, pipelined
                # over chunks (H2D / sharded search / D2H overlap)
                return D.query_knn_distributed_host(sharded["t"], pin, k,
                                                    out=(h_off, h_gid, h_dd))
            rs = lb.query_knn(tree, (host_q, k))
            assert rs.indices.shape[0] == nq * min(k, m)
            return rs

        e2e_tot, _, _ = timed_loop(e2e_step, max(2, args.steps // 2), 2)
        e2e_steps = max(2, args.steps // 2)
        span = min(k, m)
        out["e2e"] = {"value": round(world * nq * e2e_steps / (e2e_tot / 1e3), 1),
                      "unit": "queries/s",
                      "h2d_bytes_per_step": nq * 12,
                      # offsets (uniform spans) are written by host threads
                      "d2h_bytes_per_step": (nq * span * 8 + 4 if sharded is None
                                             else nq * min(k, world * m)
                                             * (4 + h_gid.element_size())),
                      "ms_per_step": round(e2e_tot / e2e_steps, 3),
                      "api": ("paper_1908_11807_b200.query_knn(tree, (pinned numpy centers, k))"
                              if sharded is None else
                              "paper_1908_11807_b200.distributed.query_knn_distributed("
                              "sharded tree, pinned centers, k) -> pinned host arrays")}

    if sharded is not None:
        out["extra"] = {"sharded_build_ms": round(sharded["build_ms"], 3),
                        "sharded_build_prims_per_sec": round(world * m / (sharded["build_ms"] / 1e3), 1),
                        "local_prims_this_rank": int(sharded["t"].counts[rank])}
    elif not args.no_extra and not args.profile:
        out["extra"] = extra_metrics(args, lb, tree, pts_d, qs_d, qs, r, timed_loop, world, rank,
                                     dev, peak_gbs)

    if world == 1 and not args.no_cpu and not args.profile:
        out["cpu_baseline"] = cpu_baseline(args, pts, qs, k)

    traversal.KERNEL_TIMER = None
    tree_mod.KERNEL_TIMER = None
    if dist_mode:
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def extra_metrics(args, lb, tree, pts_d, qs_d, qs, r, timed_loop, world, rank, dev, peak_gbs):
    import torch

    m = int(pts_d.shape[0])
    nq = int(qs_d.shape[0])
    steps, warm = args.steps, args.warmup
    ex = {}

    # build prims/s (device-resident input, full pipeline)
    def build_step():
        return lb.build(pts_d)

    tot, launches, bms = timed_loop(build_step, steps, warm, "build")
    ex["build_prims_per_sec"] = round(world * m * steps / (tot / 1e3), 1)
    ex["build_ms"] = round(tot / steps, 3)
    t63, _, _ = timed_loop(lambda: lb.build(pts_d, morton_bits=63), steps, warm)
    ex["build63_prims_per_sec"] = round(world * m * steps / (t63 / 1e3), 1)
    ex["build_roofline_frac"] = round(m * BUILD_BYTES_PER_PRIM / (bms / 1e3) / 1e9 / peak_gbs, 4)
    ex["build_launches_per_step"] = launches / steps

    # radius 2P, filled/filled
    counts_box = {}

    def rad_step():
        rs = lb.query_spatial_2p(tree, (qs_d, r))
        counts_box["total"] = rs.offsets[-1]
        return rs

    tot, _, cms = timed_loop(rad_step, steps, warm, "spatial_count")
    hits = float(counts_box["total"]) / nq
    ex["radius_2p_queries_per_sec"] = round(world * nq * steps / (tot / 1e3), 1)
    ex["radius_2p_ms"] = round(tot / steps, 3)
    ex["radius_mean_hits"] = round(hits, 3)
    if cms:
        ex["radius_count_kernel_frac"] = round(
            nq * radius_bytes_per_query(hits, T_RAD_FILLED_1E7) / (cms / 1e3) / 1e9 / peak_gbs, 4)

    # radius 2P end to end: pinned host centers in, numpy CRS out (the
    # reference's call), chunk-pipelined H2D / count / fill / D2H
    pin_q = torch.empty((nq, 3), dtype=torch.float32, pin_memory=True)
    pin_q.copy_(qs_d)
    host_q = pin_q.numpy()

    def rad_e2e_step():
        rs = lb.query_spatial_2p(tree, (host_q, r))
        counts_box["e2e_total"] = int(rs.offsets[-1])
        return rs

    tot, _, _ = timed_loop(rad_e2e_step, max(2, steps // 2), 2)
    ex["radius_2p_e2e_queries_per_sec"] = round(world * nq * max(2, steps // 2) / (tot / 1e3), 1)
    ex["radius_2p_e2e_d2h_bytes_per_step"] = (nq + 1) * 8 + counts_box["e2e_total"] * 4
    del pin_q, host_q

    # radius 1P, B=64 (max count at 1e7 is 33, so B=32 would fall back)
    fb = {}

    def rad1_step():
        rs, f = lb.query_spatial_1p(tree, (qs_d, r), 64)
        fb["f"] = f
        return rs

    tot, _, _ = timed_loop(rad1_step, steps, warm)
    ex["radius_1p_b64_queries_per_sec"] = round(world * nq * steps / (tot / 1e3), 1)
    ex["radius_1p_b64_fell_back"] = bool(fb["f"])

    # C3: hollow-sphere sources vs filled queries, radius 2P
    hs_d = lb.datasets.generate_device(lb.CloudSpec("sphere", "hollow", m, 2 * rank), dev)
    htree = lb.build(hs_d)

    def c3_step():
        rs = lb.query_spatial_2p(htree, (qs_d, r))
        counts_box["h"] = rs.offsets[-1]
        return rs

    tot, _, _ = timed_loop(c3_step, steps, warm)
    ex["c3_hollow_radius_2p_queries_per_sec"] = round(world * nq * steps / (tot / 1e3), 1)
    ex["c3_mean_hits"] = round(float(counts_box["h"]) / nq, 3)

    # kNN against the hollow sphere (the reference replay needs ~6,000 box
    # tests per query here): a stress case for the search bound
    def c3_knn_step():
        return lb.query_knn(htree, (qs_d, args.k))

    tot, _, _ = timed_loop(c3_knn_step, 2, 1)
    ex["c3_hollow_knn_queries_per_sec"] = round(world * nq * 2 / (tot / 1e3), 1)
    del htree, hs_d

    # C5: construction-only sweep, filled cube seed 0 (device-resident input)
    sweep = {}
    for n_b in (10_000, 100_000, 1_000_000, 10_000_000, 100_000_000):
        if n_b > args.sweep_max:
            break
        p_b = lb.datasets.generate_device(lb.CloudSpec("cube", "filled", n_b, 0), dev)
        reps = 10 if n_b <= 1_000_000 else 3
        tot, _, _ = timed_loop(lambda: lb.build(p_b), reps, 2)
        sweep[str(n_b)] = {"ms": round(tot / reps, 4),
                           "prims_per_sec": round(n_b * reps / (tot / 1e3), 1)}
        del p_b
        torch.cuda.empty_cache()
    ex["c5_build_sweep"] = sweep
    return ex


def cpu_baseline(args, pts, qs, k):
    """Oracle port (oracle/lbvh_oracle.c, OpenMP, all host threads) beside
    every workload the GPU run reports, each on a bounded
    sample: kNN C2 (headline, ``value``), radius 2P C2, radius 2P C3
    (hollow-sphere sources) and the C5 construction sweep up to 1e7."""
    from oracle import oracle
    import paper_1908_11807_b200.datasets as ds

    threads = host_threads(oracle)
    sample_n = min(args.cpu_sample, qs.shape[0])
    sample = qs[:sample_n]
    ref = oracle.build(pts, threads=threads)
    oracle.query_knn(ref, sample[:1000], k, threads=threads)  # warm
    t0 = time.perf_counter()
    oracle.query_knn(ref, sample, k, threads=threads)
    dt = time.perf_counter() - t0
    legs = {}
    r = ds.default_radius(k)
    t0 = time.perf_counter()
    off, _ = oracle.query_spatial_2p(ref, sample, r, threads=threads)
    legs["radius_2p_c2_queries_per_sec"] = round(sample_n / (time.perf_counter() - t0), 1)
    del off, ref
    t0 = time.perf_counter()
    oracle.build(pts, threads=threads)
    bdt = time.perf_counter() - t0
    hs = ds.generate(ds.CloudSpec("sphere", "hollow", pts.shape[0], 0))
    href = oracle.build(hs, threads=threads)
    t0 = time.perf_counter()
    oracle.query_spatial_2p(href, sample, r, threads=threads)
    legs["radius_2p_c3_queries_per_sec"] = round(sample_n / (time.perf_counter() - t0), 1)
    del href, hs
    sweep = {}
    for n_b in (10_000, 100_000, 1_000_000, 10_000_000):
        p_b = pts if n_b == pts.shape[0] else ds.generate(ds.CloudSpec("cube", "filled", n_b, 0))
        reps = 5 if n_b <= 100_000 else 1
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.build(p_b, threads=threads)
        sweep[str(n_b)] = round(n_b * reps / (time.perf_counter() - t0), 1)
    legs["c5_build_prims_per_sec"] = sweep
    return {"value": round(sample_n / dt, 1), "unit": "queries/s", "cores": threads,
            "kind": "port",
            "sample": f"kNN k={k}: first {sample_n} of the {qs.shape[0]} queries "
                      f"(Morton pre-sort included) against the full {pts.shape[0]}-point tree; "
                      f"legs: radius 2P on the same {sample_n} queries against the C2 tree and "
                      f"the {pts.shape[0]}-point hollow-sphere (C3) tree; C5 builds 1e4-1e7 "
                      "(1e8 omitted: ~20 s)",
            "build_prims_per_sec": round(pts.shape[0] / bdt, 1),
            "legs": legs}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def host_threads(oracle) -> int:
    """All host cores this process may use (torchrun exports OMP_NUM_THREADS=1,
    which the oracle's num_threads clause overrides)."""
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count() or 1
    return max(avail, oracle.max_threads())


def run_reference(args):
    """The reference's CPU path on this box's host cores: the oracle port
    (OpenMP, every host thread), same workload and config as the GPU arm.  At
    N=1 every step answers the whole C2 query batch (1e7 queries, ~2.5 s on
    16 cores); with N>1 (rank 0 only) the global cloud is built and each step
    answers a rotating window of cpu_sample queries of the global batch."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    import paper_1908_11807_b200.datasets as ds

    world = world_size(args)
    m, nq, gm, gq = shape_of(args, world)
    k = args.k
    pts = ds.generate(ds.CloudSpec("cube", "filled", gm, 0))
    qs = ds.generate(ds.CloudSpec("cube", "filled", gq, 1))
    threads = host_threads(oracle)
    ref = oracle.build(pts, threads=threads)
    sample = gq if world == 1 else max(1000, min(args.cpu_sample, gq))

    def window(s):
        lo = (s * sample) % max(1, gq - sample + 1)
        return qs[lo:lo + sample]

    for w in range(args.warmup):
        oracle.query_knn(ref, window(w), k, threads=threads)
    total = 0.0
    for s in range(args.steps):
        q = window(args.warmup + s)
        t0 = time.perf_counter()
        oracle.query_knn(ref, q, k, threads=threads)
        total += time.perf_counter() - t0
    value = args.steps * sample / total
    out = {
        "impl": "reference",
        "metric": f"knn_queries_per_sec (k={k}, {m:.0e} filled-box points, {nq:.0e} queries)",
        "value": round(value, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if args.global_points else "weak",
        "vs_baseline": None, "dtype": "f32",
        "dtype_note": "fp32 box distances (reference recipe, unfused); f64 Morton normalisation",
        "data": "synthetic: paper_1908_11807_b200.datasets PCG64 clouds (reference generators)",
        "config": workload(args, world),
        "cpu_baseline": {"value": round(value, 1), "unit": "queries/s", "cores": threads,
                         "kind": "port",
                         "sample": (f"every step: all {gq} queries (query Morton pre-sort "
                                    f"included) against the full {gm}-point tree"
                                    if sample == gq else
                                    f"every step: a {sample}-query window of the {gq} global "
                                    f"queries against the full {gm}-point tree")},
        "e2e": {"value": round(value, 1), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
