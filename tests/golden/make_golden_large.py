"""Reference digests at BASELINE scale (C2, C3, C5) — test infrastructure.

Runs the REFERENCE implementation (``lbvh`` under /root/reference/pkg/src,
imported read-only, all host threads) on the BASELINE.json configurations and
stores sha256 prefixes of every output in ``digests_large.json``.  The arrays
themselves are GBs, so only their digests are committed; the GPU tests
(``tests/test_gpu_scale.py``) regenerate the same inputs, run the CUDA path and
hash its outputs.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_large.py [c2] [c3] [c3knn] [c5]

Reference call sites: ``tree.build`` (pkg/src/lbvh/tree.py:177-209),
``query_spatial_2p`` (traversal.py:184-211), ``query_knn`` (traversal.py:251-272),
``query_sort_order`` (traversal.py:146-159), generators (datasets.py:99-172).
Cost here (8 cores): C2 ~1 min, C3 radius ~30 s, C3 kNN ~8 min, C5 to 1e8 ~3 min
and ~25 GB of host RAM.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from lbvh import datasets as ref_datasets  # noqa: E402
from lbvh import morton as ref_morton  # noqa: E402
from lbvh import traversal as ref_trav  # noqa: E402
from lbvh import tree as ref_tree  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "digests_large.json")
THREADS = os.cpu_count() or 1


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def per_query_sorted(offsets: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """Indices sorted inside each query's span (spatial order is free, A.6)."""
    counts = np.diff(offsets)
    qid = np.repeat(np.arange(counts.shape[0], dtype=np.int64), counts)
    key = (qid << 32) | indices.astype(np.int64)
    key.sort()
    return (key & 0xFFFFFFFF).astype(np.int32)


def tree_digest(t, pts) -> dict:
    codes = ref_morton.morton_codes(
        (pts.astype(np.float64) + pts) * 0.5, t.scene_min, t.scene_max)
    return {
        "points": h(pts),
        "scene_min": t.scene_min.tolist(), "scene_max": t.scene_max.tolist(),
        "codes": h(codes), "leaf_obj": h(t.leaf_obj), "left": h(t.left),
        "right": h(t.right), "node_mins": h(t.node_mins), "node_maxs": h(t.node_maxs),
    }


def spatial_digest(t, q, r) -> dict:
    t0 = time.time()
    sp = ref_trav.query_spatial_2p(t, (q, r), threads=THREADS)
    dt = time.time() - t0
    cnt = sp.counts()
    return {
        "radius": r, "sp_offsets": h(sp.offsets), "sp_total": int(sp.offsets[-1]),
        "sp_indices_fill_order": h(sp.indices),
        "sp_sorted_indices": h(per_query_sorted(sp.offsets, sp.indices)),
        "sp_counts_min_mean_max": [int(cnt.min()), float(cnt.mean()), int(cnt.max())],
        "sp_ref_seconds": round(dt, 2),
    }


def knn_digest(t, q, k) -> dict:
    t0 = time.time()
    kn = ref_trav.query_knn(t, (q, k), threads=THREADS)
    dt = time.time() - t0
    return {
        "k": k, "knn_offsets": h(kn.offsets), "knn_indices": h(kn.indices),
        "knn_distances": h(kn.distances),
        "knn_dist_sum": float(kn.distances.astype(np.float64).sum()),
        "knn_ref_seconds": round(dt, 2),
    }


def pair(src: str, tgt: str, m: int, nq: int):
    pts = ref_datasets.generate(ref_datasets.CloudSpec.parse(src, m, 0))
    q = ref_datasets.generate(ref_datasets.CloudSpec.parse(tgt, nq, 1))
    t0 = time.time()
    t = ref_tree.build(pts, threads=THREADS)
    bt = time.time() - t0
    d = {"source": src, "target": tgt, "m": m, "nq": nq, "seed": 0, "target_seed": 1,
         "queries": h(q), "build_ref_seconds": round(bt, 2)}
    d.update(tree_digest(t, pts))
    d["query_order"] = h(ref_trav.query_sort_order(q, (t.scene_min, t.scene_max)))
    return pts, q, t, d


def main(which) -> None:
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            out = json.load(fh)
    out["threads"] = THREADS
    r = ref_datasets.default_radius(10)
    if "c2" in which:
        _, q, t, d = pair("cube:filled", "cube:filled", 10_000_000, 10_000_000)
        d.update(spatial_digest(t, q, r))
        d.update(knn_digest(t, q, 10))
        out["c2_filled"] = d
        print("c2", d, flush=True)
    if "c3" in which or "c3knn" in which:
        _, q, t, d = pair("sphere:hollow", "cube:filled", 10_000_000, 10_000_000)
        prev = out.get("c3_hollow_sphere", {})
        if "c3" in which:
            d.update(spatial_digest(t, q, r))
        else:
            d.update({k: v for k, v in prev.items() if k.startswith("sp_") or k == "radius"})
        if "c3knn" in which:
            d.update(knn_digest(t, q, 10))
        else:
            d.update({k: v for k, v in prev.items() if k.startswith("knn_") or k == "k"})
        out["c3_hollow_sphere"] = d
        print("c3", d, flush=True)
    if "c5" in which:
        sweep = {}
        for m in (10_000, 100_000, 1_000_000, 10_000_000, 100_000_000):
            pts = ref_datasets.generate(ref_datasets.CloudSpec("cube", "filled", m, 0))
            t0 = time.time()
            t = ref_tree.build(pts, threads=THREADS)
            e = tree_digest(t, pts)
            e["build_ref_seconds"] = round(time.time() - t0, 2)
            sweep[str(m)] = e
            print("c5", m, e, flush=True)
            del t, pts
        out["c5_build_sweep"] = sweep
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("written", OUT)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c2", "c3", "c5"})
