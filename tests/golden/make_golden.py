"""Generate the golden fixtures that pin the oracle and the CUDA path.

Runs the REFERENCE implementation (the ``lbvh`` package under
/root/reference/pkg/src, imported read-only) on small seeded inputs and
stores its outputs.  This script runs only in the build container, where the
reference is present; the fixtures it writes are committed and travel to the
GPU box, which never reads /root/reference.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (in this directory):
  small_cases.npz   full inputs/outputs of the hand-sized cases the
                    reference tests use (LINE4, the seed-42 1000-point cloud,
                    +-3e38 extremes, duplicates, volumetric boxes, integer
                    clouds with heavy ties, Morton KAT points)
  digests.json      sha256 prefixes of the reference outputs on the
                    BASELINE C1-shaped configs (1e5 points / 1e5 queries),
                    which are too large to commit in full
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

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


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def sorted_concat(offsets, indices):
    out = np.empty_like(indices)
    for q in range(offsets.shape[0] - 1):
        s, e = offsets[q], offsets[q + 1]
        out[s:e] = np.sort(indices[s:e])
    return out


def put_tree(d, prefix, t):
    d[prefix + "node_mins"] = t.node_mins
    d[prefix + "node_maxs"] = t.node_maxs
    d[prefix + "left"] = t.left
    d[prefix + "right"] = t.right
    d[prefix + "leaf_obj"] = t.leaf_obj
    d[prefix + "scene_min"] = t.scene_min
    d[prefix + "scene_max"] = t.scene_max


def put_spatial(d, prefix, rs):
    d[prefix + "offsets"] = rs.offsets
    d[prefix + "sorted_indices"] = sorted_concat(rs.offsets, rs.indices)


def put_knn(d, prefix, rs):
    d[prefix + "offsets"] = rs.offsets
    d[prefix + "indices"] = rs.indices
    d[prefix + "distances"] = rs.distances


def small_cases():
    d = {}
    # LINE4 (pkg/tests/test_traversal.py:20)
    line4 = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]], dtype=np.float32)
    d["line4_pts"] = line4
    put_tree(d, "line4_", ref_tree.build(line4))

    # 1000-point uniform(-5,5) seed 42 cloud (pkg/tests/test_traversal.py:28-31)
    cloud = np.random.default_rng(42).uniform(-5, 5, size=(1000, 3)).astype(np.float32)
    d["cloud_pts"] = cloud
    t = ref_tree.build(cloud)
    put_tree(d, "cloud_", t)
    centers = np.random.default_rng(0).uniform(-6, 6, size=(200, 3)).astype(np.float32)
    d["cloud_sp_centers"] = centers
    put_spatial(d, "cloud_sp_", ref_trav.query_spatial_2p(t, (centers, 1.5)))
    kc = np.random.default_rng(9).uniform(-6, 6, size=(150, 3)).astype(np.float32)
    d["cloud_knn_centers"] = kc
    put_knn(d, "cloud_knn_", ref_trav.query_knn(t, (kc, 10)))
    # per-query radii and ks
    pr = np.random.default_rng(3).uniform(0, 2.5, size=200).astype(np.float32)
    d["cloud_spr_radii"] = pr
    put_spatial(d, "cloud_spr_", ref_trav.query_spatial_2p(t, (centers, pr)))
    pk = np.random.default_rng(4).integers(1, 40, size=150).astype(np.int64)
    d["cloud_knnk_ks"] = pk
    put_knn(d, "cloud_knnk_", ref_trav.query_knn(t, (kc, pk)))
    # large k (general path)
    put_knn(d, "cloud_knn100_", ref_trav.query_knn(t, (kc[:40], 100)))
    # 1P with small buffers
    for b in (1, 4, 32):
        rs, fb = ref_trav.query_spatial_1p(t, (centers, 1.5), b)
        put_spatial(d, f"cloud_1p{b}_", rs)
        d[f"cloud_1p{b}_fellback"] = np.array(fb)
    d["cloud_order"] = ref_trav.query_sort_order(centers, (t.scene_min, t.scene_max))

    # +-3e38 extremes (pkg/tests/test_build.py:220-233)
    big = 3e38
    ext = np.float32([[-big, -big, -big], [big, big, big], [0, 0, 0], [big, -big, 0]])
    d["ext_pts"] = ext
    te = ref_tree.build(ext)
    put_tree(d, "ext_", te)
    d["ext_codes"] = ref_morton.morton_codes(ext, te.scene_min, te.scene_max)

    # duplicates (pkg/tests/test_build.py:210-213, test_traversal.py:258-266)
    dup = np.tile(np.float32([2.5, -1.0, 0.25]), (64, 1))
    d["dup_pts"] = dup
    put_tree(d, "dup_", ref_tree.build(dup))

    # volumetric boxes (pkg/tests/test_traversal.py:350-361)
    rng = np.random.default_rng(31)
    lows = rng.uniform(-8, 8, size=(400, 3)).astype(np.float32)
    mins = np.minimum(lows, lows + 1)
    maxs = mins + rng.uniform(0, 2, size=(400, 3)).astype(np.float32)
    vc = rng.uniform(-9, 9, size=(60, 3)).astype(np.float32)
    d["vol_mins"], d["vol_maxs"], d["vol_centers"] = mins, maxs, vc
    tv = ref_tree.build((mins, maxs))
    put_tree(d, "vol_", tv)
    put_spatial(d, "vol_sp_", ref_trav.query_spatial_2p(tv, (vc, np.float32(1.7))))
    put_knn(d, "vol_knn_", ref_trav.query_knn(tv, (vc, 7)))

    # integer clouds with heavy ties (cf. pkg/tests/test_traversal.py:393-418)
    rng = np.random.default_rng(2024)
    ncases = 40
    d["int_ncases"] = np.array(ncases)
    for i in range(ncases):
        m = int(rng.integers(1, 120))
        pts = rng.integers(-10, 11, size=(m, 3)).astype(np.float32)
        cs = rng.integers(-12, 13, size=(int(rng.integers(1, 30)), 3)).astype(np.float32)
        r = float(rng.integers(0, 8))
        k = int(rng.integers(1, 14))
        ti = ref_tree.build(pts)
        d[f"int{i}_pts"], d[f"int{i}_centers"] = pts, cs
        d[f"int{i}_r"], d[f"int{i}_k"] = np.float32(r), np.int64(k)
        put_tree(d, f"int{i}_", ti)
        put_spatial(d, f"int{i}_sp_", ref_trav.query_spatial_2p(ti, (cs, r)))
        put_knn(d, f"int{i}_knn_", ref_trav.query_knn(ti, (cs, k)))

    # Morton KAT points (pkg/tests/test_morton.py:92-99 style)
    mp = np.random.default_rng(7).uniform(-1, 2, size=(4096, 3)).astype(np.float32)
    d["morton_pts"] = mp
    d["morton_codes_unit"] = ref_morton.morton_codes(mp, np.zeros(3, np.float32),
                                                     np.ones(3, np.float32))
    flat_max = np.float32([1, 0, 1])
    d["morton_codes_flat"] = ref_morton.morton_codes(mp, np.zeros(3, np.float32), flat_max)

    # random uniform codes -> topology (pkg/tests/test_build.py:139-146)
    codes = np.sort(np.random.default_rng(3).integers(0, 1 << 30, size=777).astype(np.uint32))
    topo = ref_tree.generate_topology(codes)
    d["topo_codes"] = codes
    d["topo_left"], d["topo_right"], d["topo_parent"] = topo.left, topo.right, topo.parent
    dcodes = np.sort(np.random.default_rng(5).integers(0, 50, size=999).astype(np.uint32))
    topo = ref_tree.generate_topology(dcodes)
    d["topod_codes"] = dcodes
    d["topod_left"], d["topod_right"], d["topod_parent"] = topo.left, topo.right, topo.parent
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **d)
    print("small_cases.npz:", len(d), "arrays")


def digests():
    out = {}
    r = ref_datasets.default_radius(10)
    cfgs = [
        ("c1_filled", "cube:filled", "cube:filled", 100_000),
        ("c3_hollow_sphere", "sphere:hollow", "cube:filled", 100_000),
        ("hollow_cube", "cube:hollow", "sphere:filled", 50_000),
    ]
    for name, src, tgt, m in cfgs:
        pts = ref_datasets.generate(ref_datasets.CloudSpec.parse(src, m, 0))
        q = ref_datasets.generate(ref_datasets.CloudSpec.parse(tgt, m, 1))
        t = ref_tree.build(pts)
        codes = ref_morton.morton_codes(pts, t.scene_min, t.scene_max)
        sp = ref_trav.query_spatial_2p(t, (q, r))
        kn = ref_trav.query_knn(t, (q, 10))
        cnt = sp.counts()
        out[name] = {
            "source": src, "target": tgt, "m": m, "seed": 0, "target_seed": 1,
            "radius": r, "k": 10,
            "points": h(pts), "queries": h(q),
            "scene_min": t.scene_min.tolist(), "scene_max": t.scene_max.tolist(),
            "codes": h(codes), "leaf_obj": h(t.leaf_obj), "left": h(t.left),
            "right": h(t.right), "node_mins": h(t.node_mins), "node_maxs": h(t.node_maxs),
            "sp_offsets": h(sp.offsets), "sp_total": int(sp.offsets[-1]),
            "sp_sorted_indices": h(sorted_concat(sp.offsets, sp.indices)),
            "sp_counts_min_mean_max": [int(cnt.min()), float(cnt.mean()), int(cnt.max())],
            "knn_indices": h(kn.indices), "knn_distances": h(kn.distances),
            "knn_dist_sum": float(kn.distances.astype(np.float64).sum()),
            "query_order": h(ref_trav.query_sort_order(q, (t.scene_min, t.scene_max))),
        }
        print(name, out[name]["sp_counts_min_mean_max"])
    # dataset generators for every shape (pins paper_1908_11807_b200.datasets)
    gens = {}
    for shape in ("cube", "sphere"):
        for variant in ("filled", "hollow"):
            for n, seed in ((1, 0), (7, 3), (1000, 17), (20_000, 5)):
                spec = ref_datasets.CloudSpec(shape, variant, n, seed)
                gens[f"{shape}:{variant}:{n}:{seed}"] = h(ref_datasets.generate(spec))
    out["datasets"] = gens
    out["default_radius_10"] = ref_datasets.default_radius(10)
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("digests.json written")


if __name__ == "__main__":
    small_cases()
    digests()
