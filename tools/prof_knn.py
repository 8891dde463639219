"""Driver for ncu / A/B timing of the kNN kernel at C2 (1e7 filled-cube points,
1e7 filled-cube queries, k=10): builds the tree, runs `reps` kNN batches on
device-resident queries and prints the median ms of the query call (CUDA
events, L2 flushed before each rep).

    python tools/prof_knn.py [n] [reps] [k] [source] [op]
        source: cube | sphere;  op: knn | radius (2P, default_radius(k)) | build
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
src = sys.argv[4] if len(sys.argv) > 4 else "cube"
op = sys.argv[5] if len(sys.argv) > 5 else "knn"
kind = "hollow" if src == "sphere" else "filled"
pts = torch.from_numpy(lb.generate(lb.CloudSpec(src, kind, n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
t = lb.build(pts)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
times = []
for _ in range(reps):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if op == "knn":
        rs = lb.query_knn(t, (qs, k))
    elif op == "radius":
        rs = lb.query_spatial_2p(t, (qs, lb.default_radius(k)))
    else:
        t = lb.build(pts)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
times.sort()
if op == "build":
    lo = t.device_arrays()["leaf_obj"].long()
    chk = f"check={int((lo * torch.arange(lo.numel(), device=lo.device) % 1000003).sum())}"
else:
    chk = (f"check={float(rs.distances.double().sum()):.6f}" if op == "knn"
           else f"check={int(rs.offsets[-1])}:{int((rs.indices.long() % 1000003).sum())}")
print(f"{op} n={n} k={k} src={src} median_ms={times[len(times) // 2]:.4f} min_ms={times[0]:.4f} "
      f"{chk}")
