"""How much a better kNN search-radius seed could save (instrumentation).

    python tools/knn_bound_study.py save [n]          # default lib: exact k-th d^2 -> /tmp
    LBVH_LIB=.../visits.so     python tools/knn_bound_study.py stats [n]
    LBVH_LIB=.../visits_kth.so python tools/knn_bound_study.py stats_kth [n]

`stats` prints node visits and kept insertions per query with the exact
Morton-window seed; `stats_kth` the same when every query starts from its
exact k-th distance (the floor any seed can reach).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200 import _device as dv, _lib, traversal  # noqa: E402

mode = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
src = sys.argv[3] if len(sys.argv) > 3 else "cube"
kind = "hollow" if src == "sphere" else "filled"
pts = torch.from_numpy(lb.generate(lb.CloudSpec(src, kind, n, 0))).cuda()
qs = torch.from_numpy(lb.generate(lb.CloudSpec("cube", "filled", n, 1))).cuda()
t = lb.build(pts)
path = f"/tmp/kth_{src}_{n}.pt"
if mode == "save":
    _, _, kth = traversal.knn_with_kth(t, qs, 10)
    torch.save(kth.cpu(), path)
    print("saved", path)
    sys.exit(0)
kth = torch.load(path).cuda() if mode == "stats_kth" else dv.empty(n, torch.float32)
b = traversal._knn_batch((qs, 10))
l = _lib.lib()
out_idx = dv.empty(n * 10, torch.int32)
out_dist = dv.empty(n * 10, torch.float32)
status = dv.Status()
offsets = dv.empty(n + 1, torch.int64)
ws = dv.workspace(l.lbvh_knn_batch_workspace_bytes(n))
evs = traversal._kernel_events("knn")
_lib.check(l.lbvh_knn_batch(t.ctree(), dv.ptr(b.centers), n, 10, traversal._ORDER_BITS,
                            dv.ptr(offsets), dv.ptr(out_idx), dv.ptr(out_dist), 0, dv.ptr(ws),
                            ws.numel(), status.ptr, dv.ptr(kth), evs[0], evs[1], dv.stream()))
torch.cuda.synchronize()
d = out_dist.view(n, 10)
v, k = d[:, 0].double().cpu().numpy(), d[:, 1].double().cpu().numpy()
print(f"{mode} n={n} src={src}: visits mean={v.mean():.1f} p50={np.median(v):.0f} "
      f"p99={np.percentile(v, 99):.0f}; kept insertions mean={k.mean():.2f} "
      f"p50={np.median(k):.0f} p99={np.percentile(k, 99):.0f}")
