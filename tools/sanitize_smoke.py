"""Small end-to-end run of every kernel, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200.tree import Topology, refit_bounds  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
pts = lb.generate(lb.CloudSpec("cube", "filled", n, 0))
qs = lb.generate(lb.CloudSpec("sphere", "hollow", n // 2, 1))
t = lb.build(pts)
rows = np.concatenate([pts, pts + 0.5], axis=1)
tb = lb.build(rows)
r = lb.default_radius(10)
rs = lb.query_spatial_2p(t, (qs, r))
rs1, fb = lb.query_spatial_1p(t, (qs, r), 4)
rs2, fb2 = lb.query_spatial_1p(t, (qs, r), 64)
rk = lb.query_knn(t, (qs, 10))
rk2 = lb.query_knn(t, (qs, np.arange(1, qs.shape[0] + 1) % 40 + 1))
rk3 = lb.query_knn(tb, (qs, 50))
topo = lb.generate_topology(np.sort(lb.morton_codes(pts, t.scene_min, t.scene_max)))
mins, maxs = t.node_mins.copy(), t.node_maxs.copy()
refit_bounds(mins, maxs, topo)
user = lb.Bvh(t.node_mins, t.node_maxs, t.left, t.right, t.leaf_obj, t.scene_min, t.scene_max)
ru = lb.query_knn(user, (qs, 7))
order = lb.query_sort_order(qs, t.scene)
# device-resident batches (fused C calls), heap paths, 63-bit build, datagen
qd = torch.from_numpy(qs).cuda()
rkd = lb.query_knn(t, (qd, 10))
rkh = lb.query_knn(t, (qd, 20))       # shared-memory heap
rkg = lb.query_knn(t, (qs[:500], 450))  # global-memory heap
rsd = lb.query_spatial_2p(t, (qd, r))
t63 = lb.build(pts, morton_bits=63)
rk63 = lb.query_knn(t63, (qd, 10))
gd = lb.datasets.generate_device(lb.CloudSpec("sphere", "hollow", 3000, 4))
gc = lb.datasets.generate_device(lb.CloudSpec("cube", "hollow", 3000, 4))
bk = lb.brute_knn_batch(pts, qs[:200], 5)
# sharded protocol on one rank with the routing forced (partition, exchanges,
# gather / scatter, forward masks, leaf remap, fused local search)
import socket  # noqa: E402
import torch.distributed as dist  # noqa: E402
from paper_1908_11807_b200 import distributed as D  # noqa: E402
sock = socket.socket()
sock.bind(("127.0.0.1", 0))
port = sock.getsockname()[1]
sock.close()
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
D._FORCE_ROUTE = True
st = D.build_distributed(pts, 0)
off, gid, dd = D.query_knn_distributed(st, qd, 10)
soff, sgid = D.query_spatial_distributed(st, qs, r)
dist.destroy_process_group()
torch.cuda.synchronize()
print("sanitize smoke ok", int(rs.offsets[-1]), fb, fb2, rk.indices.shape, rk3.indices.shape)
