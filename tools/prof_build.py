"""Driver for profiling the build pipeline under ncu: builds an n-point
filled-cube tree `reps` times from device-resident points.

    ncu --set full -k regex:hierarchy_kernel -s 1 -c 1 -o prof python tools/prof_build.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shape = sys.argv[3] if len(sys.argv) > 3 else "cube:filled"
pts = torch.from_numpy(lb.generate(lb.CloudSpec.parse(shape, n, 0))).cuda()
for _ in range(reps):
    t = lb.build(pts)
torch.cuda.synchronize()
print("built", t)
