"""Where the sharded build's time goes at world size 1 (NCCL, one GPU):
torch.profiler over build_distributed, kernels and host ops by total time.

    torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/prof_sharded_build.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1908_11807_b200 as lb  # noqa: E402
from paper_1908_11807_b200 import distributed as D  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
pts = lb.datasets.generate_device(lb.CloudSpec("cube", "filled", 10_000_000, 0))
t = None
for _ in range(3):
    t = None
    t = D.build_distributed(pts, 0)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    t = None
    ev[0].record()
    t = D.build_distributed(pts, 0)
    ev[1].record()
    torch.cuda.synchronize()
print("build_distributed ms", ev[0].elapsed_time(ev[1]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lb.build(pts)
e1.record()
torch.cuda.synchronize()
print("local build ms", e0.elapsed_time(e1))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
dist.destroy_process_group()
