# compute-sanitizer memcheck over GPU builds at 300..1e5 points, trees compared
# with the C oracle (run on the GPU box: bash tools/sanitize_build.sh)
cd $GRAFT_REPO_ROOT
cat > /tmp/b.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, numpy as np
import paper_1908_11807_b200 as lb
from oracle import oracle
for n in (300, 700, 5000, 100000, 300000):
    pts = lb.generate(lb.CloudSpec("cube","filled",n,0))
    t = lb.build(torch.from_numpy(pts).cuda())
    ref = oracle.build(pts)
    for name in ("left","right","leaf_obj","node_mins","node_maxs"):
        a=getattr(t,name); b=getattr(ref,name)
        print(n, name, a.tobytes()==b.tobytes(), flush=True)
PY
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/b.py > gpurun_out/san.txt 2>&1
