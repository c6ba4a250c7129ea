"""The config-3 mapping step in steady state, bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off`: a clean per-step
launch list (depth-limited binning, graph replay off so each launch is seen).

  ncu --profile-from-start off --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file out.csv python tools/step_launches.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scene = synthetic.config(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
mp, entry = bench.build_mapper(scene, sb, torch)
mp.use_graphs = False
mp.engine.deterministic = os.environ.get("SB_ATOMIC_BWD", "0") != "1"
mp.engine.use_caps = os.environ.get("SB_FULL_LISTS", "0") != "1"   # full tile lists
for _ in range(5):
    mp._step_device(entry)
torch.cuda.synchronize()
if os.environ.get("SB_RENDER"):      # the render path (bench.py's render FPS) instead
    kf = entry.frame
    for _ in range(3):
        mp.render_image(kf.pose, kf.intrinsics, key="bench")
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(steps):
        mp.engine.render(mp.map, kf.pose, kf.intrinsics, key="bench")
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    sys.exit(0)
torch.cuda.cudart().cudaProfilerStart()
rows = [mp._step_device(entry) for _ in range(steps)]
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("invalid", [bool(r[3][7].view(torch.int64).item()) for r in rows])
