"""The bench's e2e leg repeated several times in one process (config 3), to
separate per-process effects from run-to-run noise."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402
from paper_2404_06926_b200.hostmem import pinned_from  # noqa: E402

scene = synthetic.config(3)
mp, entry = bench.build_mapper(scene, sb, torch)
gt_host = pinned_from(scene.image.astype(np.float32))
gt_plain = torch.from_numpy(scene.image.astype(np.float32)).pin_memory()
out_host = torch.empty(8, dtype=torch.float64).pin_memory()
for _ in range(4):
    mp.optimize_keyframe(entry, gt_host, log_host=out_host)
snap = bench.snapshot(mp, entry)
st = torch.cuda.current_stream()
REPS = int(os.environ.get("E2E_REPS", "6"))
for rep in range(REPS):
    for name, host in (("hugepage", gt_host), ("pin_memory", gt_plain)):
        bench.restore(mp, entry, snap)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(50):
            mp.optimize_keyframe(entry, host, log_host=out_host)
        st.wait_stream(mp.readback_stream())
        b.record(st)
        torch.cuda.synchronize()
        print(rep, name, round(50 / (a.elapsed_time(b) / 1e3), 1))
