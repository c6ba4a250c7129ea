"""The bench's sequence (warm-up, device-timed loop, restore, e2e leg) with
switches, to find what makes the e2e leg slower in some processes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402
from paper_2404_06926_b200.hostmem import pinned_from  # noqa: E402

use_sampler = os.environ.get("SAMPLER", "1") == "1"
warm_uploads = int(os.environ.get("WARM_UPLOADS", "1"))
scene = synthetic.config(3)
mp, entry = bench.build_mapper(scene, sb, torch)
gt_host = pinned_from(scene.image.astype(np.float32))
out_host = torch.empty(8, dtype=torch.float64).pin_memory()
for i in range(3):
    up = i >= 3 - warm_uploads
    mp.optimize_keyframe(entry, gt_host if up else None, log_host=out_host if up else None)
snap = bench.snapshot(mp, entry)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if use_sampler:
    clk = bench.ClockSampler(0)
    clk.__enter__()
e0.record(st)
rows = [mp._step_device(entry) for _ in range(50)]
e1.record(st)
torch.cuda.synchronize()
if use_sampler:
    clk.__exit__(None, None, None)
dev = 50 / (e0.elapsed_time(e1) / 1e3)
bench.restore(mp, entry, snap)
torch.cuda.synchronize()
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f0.record(st)
for _ in range(50):
    mp.optimize_keyframe(entry, gt_host, log_host=out_host)
st.wait_stream(mp.readback_stream())
f1.record(st)
torch.cuda.synchronize()
print(f"sampler={int(use_sampler)} warm_uploads={warm_uploads} device {dev:.1f} e2e {50 / (f0.elapsed_time(f1) / 1e3):.1f}")
