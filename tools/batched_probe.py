"""Time the batched (keyframe-batch) step loops at world size 1: device loop
vs host-image loop, for both exchanges."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402
from paper_2404_06926_b200.batch import BatchStep, DeviceBatchCompute, ShardedBatchStep  # noqa: E402

scene = synthetic.config(3)
mp, _ = bench.build_mapper(scene, sb, torch)
intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
frame = sb.CameraFrame(pose=sb.CameraPose(np.eye(3), np.zeros(3)), intrinsics=intr,
                       image=scene.image, frame_index=1)
entry = mp.store.add(frame, mp.cfg.lr_exposure, torch.float32)
gt_host = torch.from_numpy(scene.image.astype(np.float32)).pin_memory()
out_host = torch.empty(4, dtype=torch.float64).pin_memory()
for name, step in (("allreduce", BatchStep(DeviceBatchCompute(mp))),
                   ("sharded", ShardedBatchStep(DeviceBatchCompute(mp)))):
    for _ in range(2):
        step.step([entry])
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        step.step([entry])
    torch.cuda.synchronize()
    a = (time.perf_counter() - t) / 10
    t = time.perf_counter()
    for _ in range(10):
        mp.upload_image(entry, gt_host)
        parts = step.step([entry])[0]
        out_host.copy_(parts, non_blocking=True)
    torch.cuda.synchronize()
    b = (time.perf_counter() - t) / 10
    print(f"{name}: device loop {1e3 * a:.3f} ms/step, host-image loop {1e3 * b:.3f} ms/step")
