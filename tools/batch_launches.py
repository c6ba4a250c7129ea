"""The config-5 keyframe batch (4M-Gaussian map, 8 views, one sparse Adam
per batch) through PackedBatchStep(DeviceBatchCompute) at world 1 (exchange
forced on), eager launches, bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off`: a per-batch launch list.

  ncu --profile-from-start off --metrics gpu__time_duration.sum \\
      --cache-control none --clock-control none --csv --log-file out.csv \\
      python tools/batch_launches.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402
from paper_2404_06926_b200.batch import DeviceBatchCompute, PackedBatchStep  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                         device_id=torch.device("cuda", 0))
scene, views = synthetic.config5()
mp, _ = bench.build_mapper(scene, sb, torch)
intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
entries = []
for k, v in enumerate(views):
    e = mp.store.add(sb.CameraFrame(pose=sb.CameraPose(v.W, v.t), intrinsics=intr, image=v.image,
                                    frame_index=k + 1), mp.cfg.lr_exposure, torch.float32)
    e.exposure.matrix = v.E
    entries.append(e)
step = PackedBatchStep(DeviceBatchCompute(mp), always_reduce=True, lazy=True)
step.use_graphs = False
for _ in range(4):
    step.step(entries)
step.flush()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(steps):
    step.step(entries)
step.flush()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
tdist.destroy_process_group()
