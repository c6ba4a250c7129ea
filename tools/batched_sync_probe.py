import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29577")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import bench, paper_2404_06926_b200 as sb
from paper_2404_06926_b200 import synthetic
from paper_2404_06926_b200.batch import PackedBatchStep, DeviceBatchCompute
scene = synthetic.config(3)
mp, entry = bench.build_mapper(scene, sb, torch)
comp = DeviceBatchCompute(mp)
step = PackedBatchStep(comp)
for _ in range(4): step.step([entry])
torch.cuda.synchronize()
for mode in ("sync", "nosync", "sync"):
    if mode == "nosync":
        orig = comp.step_invalid; comp.step_invalid = lambda: False
    t = time.perf_counter()
    for _ in range(40): step.step([entry])
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 40
    if mode == "nosync": comp.step_invalid = orig
    print(mode, round(1e3 * dt, 3), "ms/step")
dist.destroy_process_group()
