"""Batched-path host-sync cost at config 3, world 1 (NCCL): PackedBatchStep
with the exchange forced on (always_reduce), validity checked on the host
after every step (sync) vs two steps later (lazy, sync-free packing).
Wall clock over 40 steps after warm-up, synchronised on both sides."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29577")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import bench, paper_2404_06926_b200 as sb
from paper_2404_06926_b200 import synthetic
from paper_2404_06926_b200.batch import PackedBatchStep, DeviceBatchCompute
scene = synthetic.config(int(os.environ.get("CONFIG", "3")))
mp, entry = bench.build_mapper(scene, sb, torch)
comp = DeviceBatchCompute(mp)
for reduce_ in (False, True):
    for lazy in (False, True, False, True):
        step = PackedBatchStep(comp, always_reduce=reduce_, lazy=lazy)
        comp.deferred = lazy
        for _ in range(5):
            step.step([entry])
        step.flush()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(40):
            step.step([entry])
        step.flush()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 40
        print("exchange" if reduce_ else "no-exchange", "lazy" if lazy else "sync",
              round(1e3 * dt, 3), "ms/step", "packed_rows", getattr(step, "packed_rows", None),
              flush=True)
dist.destroy_process_group()
