"""How many rows does the coarse depth-limit drop remove at config 3?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402

scene = synthetic.config(3)
mp, entry = bench.build_mapper(scene, sb, torch)
for i in range(6):
    mp._step_device(entry)
    torch.cuda.synchronize()
    last = mp.engine.last
    lim = next(iter(mp.engine.caps.values()))
    n_tiles = 3600
    coarse = lim[n_tiles:]
    print(f"step {i}: valid rows {int(last['valid'].sum())}, kept pairs {int(last['status'][0])}, "
          f"finite coarse cells {int(torch.isfinite(coarse).sum())}/{coarse.numel()}, "
          f"finite tiles {int(torch.isfinite(lim[:n_tiles]).sum())}")
