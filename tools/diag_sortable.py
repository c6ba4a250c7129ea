"""Config 3: rows with a valid sort key (sortable) after the full-list sizing
step and in steady state (depth limits + coarse drop)."""
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
    e = mp.engine
    n = mp.map.count
    k = e.bufs["keys"][:n]
    print(f"step {i}: valid {int(e.bufs['valid'][:n].sum())}, sortable {int((k != -1).sum())}, "
          f"kept pairs {int(e.last['status'][0])}, sort_cap {e.sort_cap}, fresh {e._fresh} {e.sort_cap_fresh}")
