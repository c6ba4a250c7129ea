"""Which early iterations of a config are invalid (pair overflow or a
depth-limited tile that did not terminate)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402
from paper_2404_06926_b200.engine import log_dict  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scene = synthetic.config(cfgi)
mp, entry = bench.build_mapper(scene, sb, torch)
mp.use_graphs = os.environ.get("GRAPHS", "0") == "1"
for i in range(8):
    row = mp._step_device(entry)[3]
    torch.cuda.synchronize()
    d = log_dict(row.cpu().numpy(), scene.width * scene.height)
    caps = mp.engine.caps.get(id(entry) if mp.use_graphs else "eager")
    fin = int(torch.isfinite(caps).sum()) if caps is not None else -1
    print(i, "P", d["n_pairs"], "invalid", d["overflow"], "finite limits", fin,
          "halt", int(mp.engine.halt.item()) if mp.engine.halt is not None else None)
    if d["overflow"]:
        mp.engine.resume()

# the bench's warm-up: every step through the upload path
import numpy as np  # noqa: E402
from paper_2404_06926_b200.hostmem import pinned_from  # noqa: E402
mp, entry = bench.build_mapper(scene, sb, torch)
gt_host = pinned_from(scene.image.astype(np.float32))
out_host = torch.empty(8, dtype=torch.float64).pin_memory()
for i in range(8):
    h = mp.optimize_keyframe(entry, gt_host, log_host=out_host)
    torch.cuda.synchronize()
    d = log_dict(h[3].cpu().numpy(), scene.width * scene.height)
    print("upload", i, "P", d["n_pairs"], "invalid", d["overflow"], "gt ptr", entry.gt.data_ptr() % 100000,
          "halt", int(mp.engine.halt.item()))
    if d["overflow"]:
        mp.engine.resume()

# exactly the bench's sequence, asynchronous
mp, entry = bench.build_mapper(scene, sb, torch)
for i in range(3):
    mp.optimize_keyframe(entry, gt_host, log_host=out_host)
snap = bench.snapshot(mp, entry)
torch.cuda.synchronize()
rows = [mp._step_device(entry) for _ in range(60)]
flags = torch.stack([r[3][6:8].view(torch.int64)[1] for r in rows]).cpu().numpy()
Ps = torch.stack([r[3][6:8].view(torch.int64)[0] for r in rows]).cpu().numpy()
print("bench-seq invalid at", list(np.nonzero(flags)[0][:10]), "P", Ps[:6])
