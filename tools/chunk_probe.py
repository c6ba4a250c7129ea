import sys
sys.path.insert(0, ".")
import torch, numpy as np
import bench
import paper_2404_06926_b200 as sb
scene = bench.scene_of(3)
mp, entry = bench.build_mapper(scene, sb, torch)
for _ in range(6):
    mp._step_device(entry)
torch.cuda.synchronize()
eng = mp.engine
off = eng.binout["offsets"].cpu().numpy().astype(np.int64)
P = int(off[-1])
pg = eng.binout["a_pg"][:P].cpu().numpy().astype(np.int64)
n = mp.map.count
rec = eng.bufs["records"][:n].cpu().numpy()
valid = eng.bufs["valid"][:n].cpu().numpy() != 0
dep = np.where(valid, rec[:, 11], np.inf)
order = np.argsort(dep, kind="stable")
rank = np.empty(n, np.int64); rank[order] = np.arange(n)
ch = rank[pg] // 1024
cnt = np.bincount(ch, minlength=(n + 1023) // 1024)
nz = cnt[cnt > 0]
print("P", P, "chunks", len(cnt), "nonempty", len(nz), "max", cnt.max(), "argmax", cnt.argmax())
print("windows total", int(np.ceil(nz / 4096).sum()), "max windows", int(np.ceil(cnt.max() / 4096)))
print("top chunks", sorted(cnt.tolist(), reverse=True)[:20])
print("pct", np.percentile(nz, [50, 90, 99]))
