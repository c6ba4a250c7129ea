import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_2404_06926_b200 as sb
from paper_2404_06926_b200 import synthetic
scene = synthetic.config(3)
mp, entry = bench.build_mapper(scene, sb, torch)
kf = entry.frame
for _ in range(5):
    mp.render_image(kf.pose, kf.intrinsics, key="bench")
torch.cuda.synchronize()
st = torch.zeros((200, 2), dtype=torch.int64, device="cuda")
t0 = time.perf_counter()
for i in range(200):
    mp.engine.render(mp.map, kf.pose, kf.intrinsics, key="bench", status=st[i])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host us/render", (t1 - t0) / 200 * 1e6, "total us/render", (t2 - t0) / 200 * 1e6)
pr = cProfile.Profile(); pr.enable()
for i in range(200):
    mp.engine.render(mp.map, kf.pose, kf.intrinsics, key="bench", status=st[i])
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
