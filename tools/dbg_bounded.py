import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2404_06926_b200 as sb
from paper_2404_06926_b200 import _native as N
from paper_2404_06926_b200.synthetic import ring_map
from test_gpu_bounded_sort import _preprocess
W, H, f = 320, 240, 250.0
rng = np.random.default_rng(21)
arrays = [x.astype(np.float32) if x.dtype != bool else x for x in ring_map(rng, 40_000, f)]
R = np.array([[0.0, -1.0, 0.0], [0.0, 0.0, -1.0], [1.0, 0.0, 0.0]])
pose = sb.CameraPose(R, np.zeros(3)); intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
rec, valid, keys, vals = _preprocess(sb, N, torch, arrays, pose, intr)
n = arrays[0].shape[0]
k = keys.cpu().numpy().view(np.uint32)
sortable = int((k != 0xFFFFFFFF).sum())
print("n", n, "valid", int(valid.sum()), "sortable", sortable)
a256 = lambda x: (x + 255) // 256 * 256
cap = 4 * n + 1024
nt = 300; nch = (n + 1023) // 1024
o = 0; lay = {}
for name, sz in (("keys_sorted", 8 * n), ("order", 4 * n), ("counts", 4 * n), ("masks", 8 * n), ("geo", 4 * n), ("big", 2 * cap), ("big_total", 256 - 0), ("hist", 4 * (nt * nch + 1)), ("keys_c", 8 * n), ("vals_c", 4 * n), ("n_sel", 256)):
    lay[name] = o; o += a256(sz) if name != "big_total" else 256
dev = rec.device
bound = sortable + 100
pg = torch.empty(cap, dtype=torch.int32, device=dev)
off = torch.empty(nt + 1, dtype=torch.int32, device=dev)
status = torch.zeros(2, dtype=torch.int64, device=dev)
lib = N.load()
ws = torch.zeros(lib.sb_bin_workspace_bytes(n, cap, W, H), dtype=torch.uint8, device=dev)
npairs = N.C.c_int64(0)
kk, vv = keys.clone(), vals.clone()
N.check(lib.sb_bin(N.SB_F32, n, N.ptr(rec), N.ptr(valid), N.ptr(kk), N.ptr(vv), W, H, 16, 1, cap, N.ptr(pg), None, N.ptr(off), N.C.byref(npairs), N.ptr(ws), ws.numel(), N.ptr(status), None, bound, N.stream_ptr()), "sb_bin")
torch.cuda.synchronize()
w = ws.cpu().numpy()
nsel = w[lay["n_sel"]:lay["n_sel"] + 4].view(np.int32)[0]
kc = w[lay["keys_c"]:lay["keys_c"] + 4 * bound].view(np.uint32)
vc = w[lay["vals_c"]:lay["vals_c"] + 4 * bound].view(np.uint32)
print("n_sel", nsel, "valid keys in keys_c", int((kc != 0xFFFFFFFF).sum()), "vals_c[:8]", vc[:8], "expected rows[:8]", np.nonzero(k != 0xFFFFFFFF)[0][:8])
ks = w[lay["keys_sorted"]:lay["keys_sorted"] + 4 * bound].view(np.uint32)
od = w[lay["order"]:lay["order"] + 4 * bound].view(np.uint32)
print("sorted keys monotone", bool(np.all(np.diff(ks.astype(np.int64)) >= 0)), "order[:8]", od[:8], "status", status.cpu().numpy())
exp = np.argsort(k.astype(np.int64), kind="stable")[:bound]
print("order matches numpy", bool(np.array_equal(od[:sortable], exp[:sortable])))
