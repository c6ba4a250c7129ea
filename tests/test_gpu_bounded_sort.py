"""GPU: sb_bin's bounded depth sort (sort_capacity) on a view that sees a
minority of the map gives exactly the unbounded pair lists, and flags an
undersized bound in the device status."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _preprocess(sb, N, torch, arrays, pose, intr):
    n = arrays[0].shape[0]
    dev = torch.device("cuda")
    a = [torch.as_tensor(x).to(dev, torch.float32).contiguous() for x in arrays[:5]]
    rec = torch.empty((n, N.RECORD_REALS), dtype=torch.float32, device=dev)
    valid = torch.empty(n, dtype=torch.uint8, device=dev)
    keys = torch.empty(n, dtype=torch.int32, device=dev)
    vals = torch.empty(n, dtype=torch.int32, device=dev)
    fr = torch.empty(n, dtype=torch.uint8, device=dev)
    cam = N.camera(pose, intr)
    N.call("sb_preprocess_fwd", N.SB_F32, n, *[N.ptr(t) for t in a], None, N.C.byref(cam),
           0.01, 0.3, 0.1, N.ptr(rec), N.ptr(valid), N.ptr(keys), N.ptr(vals), N.ptr(fr),
           None, None, N.stream_ptr())
    return rec, valid, keys, vals


def _bin(N, torch, n, rec, valid, keys, vals, W, H, bound):
    dev = rec.device
    cap = 4 * n + 1024
    pg = torch.empty(cap, dtype=torch.int32, device=dev)
    off = torch.empty(((W + 15) // 16) * ((H + 15) // 16) + 1, dtype=torch.int32, device=dev)
    status = torch.zeros(2, dtype=torch.int64, device=dev)
    lib = N.load()
    ws = torch.empty(lib.sb_bin_workspace_bytes(n, cap, W, H), dtype=torch.uint8, device=dev)
    npairs = N.C.c_int64(0)
    k, v = keys.clone(), vals.clone()   # sb_bin sorts in scratch; keep the copies alive
    N.check(lib.sb_bin(N.SB_F32, n, N.ptr(rec), N.ptr(valid), N.ptr(k),
                       N.ptr(v), W, H, 16, 1, cap, N.ptr(pg), None, N.ptr(off),
                       N.C.byref(npairs), N.ptr(ws), ws.numel(), N.ptr(status), None, bound,
                       None, N.stream_ptr()), "sb_bin")
    torch.cuda.synchronize()
    P = int(status[0].item())
    return pg[:P].cpu().numpy(), off.cpu().numpy(), int(status[1].item())


def test_bounded_sort_matches_full_sort():
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.synthetic import ring_map
    W, H, f = 320, 240, 250.0
    rng = np.random.default_rng(21)
    arrays = [x.astype(np.float32) if x.dtype != bool else x for x in ring_map(rng, 40_000, f)]
    # a camera at the origin looking along +x: most of the ring is behind or
    # beside it (invalid or off-screen rows)
    R = np.array([[0.0, -1.0, 0.0], [0.0, 0.0, -1.0], [1.0, 0.0, 0.0]])
    pose = sb.CameraPose(R, np.zeros(3))
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    rec, valid, keys, vals = _preprocess(sb, N, torch, arrays, pose, intr)
    n = arrays[0].shape[0]
    sortable = int((keys != -1).sum().item())
    assert 0 < sortable < n // 3, sortable
    assert int(valid.sum().item()) > sortable      # off-screen valid rows left out of the sort
    pg0, off0, bad0 = _bin(N, torch, n, rec, valid, keys, vals, W, H, 0)
    assert bad0 == 0 and len(pg0) > 0
    for bound in (sortable, sortable + 777):
        pg1, off1, bad1 = _bin(N, torch, n, rec, valid, keys, vals, W, H, bound)
        assert bad1 == 0
        np.testing.assert_array_equal(off1, off0)
        np.testing.assert_array_equal(pg1, pg0)
    _, _, bad2 = _bin(N, torch, n, rec, valid, keys, vals, W, H, sortable - 1)
    assert bad2 == 1
