"""Binning-only timing at config 3: K1 (preprocess) + K3-K5 (sb_bin, async
mode) repeated on the engine's buffers.  Used with an ncu launch list to split
sb_bin into its kernels.

    python tools/bin_bench.py [--iters K]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import _native as N, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--full", action="store_true", help="full tile lists (no depth limits)")
    a = ap.parse_args()
    scene = synthetic.config(a.config)
    mp, entry = bench.build_mapper(scene, sb, torch)
    for _ in range(3):
        mp._step_device(entry)
    torch.cuda.synchronize()
    eng = mp.engine
    kf = entry.frame
    W, H = kf.intrinsics.width, kf.intrinsics.height
    n = mp.map.count
    arrays = mp.map.arrays()
    cam = N.camera(kf.pose, kf.intrinsics)
    rec, valid = eng.bufs["records"], eng.bufs["valid"]
    keys, vals = eng.bufs["keys"], eng.bufs["vals"]
    status = torch.zeros(2, dtype=torch.int64, device="cuda")
    lim = next(iter(eng.caps.values())) if eng.caps and not a.full else None
    n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
    caps = lim[:n_tiles] if lim is not None else None
    coarse = lim[n_tiles:] if lim is not None else None

    def once():
        N.call("sb_preprocess_fwd", N.SB_F32, n, *[N.ptr(arrays[k]) for k in (
            "positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")], None,
            N.C.byref(cam), 0.01, 0.3, 0.1, N.ptr(rec), N.ptr(valid), N.ptr(keys), N.ptr(vals),
            None, None, N.ptr(coarse), N.stream_ptr())
        eng._bin_async(torch.float32, n, rec, valid, keys, vals, W, H, status, caps)

    for _ in range(3):
        once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        once()
    e1.record()
    torch.cuda.synchronize()
    print(f"preprocess+bin {e0.elapsed_time(e1) / a.iters:.4f} ms/iter, P = {int(status[0])}")


if __name__ == "__main__":
    main()
