"""Where does the e2e leg lose time against the device-resident loop?  Times
(config 3) the step loop alone, + log-row D2H, + host-image upload, and the
host-side cost of each call; every variant replays the same iterations from a
snapshot.  Finding (B200): the 11 MB host->device copy takes ~0.22 ms on an
idle GPU but is starved to ~7 GB/s while the HBM-bound step runs beside it,
so an overlapped upload still costs ~45 us per step (an SM-driven zero-copy
upload measured the same with 8 CTAs and worse with more)."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import synthetic  # noqa: E402


def timed(fn, steps):
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h = 0.0
    e0.record(st)
    for _ in range(steps):
        t = time.perf_counter()
        fn()
        h += time.perf_counter() - t
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, 1e3 * h / steps


def main():
    scene = synthetic.config(3)
    mp, entry = bench.build_mapper(scene, sb, torch)
    for _ in range(3):
        mp._step_device(entry)
    gt_host = torch.from_numpy(scene.image.astype(np.float32)).pin_memory()
    out_host = torch.empty(8, dtype=torch.float64).pin_memory()

    def a():
        mp._step_device(entry)

    def b():
        row = mp._step_device(entry)[3]
        out_host.copy_(row, non_blocking=True)

    def c():
        mp.optimize_keyframe(entry, gt_host, log_host=out_host)

    def c2():   # upload without the 8-bit target refresh
        gt8 = entry.gt8
        entry.gt8 = None
        mp.upload_image(entry, gt_host)
        entry.gt8 = gt8
        mp._step_device(entry)

    def c3():   # only the device-to-device refresh
        entry.gt.copy_(entry.gt.clone()) if False else entry.gt.add_(0)
        mp._step_device(entry)

    def d():
        entry.gt.copy_(gt_host, non_blocking=True)
        row = mp._step_device(entry)[3]
        out_host.copy_(row, non_blocking=True)

    cs = torch.cuda.Stream()
    spare = torch.empty_like(entry.gt)
    ev_c, ev_k = torch.cuda.Event(), torch.cuda.Event()

    def c4():   # side-stream H2D into a spare buffer, main waits for it, no D2D
        main = torch.cuda.current_stream()
        cs.wait_event(ev_k)
        with torch.cuda.stream(cs):
            spare.copy_(gt_host.reshape(spare.shape), non_blocking=True)
            ev_c.record(cs)
        main.wait_event(ev_c)
        ev_k.record(main)
        mp._step_device(entry)

    def c5():   # side-stream H2D nobody waits for (pure traffic)
        with torch.cuda.stream(cs):
            spare.copy_(gt_host.reshape(spare.shape), non_blocking=True)
        mp._step_device(entry)

    def c6():   # a cross-stream event wait with no copy behind it
        main = torch.cuda.current_stream()
        cs.wait_event(ev_k)
        ev_c.record(cs)
        main.wait_event(ev_c)
        ev_k.record(main)
        mp._step_device(entry)

    spares = [torch.empty_like(entry.gt) for _ in range(2)]
    evs = [(torch.cuda.Event(), torch.cuda.Event()) for _ in range(2)]
    cnt = [0]

    def c7():   # double-buffered: this step waits for the copy issued one call earlier
        main = torch.cuda.current_stream()
        i = cnt[0]
        cnt[0] += 1
        buf, (e_c, e_k) = spares[i % 2], evs[i % 2]
        cs.wait_event(e_k)
        with torch.cuda.stream(cs):
            buf.copy_(gt_host.reshape(buf.shape), non_blocking=True)
            e_c.record(cs)
        pb, (pc, pk) = spares[(i + 1) % 2], evs[(i + 1) % 2]
        if i > 0:
            main.wait_event(pc)
            pk.record(main)
        mp._step_device(entry)

    cs2 = [torch.cuda.Stream() for _ in range(4)]
    ev2 = [(torch.cuda.Event(), torch.cuda.Event()) for _ in range(4)]

    def split(k):
        def f():   # the upload split over k side streams (copy engines), main waits all
            main = torch.cuda.current_stream()
            flat_dst = spare.view(-1)
            flat_src = gt_host.view(-1)
            n = flat_dst.numel()
            for q in range(k):
                lo, hi = q * n // k, (q + 1) * n // k
                c_s, (e_c2, e_k2) = cs2[q], ev2[q]
                c_s.wait_event(e_k2)
                with torch.cuda.stream(c_s):
                    flat_dst[lo:hi].copy_(flat_src[lo:hi], non_blocking=True)
                    e_c2.record(c_s)
            for q in range(k):
                main.wait_event(ev2[q][0])
            for q in range(k):
                ev2[q][1].record(main)
            mp._step_device(entry)
        return f

    snap = bench.snapshot(mp, entry)
    for rep in range(2):
        for name, fn in (("step", a), ("step+d2h", b), ("upload+step+d2h", c),
                         ("upload-no-q", c2), ("d2d-only", c3), ("inline h2d", d),
                         ("h2d+wait no d2d", c4), ("h2d no wait", c5), ("event wait only", c6),
                         ("h2d one call ahead", c7), ("split 2", split(2)),
                         ("split 4", split(4))):
            bench.restore(mp, entry, snap)     # every variant runs the same iterations
            fn()
            bench.restore(mp, entry, snap)
            ms, host = timed(fn, 30)
            print(f"{name:18s} device {ms:.4f} ms/step  host {host:.4f} ms/call")


if __name__ == "__main__":
    main()
