"""The flat Adam element pass (touched = NULL) against the live-row list pass
(touched-row skip) on config-3 sized groups: sb_sparse_adam_flat, device
timed, dense (every active row live) and sparse (a mapping step's ~8%)."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200 import _native as N  # noqa: E402
from paper_2404_06926_b200.adam import lr_vector  # noqa: E402
from paper_2404_06926_b200.synthetic import default_lrs  # noqa: E402


def main(n=1_000_000, reps=20, act_frac=0.91, sparse_frac=0.08):
    dt = torch.float32
    code = N.dtype_code(dt)
    shapes = {"position": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (),
              "sh": (16, 3)}
    g = torch.Generator(device="cuda").manual_seed(0)
    params = {k: torch.randn((n,) + s, device="cuda", generator=g) for k, s in shapes.items()}
    grads = {k: torch.randn((n,) + s, device="cuda", generator=g) * 1e-3
             for k, s in shapes.items()}
    st = sb.AdamState(n, default_lrs(), dtype=dt)
    active = (torch.rand(n, device="cuda", generator=g) < act_frac).to(torch.uint8)
    ws = torch.empty(N.load().sb_sparse_adam_workspace_bytes(code, n), dtype=torch.uint8,
                     device="cuda")
    G = st.groups(params, grads)
    lrs = lr_vector(st.lrs)

    def run(rows, touched):
        N.call("sb_sparse_adam_flat", code, n, N.C.byref(G), N.ptr(st._steps), N.ptr(active),
               N.ptr(rows), N.ptr(touched), lrs.ctypes.data_as(N.vp), N.ptr(ws), ws.numel(),
               None, N.stream_ptr())

    def timeit(rows, touched_fn):
        for _ in range(3):
            run(rows, touched_fn())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            t = touched_fn()
            e0.record()
            run(rows, t)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(ts))

    allrows = torch.ones(n, dtype=torch.uint8, device="cuda")
    sparse = (torch.rand(n, device="cuda", generator=g) < sparse_frac).to(torch.uint8)
    ones = torch.ones(n, dtype=torch.uint8, device="cuda")
    zeros = torch.zeros(n, dtype=torch.uint8, device="cuda")
    res = {
        "flat_dense_us": timeit(allrows, lambda: None),
        "list_dense_us": timeit(allrows, lambda: ones),
        "flat_sparse_grad_us": timeit(sparse, lambda: None),
        "list_sparse_us": timeit(sparse, lambda: zeros.zero_()),
    }
    live_dense = int(active.sum())
    live_sparse = int((active.bool() & sparse.bool()).sum())
    for k, rows in (("flat_dense_us", live_dense), ("list_dense_us", live_dense),
                    ("list_sparse_us", live_sparse)):
        res[k.replace("_us", "_GBps")] = round(1416 * rows / (res[k] * 1e-6) / 1e9, 1)
    res.update(n=n, live_dense=live_dense, live_sparse=live_sparse)
    print(res)


if __name__ == "__main__":
    main()
    # the config-4 stream's shape: 4M rows, ~21 % frustum-active, all live
    main(n=4_000_000, act_frac=0.21, sparse_frac=0.05)
