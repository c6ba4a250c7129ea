"""Lazy validity checks of the batched step (batch.BatchStep(lazy=True)):
no host sync per step, the invalid flag read two steps later, invalid steps
(and the no-op steps queued behind them) re-run in order.  The result must be
the synchronous path's, including when the fixed-capacity
packing of PackedBatchStep overflows -- bitwise (_same)."""

import numpy as np
import pytest

from test_gpu_batch_growth import _mapper, _views


def _run(sb, lazy, steps=6, overflow_at=None, graphs=False, always_reduce=True, packed=True):
    import torch
    from paper_2404_06926_b200.batch import BatchStep, DeviceBatchCompute, PackedBatchStep
    mp, _ = _mapper(sb)
    entries = []
    for i, (pose, intr, img) in enumerate(_views(sb, 3)):
        entries.append(mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=img,
                                                   frame_index=i), mp.cfg.lr_exposure))
    cls = PackedBatchStep if packed else BatchStep
    step = cls(DeviceBatchCompute(mp), always_reduce=always_reduce, lazy=lazy)
    step.use_graphs = graphs
    logs, caps = [], []
    for i in range(steps):
        logs.append(step.step(entries))
        if overflow_at is not None and i == overflow_at:
            step.k_cap = 16          # the next step's reached rows do not fit
        caps.append(getattr(step, "k_cap", 0))
    step.flush()
    a = mp.map.arrays()
    out = {k: a[k].cpu().numpy().copy() for k in a}
    out["steps"] = mp.adam.steps.cpu().numpy().copy()
    out["logs"] = torch.stack([torch.cat([p.double() for p in l]) for l in logs]).cpu().numpy()
    return out, step, caps


def _same(got, ref):
    # bitwise: every no-op step was re-run exactly once, and the step is
    # deterministic (no float atomics; re-runs with full lists replay the
    # same prefixes as the depth-limited lists)
    for k in ref:
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


@pytest.mark.gpu
def test_lazy_packed_step_equals_sync_with_overflow():
    import torch
    import torch.distributed as dist
    import paper_2404_06926_b200 as sb
    init = not dist.is_initialized()
    if init:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        ref, _, _ = _run(sb, lazy=False)
        got, step, caps = _run(sb, lazy=True, overflow_at=1)
        assert step.lazy and not step._pending
        assert caps[1] == 16 and step.k_cap > 16       # the overflow was seen and resized
        _same(got, ref)
        # no overflow: the fixed-capacity packing carries spare dump-row slots
        got2, step2, _ = _run(sb, lazy=True)
        assert step2.packed_rows == min(step2.k_cap, got2["steps"].shape[0])
        _same(got2, ref)
    finally:
        if init:
            dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", [True, False])
@pytest.mark.parametrize("packed", [True, False])
def test_graphed_batched_step_equals_eager(exchange, packed):
    """The batched step replayed as ONE CUDA graph (NCCL collectives, the
    fixed-capacity packing, first-touch accumulation and the sparse Adam
    step captured) gives bitwise the eager steps' map and logs, including
    a packing overflow (eager re-run, graphs re-captured after it)."""
    import torch
    import torch.distributed as dist
    import paper_2404_06926_b200 as sb
    init = not dist.is_initialized()
    if init:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        kw = dict(always_reduce=exchange, packed=packed, steps=8)
        ref, _, _ = _run(sb, lazy=True, **kw)
        got, step, _ = _run(sb, lazy=True, graphs=True, **kw)
        assert step.graphs, "no step was graph-replayed"
        _same(got, ref)
        if packed and exchange:
            got2, step2, _ = _run(sb, lazy=True, graphs=True, overflow_at=3, **kw)
            _same(got2, ref)
    finally:
        if init:
            dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_pack_unpack_rows_match_torch_gather(dtype):
    """sb_pack_rows / sb_unpack_rows (csrc/exchange.cu) against torch
    indexing on the group-major flat layout, bit for bit, with repeated dump
    slots."""
    import torch
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.batch import GROUP_WIDTHS, ROW_REALS, group_views
    dt = getattr(torch, dtype)
    n_pad, n = 1000, 997
    g = torch.Generator().manual_seed(3)
    flat = torch.randn(ROW_REALS * n_pad, generator=g, dtype=torch.float64).to(dt).cuda()
    full = group_views(flat, n_pad)
    for name, _ in GROUP_WIDTHS:
        full[name][n:] = 0        # dump rows hold zeros
    rows = torch.randperm(n, generator=g)[:300].sort().values
    pos = torch.cat([rows, torch.full((50,), n)]).cuda()
    packed = torch.empty((pos.numel(), ROW_REALS), dtype=dt, device="cuda")
    st = N.stream_ptr()
    N.call("sb_pack_rows", N.dtype_code(dt), n_pad, N.ptr(flat), N.ptr(pos), pos.numel(),
           N.ptr(packed), None, st)
    want = torch.cat([full[k].reshape(n_pad, -1)[pos] for k, _ in GROUP_WIDTHS], 1)
    torch.testing.assert_close(packed, want, rtol=0, atol=0)
    before = torch.cat([full[k].reshape(n_pad, -1) for k, _ in GROUP_WIDTHS], 1).clone()
    new = packed * 3
    new[300:] = 0                 # the dump slots carry the dump row's zeros
    N.call("sb_unpack_rows", N.dtype_code(dt), n_pad, N.ptr(flat), N.ptr(pos), pos.numel(),
           N.ptr(new), st)
    after = torch.cat([group_views(flat, n_pad)[k].reshape(n_pad, -1) for k, _ in GROUP_WIDTHS],
                      1)
    rows = rows.cuda()
    torch.testing.assert_close(after[rows], new[:300], rtol=0, atol=0)
    other = torch.ones(n_pad, dtype=torch.bool, device="cuda")
    other[rows] = False
    torch.testing.assert_close(after[other], before[other], rtol=0, atol=0)
