"""GPU: keyframe-batch step and map growth (§8f row 1)."""

import numpy as np
import pytest

from parity import oracle

pytestmark = pytest.mark.gpu


def _mapper(sb, n=400, seed=5, W=64, H=48, f=56.0):
    import torch
    from paper_2404_06926_b200.synthetic import view_map
    rng = np.random.default_rng(seed)
    arrays = [a.astype(np.float32) if a.dtype != bool else a
              for a in view_map(rng, n, W, H, f)]
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs(), dtype=torch.float32)
    return mp, arrays


def _views(sb, k, W=64, H=48, f=56.0):
    out = []
    for i in range(k):
        a = 0.06 * (i - 1)
        R = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
        pose = sb.CameraPose(R, np.array([0.05 * i, 0.0, 0.0]))
        intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
        img = np.random.default_rng(30 + i).uniform(0, 1, (H, W, 3))
        out.append((pose, intr, img))
    return out


@pytest.mark.parametrize("sharded", [False, True, "packed", "packed_ar"])
def test_batch_step_matches_batched_oracle(sharded):
    """BatchStep (all-reduce exchange) and ShardedBatchStep (row-block Adam,
    here at world size 1) against the batched oracle."""
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200.batch import (BatchStep, DeviceBatchCompute, PackedBatchStep,
                                             PackedShardedBatchStep, ShardedBatchStep)
    o = oracle()
    mp, arrays = _mapper(sb)
    views = _views(sb, 3)
    entries = []
    for i, (pose, intr, img) in enumerate(views):
        e = mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=img, frame_index=i),
                         mp.cfg.lr_exposure)
        entries.append(e)
    cls = {"packed": PackedShardedBatchStep, "packed_ar": PackedBatchStep,
           True: ShardedBatchStep, False: BatchStep}[sharded]
    cls(DeviceBatchCompute(mp)).step(entries)
    # batched oracle: f32 per-view gradient sum, one Adam step on the union
    g = {"positions": arrays[0].copy(), "log_scales": arrays[1].copy(),
         "rotations": arrays[2].copy(), "opacity_logits": arrays[3].copy(),
         "sh_coeffs": arrays[4].copy()}
    n = g["positions"].shape[0]
    tot = {k: 0 for k in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")}
    union = np.zeros(n, bool)
    for pose, intr, img in views:
        cam = o.Camera(W=pose.rotation_wc, t=pose.translation_wc, fx=intr.fx, fy=intr.fy,
                       cx=intr.cx, cy=intr.cy, width=intr.width, height=intr.height)
        sc, (pg, pt, off), t = o.render_view(g, cam)
        _, d_r, _, _ = o.photometric_loss(t["color"], img.astype(np.float32),
                                          np.concatenate([np.eye(3), np.zeros((3, 1))], 1), 0.2)
        adj = o.backward_tiles(pg, off, sc, d_r, t["color"], intr.width, intr.height)
        gr = o.chain(adj, sc, g, cam)
        for k in tot:
            tot[k] = tot[k] + gr[k]
        union |= o.frustum_mask(cam, g["positions"])
    arrs = [g[k] for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")]
    m = {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)}
    v = {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)}
    steps = np.zeros(n, np.int64)
    params = dict(zip(o.GROUPS, arrs))
    grads = dict(zip(o.GROUPS, [tot["d_position"], tot["d_log_scale"], tot["d_rotation"],
                                tot["d_opacity_logit"], tot["d_sh"]]))
    o.adam_step(params, grads, m, v, steps, mp.adam.lrs, active=union)
    np.testing.assert_array_equal(mp.adam.steps.cpu().numpy(), steps)
    a = mp.map.arrays()
    lrs = mp.adam.lrs
    for key, gk, lr in (("positions", "position", lrs["position"]),
                        ("log_scales", "log_scale", lrs["log_scale"]),
                        ("rotations", "rotation", lrs["rotation"]),
                        ("opacity_logits", "opacity_logit", lrs["opacity_logit"]),
                        ("sh_coeffs", "sh", max(lrs["sh0"], lrs["sh_rest"]))):
        gref = np.abs(grads[gk].astype(np.float64))
        noisy = gref <= 1e-6 * max(gref.max(), 1e-30) + 1e-12
        d = np.abs(a[key].cpu().numpy().astype(np.float64) - g[key])
        assert d[~noisy].max(initial=0) <= 1e-5 * (1 + np.abs(g[key]).max()), key
        assert d[noisy].max(initial=0) <= 2 * lr * 1.0001 + 1e-7, key


def test_expand_selects_like_reference():
    """Mapper.expand (mapper.py:252-281): f64 projection, nearest pixel
    floor(u + 0.5), opacity < 0.99 of the keyframe render; bit-exact count
    and seeded rows."""
    import paper_2404_06926_b200 as sb
    mp, _ = _mapper(sb, n=150)
    pose, intr, img = _views(sb, 1)[0]
    frame = sb.CameraFrame(pose=pose, intrinsics=intr, image=img, frame_index=0)
    rng = np.random.default_rng(9)
    k = 3000
    z = rng.uniform(-1.0, 9.0, k)
    pts = np.stack([rng.uniform(-4, 4, k) * np.abs(z) / 6, rng.uniform(-3, 3, k) * np.abs(z) / 6,
                    z], 1)
    rgb = rng.uniform(0, 1, (k, 3))
    merged = np.concatenate([pts, rgb], 1)
    _, _, t = mp.render_view(pose, intr)
    mask = (t.opacity < np.float32(0.99)).cpu().numpy()
    n0 = mp.map.count
    added = mp.expand(frame, merged)
    # numpy restatement of mapper.py:262-274
    pc = pts @ pose.rotation_wc.T + pose.translation_wc
    zc = pc[:, 2]
    ok = zc > mp.cfg.near
    with np.errstate(divide="ignore", invalid="ignore"):
        u = intr.fx * pc[:, 0] / zc + intr.cx
        v = intr.fy * pc[:, 1] / zc + intr.cy
    col = np.floor(u + 0.5)
    row = np.floor(v + 0.5)
    ok &= (col >= 0) & (col < intr.width) & (row >= 0) & (row < intr.height)
    sel = np.nonzero(ok)[0]
    sel = sel[mask[row[sel].astype(int), col[sel].astype(int)]]
    assert added == sel.size > 0
    assert mp.map.count == n0 + added
    assert mp.adam.count == mp.map.count
    new = {k: v.cpu().numpy() for k, v in mp.map.arrays().items()}
    np.testing.assert_allclose(new["positions"][n0:], pts[sel].astype(np.float32))
    scale = pc[sel, 2] / intr.fx
    np.testing.assert_allclose(new["log_scales"][n0:, 0], np.log(scale).astype(np.float32),
                               rtol=1e-6)
    np.testing.assert_allclose(new["sh_coeffs"][n0:, 0, :],
                               ((rgb[sel] - 0.5) / 0.28209479177387814).astype(np.float32),
                               rtol=1e-6)
    assert (mp.adam.steps[n0:] == 0).all()


def test_capacity_error():
    import paper_2404_06926_b200 as sb
    m = sb.GaussianMap(capacity=10)
    arr = [np.zeros((11, 3)), np.zeros((11, 3)), np.tile([1.0, 0, 0, 0], (11, 1)), np.zeros(11),
           np.zeros((11, 16, 3)), np.zeros(11, bool)]
    with pytest.raises(sb.CapacityError):
        m.append_arrays(*arr)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_chain_accumulate_equals_row_kernel(dtype):
    """sb_chain_accumulate (compacted list of reached rows) is bit-identical
    to sb_preprocess_bwd_rows(accumulate=1) (one thread per map row)."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.synthetic import view_map
    dt = torch.float32 if dtype == "f32" else torch.float64
    code = N.dtype_code(dt)
    n, W, H, f = 3000, 96, 64, 80.0
    rng = np.random.default_rng(11)
    arrs = [torch.as_tensor(a).to("cuda", dt) for a in view_map(rng, n, W, H, f)[:5]]
    valid = torch.as_tensor(rng.uniform(size=n) < 0.8).to("cuda", torch.uint8)
    reached = torch.as_tensor(rng.uniform(size=n) < 0.3, device="cuda")
    adj = [torch.as_tensor(rng.normal(size=(n,) + s) * 1e-3).to("cuda", dt)
           for s in ((2,), (3,), (), (3,))]
    for t in adj:
        t.mul_(reached.view((n,) + (1,) * (t.dim() - 1)).to(dt))
    adj[2][:7] = 0.0   # rows with only some adjoints zero
    cam = N.camera(sb.CameraPose(np.eye(3), np.zeros(3)), sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H))
    base = [torch.as_tensor(rng.normal(size=(n,) + s)).to("cuda", dt)
            for s in ((3,), (3,), (4,), (), (16, 3))]
    outs = []
    for variant in ("rows", "list"):
        g = [b.clone() for b in base]
        st = N.stream_ptr()
        if variant == "rows":
            N.call("sb_preprocess_bwd_rows", code, n, N.ptr(valid), *[N.ptr(a) for a in arrs],
                   N.C.byref(cam), 0.3, *[N.ptr(t) for t in adj], *[N.ptr(t) for t in g], 1, st)
        else:
            ws = torch.empty(N.load().sb_chain_accumulate_workspace_bytes(code, n),
                             dtype=torch.uint8, device="cuda")
            hit = torch.zeros(n, dtype=torch.uint8, device="cuda")
            N.call("sb_chain_accumulate", code, n, N.ptr(valid), *[N.ptr(a) for a in arrs],
                   N.C.byref(cam), 0.3, *[N.ptr(t) for t in adj], *[N.ptr(t) for t in g],
                   N.ptr(hit), 0, None, N.ptr(ws), ws.numel(), st)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in g])
    # the reached mask: valid rows with some non-zero adjoint
    nz = torch.zeros(n, dtype=torch.bool, device="cuda")
    for t in adj:
        nz |= (t.reshape(n, -1) != 0).any(dim=1)
    np.testing.assert_array_equal(hit.bool().cpu().numpy(), (nz & valid.bool()).cpu().numpy())
    for a, b, b0 in zip(outs[0], outs[1], base):
        assert np.array_equal(a, b)
    assert not np.array_equal(outs[1][4], base[4].cpu().numpy())   # something accumulated


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_sparse_adam_flat_equals_row_kernel(dtype):
    """sb_sparse_adam_flat (the batched step's and adam_step's path) is
    bit-identical to the per-row sb_sparse_adam kernel over several steps."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.adam import lr_vector
    from paper_2404_06926_b200.synthetic import default_lrs
    dt = torch.float32 if dtype == "f32" else torch.float64
    code = N.dtype_code(dt)
    n = 5003
    rng = np.random.default_rng(3)
    shapes = {"position": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (),
              "sh": (16, 3)}
    p0 = {k: torch.as_tensor(rng.normal(size=(n,) + s)).to("cuda", dt) for k, s in shapes.items()}
    results = []
    for variant in ("rows", "flat"):
        params = {k: v.clone() for k, v in p0.items()}
        st = sb.AdamState(n, default_lrs(), dtype=dt)
        grng = np.random.default_rng(9)
        for step in range(3):
            grads = {k: torch.as_tensor(grng.normal(size=(n,) + s) * 10.0 ** grng.integers(-8, 1))
                     .to("cuda", dt) for k, s in shapes.items()}
            active = torch.as_tensor(grng.uniform(size=n) < 0.7).to("cuda", torch.uint8)
            G = st.groups(params, grads)
            lrs = lr_vector(st.lrs)
            if variant == "rows":
                N.call("sb_sparse_adam", code, n, N.C.byref(G), N.ptr(st._steps), N.ptr(active),
                       lrs.ctypes.data_as(N.vp), N.stream_ptr())
            else:
                ws = torch.empty(N.load().sb_sparse_adam_workspace_bytes(code, n),
                                 dtype=torch.uint8, device="cuda")
                N.call("sb_sparse_adam_flat", code, n, N.C.byref(G), N.ptr(st._steps),
                       N.ptr(active), None, None, lrs.ctypes.data_as(N.vp), N.ptr(ws),
                       ws.numel(), None, N.stream_ptr())
        torch.cuda.synchronize()
        results.append(({k: v.cpu().numpy() for k, v in params.items()},
                        st._steps.cpu().numpy()))
    (pa, sa), (pb, sb_) = results
    assert np.array_equal(sa, sb_)
    for k in pa:
        assert np.array_equal(pa[k], pb[k]), k


def test_batched_depth_limits_match_full_lists():
    """Repeated keyframe-batch steps with the per-view tile depth limits
    (async binning, validated truncated lists) follow the same trajectory as
    full lists: bitwise the same losses and map (the backward is
    deterministic), identical Adam step counters, and fewer pairs kept once
    the limits apply."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200.batch import BatchStep, DeviceBatchCompute
    runs = []
    for use_limits in (True, False):
        mp, _ = _mapper(sb, n=6000, seed=8)
        views = _views(sb, 3)
        entries = [mp.store.add(sb.CameraFrame(pose=p, intrinsics=i, image=img, frame_index=k),
                                mp.cfg.lr_exposure) for k, (p, i, img) in enumerate(views)]
        comp = DeviceBatchCompute(mp)
        comp.use_limits = use_limits
        step = BatchStep(comp)
        losses = []
        for _ in range(5):
            parts = step.step(entries)
            losses.append(torch.stack(parts).cpu().numpy())
        kept = [int(comp.bufs[("status", id(e))][0].item()) for e in entries]
        runs.append((np.array(losses), mp.adam.steps.cpu().numpy(), kept,
                     {k: v.cpu().numpy() for k, v in mp.map.arrays().items()}))
    (l_lim, s_lim, k_lim, m_lim), (l_full, s_full, k_full, m_full) = runs
    np.testing.assert_array_equal(s_lim, s_full)
    np.testing.assert_array_equal(l_lim, l_full)
    for k in m_lim:
        np.testing.assert_array_equal(m_lim[k], m_full[k], err_msg=k)
    assert sum(k_lim) < sum(k_full), (k_lim, k_full)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_chain_accumulate_first_touch(dtype):
    """first_touch: two views accumulated into an UNZEROED buffer (a row's
    first reach stores, later views add) equal the zeroed buffer's sums on
    every reached row, bit for bit; sb_sparse_adam_flat with grad_rows =
    those rows then equals the zero-filled gradient's update."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.adam import lr_vector
    from paper_2404_06926_b200.synthetic import default_lrs, view_map
    dt = torch.float32 if dtype == "f32" else torch.float64
    code = N.dtype_code(dt)
    n, W, H, f = 3000, 96, 64, 80.0
    rng = np.random.default_rng(12)
    arrs = [torch.as_tensor(a).to("cuda", dt) for a in view_map(rng, n, W, H, f)[:5]]
    valid = torch.ones(n, dtype=torch.uint8, device="cuda")
    views = []
    for _ in range(2):
        reached = torch.as_tensor(rng.uniform(size=n) < 0.3, device="cuda")
        adj = [torch.as_tensor(rng.normal(size=(n,) + s) * 1e-3).to("cuda", dt)
               for s in ((2,), (3,), (), (3,))]
        for t in adj:
            t.mul_(reached.view((n,) + (1,) * (t.dim() - 1)).to(dt))
        views.append(adj)
    cam = N.camera(sb.CameraPose(np.eye(3), np.zeros(3)), sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H))
    shapes = ((3,), (3,), (4,), (), (16, 3))
    ws = torch.empty(N.load().sb_chain_accumulate_workspace_bytes(code, n), dtype=torch.uint8,
                     device="cuda")
    outs = []
    for first in (0, 1):
        g = [torch.zeros((n,) + s, dtype=dt, device="cuda") if not first else
             torch.full((n,) + s, float("nan"), dtype=dt, device="cuda") for s in shapes]
        hit = torch.zeros(n, dtype=torch.uint8, device="cuda")
        for adj in views:
            N.call("sb_chain_accumulate", code, n, N.ptr(valid), *[N.ptr(a) for a in arrs],
                   N.C.byref(cam), 0.3, *[N.ptr(t) for t in adj], *[N.ptr(t) for t in g],
                   N.ptr(hit), first, None, N.ptr(ws), ws.numel(), N.stream_ptr())
        outs.append((g, hit))
    (gz, hz), (gf, hf) = outs
    assert torch.equal(hz, hf)
    rows = hz.bool()
    for a, b in zip(gz, gf):
        assert torch.equal(a[rows], b[rows])
        assert bool(torch.isnan(b[~rows]).all())       # untouched: never read
    # the sparse Adam reads only grad_rows
    params0 = [torch.as_tensor(rng.normal(size=(n,) + s)).to("cuda", dt) for s in shapes]
    active = torch.as_tensor(rng.uniform(size=n) < 0.8).to("cuda", torch.uint8)
    res = []
    for grads, grows in ((gz, None), (gf, hz)):
        params = {k: p.clone() for k, p in zip(("position", "log_scale", "rotation",
                                                "opacity_logit", "sh"), params0)}
        st = sb.AdamState(n, default_lrs(), dtype=dt)
        G = st.groups(params, dict(zip(params, grads)))
        w2 = torch.empty(N.load().sb_sparse_adam_workspace_bytes(code, n), dtype=torch.uint8,
                         device="cuda")
        N.call("sb_sparse_adam_flat", code, n, N.C.byref(G), N.ptr(st._steps), N.ptr(active),
               N.ptr(grows), None, lr_vector(st.lrs).ctypes.data_as(N.vp), N.ptr(w2), w2.numel(),
               None, N.stream_ptr())
        res.append(params)
    for k in res[0]:
        assert torch.equal(res[0][k], res[1][k]), k


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("grad_frac", [0.03, 0.2])
def test_touched_row_skip_bitwise(dtype, grad_frac):
    """The touched-row skip (sb_sparse_adam_flat with a touched mask) equals
    the full pass bit for bit over several steps: params, both moments and the
    step counters -- with rows whose moments were written from outside
    (AdamState.m, a signed zero among them) and a gradient whose rows change
    from step to step; the mask the kernels keep then matches the one rebuilt
    from the moments' bits.  grad_frac 0.03 keeps the live rows under n/6
    (the live-row list pass), 0.2 takes them over it within two steps (the
    flat pass; the pass is chosen from the previous step's live count)."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import _native as N
    from paper_2404_06926_b200.adam import lr_vector
    from paper_2404_06926_b200.synthetic import default_lrs
    dt = torch.float32 if dtype == "f32" else torch.float64
    code = N.dtype_code(dt)
    n = 7001
    rng = np.random.default_rng(5)
    shapes = {"position": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (),
              "sh": (16, 3)}
    p0 = {k: torch.as_tensor(rng.normal(size=(n,) + s)).to("cuda", dt) for k, s in shapes.items()}
    p0["position"][5, 0] = -0.0
    out = []
    for skip in (False, True):
        params = {k: v.clone() for k, v in p0.items()}
        st = sb.AdamState(n, default_lrs(), dtype=dt)
        st.m["sh"][100:110] = 1e-3        # outside writes: the mask is rebuilt
        st.v["rotation"][200, 1] = -0.0   # a signed zero counts as touched
        grng = np.random.default_rng(11)
        kept = []
        for step in range(5):
            grads = {k: torch.as_tensor(grng.normal(size=(n,) + s) * 10.0 ** grng.integers(-8, 1))
                     .to("cuda", dt) for k, s in shapes.items()}
            active = torch.as_tensor(grng.uniform(size=n) < 0.8).to("cuda", torch.uint8)
            rows = torch.as_tensor(grng.uniform(size=n) < grad_frac).to("cuda", torch.uint8)
            G = st.groups(params, grads)
            if step == 0:   # one workspace for the run: it carries the live count
                ws = torch.zeros(N.load().sb_sparse_adam_workspace_bytes(code, n),
                                 dtype=torch.uint8, device="cuda")
            touched = st.touched() if skip else None
            N.call("sb_sparse_adam_flat", code, n, N.C.byref(G), N.ptr(st._steps), N.ptr(active),
                   N.ptr(rows), N.ptr(touched), lr_vector(st.lrs).ctypes.data_as(N.vp),
                   N.ptr(ws), ws.numel(), None, N.stream_ptr())
            if skip:
                kept.append(st._touched[:n].clone())
        torch.cuda.synchronize()
        if skip:
            st.moments_written()
            rebuilt = st.touched()[:n]
            # the kernels' mask: a superset of the rows with non-zero moments
            assert bool((kept[-1] >= rebuilt).all())
            assert int(kept[-1].sum()) < n      # something was skipped
        out.append(({k: v.cpu().numpy() for k, v in params.items()},
                    {k: t.cpu().numpy() for k, t in st._m.items()},
                    {k: t.cpu().numpy() for k, t in st._v.items()},
                    st._steps.cpu().numpy()))
    a, b = out
    for i in range(3):
        for k in a[i]:
            assert np.array_equal(a[i][k].view(np.uint8), b[i][k].view(np.uint8)), (i, k)
    assert np.array_equal(a[3], b[3])
