"""GPU edge cases of the binning and blend path against the oracle (the
reference's own tests cover empty maps, rows behind the camera and odd image
sizes; the explicit-list path for splats with more than 64 candidate tiles
and the engine's depth-limited lists have no golden vector of their own)."""

import numpy as np
import pytest
import torch

from parity import COLOR_TOL, assert_image_close, oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2404_06926_b200 as sb
    return sb


@pytest.fixture(scope="module")
def o():
    return oracle()


def _np(t):
    return t.detach().cpu().numpy()


def _map(rng, n, W, H, f, scale_lo=0.02, scale_hi=0.3, zlo=2.0, zhi=8.0):
    z = rng.uniform(zlo, zhi, n)
    x = (rng.uniform(0, W, n) - W / 2) * z / f
    y = (rng.uniform(0, H, n) - H / 2) * z / f
    pos = np.stack([x, y, z], 1)
    ls = np.log(rng.uniform(scale_lo, scale_hi, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.normal(0.5, 1.5, n)
    sh = rng.normal(0, 0.3, (n, 16, 3))
    return [a.astype(np.float32) for a in (pos, ls, q, op, sh)]


def _bin_both(sb, o, arrays, W, H, f):
    pose = sb.CameraPose.identity()
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    scr = sb.project_gaussians(*arrays, pose, intr)
    grid = sb.bin_and_sort(scr, intr)
    sd = {k: _np(getattr(scr, k)) for k in scr.FIELDS}
    pg, pt, off = o.bin_and_sort(sd, W, H)
    return scr, intr, grid, sd, (pg, pt, off)


def _check(grid, ref):
    pg, pt, off = ref
    np.testing.assert_array_equal(_np(grid.pair_gaussian), pg)
    np.testing.assert_array_equal(_np(grid.pair_tile), pt)
    np.testing.assert_array_equal(_np(grid.offsets), off)


def test_big_splats_explicit_lists(sb, o):
    """Splats covering well over 64 tiles go through the explicit tile-list
    path of the binning; order and ranges stay bit-exact."""
    rng = np.random.default_rng(11)
    W, H, f = 320, 240, 200.0
    small = _map(rng, 300, W, H, f)
    big = _map(rng, 12, W, H, f, scale_lo=0.8, scale_hi=2.0, zlo=3.0, zhi=5.0)
    arrays = [np.concatenate([a, b]) for a, b in zip(small, big)]
    scr, intr, grid, sd, ref = _bin_both(sb, o, arrays, W, H, f)
    r = sd["radius_cut"]
    assert ((2 * r / 16 + 1) ** 2 > 64).sum() >= 5, "scene lacks >64-candidate splats"
    _check(grid, ref)
    t = sb.render(grid, scr, intr)
    ot = o.composite(_np(grid.pair_gaussian), _np(grid.offsets), sd, W, H)
    assert_image_close(_np(t.color), ot["color"], tol=1e-6)
    np.testing.assert_array_equal(_np(t.n_contrib), ot["n_contrib"])


@pytest.mark.parametrize("W,H", [(16, 16), (17, 9), (33, 47), (100, 7)])
def test_odd_image_sizes(sb, o, W, H):
    rng = np.random.default_rng(W * 100 + H)
    f = 0.8 * max(W, H)
    arrays = _map(rng, 120, W, H, f)
    scr, intr, grid, sd, ref = _bin_both(sb, o, arrays, W, H, f)
    _check(grid, ref)
    t = sb.render(grid, scr, intr)
    ot = o.composite(_np(grid.pair_gaussian), _np(grid.offsets), sd, W, H)
    assert_image_close(_np(t.color), ot["color"], tol=COLOR_TOL)


def test_rows_behind_camera_and_empty(sb, o):
    rng = np.random.default_rng(4)
    W, H, f = 64, 48, 50.0
    arrays = _map(rng, 50, W, H, f)
    arrays[0][:, 2] = -np.abs(arrays[0][:, 2])       # everything behind the camera
    scr, intr, grid, sd, ref = _bin_both(sb, o, arrays, W, H, f)
    assert len(scr) == 0
    _check(grid, ref)
    assert int(_np(grid.offsets)[-1]) == 0
    t = sb.render(grid, scr, intr)
    assert float(np.abs(_np(t.color)).max()) == 0.0
    assert float(_np(t.transmittance).min()) == 1.0


def test_engine_depth_limits_with_big_splats(sb):
    """The engine's depth-limited lists on a scene with explicit-list splats:
    bitwise the same iterations as full lists (the iteration is flagged and
    re-run whenever a limited tile fails to terminate)."""
    from parity import assert_logs_identical, assert_maps_identical
    rng = np.random.default_rng(21)
    W, H, f = 160, 128, 120.0
    small = _map(rng, 1500, W, H, f, zlo=2.0, zhi=9.0)
    big = _map(rng, 8, W, H, f, scale_lo=0.8, scale_hi=1.5, zlo=6.0, zhi=9.0)
    arrays = [np.concatenate([a, b]) for a, b in zip(small, big)]
    img = rng.uniform(0, 1, (H, W, 3))
    mps = []
    for caps in (True, False):
        cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False)
        mp = sb.Mapper(cfg)
        mp.map.append_arrays(*arrays, np.zeros(len(arrays[0]), bool))
        mp.scene_extent = 1.0
        mp.adam = sb.AdamState(mp.map.count, mp._lrs())
        intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
        e = mp.store.add(sb.CameraFrame(pose=sb.CameraPose.identity(), intrinsics=intr,
                                        image=img), cfg.lr_exposure)
        mp.engine.use_caps = caps
        logs = mp.collect([mp.optimize_keyframe(e) for _ in range(5)])
        mps.append((mp, logs))
    (a, la), (b, lb) = mps
    assert_logs_identical(la, lb)
    assert_maps_identical(a, b)


def test_many_big_splats_in_one_warp(sb, o):
    """Several explicit-list rows per 32-row warp (walked by the whole warp,
    one row at a time) and a splat over the whole image: bit-exact lists."""
    rng = np.random.default_rng(12)
    W, H, f = 320, 240, 200.0
    small = _map(rng, 200, W, H, f)
    big = _map(rng, 160, W, H, f, scale_lo=0.6, scale_hi=1.5, zlo=3.0, zhi=6.0)
    huge = _map(rng, 2, W, H, f, scale_lo=6.0, scale_hi=8.0, zlo=4.0, zhi=4.5)
    arrays = [np.concatenate([a, b, c]) for a, b, c in zip(small, big, huge)]
    scr, intr, grid, sd, ref = _bin_both(sb, o, arrays, W, H, f)
    ncand = (2 * sd["radius_cut"] / 16 + 1) ** 2
    assert (ncand > 64).sum() >= 100 and (ncand >= 300).any()
    _check(grid, ref)


def test_long_rank_adjoints_vs_oracle(o):
    """The deterministic merge of ranks with more than 64 kept pairs (one warp
    per queued rank, pair-order sums) on the engine's own screen, pairs,
    render and dC: against the oracle's serial per-pair merge
    (backward.py:91-213), 1e-3 rel / 1e-5 abs, f64-calibrated."""
    import paper_2404_06926_b200 as sb
    from parity import assert_grads_calibrated
    rng = np.random.default_rng(13)
    W, H, f = 320, 240, 200.0
    small = _map(rng, 400, W, H, f)
    big = _map(rng, 120, W, H, f, scale_lo=0.6, scale_hi=1.5, zlo=3.0, zhi=6.0)
    arrays = [np.concatenate([a, b]) for a, b in zip(small, big)]
    arrays[3][:] = np.float32(-1.0)          # translucent: long replays
    n = arrays[0].shape[0]
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=n)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*arrays, np.zeros(n, dtype=bool))
    mp.adam = sb.AdamState(n, mp._lrs())
    pose = sb.CameraPose.identity()
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    img = np.random.default_rng(14).uniform(0, 1, (H, W, 3))
    entry = mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=img),
                         cfg.lr_exposure, torch.float32)
    mp.use_graphs = False
    mp.collect([mp.optimize_keyframe(entry) for _ in range(3)])
    mp.collect([mp.optimize_keyframe(entry)])
    assert mp.reruns == 0
    torch.cuda.synchronize()
    eng = mp.engine
    b = eng.bufs
    P = int(eng.binout["offsets"][-1].item())
    pg = _np(eng.binout["a_pg"][:P]).astype(np.int64)
    off = _np(eng.binout["offsets"]).astype(np.int64)
    assert np.bincount(pg, minlength=n).max() > 64, "no long rank"
    r = _np(b["records"][:n]).astype(np.float32)
    inv = np.stack([np.stack([r[:, 2], r[:, 3]], 1), np.stack([r[:, 3], r[:, 4]], 1)], 1)
    screen = {"mean2d": r[:, 0:2].copy(), "inv_cov2d": inv, "opacity": r[:, 5].copy(),
              "q_cut": r[:, 6].copy(), "radius_cut": r[:, 7].copy(),
              "color": r[:, 8:11].copy(), "depth": r[:, 11].copy()}
    dr = _np(eng.loss["d_rendered"]).copy()
    color = _np(eng.fwd["color"]).copy()
    a32 = o.backward_tiles(pg, off, screen, dr, color, W, H)
    up = {k: v.astype(np.float64) for k, v in screen.items()}
    a64 = o.backward_tiles(pg, off, up, dr.astype(np.float64), color.astype(np.float64), W, H)
    # rows the gather reached carry merged adjoints; the others are zero by
    # definition (the engine does not zero them)
    ws = b["ws_chain_adam"]
    a256 = lambda x: (x + 255) & ~255  # noqa: E731
    offb = sum(a256(w * 4 * n) for w in (3, 3, 4, 1, 48))
    reached = (_np(ws[offb:offb + n]) & 2) != 0
    rows = np.nonzero(_np(b["valid"][:n]))[0]
    long_rows = np.nonzero(np.bincount(pg, minlength=n) > 64)[0]
    for k in ("d_mean2d", "d_conic", "d_opacity", "d_color"):
        g = _np(b[k][:n]).astype(np.float32)
        g = np.where(reached.reshape((-1,) + (1,) * (g.ndim - 1)), g, 0)
        assert_grads_calibrated(g[rows], a32[k][rows], a64[k][rows], k)
        assert_grads_calibrated(g[long_rows], a32[k][long_rows], a64[k][long_rows], k)


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
def test_long_rank_gradients_stage_api(sb, o, dt):
    """backward_per_gaussian (sb_blend_bwd_det: per-pair records, the long
    ranks merged one warp per rank) on a scene whose ranks hold well over 64
    pairs, in both dtypes: against the oracle's serial merge + chain on the
    GPU's own screen, grid and render (backward.py:91-213, 415-500)."""
    from parity import assert_grads_calibrated
    rng = np.random.default_rng(15)
    W, H, f = 320, 240, 200.0
    small = _map(rng, 300, W, H, f)
    big = _map(rng, 80, W, H, f, scale_lo=0.6, scale_hi=1.5, zlo=3.0, zhi=6.0)
    arrays = [np.concatenate([a, b]).astype(dt) for a, b in zip(small, big)]
    arrays[3][:] = dt(-1.0)
    pose = sb.CameraPose.identity()
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    scr = sb.project_gaussians(*arrays, pose, intr)
    grid = sb.bin_and_sort(scr, intr)
    pg = _np(grid.pair_gaussian).astype(np.int64)
    assert np.bincount(pg).max() > 64, "no long rank"
    t = sb.render(grid, scr, intr)
    dC = np.random.default_rng(16).normal(0, 1e-3, (H, W, 3)).astype(dt)
    gm = sb.GaussianMap(dtype=dt)
    gm.append_arrays(*arrays, np.zeros(arrays[0].shape[0], dtype=bool))
    buf = sb.backward_per_gaussian(t, torch.as_tensor(dC).cuda(), scr, grid, gm, pose, intr)
    sd = {k: _np(getattr(scr, k)) for k in scr.FIELDS}
    off = _np(grid.offsets)
    cam = o.Camera(W=np.eye(3), t=np.zeros(3), fx=f, fy=f, cx=W / 2, cy=H / 2, width=W,
                   height=H)
    gmap = {"positions": arrays[0], "log_scales": arrays[1], "rotations": arrays[2],
            "opacity_logits": arrays[3], "sh_coeffs": arrays[4], "is_sky": None}
    adj = o.backward_tiles(pg, off, sd, dC, _np(t.color), W, H)
    og = o.chain(adj, sd, gmap, cam)
    up = lambda v: v.astype(np.float64) if getattr(v, "dtype", None) == np.float32 else v  # noqa: E731
    s64 = {k: up(v) for k, v in sd.items()}
    adj64 = o.backward_tiles(pg, off, s64, up(dC), up(_np(t.color)), W, H)
    truth = o.chain(adj64, s64, {k: up(v) for k, v in gmap.items() if v is not None}, cam)
    for k in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        assert_grads_calibrated(_np(getattr(buf, k)), og[k], truth[k], k)
