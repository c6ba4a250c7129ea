"""GPU parity at BASELINE.json's other configs (parity cases, not bench lines)
and the reference's float64 finite-difference gate (gradcheck.py:80-117).

* config 1 (10k, 320x240): one full step against the oracle's step;
* config 2 (100k, 640x480, repeated steps on one keyframe): per-step parity
  with the CPU reseeded from the GPU state each step, plus a
  GPU-only trajectory whose loss must descend;
* config 3 (1M, 1280x720, sky + exposure) at full size: binning bit-exact
  against the oracle on the GPU's own splat floats, render within the
  explained-flip budget, and size-independent properties;
* config 4 shape (incremental stream with map growth): a small teacher-map
  stream through Mapper.process_frame;
* f64: central finite differences of the full loss on the gradcheck scenes.
"""

import numpy as np
import pytest

from parity import (COLOR_TOL, assert_image_close, explained_pixel_budget, max_abs, oracle)

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _setup(sb, scene, dtype=np.float32):
    import torch
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=max(scene.n, 1))
    mp = sb.Mapper(cfg, dtype=torch.float32 if dtype == np.float32 else torch.float64)
    mp.map.append_arrays(*scene.arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs(), dtype=mp.dtype)
    pose = sb.CameraPose(scene.W, scene.t)
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    entry = mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=scene.image),
                         cfg.lr_exposure, mp.dtype)
    entry.exposure.matrix = scene.E
    return mp, entry, pose, intr


def _oracle_state(o, arrays):
    gm = {"positions": arrays[0].copy(), "log_scales": arrays[1].copy(),
          "rotations": arrays[2].copy(), "opacity_logits": arrays[3].copy(),
          "sh_coeffs": arrays[4].copy(), "is_sky": arrays[5]}
    arrs = [gm[k] for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")]
    adam = {"m": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "v": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "steps": np.zeros(arrs[0].shape[0], np.int64)}
    return gm, adam


def test_config1_step_vs_oracle():
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    o = oracle()
    scene = synthetic.config(1)
    mp, entry, pose, intr = _setup(sb, scene)
    log = mp._optimize_step(entry)
    gm, adam = _oracle_state(o, scene.arrays)
    cam = o.Camera(W=scene.W, t=scene.t, fx=scene.fx, fy=scene.fy, cx=scene.cx, cy=scene.cy,
                   width=scene.width, height=scene.height)
    E = scene.E.copy()
    ref = o.optimize_step(gm, adam, synthetic.default_lrs(), cam, scene.image, E,
                          o.ScalarAdam((3, 4), 1e-2))
    assert log["loss"] == pytest.approx(ref["loss"], rel=1e-6)
    np.testing.assert_array_equal(_np(mp.adam.steps), adam["steps"])
    # params: equal except Adam's first-step sign on noise-level gradients
    a = mp.map.arrays()
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        d = np.abs(_np(a[k]).astype(np.float64) - gm[k])
        frac_big = float((d > 1e-6).mean())
        assert frac_big < 5e-3, (k, frac_big)
    np.testing.assert_allclose(entry.exposure.matrix, E, atol=1e-7)


def test_config2_trajectory_reseeded_per_step():
    """each GPU step compared with the oracle's step from
    the same (GPU) state; loss agrees to 1e-3 relative at every step."""
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    o = oracle()
    scene = synthetic.config(2)
    mp, entry, pose, intr = _setup(sb, scene)
    mp.use_graphs = True
    cam = o.Camera(W=scene.W, t=scene.t, fx=scene.fx, fy=scene.fy, cx=scene.cx, cy=scene.cy,
                   width=scene.width, height=scene.height)
    losses = []
    for it in range(4):
        # reseed the CPU from the GPU state
        a = mp.map.arrays()
        gm = {k: _np(v).copy() for k, v in a.items()}
        gm["is_sky"] = _np(mp.map.is_sky)
        adam = {"m": {g: _np(t).copy() for g, t in mp.adam.m.items()},
                "v": {g: _np(t).copy() for g, t in mp.adam.v.items()},
                "steps": _np(mp.adam.steps).copy()}
        for g in adam["m"]:
            adam["m"][g] = np.ascontiguousarray(adam["m"][g])
            adam["v"][g] = np.ascontiguousarray(adam["v"][g])
        E = entry.exposure.matrix.copy()
        ex = o.ScalarAdam((3, 4), 1e-2)
        st = _np(entry.exposure.state)
        ex.m, ex.v, ex.t = st[:12].reshape(3, 4).copy(), st[12:24].reshape(3, 4).copy(), int(st[24])
        ref = o.optimize_step(gm, adam, synthetic.default_lrs(), cam, scene.image, E, ex)
        log = mp._optimize_step(entry)
        assert log["loss"] == pytest.approx(ref["loss"], rel=1e-3), it
        losses.append(log["loss"])
        np.testing.assert_allclose(entry.exposure.matrix, E, atol=1e-6)
    # GPU-only continuation: 100 iterations on the keyframe descend
    rows = [mp._step_device(entry) for _ in range(96)]
    final = mp._materialise(rows[-1:])[0]["loss"]
    assert final < losses[0]
    torch.cuda.synchronize()


def test_config3_full_size_binning_and_render():
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    o = oracle()
    scene = synthetic.config(3)
    pose = sb.CameraPose(scene.W, scene.t)
    intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width, scene.height)
    scr = sb.project_gaussians(*scene.arrays[:5], pose, intr)
    assert len(scr) >= 999_990
    grid = sb.bin_and_sort(scr, intr)
    sd = {k: _np(getattr(scr, k)) for k in ("mean2d", "inv_cov2d", "depth", "radius_cut", "q_cut",
                                            "color", "opacity")}
    pg, pt, off = o.bin_and_sort(sd, intr.width, intr.height)
    np.testing.assert_array_equal(_np(grid.offsets), off)
    np.testing.assert_array_equal(_np(grid.pair_gaussian), pg)
    assert grid.n_pairs > 10_000_000
    t = sb.render(grid, scr, intr)
    ot = o.composite(pg, off, sd, intr.width, intr.height)
    assert_image_close(_np(t.color), ot["color"], tol=1e-6,
                       budget=explained_pixel_budget(intr.width * intr.height))
    # properties: opacity = 1 - T, T monotone-bounded, contributor counts agree
    assert np.all(_np(t.transmittance) <= 1) and np.all(_np(t.transmittance) >= 0)
    assert float(np.mean(_np(t.n_contrib) != ot["n_contrib"])) < 1e-5
    d = _np(t.depth)
    assert d.max() > 1000.0  # sky depths reach ~1e4 m
    assert max_abs(d / d.max(), ot["depth"] / d.max()) <= 1e-4


def test_config4_stream_with_growth():
    """Incremental mapping (mapper.py:332-374) on a small teacher stream:
    bootstrap from frame points, keyframes every 5 frames expand the map from
    LiDAR-like points on unreliable pixels, then optimise."""
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200.synthetic import view_map
    rng = np.random.default_rng(4)
    W, H, f = 96, 64, 80.0
    teacher = [a.astype(np.float32) if a.dtype != bool else a for a in view_map(rng, 4000, W, H, f)]
    cfg = sb.MapperConfig(sky_count=500, sky_radius=100.0, keyframe_interval=5,
                          replay_keyframes=4, capacity=20_000)
    mp = sb.Mapper(cfg, seed=0)
    counts = []
    for i in range(16):
        yaw = 0.01 * i
        R = np.array([[np.cos(yaw), 0, np.sin(yaw)], [0, 1, 0], [-np.sin(yaw), 0, np.cos(yaw)]])
        pose = sb.CameraPose(R, np.zeros(3))
        intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
        img = np.random.default_rng(100 + i).uniform(0, 1, (H, W, 3))
        sel = rng.choice(teacher[0].shape[0], 150, replace=False)
        pts = [sb.ColoredPoint(teacher[0][k], np.clip(0.5 + 0.28 * teacher[4][k, 0], 0, 1))
               for k in sel]
        mp.process_frame(sb.CameraFrame(pose=pose, intrinsics=intr, image=img, points=pts,
                                        frame_index=i))
        counts.append(mp.map.count)
    assert counts[0] > 500                      # bootstrap points + sky
    assert counts[-1] > counts[0]               # keyframes grew the map
    assert len(mp.store) == 4                   # frames 0, 5, 10, 15
    assert mp.adam.count == mp.map.count
    assert len(mp.training_log) == 1 + 2 + 3 + 4   # min(replay, store) per keyframe
    assert all(np.isfinite(r["loss"]) for r in mp.training_log)


def _fd_scene_loss(sb, gmap_arrays, pose, intr, target, E, lam=0.2):
    import torch
    scr = sb.project_gaussians(*gmap_arrays, pose, intr)
    grid = sb.bin_and_sort(scr, intr)
    t = sb.render(grid, scr, intr)
    loss, _, _, _ = sb.photometric_loss(t.color, target, sb.ExposureAffine(E), lam)
    del torch
    return loss


@pytest.mark.parametrize("seed", [0, 1])
def test_f64_finite_difference_gate(seed):
    """gradcheck.py:80-117: every analytic gradient (float64 GPU path) within
    1e-4 relative of central finite differences (relative_error with the
    1e-7 absolute floor, backward.py:547-551)."""
    import torch
    import paper_2404_06926_b200 as sb
    rng = np.random.default_rng(seed)
    size = 24
    n = int(rng.integers(6, 13))
    intr = sb.CameraIntrinsics(size, size, size / 2.0, size / 2.0, size, size)
    pose = sb.CameraPose.identity()
    pos, ls, rot, op, sh = [], [], [], [], []
    for _ in range(n):
        depth = rng.uniform(3.0, 7.0)
        s_world = rng.uniform(25.0, 60.0) * depth / intr.fx
        pos.append([rng.uniform(-0.3, 0.3) * depth, rng.uniform(-0.3, 0.3) * depth, depth])
        q = rng.normal(size=4)
        rot.append(q / np.linalg.norm(q))
        ls.append(np.log(s_world * rng.uniform(0.7, 1.4, 3)))
        p = rng.uniform(0.05, 0.25)
        op.append(np.log(p) - np.log1p(-p))
        sh.append(rng.normal(0.0, 0.3, (16, 3)))
    arrays = [np.array(a, np.float64) for a in (pos, ls, rot, op, sh)]
    target = rng.uniform(0.0, 1.0, (size, size, 3))
    E = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) + rng.normal(0.0, 0.02, (3, 4))
    gm = sb.GaussianMap(dtype=np.float64)
    gm.append_arrays(*arrays, np.zeros(n, bool))
    scr = sb.project_gaussians(*gm.arrays().values(), pose, intr)
    grid = sb.bin_and_sort(scr, intr)
    t = sb.render(grid, scr, intr)
    _, d_r, d_E, _ = sb.photometric_loss(t.color, target, sb.ExposureAffine(E), 0.2)
    buf = sb.backward_per_gaussian(t, d_r, scr, grid, gm, pose, intr)
    analytic = [_np(buf.d_position), _np(buf.d_log_scale), _np(buf.d_rotation),
                _np(buf.d_opacity_logit), _np(buf.d_sh)]
    eps = 1e-5
    worst = 0.0
    for gi, (arr, an) in enumerate(zip(arrays, analytic)):
        flat = arr.reshape(-1)
        for i in range(0, flat.size, max(1, flat.size // 40)):
            orig = flat[i]
            flat[i] = orig + eps
            lp = _fd_scene_loss(sb, arrays, pose, intr, target, E)
            flat[i] = orig - eps
            lm = _fd_scene_loss(sb, arrays, pose, intr, target, E)
            flat[i] = orig
            fd = (lp - lm) / (2 * eps)
            a = float(an.reshape(-1)[i])
            diff = abs(a - fd)
            err = 0.0 if diff <= 1e-7 else diff / max(abs(a), abs(fd), 1e-7)
            worst = max(worst, err)
    # exposure gradient
    for i in range(12):
        Ep, Em = E.copy(), E.copy()
        Ep.reshape(-1)[i] += eps
        Em.reshape(-1)[i] -= eps
        fd = (_fd_scene_loss(sb, arrays, pose, intr, target, Ep)
              - _fd_scene_loss(sb, arrays, pose, intr, target, Em)) / (2 * eps)
        a = float(d_E.reshape(-1)[i])
        diff = abs(a - fd)
        worst = max(worst, 0.0 if diff <= 1e-7 else diff / max(abs(a), abs(fd), 1e-7))
    assert worst <= 1e-4, worst
    del torch
