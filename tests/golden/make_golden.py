"""Generate golden vectors from the REFERENCE implementation (splatmap).

Run in the build container only (the reference lives at /root/reference and
does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py

Each scene is recorded as ``tests/golden/<name>.npz`` holding the inputs (map
arrays, camera, target image, exposure, learning rates) and the reference's
outputs for every hot-path stage, produced by calling the reference functions
exactly as ``Mapper._optimize_step`` does (mapper.py:299-328):

  frustum mask        scene.frustum_mask          (scene.py:283-298)
  SplatScreen         projection.project_gaussians (projection.py:307-392)
  TileGrid            forward.bin_and_sort        (forward.py:184-255)
  RenderTargets       forward.render              (forward.py:345-368)
  loss / dC / dE      loss.photometric_loss       (loss.py:143-177)
  pair adjoints       backward._pixel_stage_per_gaussian (backward.py:216-244)
  GradientBuffer      backward.backward_per_gaussian     (backward.py:516-527)
  Adam + exposure     mapper.Mapper._optimize_step       (mapper.py:299-328)

The scene recipes follow SURVEY.md §8(d) (build_view_map, bench.py:20-44, with
per-axis anisotropy and small higher-order SH) at sizes the CPU oracle runs in
well under a second, plus the reference test-suite scene builders
(helpers.random_map, gradcheck.build_gradcheck_scene).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from splatmap import adam as ref_adam  # noqa: E402
from splatmap import backward as ref_bwd  # noqa: E402
from splatmap import forward as ref_fwd  # noqa: E402
from splatmap import loss as ref_loss  # noqa: E402
from splatmap import mapper as ref_mapper  # noqa: E402
from splatmap import projection as ref_proj  # noqa: E402
from splatmap import scene as ref_scene  # noqa: E402
from splatmap.gradcheck import build_gradcheck_scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def view_map(rng, n, width, height, f, depth=(4.0, 12.0), sigma_px=(3.0, 9.0),
             opacity=(0.55, 0.95), v_frac=(0.0, 1.0), aniso=(0.7, 1.4), sh_rest=0.05,
             dtype=np.float32):
    """build_view_map recipe (bench.py:20-44) + SURVEY §8(d) anisotropy."""
    cx, cy = width / 2, height / 2
    z = rng.uniform(*depth, n)
    u = rng.uniform(0, width - 1, n)
    v = rng.uniform(v_frac[0] * (height - 1), v_frac[1] * (height - 1), n)
    x = (u - cx) * z / f
    y = (v - cy) * z / f
    pos = np.stack([x, y, z], axis=1)
    sig = rng.uniform(*sigma_px, n)
    s_world = sig * z / f
    ls = np.log(np.repeat(s_world[:, None], 3, axis=1)) + np.log(rng.uniform(*aniso, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ops = np.array([ref_proj.logit(o) for o in rng.uniform(*opacity, n)])
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = rng.uniform(-1.0, 1.5, (n, 3))
    sh[:, 1:, :] = rng.normal(0.0, sh_rest, (n, 15, 3))
    return [a.astype(dtype) for a in (pos, ls, q, ops, sh)] + [np.zeros(n, bool)]


def sky(rng, count, radius, dtype=np.float32):
    cfg = ref_mapper.MapperConfig(sky_count=count, sky_radius=radius)
    arrs = ref_mapper._sky_arrays(cfg, rng)
    return [np.asarray(a).astype(dtype) for a in arrs[:5]] + [np.ones(count, bool)]


def cat(a, b):
    return [np.concatenate([x, y]) for x, y in zip(a, b)]


def record(name, arrays, pose, intr, image, E, lam=0.2, exposure=True, margin=0.1,
           near=0.01, lrs=None, extra_bin=False):
    pos, ls, rot, op, sh, is_sky = arrays
    dt = pos.dtype
    gmap = ref_scene.GaussianMap(capacity=max(len(pos), 1), dtype=dt)
    gmap.append_arrays(pos, ls, rot, op, sh, is_sky)
    out = {"positions": pos, "log_scales": ls, "rotations": rot, "opacity_logits": op,
           "sh_coeffs": sh, "is_sky": is_sky, "W": pose.rotation_wc, "t": pose.translation_wc,
           "intr": np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], np.float64),
           "image": image, "E": E.matrix.copy(), "lam": np.float64(lam),
           "near": np.float64(near), "margin": np.float64(margin)}
    # --- stages, exactly as _optimize_step -> render_view ---------------
    screen = ref_proj.project_gaussians(pos, ls, rot, op, sh, pose, intr, near=near)
    grid = ref_fwd.bin_and_sort(screen, intr)
    targets = ref_fwd.render(grid, screen, intr)
    loss, d_r, d_E, parts = ref_loss.photometric_loss(targets.color, image.astype(dt), E, lam)
    acc = ref_bwd._pixel_stage_per_gaussian(targets, d_r, screen, grid, intr, True, 1e-4)
    buf = ref_bwd.backward_per_gaussian(targets, d_r, screen, grid, gmap, pose, intr)
    mask = ref_scene.frustum_mask(pose, intr, pos, near=near, margin=margin)
    for f in ("mean2d", "cov2d", "inv_cov2d", "depth", "color", "opacity", "source_index",
              "t_cam", "t_clamped", "clamped_x", "clamped_y", "view_dir", "basis", "color_raw",
              "radius_cut", "q_cut"):
        out[f"screen_{f}"] = getattr(screen, f)
    out["pair_gaussian"] = grid.pair_gaussian.astype(np.int32)
    out["pair_tile"] = grid.pair_tile.astype(np.int32)
    out["offsets"] = grid.offsets.astype(np.int64)
    if extra_bin:
        g_off = ref_fwd.bin_and_sort(screen, intr, cull=False)
        out["nocull_pair_gaussian"] = g_off.pair_gaussian.astype(np.int32)
        out["nocull_offsets"] = g_off.offsets.astype(np.int64)
        t_noterm = ref_fwd.render(grid, screen, intr, early_termination=False)
        out["noterm_color"] = t_noterm.color
        out["refrender_color"] = ref_fwd.reference_render(screen, intr).color
    out["color"] = targets.color
    out["depth"] = targets.depth
    out["transmittance"] = targets.transmittance
    out["n_contrib"] = targets.n_contrib
    out["loss"] = np.array([loss, parts["l1"], parts["dssim"], parts["ssim"]], np.float64)
    out["d_rendered"] = d_r
    out["d_E"] = d_E
    out["adj_mean2d"] = acc.d_mean2d
    out["adj_conic"] = acc.d_conic
    out["adj_opacity"] = acc.d_opacity
    out["adj_color"] = acc.d_color
    for f in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        out[f"grad_{f}"] = getattr(buf, f)
    out["frustum"] = mask
    # --- the literal reference step: Mapper._optimize_step --------------
    cfg = ref_mapper.MapperConfig(sky_enabled=False, exposure_mode="per_keyframe"
                                  if exposure else "off", loss_lambda=lam, near=near,
                                  frustum_margin=margin, scene_extent=1.0)
    mp = ref_mapper.Mapper(cfg, seed=0, dtype=dt)
    mp.map = gmap
    mp.scene_extent = 1.0
    lr = mp._lrs() if lrs is None else lrs
    mp.adam = ref_adam.AdamState(gmap.count, lr, dtype=dt)
    out["lrs"] = np.array([lr["position"], lr["log_scale"], lr["rotation"], lr["opacity_logit"],
                           lr["sh0"], lr["sh_rest"]], np.float64)
    frame = ref_scene.CameraFrame(pose=pose, intrinsics=intr, image=image, frame_index=0,
                                  is_keyframe=True)
    entry = ref_mapper.KeyframeEntry(frame, ref_loss.ExposureAffine(E.matrix.copy()),
                                     ref_adam.ScalarAdam((3, 4), cfg.lr_exposure))
    log = mp._optimize_step(entry)
    out["step_loss"] = np.float64(log["loss"])
    out["step_psnr"] = np.float64(log["psnr"])
    out["after_positions"] = gmap.positions
    out["after_log_scales"] = gmap.log_scales
    out["after_rotations"] = gmap.rotations
    out["after_opacity_logits"] = gmap.opacity_logits
    out["after_sh_coeffs"] = gmap.sh_coeffs
    out["after_steps"] = mp.adam.steps
    out["after_m_position"] = mp.adam.m["position"]
    out["after_v_sh"] = mp.adam.v["sh"]
    out["after_E"] = entry.exposure.matrix
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: N={len(pos)} M={len(screen)} P={grid.n_pairs} loss={loss:.6f}")


def intrinsics(width, height, f):
    return ref_scene.CameraIntrinsics(fx=f, fy=f, cx=width / 2, cy=height / 2, width=width,
                                      height=height)


def main():
    from helpers import random_map

    # 1. the reference test-suite scene (helpers.random_map), f32 and f64
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        rng = np.random.default_rng(77)
        m = random_map(rng, 300, dtype=dt)
        arrays = [m.positions, m.log_scales, m.rotations, m.opacity_logits, m.sh_coeffs, m.is_sky]
        intr = intrinsics(64, 64, 64)
        img = np.random.default_rng(1).uniform(0, 1, (64, 64, 3))
        E = ref_loss.ExposureAffine.identity()
        E.matrix = E.matrix + np.random.default_rng(2).normal(0, 0.02, (3, 4))
        record(f"random64_{tag}", arrays, ref_scene.CameraPose.identity(), intr, img, E,
               extra_bin=True)

    # 2. the gradcheck scene (gradcheck.py:36-65), f64, 24x24
    sc = build_gradcheck_scene(0, n_gaussians=12)
    m = sc.gmap
    record("gradcheck_f64", [m.positions, m.log_scales, m.rotations, m.opacity_logits,
                             m.sh_coeffs, m.is_sky], sc.pose, sc.intr, sc.target, sc.exposure)

    # 3. config-1 recipe at reduced size: 4000 Gaussians, 160x120, f=125
    rng = np.random.default_rng(0)
    intr = intrinsics(160, 120, 125.0)
    arrays = view_map(rng, 4000, 160, 120, 125.0)
    img = np.random.default_rng(1).uniform(0, 1, (120, 160, 3))
    E = ref_loss.ExposureAffine.identity()
    E.matrix = E.matrix + np.random.default_rng(2).normal(0, 0.02, (3, 4))
    record("view160_f32", arrays, ref_scene.CameraPose.identity(), intr, img, E)

    # 4. config-3 recipe at reduced size: 3000 fg in the lower 65% + 1000 sky
    #    (radius 1e4), 200x112 (partial tiles on both axes), exposure on,
    #    a rotated + translated pose
    rng = np.random.default_rng(3)
    intr = intrinsics(200, 112, 150.0)
    fg = view_map(rng, 3000, 200, 112, 150.0, v_frac=(0.35, 1.0))
    sk = sky(np.random.default_rng(1), 1000, 1e4)
    arrays = cat(fg, sk)
    img = np.random.default_rng(1).uniform(0, 1, (112, 200, 3))
    E = ref_loss.ExposureAffine.identity()
    E.matrix = E.matrix + np.random.default_rng(2).normal(0, 0.02, (3, 4))
    # pose: small rotation about y and x, camera moved; world->camera
    ang = 0.05
    Ry = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    Rx = np.array([[1, 0, 0], [0, np.cos(-ang), -np.sin(-ang)], [0, np.sin(-ang), np.cos(-ang)]])
    pose = ref_scene.CameraPose(Rx @ Ry, np.array([0.1, -0.05, 0.2]))
    record("sky200_f32", arrays, pose, intr, img, E)

    # 5. slim-Gaussian culling stress (bench_culling recipe, bench.py:113-145)
    rng = np.random.default_rng(5)
    intr = intrinsics(128, 96, 104.0)
    arrays = view_map(rng, 2000, 128, 96, 104.0, sigma_px=(0.8, 2.0), aniso=(1.0, 1.0))
    arrays[1][:, 0] += np.float32(np.log(30.0))
    img = np.random.default_rng(1).uniform(0, 1, (96, 128, 3))
    record("slim128_f32", arrays, ref_scene.CameraPose.identity(), intr, img,
           ref_loss.ExposureAffine.identity(), extra_bin=True)

    # 6. deep stack that terminates everywhere (test_backward.py:179-211 shape),
    #    odd image size 50x37
    rng = np.random.default_rng(21)
    intr = intrinsics(50, 37, 40.0)
    n = 40
    z = 2.0 + 0.25 * np.arange(n)
    pos = np.stack([rng.uniform(-0.2, 0.2, n) * z, rng.uniform(-0.2, 0.2, n) * z, z], 1)
    ls = np.log(np.repeat((60.0 * z / 40.0)[:, None], 3, 1)) + np.log(rng.uniform(0.7, 1.4, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = np.full(n, ref_proj.logit(0.85))
    sh = rng.normal(0, 0.3, (n, 16, 3))
    arrays = [a.astype(np.float32) for a in (pos, ls, q, op, sh)] + [np.zeros(n, bool)]
    img = np.random.default_rng(1).uniform(0, 1, (37, 50, 3))
    record("stack50_f32", arrays, ref_scene.CameraPose.identity(), intr, img,
           ref_loss.ExposureAffine.identity())


if __name__ == "__main__":
    main()
