"""Seeded synthetic scenes of BASELINE.json's configs.

Foreground splats follow the reference's build_view_map recipe (bench.py:20-44:
depth U[4,12] m, uniform screen position, sigma_px U[3,9], opacity U[.55,.95],
random unit quaternions, SH0 U[-1,1.5]) with the survey's per-axis anisotropy
U[0.7,1.4] and SH rows 1-15 ~ N(0, 0.05).  Config 3 adds the 100k-Gaussian
sky shell of init_sky (mapper.py:124-161, radius 1e4) seen by an identity
camera looking at the zenith, and restricts the foreground to the lower 65% of
the rows.  All draws are host numpy with fixed seeds.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _logit(p):
    return np.log(p) - np.log1p(-p)


def view_map(rng, n, width, height, f, depth=(4.0, 12.0), sigma_px=(3.0, 9.0),
             opacity=(0.55, 0.95), v_frac=(0.0, 1.0), aniso=(0.7, 1.4), sh_rest=0.05):
    cx, cy = width / 2, height / 2
    z = rng.uniform(*depth, n)
    u = rng.uniform(0, width - 1, n)
    v = rng.uniform(v_frac[0] * (height - 1), v_frac[1] * (height - 1), n)
    pos = np.stack([(u - cx) * z / f, (v - cy) * z / f, z], axis=1)
    s_world = rng.uniform(*sigma_px, n) * z / f
    ls = np.log(np.repeat(s_world[:, None], 3, axis=1)) + np.log(rng.uniform(*aniso, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ops = _logit(rng.uniform(*opacity, n))
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = rng.uniform(-1.0, 1.5, (n, 3))
    sh[:, 1:, :] = rng.normal(0.0, sh_rest, (n, 15, 3))
    return [pos, ls, q, ops, sh, np.zeros(n, bool)]


def sky_shell(count, radius, seed=1, opacity=0.7):
    """init_sky's draws (mapper.py:124-161)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    z = rng.uniform(0.0, 1.0, count) * radius
    phi = rng.uniform(0.0, 2.0 * np.pi, count)
    rxy = np.sqrt(np.maximum(radius * radius - z * z, 0.0))
    pos = np.stack([rxy * np.cos(phi), rxy * np.sin(phi), z], axis=1)
    dist, _ = cKDTree(pos).query(pos, k=2)
    scales = 1.1 * dist[:, 1]
    ls = np.repeat(np.log(scales)[:, None], 3, axis=1)
    rot = np.zeros((count, 4))
    rot[:, 0] = 1.0
    sh = np.zeros((count, 16, 3))
    sh[:, 0, :] = (1.0 - 0.5) / 0.28209479177387814
    ops = np.full(count, _logit(opacity))
    return [pos, ls, rot, ops, sh, np.ones(count, bool)]


@dataclass
class Scene:
    name: str
    arrays: list          # positions, log_scales, rotations, opacity_logits, sh_coeffs, is_sky
    W: np.ndarray
    t: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    image: np.ndarray     # ground truth (H, W, 3) float64
    E: np.ndarray         # exposure 3x4 float64
    exposure: bool

    @property
    def n(self) -> int:
        return self.arrays[0].shape[0]


def config(idx: int, dtype=np.float32) -> Scene:
    """BASELINE.json configs[idx-1] as concrete seeded inputs."""
    if idx == 1:
        n, w, h, sky = 10_000, 320, 240, 0
    elif idx == 2:
        n, w, h, sky = 100_000, 640, 480, 0
    elif idx == 3:
        n, w, h, sky = 900_000, 1280, 720, 100_000
    else:
        raise ValueError(f"config {idx} has no single-view synthetic scene")
    f = 500.0 * w / 640.0 if idx != 3 else 1000.0
    rng = np.random.default_rng(0)
    fg = view_map(rng, n, w, h, f, v_frac=(0.35, 1.0) if idx == 3 else (0.0, 1.0))
    arrays = fg
    if sky:
        sk = sky_shell(sky, 1e4)
        arrays = [np.concatenate([a, b]) for a, b in zip(fg, sk)]
    arrays = [a.astype(dtype) if a.dtype != bool else a for a in arrays]
    image = np.random.default_rng(1).uniform(0.0, 1.0, (h, w, 3))
    E = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) + np.random.default_rng(2).normal(
        0.0, 0.02, (3, 4))
    return Scene(f"config{idx}", arrays, np.eye(3), np.zeros(3), f, f, w / 2, h / 2, w, h,
                 image, E, exposure=True)


def look_at(position, target, up=(0.0, 0.0, 1.0)):
    """World-to-camera (R, t), z forward, x right, y down (sim.py:476-487)."""
    c = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - c
    fwd /= np.linalg.norm(fwd)
    x = np.cross(fwd, np.asarray(up, dtype=np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(fwd, x)
    r_wc = np.stack([x, y, fwd], axis=1).T
    return r_wc, -r_wc @ c


@dataclass
class View:
    W: np.ndarray
    t: np.ndarray
    image: np.ndarray     # ground truth (H, W, 3) float64
    E: np.ndarray         # exposure 3x4 float64


def ring_map(rng, n, f, radius=(6.0, 14.0), height=(-4.0, 4.0), sigma_px=(3.0, 9.0),
             opacity=(0.55, 0.95), aniso=(0.7, 1.4), sh_rest=0.05):
    """Config 5's foreground: a ring around the origin, radius
    U[6,14] m, height U[-4,4] m, sigma_px U[3,9] at the ring radius; the other
    attributes follow view_map."""
    r = rng.uniform(*radius, n)
    th = rng.uniform(0.0, 2.0 * np.pi, n)
    pos = np.stack([r * np.cos(th), r * np.sin(th), rng.uniform(*height, n)], axis=1)
    s_world = rng.uniform(*sigma_px, n) * r / f
    ls = np.log(np.repeat(s_world[:, None], 3, axis=1)) + np.log(rng.uniform(*aniso, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ops = _logit(rng.uniform(*opacity, n))
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = rng.uniform(-1.0, 1.5, (n, 3))
    sh[:, 1:, :] = rng.normal(0.0, sh_rest, (n, 15, 3))
    return [pos, ls, q, ops, sh, np.zeros(n, bool)]


def config5(n_fg: int = 3_900_000, sky: int = 100_000, n_views: int = 8, width: int = 1280,
            height: int = 720, f: float = 1000.0, dtype=np.float32):
    """BASELINE.json configs[4]: the 4M-Gaussian ring map plus the sky shell,
    seen by n_views cameras at the origin with yaw k*360/n_views degrees
    (look_at, up = +z).  Returns (Scene of view 0, [View] for every view)."""
    rng = np.random.default_rng(0)
    fg = ring_map(rng, n_fg, f)
    arrays = fg
    if sky:
        sk = sky_shell(sky, 1e4)
        arrays = [np.concatenate([a, b]) for a, b in zip(fg, sk)]
    arrays = [a.astype(dtype) if a.dtype != bool else a for a in arrays]
    views = []
    for k in range(n_views):
        yaw = 2.0 * np.pi * k / n_views
        R, t = look_at(np.zeros(3), np.array([np.cos(yaw), np.sin(yaw), 0.0]))
        image = np.random.default_rng(10 + k).uniform(0.0, 1.0, (height, width, 3))
        E = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) + np.random.default_rng(
            20 + k).normal(0.0, 0.02, (3, 4))
        views.append(View(R, t, image, E))
    v0 = views[0]
    scene = Scene("config5", arrays, v0.W, v0.t, f, f, width / 2, height / 2, width, height,
                  v0.image, v0.E, exposure=True)
    return scene, views


def default_lrs(scene_extent=1.0) -> dict:
    """MapperConfig defaults (mapper.py:48-54, 239-243)."""
    return {"position": 1.6e-4 * scene_extent, "log_scale": 5e-3, "rotation": 1e-3,
            "opacity_logit": 5e-2, "sh0": 2.5e-3, "sh_rest": 1.25e-4}
