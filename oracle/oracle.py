"""CPU oracle for the Gaussian-LIC mapping hot path -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end over ``oracle/splat_oracle.c`` (a scalar C
restatement of the reference package ``splatmap``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import
this module; the product package ``paper_2404_06926_b200`` never does, and its
CUDA path fails loudly when its own extension is missing.

Every function cites the reference file:line it restates.  Arrays are plain
numpy, in the reference's layouts, dtype float32 or float64.

Parity pinned: ``tests/test_oracle_golden.py`` checks this module against
golden vectors recorded from the reference itself (``tests/golden/``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")

ALPHA_CUTOFF = 1.0 / 255.0
ALPHA_CLAMP = 0.99
TERMINATION_THRESHOLD = 1e-4
BETA1, BETA2, EPS = 0.9, 0.999, 1e-15


class OCam(C.Structure):
    _fields_ = [("W", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


@dataclass
class Camera:
    """Pose (world->camera, scene.py:67-80) + intrinsics (scene.py:51-64)."""

    W: np.ndarray
    t: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def struct(self) -> OCam:
        s = OCam()
        s.W[:] = [float(v) for v in np.asarray(self.W, np.float64).reshape(9)]
        s.t[:] = [float(v) for v in np.asarray(self.t, np.float64).reshape(3)]
        s.fx, s.fy, s.cx, s.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        s.width, s.height = int(self.width), int(self.height)
        return s

    def center(self) -> np.ndarray:
        W = np.asarray(self.W, np.float64)
        return -W.T @ np.asarray(self.t, np.float64)


def build(force: bool = False) -> None:
    """Compile the oracle libraries with the committed Makefile."""
    libs = [os.path.join(_BUILD, f"liboracle_{s}.so") for s in ("f32", "f64")]
    src = os.path.join(_HERE, "splat_oracle.c")
    if not force and all(os.path.exists(p) and os.path.getmtime(p) >= os.path.getmtime(src)
                         for p in libs):
        return
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_LIBS: dict = {}


def _lib(dtype):
    key = "f64" if np.dtype(dtype) == np.float64 else "f32"
    if key not in _LIBS:
        build()
        _LIBS[key] = C.CDLL(os.path.join(_BUILD, f"liboracle_{key}.so"))
    return _LIBS[key], key


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's parallel blend (both precisions)."""
    for dt in (np.float32, np.float64):
        lib, k = _lib(dt)
        getattr(lib, f"oracle_set_threads_{k}")(C.c_int32(int(n)))


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# a1: frustum_mask (scene.py:283-298)
# --------------------------------------------------------------------------
def frustum_mask(cam: Camera, points, near=0.01, margin=0.1) -> np.ndarray:
    pts = np.asarray(points)
    dt = pts.dtype
    lib, k = _lib(dt)
    pts = _c(pts, dt)
    out = np.zeros(pts.shape[0], np.uint8)
    s = cam.struct()
    getattr(lib, f"oracle_frustum_mask_{k}")(C.c_int64(pts.shape[0]), _p(pts), C.byref(s),
                                             C.c_double(near), C.c_double(margin), _p(out))
    return out.astype(bool)


# --------------------------------------------------------------------------
# a2: project_gaussians (projection.py:307-392) -> compacted screen dict
# --------------------------------------------------------------------------
SCREEN_FIELDS = ("mean2d", "cov2d", "inv_cov2d", "depth", "color", "opacity", "t_cam",
                 "t_clamped", "clamped_x", "clamped_y", "view_dir", "basis", "color_raw",
                 "radius_cut", "q_cut", "source_index")


def project(positions, log_scales, rotations, opacity_logits, sh_coeffs, cam: Camera,
            near=0.01, dilation=0.3, select=None) -> dict:
    dt = np.asarray(positions).dtype
    lib, k = _lib(dt)
    n = int(np.asarray(positions).shape[0])
    pos = _c(positions, dt)
    ls = _c(log_scales, dt)
    rot = _c(rotations, dt)
    ol = _c(opacity_logits, dt)
    sh = _c(sh_coeffs, dt)
    sel = None
    if select is not None:
        select = np.asarray(select)
        if select.dtype == bool:
            sel = select.astype(np.uint8)
        else:
            sel = np.zeros(n, np.uint8)
            sel[select] = 1
    o = {
        "valid": np.zeros(n, np.uint8), "mean2d": np.zeros((n, 2), dt),
        "cov2d": np.zeros((n, 2, 2), dt), "inv_cov2d": np.zeros((n, 2, 2), dt),
        "depth": np.zeros(n, dt), "color": np.zeros((n, 3), dt), "opacity": np.zeros(n, dt),
        "t_cam": np.zeros((n, 3), dt), "t_clamped": np.zeros((n, 3), dt),
        "clamped_x": np.zeros(n, np.uint8), "clamped_y": np.zeros(n, np.uint8),
        "view_dir": np.zeros((n, 3), dt), "basis": np.zeros((n, 16), dt),
        "color_raw": np.zeros((n, 3), dt), "radius_cut": np.zeros(n, dt),
        "q_cut": np.zeros(n, dt),
    }
    s = cam.struct()
    getattr(lib, f"oracle_project_{k}")(
        C.c_int64(n), _p(pos), _p(ls), _p(rot), _p(ol), _p(sh),
        _p(sel) if sel is not None else None, C.byref(s), C.c_double(near),
        C.c_double(dilation), _p(o["valid"]), _p(o["mean2d"]), _p(o["cov2d"]),
        _p(o["inv_cov2d"]), _p(o["depth"]), _p(o["color"]), _p(o["opacity"]), _p(o["t_cam"]),
        _p(o["t_clamped"]), _p(o["clamped_x"]), _p(o["clamped_y"]), _p(o["view_dir"]),
        _p(o["basis"]), _p(o["color_raw"]), _p(o["radius_cut"]), _p(o["q_cut"]))
    idx = np.nonzero(o.pop("valid"))[0]
    screen = {f: v[idx] for f, v in o.items()}
    screen["clamped_x"] = screen["clamped_x"].astype(bool)
    screen["clamped_y"] = screen["clamped_y"].astype(bool)
    screen["source_index"] = idx.astype(np.int64)
    return screen


# --------------------------------------------------------------------------
# a3: bin_and_sort (forward.py:184-255) -> (pair_gaussian, pair_tile, offsets)
# --------------------------------------------------------------------------
def bin_and_sort(screen: dict, width: int, height: int, tile_size: int = 16, cull: bool = True):
    mean2d = np.asarray(screen["mean2d"])
    dt = mean2d.dtype
    lib, k = _lib(dt)
    m = mean2d.shape[0]
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    args = [_c(screen["mean2d"], dt), _c(np.asarray(screen["inv_cov2d"]).reshape(-1, 4), dt),
            _c(screen["depth"], dt), _c(screen["radius_cut"], dt), _c(screen["q_cut"], dt)]
    fn = getattr(lib, f"oracle_bin_{k}")
    fn.restype = C.c_int64
    offsets = np.zeros(tiles_x * tiles_y + 1, np.int64)
    cap = 0
    dummy = np.zeros(1, np.int64)
    total = fn(C.c_int64(m), *[_p(a) for a in args], C.c_int32(width), C.c_int32(height),
               C.c_int32(tile_size), C.c_int32(int(cull)), C.c_int64(cap), _p(dummy), _p(dummy),
               _p(offsets))
    pg = np.zeros(max(total, 1), np.int64)
    pt = np.zeros(max(total, 1), np.int64)
    total2 = fn(C.c_int64(m), *[_p(a) for a in args], C.c_int32(width), C.c_int32(height),
                C.c_int32(tile_size), C.c_int32(int(cull)), C.c_int64(total), _p(pg), _p(pt),
                _p(offsets))
    assert total2 == total
    return pg[:total], pt[:total], offsets


# --------------------------------------------------------------------------
# a4: render / _composite_tiles (forward.py:261-368)
# --------------------------------------------------------------------------
def composite(pair_gaussian, offsets, screen: dict, width: int, height: int, tile_size: int = 16,
              early_termination: bool = True, term_threshold: float = TERMINATION_THRESHOLD) -> dict:
    dt = np.asarray(screen["mean2d"]).dtype
    lib, k = _lib(dt)
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    out_c = np.zeros((height, width, 3), dt)
    out_d = np.zeros((height, width), dt)
    out_t = np.ones((height, width), dt)
    out_nc = np.zeros((height, width), np.int32)
    pg = _c(pair_gaussian, np.int64)
    off = _c(offsets, np.int64)
    f = [_c(screen["mean2d"], dt), _c(np.asarray(screen["inv_cov2d"]).reshape(-1, 4), dt),
         _c(screen["color"], dt), _c(screen["opacity"], dt), _c(screen["depth"], dt),
         _c(screen["q_cut"], dt), _c(screen["radius_cut"], dt)]
    getattr(lib, f"oracle_composite_{k}")(
        _p(pg), _p(off), C.c_int32(tiles_x), C.c_int32(tiles_y), C.c_int32(tile_size),
        C.c_int32(width), C.c_int32(height), *[_p(a) for a in f], C.c_int32(int(early_termination)),
        C.c_double(term_threshold), _p(out_c), _p(out_d), _p(out_t), _p(out_nc))
    one = dt.type(1)
    return {"color": out_c, "depth": out_d, "transmittance": out_t, "opacity": one - out_t,
            "n_contrib": out_nc}


# --------------------------------------------------------------------------
# a6: _backward_tiles (backward.py:91-213) -> per-row screen adjoints
# --------------------------------------------------------------------------
def backward_tiles(pair_gaussian, offsets, screen: dict, d_color_image, c_final, width: int,
                   height: int, tile_size: int = 16, early_termination: bool = True,
                   term_threshold: float = TERMINATION_THRESHOLD) -> dict:
    dt = np.asarray(screen["mean2d"]).dtype
    lib, k = _lib(dt)
    m = np.asarray(screen["mean2d"]).shape[0]
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    out = {"d_mean2d": np.zeros((m, 2), dt), "d_conic": np.zeros((m, 3), dt),
           "d_opacity": np.zeros(m, dt), "d_color": np.zeros((m, 3), dt)}
    f = [_c(screen["mean2d"], dt), _c(np.asarray(screen["inv_cov2d"]).reshape(-1, 4), dt),
         _c(screen["color"], dt), _c(screen["opacity"], dt), _c(screen["radius_cut"], dt),
         _c(screen["q_cut"], dt), _c(d_color_image, dt), _c(c_final, dt)]
    getattr(lib, f"oracle_backward_tiles_{k}")(
        _p(_c(pair_gaussian, np.int64)), _p(_c(offsets, np.int64)), C.c_int32(tiles_x),
        C.c_int32(tiles_y), C.c_int32(tile_size), C.c_int32(width), C.c_int32(height),
        *[_p(a) for a in f], C.c_int32(int(early_termination)), C.c_double(term_threshold),
        _p(out["d_mean2d"]), _p(out["d_conic"]), _p(out["d_opacity"]), _p(out["d_color"]))
    return out


# --------------------------------------------------------------------------
# a7: _chain_to_parameters (backward.py:415-500) -> GradientBuffer dict
# --------------------------------------------------------------------------
def chain(adj: dict, screen: dict, gmap: dict, cam: Camera) -> dict:
    dt = np.asarray(gmap["positions"]).dtype
    lib, k = _lib(dt)
    n = np.asarray(gmap["positions"]).shape[0]
    m = np.asarray(screen["mean2d"]).shape[0]
    g = {"d_position": np.zeros((n, 3), dt), "d_log_scale": np.zeros((n, 3), dt),
         "d_rotation": np.zeros((n, 4), dt), "d_opacity_logit": np.zeros(n, dt),
         "d_sh": np.zeros((n, 16, 3), dt)}
    s = cam.struct()
    args = [_c(screen["source_index"], np.int64), _c(gmap["positions"], dt),
            _c(gmap["log_scales"], dt), _c(gmap["rotations"], dt), _c(gmap["sh_coeffs"], dt),
            _c(np.asarray(screen["inv_cov2d"]).reshape(-1, 4), dt), _c(screen["t_cam"], dt),
            _c(screen["t_clamped"], dt), _c(screen["clamped_x"], np.uint8),
            _c(screen["clamped_y"], np.uint8), _c(screen["view_dir"], dt), _c(screen["basis"], dt),
            _c(screen["color_raw"], dt), _c(screen["opacity"], dt), _c(adj["d_mean2d"], dt),
            _c(np.asarray(adj["d_conic"]).reshape(m, -1), dt), _c(adj["d_opacity"], dt),
            _c(adj["d_color"], dt)]
    if args[15].shape[1] == 4:   # (M,2,2) symmetric -> (aa, ab, cc)
        args[15] = _c(args[15][:, [0, 1, 3]], dt)
    getattr(lib, f"oracle_chain_{k}")(
        C.c_int64(m), *[_p(a) for a in args], C.byref(s), _p(g["d_position"]),
        _p(g["d_log_scale"]), _p(g["d_rotation"]), _p(g["d_opacity_logit"]), _p(g["d_sh"]))
    return g


# --------------------------------------------------------------------------
# a5: photometric_loss (loss.py:143-177)
# --------------------------------------------------------------------------
def photometric_loss(rendered, ground_truth, E, lam=0.2):
    rendered = np.asarray(rendered)
    if rendered.shape != np.asarray(ground_truth).shape:
        raise ValueError("shape mismatch")
    dt = rendered.dtype
    lib, k = _lib(dt)
    h, w, _ = rendered.shape
    r = _c(rendered, dt)
    gt = _c(ground_truth, dt)
    Em = _c(np.asarray(E, np.float64).reshape(3, 4), np.float64)
    parts = np.zeros(4, np.float64)
    d_r = np.zeros_like(r)
    d_E = np.zeros((3, 4), np.float64)
    getattr(lib, f"oracle_loss_{k}")(C.c_int32(h), C.c_int32(w), _p(r), _p(gt), _p(Em),
                                     C.c_double(lam), _p(parts), _p(d_r), _p(d_E))
    return (float(parts[0]), d_r, d_E.astype(dt),
            {"l1": float(parts[1]), "dssim": float(parts[2]), "ssim": float(parts[3])})


def apply_exposure(E, color_image):
    """loss.py:31-36: Y = C M^T + b, no clamp."""
    img = np.asarray(color_image)
    dt = img.dtype
    M = np.asarray(E, np.float64)[:, :3].astype(dt)
    b = np.asarray(E, np.float64)[:, 3].astype(dt)
    return img @ M.T + b


# --------------------------------------------------------------------------
# a8/a9: adam_step (adam.py:76-122) and ScalarAdam (adam.py:125-140)
# --------------------------------------------------------------------------
GROUPS = ("position", "log_scale", "rotation", "opacity_logit", "sh")


def adam_step(params: dict, grads: dict, m: dict, v: dict, steps: np.ndarray, lrs: dict,
              active=None) -> None:
    """In place; ``active`` None (dense), bool mask or index array."""
    dt = params["position"].dtype
    lib, k = _lib(dt)
    n = steps.shape[0]
    mask = None
    if active is not None:
        a = np.asarray(active)
        mask = np.zeros(n, np.uint8)
        if a.dtype == bool:
            mask[:] = a
        else:
            mask[a] = 1
    widths = np.array([3, 3, 4, 1, 48], np.int32)
    lr_first = np.array([lrs["position"], lrs["log_scale"], lrs["rotation"],
                         lrs["opacity_logit"], lrs["sh0"]], np.float64)
    lr_rest = np.array([lrs["position"], lrs["log_scale"], lrs["rotation"],
                        lrs["opacity_logit"], lrs["sh_rest"]], np.float64)
    first_len = np.array([3, 3, 4, 1, 3], np.int32)
    for d in (params, m, v):
        for gname in GROUPS:
            assert d[gname].flags.c_contiguous and d[gname].dtype == dt
    gr = {gname: _c(grads[gname], dt) for gname in GROUPS}
    P = (C.c_void_p * 5)(*[d.ctypes.data for d in (params[g] for g in GROUPS)])
    G = (C.c_void_p * 5)(*[gr[g].ctypes.data for g in GROUPS])
    M1 = (C.c_void_p * 5)(*[m[g].ctypes.data for g in GROUPS])
    M2 = (C.c_void_p * 5)(*[v[g].ctypes.data for g in GROUPS])
    assert steps.dtype == np.int64 and steps.flags.c_contiguous
    getattr(lib, f"oracle_adam_{k}")(C.c_int64(n), C.c_int32(5), P, G, M1, M2, _p(widths),
                                     _p(lr_first), _p(lr_rest), _p(first_len), _p(steps),
                                     _p(mask) if mask is not None else None)


class ScalarAdam:
    """adam.py:125-140, float64."""

    def __init__(self, shape, lr):
        self.lr = lr
        self.m = np.zeros(shape)
        self.v = np.zeros(shape)
        self.t = 0

    def step(self, param, grad):
        self.t += 1
        self.m = BETA1 * self.m + (1 - BETA1) * grad
        self.v = BETA2 * self.v + (1 - BETA2) * grad * grad
        mh = self.m / (1 - BETA1 ** self.t)
        vh = self.v / (1 - BETA2 ** self.t)
        param -= self.lr * mh / (np.sqrt(vh) + EPS)


# --------------------------------------------------------------------------
# a10: Mapper._optimize_step (mapper.py:299-328), whole step on the oracle
# --------------------------------------------------------------------------
def render_view(gmap: dict, cam: Camera, near=0.01, tile_size=16, early_termination=True,
                include_sky=True):
    """mapper.py:202-212."""
    select = None if include_sky else ~np.asarray(gmap["is_sky"], bool)
    screen = project(gmap["positions"], gmap["log_scales"], gmap["rotations"],
                     gmap["opacity_logits"], gmap["sh_coeffs"], cam, near=near, select=select)
    pg, pt, off = bin_and_sort(screen, cam.width, cam.height, tile_size)
    targets = composite(pg, off, screen, cam.width, cam.height, tile_size, early_termination)
    return screen, (pg, pt, off), targets


def optimize_step(gmap: dict, adam: dict, lrs: dict, cam: Camera, image, E, exposure_opt=None,
                  lam=0.2, near=0.01, margin=0.1, tile_size=16) -> dict:
    """One reference mapping iteration; mutates gmap/adam/E in place."""
    dt = gmap["positions"].dtype
    screen, (pg, pt, off), targets = render_view(gmap, cam, near, tile_size)
    E_used = np.asarray(E) if E is not None else np.concatenate([np.eye(3), np.zeros((3, 1))], 1)
    loss, d_r, d_E, parts = photometric_loss(targets["color"], np.asarray(image).astype(dt),
                                             E_used, lam)
    adj = backward_tiles(pg, off, screen, d_r, targets["color"], cam.width, cam.height, tile_size)
    grads = chain(adj, screen, gmap, cam)
    active = frustum_mask(cam, gmap["positions"], near, margin)
    params = {"position": gmap["positions"], "log_scale": gmap["log_scales"],
              "rotation": gmap["rotations"], "opacity_logit": gmap["opacity_logits"],
              "sh": gmap["sh_coeffs"]}
    g = {"position": grads["d_position"], "log_scale": grads["d_log_scale"],
         "rotation": grads["d_rotation"], "opacity_logit": grads["d_opacity_logit"],
         "sh": grads["d_sh"]}
    adam_step(params, g, adam["m"], adam["v"], adam["steps"], lrs, active=active)
    if E is not None and exposure_opt is not None:
        exposure_opt.step(E, d_E)
    return {"loss": loss, **parts, "n_pairs": int(pg.shape[0]), "n_active": int(active.sum()),
            "n_visible": int(screen["source_index"].shape[0])}
