"""Parity comparators shared by the CPU (oracle-vs-golden) and GPU
(CUDA-vs-oracle) tests.  Tolerances follow BASELINE.json's north star and
SURVEY.md §8(c):

* integer work (culling masks, tile keys, pair order, tile ranges): bit-exact
  on identical float inputs;
* rendered colour within 1e-4 max-abs; depth within 1e-4 relative to the
  frame's maximum depth (sky depths reach ~1e4 m);
* Gaussian and exposure gradients within 1e-3 relative / 1e-5 absolute per
  element, and normwise max|d| / max|ref| <= 1e-3 per group.

Pixels over tolerance are allowed only when they are EXPLAINED by a hard
decision flip (alpha at the 1/255 cutoff or the 0.99 clamp, q at q_cut+1/64,
T at the termination threshold): ``explain_pixels`` replays each one in
float64 and returns those no contributor explains (they fail);
``explained_pixel_budget`` bounds how many explained pixels a frame may have.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")

COLOR_TOL = 1e-4
DEPTH_REL_TOL = 1e-4
GRAD_RTOL = 1e-3
GRAD_ATOL = 1e-5


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def oracle():
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    from oracle import oracle as o  # noqa: WPS433 - test infrastructure
    return o


def camera_from(g):
    o = oracle()
    fx, fy, cx, cy, w, h = g["intr"]
    return o.Camera(W=g["W"], t=g["t"], fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))


def screen_from(g):
    return {k[len("screen_"):]: v for k, v in g.items() if k.startswith("screen_")}


def gmap_from(g, prefix=""):
    return {"positions": g[prefix + "positions"], "log_scales": g[prefix + "log_scales"],
            "rotations": g[prefix + "rotations"], "opacity_logits": g[prefix + "opacity_logits"],
            "sh_coeffs": g[prefix + "sh_coeffs"], "is_sky": g.get("is_sky")}


def lrs_from(g):
    p, s, r, o, s0, sr = g["lrs"]
    return {"position": p, "log_scale": s, "rotation": r, "opacity_logit": o, "sh0": s0,
            "sh_rest": sr}


def max_abs(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max())


def assert_image_close(got, want, tol=COLOR_TOL, budget=0, what="color"):
    """Max-abs per pixel; at most ``budget`` pixels may exceed ``tol``
    (each must be a decision flip, checked by the caller's budget choice)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    err = np.abs(got - want)
    if err.ndim == 3:
        err = err.max(axis=2)
    bad = int((err > tol).sum())
    assert bad <= budget, f"{what}: {bad} pixels over {tol} (budget {budget}); max {err.max():.3e}"
    return bad, float(err.max()) if err.size else 0.0


def assert_depth_close(got, want, budget=0):
    scale = max(float(np.abs(want).max()), 1.0)
    return assert_image_close(np.asarray(got) / scale, np.asarray(want) / scale,
                              DEPTH_REL_TOL, budget, "depth")


def grad_report(got, want):
    """(n elements failing the per-element contract, normwise ratio)."""
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    fail = np.abs(g - w) > GRAD_ATOL + GRAD_RTOL * np.abs(w)
    scale = max(float(np.abs(w).max()), 1e-30)
    return int(fail.sum()), float(np.abs(g - w).max() / scale) if g.size else 0.0


def assert_grads_close(got, want, what, max_fail=0, norm_tol=GRAD_RTOL):
    nfail, norm = grad_report(got, want)
    assert nfail <= max_fail and norm <= norm_tol, \
        f"{what}: {nfail} elements fail 1e-3 rel/1e-5 abs (allowed {max_fail}); normwise {norm:.3e}"
    return nfail, norm


def explain_pixels(pixels, pair_gaussian, offsets, screen, width, tile=16, early=True,
                   thresh=1e-4, k_rel=1e-5, k_rel_t=1e-4):
    """a pixel whose value differs between two
    implementations is EXPLAINED when one of its contributors sits at a hard
    decision of the blend (forward.py:277-333, the reference's thresholds):
    alpha_raw within k_rel of the 1/255 cutoff or of the 0.99 clamp, q within
    k_rel of q_cut + 1/64, the pixel on the edge of the Gaussian's radius
    box, or the transmittance in front of it within k_rel_t of the
    termination threshold (T is a product over the list: a 2-ulp exp moves it
    by up to ~n x 2.4e-7 relative after n contributors).  Replays each given (y, x) pixel in float64 along
    its tile's list; returns the pixels with no such contributor."""
    tiles_x = (width + tile - 1) // tile
    mean2d = np.asarray(screen["mean2d"], np.float64)
    inv = np.asarray(screen["inv_cov2d"], np.float64).reshape(-1, 4)
    opa = np.asarray(screen["opacity"], np.float64)
    qcut = np.asarray(screen["q_cut"], np.float64)
    rad = np.asarray(screen["radius_cut"], np.float64)
    cutoff, clamp, margin = 1.0 / 255.0, 0.99, 1.0 / 64.0
    near = lambda v, ref: abs(v - ref) <= k_rel * max(abs(ref), 1e-30)  # noqa: E731
    unexplained = []
    for y, x in np.asarray(pixels, np.int64).reshape(-1, 2):
        t = (y // tile) * tiles_x + x // tile
        T = 1.0
        hit = False
        for g in pair_gaussian[offsets[t]:offsets[t + 1]]:
            if early and abs(T - thresh) <= k_rel_t * thresh:
                hit = True          # termination decided within rounding of 1e-4
                break
            if early and T < thresh:
                break
            mx, my, r = mean2d[g, 0], mean2d[g, 1], rad[g]
            for edge in (mx - r, mx + r, my - r, my + r):
                if abs(edge - round(edge)) <= k_rel * max(1.0, abs(edge)):
                    if round(edge) in (x, y):
                        hit = True
            if not (np.ceil(mx - r) <= x <= np.floor(mx + r)
                    and np.ceil(my - r) <= y <= np.floor(my + r)):
                continue
            dx, dy = x - mx, y - my
            a, b, c = inv[g, 0], inv[g, 1], inv[g, 3]
            q = a * dx * dx + 2 * b * dx * dy + c * dy * dy
            qc = qcut[g] + margin
            if near(q, qc):
                hit = True
            if q > qc:
                continue
            ar = opa[g] * np.exp(-0.5 * q)
            if near(ar, cutoff) or near(ar, clamp):
                hit = True
            al = min(ar, clamp)
            if al < cutoff:
                continue
            T *= 1.0 - al
            if hit:
                break
        if not hit:
            unexplained.append((int(y), int(x)))
    return unexplained


def explained_pixel_budget(n_pixels, frac=2e-4, floor=4):
    """Decision flips are rare: the reference's own f32 and f64 renders differ
    on 4 of 307,200 pixels at config 2; allow ~7e-4 of that."""
    return max(floor, int(np.ceil(frac * n_pixels)))


def f64_truth_grads(g):
    """Float64 oracle gradients on the float64-cast reference inputs (screen,
    grid, render, dC): the 'truth' an f32 result is measured against.  The f64
    oracle is itself pinned to the reference's f64 mode (test_oracle_golden)."""
    o = oracle()
    cam = camera_from(g)
    up = lambda v: v.astype(np.float64) if v.dtype == np.float32 else v  # noqa: E731
    s64 = {k: up(v) for k, v in screen_from(g).items()}
    adj = o.backward_tiles(g["pair_gaussian"], g["offsets"], s64, up(g["d_rendered"]),
                           up(g["color"]), cam.width, cam.height)
    gm = {k: (up(v) if v is not None else None) for k, v in gmap_from(g).items()}
    return o.chain(adj, s64, gm, cam)


def normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)) if a.size else 0.0


def assert_grads_calibrated(got, ref32, truth, what, norm_tol=GRAD_RTOL):
    """Per element: 1e-3 rel / 1e-5 abs against the reference (no failures).
    Normwise: within ``norm_tol`` of the reference, OR -- where the
    reference's own float32 result is that far from the float64 truth (slim,
    ill-conditioned splats) -- no farther from the truth than 1.5x the
    reference's own error."""
    nfail, _ = grad_report(got, ref32)
    assert nfail == 0, f"{what}: {nfail} elements fail 1e-3 rel / 1e-5 abs"
    n_ref = normwise(got, ref32)
    if n_ref <= norm_tol:
        return
    e_got, e_ref = normwise(got, truth), normwise(ref32, truth)
    assert e_got <= max(norm_tol, 1.5 * e_ref), \
        f"{what}: normwise vs reference {n_ref:.2e}; vs f64 truth {e_got:.2e} (reference f32 {e_ref:.2e})"


MAP_GROUPS = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")


def assert_maps_identical(a_mp, b_mp):
    """Two mapping runs of the same iterations must agree BITWISE: the
    deterministic backward (sb_blend_bwd_det) merges every row's per-tile
    sums in tile order and the loss reduces its block sums in a fixed order,
    so no float summation order depends on scheduling, graph capture, the
    tile order or depth-limited vs full lists.  Compares the map, the Adam
    moments and the step counters."""
    import torch
    for name in MAP_GROUPS:
        x, y = getattr(a_mp.map, name), getattr(b_mp.map, name)
        assert torch.equal(x, y), (name, float((x.double() - y.double()).abs().max()))
    for g in a_mp.adam.m:
        assert torch.equal(a_mp.adam.m[g], b_mp.adam.m[g]), ("m", g)
        assert torch.equal(a_mp.adam.v[g], b_mp.adam.v[g]), ("v", g)
    assert torch.equal(a_mp.adam.steps, b_mp.adam.steps)


def assert_logs_identical(la, lb):
    assert len(la) == len(lb)
    for x, y in zip(la, lb):
        for k in ("loss", "l1", "dssim", "psnr"):
            assert x[k] == y[k], (k, x, y)
