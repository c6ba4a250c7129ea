"""The reference's own known-answer tests, on the GPU path.

Each test restates one of splatmap's unit tests (pkg/tests/*.py, cited per
test) against this package's device API with the reference's constants and
tolerances.  Scalar host helpers the reference exposes for its own tests
(covariance_3d, project_mean, project_covariance, alpha_weight, evaluate_sh)
are not part of the hot path; their KATs are checked through the batched
device calls that compute the same quantities (project_gaussians, render).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C0 = 0.28209479177387814


def _np(t):
    return t.detach().cpu().numpy()


def _sb():
    import paper_2404_06926_b200 as sb
    return sb


def _logit(p):
    return float(np.log(p) - np.log1p(-p))


def small_intrinsics(size=64, f=None):
    """helpers.py:37-40"""
    sb = _sb()
    f = f if f is not None else size
    return sb.CameraIntrinsics(f, f, size / 2, size / 2, size, size)


def splat_screen(mean2d, inv_cov2d, depth, color, opacity, dtype=np.float64):
    """A SplatScreen given directly in screen space (helpers.py:43-72's
    single_splat_screen: q_cut = 2 ln(255 o), radius from the largest
    covariance eigenvalue, inflated by (1 + 1e-5) and + 1e-3)."""
    sb = _sb()
    mean2d = np.atleast_2d(np.asarray(mean2d, dtype))
    n = mean2d.shape[0]
    inv = np.asarray(inv_cov2d, dtype).reshape(-1, 2, 2)
    if inv.shape[0] == 1 and n > 1:
        inv = np.repeat(inv, n, axis=0)
    cov = np.linalg.inv(inv)
    depth = np.atleast_1d(np.asarray(depth, dtype))
    color = np.atleast_2d(np.asarray(color, dtype))
    opacity = np.atleast_1d(np.asarray(opacity, dtype))
    lam = np.linalg.eigvalsh(cov).max(axis=1)
    q_cut = 2.0 * np.log(opacity * 255.0)
    radius = np.sqrt(np.maximum(q_cut, 0.0) * lam) * (1 + 1e-5) + 1e-3
    z3 = np.zeros((n, 3), dtype)
    return sb.SplatScreen(mean2d=mean2d, cov2d=cov, inv_cov2d=inv, depth=depth, color=color,
                          opacity=opacity, source_index=np.arange(n, dtype=np.int64), t_cam=z3,
                          t_clamped=z3, clamped_x=np.zeros(n, bool), clamped_y=np.zeros(n, bool),
                          view_dir=np.tile(np.array([0.0, 0.0, 1.0], dtype), (n, 1)),
                          basis=np.zeros((n, 16), dtype), color_raw=color.astype(dtype),
                          radius_cut=radius.astype(dtype), q_cut=q_cut.astype(dtype))


def random_map(rng, n, dtype=np.float64, spread=2.0, depth=(3.0, 8.0), opacity=(0.15, 0.8),
               scale=(0.05, 0.4)):
    """helpers.py:10-28 (same draws per Gaussian)."""
    sb = _sb()
    gs = []
    for _ in range(n):
        pos = np.array([rng.uniform(-spread, spread), rng.uniform(-spread, spread),
                        rng.uniform(*depth)])
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        gs.append(sb.Gaussian(position=pos, log_scale=np.log(rng.uniform(*scale, size=3)),
                              rotation=q, opacity_logit=_logit(rng.uniform(*opacity)),
                              sh_coeffs=rng.normal(0.0, 0.3, size=(16, 3))))
    m = sb.GaussianMap(dtype=dtype)
    m.append(gs)
    return m


def project_map(gmap, pose, intr):
    sb = _sb()
    return sb.project_gaussians(gmap.positions, gmap.log_scales, gmap.rotations,
                                gmap.opacity_logits, gmap.sh_coeffs, pose, intr)


def render_all(gmap, pose, intr, **kw):
    sb = _sb()
    screen = project_map(gmap, pose, intr)
    grid = sb.bin_and_sort(screen, intr)
    return screen, grid, sb.render(grid, screen, intr, **kw)


def dense_tile_max_alpha(screen, i, tx, ty, intr, tile=16):
    """test_forward.py:12-25: max alpha of row i over a tile's pixel centres."""
    x0, y0 = tx * tile, ty * tile
    x1, y1 = min(x0 + tile, intr.width), min(y0 + tile, intr.height)
    mean = _np(screen.mean2d[i]).astype(np.float64)
    inv = _np(screen.inv_cov2d[i]).astype(np.float64)
    o = float(screen.opacity[i])
    best = 0.0
    for py in range(y0, y1):
        for px in range(x0, x1):
            d = mean - [px, py]
            best = max(best, min(o * np.exp(-0.5 * float(d @ inv @ d)), 0.99))
    return best


def brute_force_composite(screen, intr):
    """helpers.py:75-100: literal front-to-back sums with a global stable
    depth sort, no tiles, no culling, no early termination."""
    H, W = intr.height, intr.width
    mean = _np(screen.mean2d).astype(np.float64)
    inv = _np(screen.inv_cov2d).astype(np.float64)
    opa = _np(screen.opacity).astype(np.float64)
    col = _np(screen.color).astype(np.float64)
    dep = _np(screen.depth).astype(np.float64)
    order = np.lexsort((_np(screen.source_index), dep))
    C, D, O = np.zeros((H, W, 3)), np.zeros((H, W)), np.zeros((H, W))
    for py in range(H):
        for px in range(W):
            T = 1.0
            for i in order:
                d = mean[i] - [px, py]
                a = min(opa[i] * np.exp(-0.5 * float(d @ inv[i] @ d)), 0.99)
                if a < 1.0 / 255.0:
                    continue
                w = a * T
                C[py, px] += w * col[i]
                D[py, px] += w * dep[i]
                O[py, px] += w
                T *= 1.0 - a
    return C, D, O


# ---------------------------------------------------------------------------
# binning (test_forward.py:28-105)
# ---------------------------------------------------------------------------
def test_small_gaussian_single_tile():
    """test_forward.py:28-35"""
    sb = _sb()
    intr = small_intrinsics(64)
    screen = splat_screen([24.0, 24.0], np.eye(2) * 4.0, 2.0, [1, 0, 0], 0.9)
    grid = sb.bin_and_sort(screen, intr)
    assert np.unique(_np(grid.pair_tile)).tolist() == [1 * grid.tiles_x + 1]


def test_corner_gaussian_four_tiles():
    """test_forward.py:37-45"""
    sb = _sb()
    intr = small_intrinsics(64)
    screen = splat_screen([16.0, 16.0], np.eye(2), 2.0, [1, 0, 0], 0.9)
    grid = sb.bin_and_sort(screen, intr)
    assert grid.n_pairs == 4
    tx = grid.tiles_x
    assert sorted(_np(grid.pair_tile).tolist()) == [0, 1, tx, tx + 1]


def test_membership_against_dense_oracle():
    """test_forward.py:47-60: culling never drops a tile where the Gaussian's
    max alpha over the tile reaches the 1/255 cutoff."""
    sb = _sb()
    rng = np.random.default_rng(12)
    intr = small_intrinsics(64)
    screen = project_map(random_map(rng, 200), sb.CameraPose.identity(), intr)
    grid = sb.bin_and_sort(screen, intr)
    members = set(zip(_np(grid.pair_gaussian).tolist(), _np(grid.pair_tile).tolist()))
    for i in range(0, len(screen), 7):
        for ty in range(grid.tiles_y):
            for tx in range(grid.tiles_x):
                if dense_tile_max_alpha(screen, i, tx, ty, intr) >= 1.0 / 255.0:
                    assert (i, ty * grid.tiles_x + tx) in members


def test_depth_sort_and_index_tiebreak():
    """test_forward.py:62-70: depth ascending, equal depths by row: [2, 0, 1]."""
    sb = _sb()
    intr = small_intrinsics(64)
    for dt in (np.float64, np.float32):
        screen = splat_screen([[24.0, 24.0], [25.0, 24.0], [24.5, 24.0]], np.eye(2),
                              [2.0, 2.0, 1.0], [[1, 0, 0]] * 3, [0.5, 0.5, 0.5], dtype=dt)
        grid = sb.bin_and_sort(screen, intr)
        assert grid.tile_list(1, 1).tolist() == [2, 0, 1]


def test_equal_depth_ties_many_rows():
    """The stable (depth, row) order at scale: 3,000 splats on 4 distinct
    depths over one tile -- within each depth, ascending row id."""
    sb = _sb()
    rng = np.random.default_rng(3)
    n = 3000
    intr = small_intrinsics(64)
    dep = rng.choice([1.0, 2.0, 3.0, 4.0], n)
    screen = splat_screen(rng.uniform(17, 30, (n, 2)), np.eye(2) * 0.5, dep,
                          np.ones((n, 3)), np.full(n, 0.3), dtype=np.float32)
    grid = sb.bin_and_sort(screen, intr)
    lst = grid.tile_list(1, 1).cpu().numpy()
    key = np.stack([dep[lst], lst], 1)
    assert np.all((np.diff(key[:, 0]) > 0) | ((np.diff(key[:, 0]) == 0) & (np.diff(key[:, 1]) > 0)))


# ---------------------------------------------------------------------------
# blend (test_forward.py:107-256)
# ---------------------------------------------------------------------------
def test_single_gaussian_closed_form():
    """test_forward.py:109-118: alpha = 0.3 at the centre pixel."""
    sb = _sb()
    intr = small_intrinsics(32)
    screen = splat_screen([16.0, 16.0], np.eye(2) * 1e-6, 2.0, [1, 0, 0], 0.3)
    t = sb.render(sb.bin_and_sort(screen, intr), screen, intr)
    np.testing.assert_allclose(_np(t.color)[16, 16], [0.3, 0, 0], atol=1e-7)
    assert float(t.depth[16, 16]) == pytest.approx(0.6, rel=1e-6)
    assert float(t.opacity[16, 16]) == pytest.approx(0.3, rel=1e-6)


def test_two_gaussian_expansion():
    """test_forward.py:120-129"""
    sb = _sb()
    intr = small_intrinsics(32)
    screen = splat_screen([[16.0, 16.0], [16.0, 16.0]], np.eye(2) * 1e-6, [1.0, 2.0],
                          [[1, 0, 0], [0, 0, 1]], [0.5, 1.0])
    t = sb.render(sb.bin_and_sort(screen, intr), screen, intr)
    want = 0.5 * np.array([1, 0, 0]) + 0.5 * 0.99 * np.array([0, 0, 1])
    np.testing.assert_allclose(_np(t.color)[16, 16], want, atol=1e-7)
    assert float(t.opacity[16, 16]) == pytest.approx(0.5 + 0.5 * 0.99, rel=1e-6)


def test_opacity_bounds_and_transmittance():
    """test_forward.py:155-163"""
    sb = _sb()
    rng = np.random.default_rng(79)
    intr = small_intrinsics(48)
    _, _, t = render_all(random_map(rng, 200, opacity=(0.3, 0.95)), sb.CameraPose.identity(),
                         intr)
    op = _np(t.opacity)
    assert op.min() >= 0.0 and op.max() <= 1.0
    np.testing.assert_allclose(_np(t.transmittance), 1 - op, atol=1e-6)


def test_blending_weights_sum_to_opacity():
    """test_forward.py:176-184 (and helpers.py's brute-force oracle for the
    colour and depth as well, test_forward.py:230-238)."""
    sb = _sb()
    rng = np.random.default_rng(81)
    intr = small_intrinsics(24)
    screen = project_map(random_map(rng, 40), sb.CameraPose.identity(), intr)
    t = sb.render(sb.bin_and_sort(screen, intr), screen, intr, early_termination=False)
    C, D, O = brute_force_composite(screen, intr)
    np.testing.assert_allclose(_np(t.opacity), O, atol=1e-9)
    np.testing.assert_allclose(_np(t.color), C, atol=1e-9)
    np.testing.assert_allclose(_np(t.depth), D, atol=1e-8)


def test_gaussian_behind_termination_is_invisible():
    """test_forward.py:186-203: bitwise."""
    sb = _sb()
    intr = small_intrinsics(32)
    n = 10
    for dt in (np.float64, np.float32):
        s0 = splat_screen([[16.0, 16.0]] * n, np.eye(2) * 1e-6, list(np.linspace(1, 2, n)),
                          [[1, 1, 1]] * n, [0.9] * n, dtype=dt)
        t0 = sb.render(sb.bin_and_sort(s0, intr), s0, intr)
        assert float(t0.transmittance[16, 16]) < 1e-4
        s1 = splat_screen([[16.0, 16.0]] * (n + 1), np.eye(2) * 1e-6,
                          list(np.linspace(1, 2, n)) + [5.0], [[1, 1, 1]] * n + [[0, 1, 0]],
                          [0.9] * (n + 1), dtype=dt)
        t1 = sb.render(sb.bin_and_sort(s1, intr), s1, intr)
        np.testing.assert_array_equal(_np(t0.color)[16, 16], _np(t1.color)[16, 16])
        np.testing.assert_array_equal(_np(t0.depth)[16, 16], _np(t1.depth)[16, 16])


def test_depth_approaches_d_when_opaque():
    """test_forward.py:205-212: alpha clamps at 0.99, so D = 0.99 d."""
    sb = _sb()
    intr = small_intrinsics(32)
    screen = splat_screen([16.0, 16.0], np.eye(2) * 1e-6, 3.0, [1, 1, 1], 0.9999)
    t = sb.render(sb.bin_and_sort(screen, intr), screen, intr)
    assert float(t.depth[16, 16]) == pytest.approx(0.99 * 3.0, rel=1e-6)


def test_culling_never_changes_output():
    """test_forward.py:243-256"""
    sb = _sb()
    rng = np.random.default_rng(84)
    intr = small_intrinsics(64)
    gmap = random_map(rng, 150, scale=(0.01, 0.6))
    gmap.log_scales[:, 0] += float(np.log(30.0))   # slim splats
    screen = project_map(gmap, sb.CameraPose.identity(), intr)
    g_on = sb.bin_and_sort(screen, intr, cull=True)
    g_off = sb.bin_and_sort(screen, intr, cull=False)
    assert g_on.n_pairs < g_off.n_pairs
    t_on = sb.render(g_on, screen, intr)
    t_off = sb.render(g_off, screen, intr)
    assert float((t_on.color - t_off.color).abs().max()) <= 2e-4


# ---------------------------------------------------------------------------
# projection KATs through project_gaussians (test_projection.py)
# ---------------------------------------------------------------------------
def _one(sb, pos, log_scale=(0.0, 0.0, 0.0), rot=(1.0, 0.0, 0.0, 0.0), opacity=0.5, sh=None):
    g = sb.Gaussian(position=pos, log_scale=log_scale, rotation=rot,
                    opacity_logit=_logit(opacity),
                    sh_coeffs=np.zeros((16, 3)) if sh is None else sh)
    m = sb.GaussianMap(dtype=np.float64)
    m.append([g])
    return m


def test_project_mean_kats():
    """test_projection.py:55-71"""
    sb = _sb()
    intr = sb.CameraIntrinsics(100, 100, 50, 50, 100, 100)
    s = project_map(_one(sb, [0, 0, 2]), sb.CameraPose.identity(), intr)
    np.testing.assert_allclose(_np(s.mean2d)[0], [50, 50])
    assert float(s.depth[0]) == 2.0
    s = project_map(_one(sb, [1, 0, 2]), sb.CameraPose.identity(), intr)
    np.testing.assert_allclose(_np(s.mean2d)[0], [100, 50])
    s = project_map(_one(sb, [0, 0, 1]), sb.CameraPose(np.eye(3), np.array([0.0, 0.0, 1.0])),
                    intr)
    np.testing.assert_allclose(_np(s.mean2d)[0], [50, 50])
    assert float(s.depth[0]) == 2.0


def test_projected_covariance_kats():
    """test_projection.py:24-36 and 75-87: cov3d diag(1, 4, 9) for the
    identity rotation, the 90-degree z rotation moving the y variance onto x,
    cov2d on axis = I + 0.3 I, and doubling the depth quarters cov2d."""
    sb = _sb()
    pose = sb.CameraPose.identity()
    intr = sb.CameraIntrinsics(1, 1, 0.5, 0.5, 1, 1)
    s = project_map(_one(sb, [0, 0, 1]), pose, intr)
    np.testing.assert_allclose(_np(s.cov2d)[0], np.eye(2) * 1.3, atol=1e-12)
    # diag(1, 4, 9) seen on axis at z = 1 with f = 1: cov2d = diag(1, 4) + 0.3
    s = project_map(_one(sb, [0, 0, 1], log_scale=(0.0, np.log(2.0), np.log(3.0))), pose, intr)
    np.testing.assert_allclose(_np(s.cov2d)[0], np.diag([1.3, 4.3]), atol=1e-12)
    q = (np.cos(np.pi / 4), 0.0, 0.0, np.sin(np.pi / 4))
    s = project_map(_one(sb, [0, 0, 1], log_scale=(0.0, np.log(2.0), 0.0), rot=q), pose, intr)
    np.testing.assert_allclose(_np(s.cov2d)[0], np.diag([4.3, 1.3]), atol=1e-12)
    intr = sb.CameraIntrinsics(50, 50, 32, 32, 64, 64)
    keys = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")
    c1 = _np(sb.project_gaussians(*[_one(sb, [0, 0, 2]).arrays()[k] for k in keys], pose, intr,
                                  dilation=0.0).cov2d)[0]
    c2 = _np(sb.project_gaussians(*[_one(sb, [0, 0, 4]).arrays()[k] for k in keys], pose, intr,
                                  dilation=0.0).cov2d)[0]
    np.testing.assert_allclose(c2, c1 / 4.0, rtol=1e-12)


def test_alpha_kats_through_render():
    """test_projection.py:124-138: alpha at the mean = opacity, exp(-1/2) at
    unit Mahalanobis distance, clamped at 0.99, zero below 1/255 -- read off
    the render of one splat over a black background (C = alpha c at T = 1)."""
    sb = _sb()
    intr = small_intrinsics(32)
    for o, pix, want in ((0.5, (10, 10), 0.5), (1.0, (11, 10), np.exp(-0.5)),
                         (1.0, (10, 10), 0.99), (0.5, (20, 10), 0.0)):
        s = splat_screen([10.0, 10.0], np.eye(2), 2.0, [1, 1, 1], o)
        t = sb.render(sb.bin_and_sort(s, intr), s, intr)
        got = float(t.opacity[pix[1], pix[0]])
        assert got == pytest.approx(want, rel=1e-12, abs=0 if want else 1e-300), (o, pix)


def test_sh_kats_through_projection():
    """test_projection.py:168-184: zero coefficients give gray 0.5; a degree-0
    coefficient k gives 0.5 + C0 k in any direction; clamped at 0."""
    sb = _sb()
    intr = sb.CameraIntrinsics(100, 100, 50, 50, 100, 100)
    pose = sb.CameraPose.identity()
    s = project_map(_one(sb, [0, 0, 2]), pose, intr)
    np.testing.assert_allclose(_np(s.color)[0], [0.5, 0.5, 0.5])
    sh = np.zeros((16, 3))
    sh[0, 0] = 0.7
    for p in ([0, 0, 2], [0.5, -0.4, 2], [-0.9, 0.3, 3]):
        c = _np(project_map(_one(sb, p, sh=sh), pose, intr).color)[0]
        assert c[0] == pytest.approx(0.5 + C0 * 0.7, rel=1e-9)
        assert c[1] == pytest.approx(0.5)
    sh = np.zeros((16, 3))
    sh[0, :] = -10.0
    np.testing.assert_array_equal(_np(project_map(_one(sb, [0, 0, 2], sh=sh), pose, intr).color)[0],
                                  0.0)


# ---------------------------------------------------------------------------
# backward (test_backward.py:34-110)
# ---------------------------------------------------------------------------
def single_gaussian_map(opacity=0.6, depth=4.0, sigma_px=40.0, intr=None):
    """test_backward.py:21-31"""
    sb = _sb()
    intr = intr or small_intrinsics(24)
    s_world = sigma_px * depth / intr.fx
    return _one(sb, [0, 0, depth], log_scale=np.log([s_world] * 3), opacity=opacity), intr


def _backward(gmap, intr, dC):
    sb = _sb()
    import torch
    pose = sb.CameraPose.identity()
    screen, grid, t = render_all(gmap, pose, intr)
    dC = torch.as_tensor(dC, dtype=torch.float64, device="cuda")
    return screen, t, sb.backward_per_gaussian(t, dC, screen, grid, gmap, pose, intr)


def test_single_gaussian_single_pixel_sh_gradient():
    """test_backward.py:34-48: d_sh[0, 0, 0] = C0 alpha at rel 1e-12."""
    m, intr = single_gaussian_map(opacity=0.6)
    dC = np.zeros((24, 24, 3))
    dC[12, 12, 0] = 1.0
    screen, _, buf = _backward(m, intr, dC)
    d = _np(screen.mean2d)[0] - [12.0, 12.0]
    q = float(d @ _np(screen.inv_cov2d)[0] @ d)
    alpha = min(float(screen.opacity[0]) * np.exp(-0.5 * q), 0.99)
    assert float(buf.d_sh[0, 0, 0]) == pytest.approx(C0 * alpha, rel=1e-12)
    assert float(buf.d_sh[0, 0, 1]) == 0.0


def test_zero_cotangent_gives_zero_gradients():
    """test_backward.py:50-60"""
    rng = np.random.default_rng(5)
    intr = small_intrinsics(32)
    m = random_map(rng, 25)
    _, _, buf = _backward(m, intr, np.zeros((32, 32, 3)))
    for a in (buf.d_position, buf.d_log_scale, buf.d_rotation, buf.d_opacity_logit, buf.d_sh):
        assert not bool(a.any())


def test_gradient_locality_for_invisible_gaussian():
    """test_backward.py:62-74: a Gaussian behind the camera gets exactly zero."""
    import torch
    rng = np.random.default_rng(6)
    intr = small_intrinsics(32)
    m = random_map(rng, 10)
    pos = _np(m.positions).copy()
    pos[3] = [0.0, 0.0, -5.0]
    m.positions.copy_(torch.as_tensor(pos))
    _, _, buf = _backward(m, intr, rng.normal(size=(32, 32, 3)))
    assert not bool(buf.d_position[3].any())
    assert not bool(buf.d_sh[3].any())
    assert float(buf.d_opacity_logit[3]) == 0.0


def test_missing_forward_state_raises():
    """test_backward.py:76-86"""
    sb = _sb()
    rng = np.random.default_rng(7)
    intr = small_intrinsics(16)
    m = random_map(rng, 5)
    pose = sb.CameraPose.identity()
    screen, grid, t = render_all(m, pose, intr)
    t.n_contrib = None
    with pytest.raises(ValueError):
        sb.backward_per_gaussian(t, np.zeros((16, 16, 3)), screen, grid, m, pose, intr)


def test_clamped_alpha_blocks_opacity_and_shape_gradients():
    """test_backward.py:89-101"""
    m, intr = single_gaussian_map(opacity=0.999, sigma_px=500.0)
    screen, _, buf = _backward(m, intr, np.ones((24, 24, 3)))
    assert min(float(screen.opacity[0]), 1.0) > 0.99
    assert float(buf.d_opacity_logit[0]) == 0.0
    np.testing.assert_allclose(_np(buf.d_log_scale)[0], 0.0, atol=1e-20)
    assert bool(buf.d_sh[0].any())


def test_cutoff_gaussian_gets_zero_gradient():
    """test_backward.py:103-110"""
    m, intr = single_gaussian_map(opacity=1.0 / 300.0)
    _, _, buf = _backward(m, intr, np.ones((24, 24, 3)))
    assert not bool(buf.d_sh[0].any())
    assert float(buf.d_opacity_logit[0]) == 0.0


# ---------------------------------------------------------------------------
# sparse Adam (test_adam.py)
# ---------------------------------------------------------------------------
LRS = {"position": 1e-2, "sh0": 1e-2, "sh_rest": 1e-2, "opacity_logit": 1e-2,
       "log_scale": 1e-2, "rotation": 1e-2}
SHAPES = {"position": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (),
          "sh": (16, 3)}


def _params(rng, n, dtype=np.float64):
    import torch
    return {k: torch.as_tensor(rng.normal(size=(n,) + s).astype(dtype), device="cuda")
            for k, s in SHAPES.items()}


def _grads(rng, n, dtype=np.float64):
    return {k: rng.normal(size=(n,) + s).astype(dtype) for k, s in SHAPES.items()}


def test_adam_single_step_closed_form():
    """test_adam.py:23-35: -lr g / (|g| + eps sqrt(1 - beta2))."""
    sb = _sb()
    rng = np.random.default_rng(0)
    p = _params(rng, 8)
    before = {k: _np(v).copy() for k, v in p.items()}
    g = _grads(rng, 8)
    st = sb.AdamState(8, LRS, dtype=np.float64)
    sb.adam_step(p, g, st)
    for k in p:
        want = before[k] - 1e-2 * g[k] / (np.abs(g[k]) + 1e-15 * np.sqrt(1 - 0.999))
        np.testing.assert_allclose(_np(p[k]), want, rtol=1e-9)


def test_adam_empty_active_is_noop():
    """test_adam.py:37-46"""
    sb = _sb()
    rng = np.random.default_rng(1)
    p = _params(rng, 5)
    before = {k: _np(v).copy() for k, v in p.items()}
    st = sb.AdamState(5, LRS, dtype=np.float64)
    sb.adam_step(p, _grads(rng, 5), st, active=np.array([], dtype=np.int64))
    for k in p:
        np.testing.assert_array_equal(_np(p[k]), before[k])
    assert not bool(st.steps.any())


def test_adam_inactive_rows_untouched():
    """test_adam.py:48-58"""
    sb = _sb()
    rng = np.random.default_rng(2)
    p = _params(rng, 6)
    before = {k: _np(v).copy() for k, v in p.items()}
    st = sb.AdamState(6, LRS, dtype=np.float64)
    sb.adam_step(p, _grads(rng, 6), st, active=np.array([1, 4]))
    for k in p:
        np.testing.assert_array_equal(_np(p[k])[0], before[k][0])
        assert not np.array_equal(_np(p[k])[1], before[k][1])
    assert _np(st.steps).tolist() == [0, 1, 0, 0, 1, 0]


def test_adam_sparse_all_equals_dense_bitwise():
    """test_adam.py:60-75 (float32, four steps)."""
    sb = _sb()
    import torch
    rng = np.random.default_rng(3)
    n = 17
    p1 = _params(rng, n, np.float32)
    p2 = {k: v.clone() for k, v in p1.items()}
    s1 = sb.AdamState(n, LRS, dtype=np.float32)
    s2 = sb.AdamState(n, LRS, dtype=np.float32)
    for _ in range(4):
        g = _grads(rng, n, np.float32)
        sb.adam_step(p1, g, s1, active=None)
        sb.adam_step(p2, g, s2, active=np.arange(n))
    for k in p1:
        assert torch.equal(p1[k], p2[k]), k
        assert torch.equal(s1.m[k], s2.m[k]) and torch.equal(s1.v[k], s2.v[k]), k


def test_adam_replay_oracle_for_intermittent_gaussian():
    """test_adam.py:77-95"""
    sb = _sb()
    rng = np.random.default_rng(4)
    p = _params(rng, 3)
    fresh = {k: v[[1]].clone() for k, v in p.items()}
    st = sb.AdamState(3, LRS, dtype=np.float64)
    fst = sb.AdamState(1, LRS, dtype=np.float64)
    for active in (True, False, False, True, True, False, True):
        g = _grads(rng, 3)
        sb.adam_step(p, g, st, active=np.array([0, 1, 2]) if active else np.array([0, 2]))
        if active:
            sb.adam_step(fresh, {k: v[[1]] for k, v in g.items()}, fst)
    for k in p:
        np.testing.assert_allclose(_np(p[k])[1], _np(fresh[k])[0], rtol=1e-14)


def test_adam_resize_preserves_and_extends():
    """test_adam.py:97-107"""
    sb = _sb()
    st = sb.AdamState(2, LRS, dtype=np.float32)
    st.m["position"][:] = 1.0
    st.steps[:] = 5
    st.resize(4)
    assert st.count == 4
    np.testing.assert_array_equal(_np(st.m["position"])[:2], 1.0)
    np.testing.assert_array_equal(_np(st.m["position"])[2:], 0.0)
    assert _np(st.steps).tolist() == [5, 5, 0, 0]
    with pytest.raises(ValueError):
        st.resize(3)


def test_adam_sh_group_uses_two_rates():
    """test_adam.py:109-118: with sh0 = 10 sh_rest the first-step updates
    differ by a factor of 10."""
    sb = _sb()
    rng = np.random.default_rng(5)
    lrs = dict(LRS, sh0=1e-2, sh_rest=1e-3)
    p = _params(rng, 1)
    before = _np(p["sh"]).copy()
    g = {k: np.ones((1,) + s) for k, s in SHAPES.items()}
    sb.adam_step(p, g, sb.AdamState(1, lrs, dtype=np.float64))
    d = before - _np(p["sh"])
    assert d[0, 0, 0] == pytest.approx(10 * d[0, 1, 0], rel=1e-6)


# ---------------------------------------------------------------------------
# loss (test_loss.py)
# ---------------------------------------------------------------------------
def _img(rng, h=12, w=14):
    return rng.uniform(0.0, 1.0, (h, w, 3))


def test_loss_zero_when_equal_and_ssim_one():
    """test_loss.py:36-40 and 73-78"""
    sb = _sb()
    rng = np.random.default_rng(5)
    img = _img(rng)
    loss, _, _, parts = sb.photometric_loss(img, img, sb.ExposureAffine.identity(), 0.2)
    assert loss == pytest.approx(0.0, abs=1e-12)
    assert parts["ssim"] == pytest.approx(1.0, abs=1e-10)
    for _ in range(3):
        x = _img(rng)
        assert sb.ssim(x, x) == pytest.approx(1.0, abs=1e-9)


def test_ssim_symmetric():
    """test_loss.py:42-45"""
    sb = _sb()
    rng = np.random.default_rng(3)
    a, b = _img(rng), _img(rng)
    assert sb.ssim(a, b) == pytest.approx(sb.ssim(b, a), abs=1e-12)


def test_pure_l1_constant_difference():
    """test_loss.py:80-85: loss 0.1 with lambda 0."""
    sb = _sb()
    a, b = np.full((6, 6, 3), 0.4), np.full((6, 6, 3), 0.5)
    loss, _, _, parts = sb.photometric_loss(a, b, sb.ExposureAffine.identity(), 0.0)
    assert loss == pytest.approx(0.1, rel=1e-9)
    assert parts["l1"] == pytest.approx(0.1, rel=1e-9)


def test_loss_shape_mismatch_raises():
    """test_loss.py:93-96"""
    sb = _sb()
    with pytest.raises(ValueError):
        sb.photometric_loss(np.zeros((8, 8, 3)), np.zeros((8, 9, 3)),
                            sb.ExposureAffine.identity(), 0.2)


def test_exposure_gradient_zero_at_optimum():
    """test_loss.py:129-139"""
    sb = _sb()
    rng = np.random.default_rng(8)
    rendered = _img(rng)
    E = sb.ExposureAffine(rng.normal(size=(3, 4)) * 0.1
                          + np.concatenate([np.eye(3), np.zeros((3, 1))], 1))
    gt = _np(sb.apply_exposure(E, rendered))
    loss, d_r, d_E, _ = sb.photometric_loss(rendered, gt, E, 0.2)
    assert loss == pytest.approx(0.0, abs=1e-12)
    np.testing.assert_allclose(np.asarray(d_E), 0.0, atol=1e-12)
    np.testing.assert_allclose(_np(d_r), 0.0, atol=1e-12)
