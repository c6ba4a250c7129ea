"""Pin the CPU oracle (oracle/) to the reference.

Golden vectors in tests/golden/ were recorded from the reference package
itself by tests/golden/make_golden.py.  Each stage of the oracle is fed the
reference's own upstream outputs, so integer stages must be bit-exact and
float stages must agree to within a few ulps (well inside the north-star
tolerances).  CPU only; runs in seconds.
"""

import numpy as np
import pytest

from parity import (assert_grads_close, assert_image_close, camera_from, gmap_from,
                    golden_names, grad_report, load_golden, lrs_from, max_abs, oracle,
                    screen_from)

NAMES = golden_names()


@pytest.fixture(scope="module")
def o():
    return oracle()


def _ulps(dt):
    return 1e-12 if dt == np.float64 else 1e-5


@pytest.mark.parametrize("name", NAMES)
def test_frustum_mask_bit_exact(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    got = o.frustum_mask(cam, g["positions"], float(g["near"]), float(g["margin"]))
    np.testing.assert_array_equal(got, g["frustum"])


@pytest.mark.parametrize("name", NAMES)
def test_projection(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    sc = o.project(g["positions"], g["log_scales"], g["rotations"], g["opacity_logits"],
                   g["sh_coeffs"], cam, float(g["near"]))
    ref = screen_from(g)
    # keep set (integer): bit-exact
    np.testing.assert_array_equal(sc["source_index"], ref["source_index"])
    np.testing.assert_array_equal(sc["clamped_x"], ref["clamped_x"])
    np.testing.assert_array_equal(sc["clamped_y"], ref["clamped_y"])
    tol = _ulps(g["positions"].dtype)
    for f in ("mean2d", "depth", "t_cam", "t_clamped", "view_dir", "basis", "color", "color_raw"):
        np.testing.assert_allclose(sc[f], ref[f], rtol=tol, atol=tol * 1e-2, err_msg=f)
    for f in ("opacity", "q_cut", "radius_cut"):
        np.testing.assert_allclose(sc[f], ref[f], rtol=10 * tol, atol=tol * 1e-2, err_msg=f)
    # 2x2 matrices: off-diagonals can be tiny, compare against each row's scale
    for f in ("cov2d", "inv_cov2d"):
        scale = np.abs(ref[f]).reshape(-1, 4).max(axis=1)[:, None, None]
        assert (np.abs(sc[f] - ref[f]) <= 10 * tol * scale + 1e-30).all(), f


@pytest.mark.parametrize("name", NAMES)
def test_binning_bit_exact_on_reference_floats(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    pg, pt, off = o.bin_and_sort(screen_from(g), cam.width, cam.height)
    np.testing.assert_array_equal(pg, g["pair_gaussian"])
    np.testing.assert_array_equal(pt, g["pair_tile"])
    np.testing.assert_array_equal(off, g["offsets"])
    if "nocull_pair_gaussian" in g:
        pg2, _, off2 = o.bin_and_sort(screen_from(g), cam.width, cam.height, cull=False)
        np.testing.assert_array_equal(pg2, g["nocull_pair_gaussian"])
        np.testing.assert_array_equal(off2, g["nocull_offsets"])


@pytest.mark.parametrize("name", NAMES)
def test_composite_on_reference_grid(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    sc = screen_from(g)
    t = o.composite(g["pair_gaussian"], g["offsets"], sc, cam.width, cam.height)
    tol = _ulps(g["positions"].dtype)
    assert_image_close(t["color"], g["color"], tol=tol)
    depth_scale = max(float(np.abs(g["depth"]).max()), 1.0)
    assert max_abs(t["depth"], g["depth"]) <= tol * depth_scale
    assert max_abs(t["transmittance"], g["transmittance"]) <= tol
    np.testing.assert_array_equal(t["n_contrib"], g["n_contrib"])
    if "noterm_color" in g:
        t2 = o.composite(g["pair_gaussian"], g["offsets"], sc, cam.width, cam.height,
                         early_termination=False)
        assert_image_close(t2["color"], g["noterm_color"], tol=tol)
        # acceptance #1 (test_acceptance.py:67-88): tiled vs reference_render
        assert max_abs(t2["color"], g["refrender_color"]) <= 1e-5


@pytest.mark.parametrize("name", NAMES)
def test_loss_on_reference_render(o, name):
    g = load_golden(name)
    dt = g["positions"].dtype
    loss, d_r, d_E, parts = o.photometric_loss(g["color"], g["image"].astype(dt), g["E"],
                                               float(g["lam"]))
    rel = 1e-12 if dt == np.float64 else 2e-6
    assert loss == pytest.approx(g["loss"][0], rel=rel, abs=1e-12)
    assert parts["l1"] == pytest.approx(g["loss"][1], rel=rel, abs=1e-12)
    assert parts["ssim"] == pytest.approx(g["loss"][3], rel=rel, abs=1e-12)
    scale = np.abs(g["d_rendered"]).max()
    assert max_abs(d_r, g["d_rendered"]) <= (1e-12 if dt == np.float64 else 1e-6) * scale
    assert max_abs(d_E, g["d_E"]) <= (1e-12 if dt == np.float64 else 1e-5) * np.abs(g["d_E"]).max()


@pytest.mark.parametrize("name", NAMES)
def test_backward_pixel_stage_on_reference_inputs(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    adj = o.backward_tiles(g["pair_gaussian"], g["offsets"], screen_from(g), g["d_rendered"],
                           g["color"], cam.width, cam.height)
    conic = g["adj_conic"].reshape(-1, 4)[:, [0, 1, 3]]
    for k, ref in (("d_mean2d", g["adj_mean2d"]), ("d_conic", conic),
                   ("d_opacity", g["adj_opacity"]), ("d_color", g["adj_color"])):
        assert_grads_close(adj[k], ref, k, norm_tol=1e-4)


@pytest.mark.parametrize("name", NAMES)
def test_chain_on_reference_adjoints(o, name):
    g = load_golden(name)
    cam = camera_from(g)
    adj = {"d_mean2d": g["adj_mean2d"], "d_conic": g["adj_conic"].reshape(-1, 4)[:, [0, 1, 3]],
           "d_opacity": g["adj_opacity"], "d_color": g["adj_color"]}
    gr = o.chain(adj, screen_from(g), gmap_from(g), cam)
    for f in ("d_position", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        assert_grads_close(gr[f], g["grad_" + f], f, norm_tol=1e-4)


def _fresh_adam(o, gm):
    arrs = [gm["positions"], gm["log_scales"], gm["rotations"], gm["opacity_logits"],
            gm["sh_coeffs"]]
    return {"m": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "v": {k: np.zeros_like(v) for k, v in zip(o.GROUPS, arrs)},
            "steps": np.zeros(arrs[0].shape[0], np.int64)}


@pytest.mark.parametrize("name", NAMES)
def test_sparse_adam_on_reference_gradients(o, name):
    g = load_golden(name)
    gm = {k: np.array(v, copy=True) for k, v in gmap_from(g).items()}
    adam = _fresh_adam(o, gm)
    params = {"position": gm["positions"], "log_scale": gm["log_scales"],
              "rotation": gm["rotations"], "opacity_logit": gm["opacity_logits"],
              "sh": gm["sh_coeffs"]}
    grads = {"position": g["grad_d_position"], "log_scale": g["grad_d_log_scale"],
             "rotation": g["grad_d_rotation"], "opacity_logit": g["grad_d_opacity_logit"],
             "sh": g["grad_d_sh"]}
    o.adam_step(params, grads, adam["m"], adam["v"], adam["steps"], lrs_from(g),
                active=g["frustum"])
    np.testing.assert_array_equal(adam["steps"], g["after_steps"])
    inactive = ~g["frustum"]
    for f in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        # inactive rows untouched (bitwise, test_adam.py:48-58)
        np.testing.assert_array_equal(gm[f][inactive], g[f][inactive])
        np.testing.assert_allclose(gm[f], g["after_" + f], rtol=1e-6, atol=1e-9, err_msg=f)
    np.testing.assert_allclose(adam["m"]["position"], g["after_m_position"], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(adam["v"]["sh"], g["after_v_sh"], rtol=1e-6, atol=1e-18)


@pytest.mark.parametrize("name", NAMES)
def test_full_step_against_reference_step(o, name):
    """End to end: the oracle's optimize_step vs Mapper._optimize_step.

    Adam's first step is -lr*sign(g): rows whose reference gradient is at the
    float noise floor may take the opposite sign, so those elements are held
    only to |delta| <= 2 lr; all others to 1e-6."""
    g = load_golden(name)
    cam = camera_from(g)
    gm = {k: np.array(v, copy=True) for k, v in gmap_from(g).items()}
    adam = _fresh_adam(o, gm)
    E = g["E"].copy()
    log = o.optimize_step(gm, adam, lrs_from(g), cam, g["image"], E, o.ScalarAdam((3, 4), 1e-2),
                          float(g["lam"]), float(g["near"]), float(g["margin"]))
    assert log["loss"] == pytest.approx(float(g["step_loss"]), rel=1e-6)
    np.testing.assert_array_equal(adam["steps"], g["after_steps"])
    lrs = lrs_from(g)
    for f, gf, lr in (("positions", "d_position", lrs["position"]),
                      ("log_scales", "d_log_scale", lrs["log_scale"]),
                      ("rotations", "d_rotation", lrs["rotation"]),
                      ("opacity_logits", "d_opacity_logit", lrs["opacity_logit"]),
                      ("sh_coeffs", "d_sh", max(lrs["sh0"], lrs["sh_rest"]))):
        gref = np.abs(g["grad_" + gf].astype(np.float64))
        noisy = gref <= 1e-6 * max(gref.max(), 1e-30) + 1e-12
        d = np.abs(gm[f].astype(np.float64) - g["after_" + f])
        assert d[~noisy].max(initial=0) <= 1e-6 * (1 + np.abs(g["after_" + f]).max()), f
        assert d[noisy].max(initial=0) <= 2 * lr * 1.0001 + 1e-7, f
    np.testing.assert_allclose(E, g["after_E"], rtol=0, atol=1e-8)


def test_grad_report_helper():
    assert grad_report(np.ones(3), np.ones(3)) == (0, 0.0)
    n, norm = grad_report(np.array([1.0, 2.0]), np.array([1.0, 1.0]))
    assert n == 1 and norm == 1.0
