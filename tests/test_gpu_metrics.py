"""Device metrics and the per-view evaluation path (SURVEY §8f row 3,
metrics.py:12-34, cli.py:_render_views) against numpy restatements of the
reference formulas and the CPU oracle's float64 SSIM."""

import numpy as np
import pytest

from parity import oracle

pytestmark = pytest.mark.gpu


def _psnr_ref(a, b):
    """metrics.py:16-27."""
    qa = np.clip(np.round(np.clip(a, 0.0, 1.0) * 255.0), 0, 255).astype(np.float64)
    qb = np.clip(np.round(np.clip(b, 0.0, 1.0) * 255.0), 0, 255).astype(np.float64)
    mse = np.mean((qa - qb) ** 2)
    return 99.0 if mse == 0.0 else min(float(10.0 * np.log10(255.0 ** 2 / mse)), 99.0)


def test_psnr_and_ssim_metrics():
    import paper_2404_06926_b200 as sb
    rng = np.random.default_rng(2)
    a = rng.uniform(-0.1, 1.1, (48, 64, 3))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    assert abs(sb.psnr_8bit(a, b) - _psnr_ref(a, b)) < 1e-9
    assert sb.psnr_8bit(b, b) == 99.0
    o = oracle()
    E = np.concatenate([np.eye(3), np.zeros((3, 1))], 1)
    _, _, _, parts = o.photometric_loss(a.astype(np.float64), b.astype(np.float64), E, 1.0)
    assert abs(sb.ssim_metric(a, b) - parts["ssim"]) < 1e-12


def test_evaluate_view_matches_manual_pipeline():
    import torch
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200.synthetic import view_map
    rng = np.random.default_rng(8)
    W, H, f = 80, 64, 70.0
    arrays = [x.astype(np.float32) if x.dtype != bool else x for x in view_map(rng, 500, W, H, f)]
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*arrays)
    pose = sb.CameraPose.identity()
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    gt = rng.uniform(0, 1, (H, W, 3))
    E = sb.ExposureAffine(np.concatenate([np.eye(3) * 1.1, np.full((3, 1), -0.02)], 1))
    r = sb.evaluate_view(mp, pose, intr, gt, E)
    _, _, t = mp.render_view(pose, intr)
    img = np.clip(sb.apply_exposure(E, t.color).cpu().numpy(), 0, 1)
    np.testing.assert_array_equal(r["image"].cpu().numpy(), img)
    assert abs(r["psnr"] - _psnr_ref(img, gt)) < 1e-9
    assert abs(r["ssim"] - sb.ssim_metric(img, gt)) < 1e-12
    torch.cuda.synchronize()
