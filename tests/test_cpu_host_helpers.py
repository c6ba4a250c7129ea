"""CPU: host-side helpers added for the config-4/5 workloads -- the bulk
frame-point path of process_frame, the config-5 scene and its look-at poses
(against the reference's look_at_pose when the reference tree is present)."""

import os
import sys

import numpy as np
import pytest


def test_points_array_accepts_colored_points_and_arrays():
    from paper_2404_06926_b200.mapper import _points_array
    from paper_2404_06926_b200.scene import ColoredPoint
    rng = np.random.default_rng(0)
    pos, rgb = rng.normal(size=(5, 3)), rng.uniform(size=(5, 3))
    pts = [ColoredPoint(p, c) for p, c in zip(pos, rgb)]
    a = _points_array(pts)
    b = _points_array(np.concatenate([pos, rgb], 1).astype(np.float32))
    assert a.shape == (5, 6) and a.dtype == np.float64
    np.testing.assert_array_equal(a, np.concatenate([pos, rgb], 1))
    np.testing.assert_allclose(b, a, rtol=1e-6, atol=1e-7)
    assert _points_array(np.zeros((0, 6))).shape == (0, 6)


def test_config5_scene_geometry():
    from paper_2404_06926_b200 import synthetic
    scene, views = synthetic.config5(n_fg=20_000, sky=500, n_views=8)
    assert scene.n == 20_500 and len(views) == 8
    pos = scene.arrays[0][:20_000].astype(np.float64)
    r = np.hypot(pos[:, 0], pos[:, 1])
    assert r.min() >= 6.0 - 1e-4 and r.max() <= 14.0 + 1e-4
    assert np.abs(pos[:, 2]).max() <= 4.0 + 1e-4
    for k, v in enumerate(views):
        R = v.W
        np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-12)
        fwd = R[2]                                    # camera z axis in world
        yaw = 2 * np.pi * k / 8
        np.testing.assert_allclose(fwd, [np.cos(yaw), np.sin(yaw), 0.0], atol=1e-12)
    # the same seed gives the same scene
    s2, _ = synthetic.config5(n_fg=20_000, sky=500, n_views=8)
    for a, b in zip(scene.arrays, s2.arrays):
        np.testing.assert_array_equal(a, b)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference tree absent")
def test_look_at_matches_reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from splatmap.sim import look_at_pose
    except Exception as e:   # numba / optional deps
        pytest.skip(f"reference import failed: {e}")
    from paper_2404_06926_b200.synthetic import look_at
    for target in ([1.0, 0.0, 0.0], [0.3, -2.0, 0.5], [-1.0, 1.0, -0.2]):
        ref = look_at_pose(np.zeros(3), np.array(target))
        R, t = look_at(np.zeros(3), np.array(target))
        np.testing.assert_allclose(R, ref.rotation_wc, atol=1e-12)
        np.testing.assert_allclose(t, ref.translation_wc, atol=1e-12)


def test_hostmem_falls_back_without_cuda():
    """pinned_empty returns a CPU tensor of the right shape and dtype (pinned
    when CUDA is available, a pin_memory fallback otherwise)."""
    import torch
    from paper_2404_06926_b200 import hostmem
    if not torch.cuda.is_available():
        pytest.skip("needs the CUDA runtime to register host memory")
    t = hostmem.pinned_from(np.arange(12, dtype=np.float32).reshape(3, 4))
    assert t.shape == (3, 4) and t.dtype == torch.float32 and t.is_pinned()
    np.testing.assert_array_equal(t.numpy(), np.arange(12, dtype=np.float32).reshape(3, 4))
