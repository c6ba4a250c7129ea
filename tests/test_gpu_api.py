"""Host-buffer entry point of the mapping step (Mapper.optimize_keyframe with a
pinned host image, the call bench.py's e2e leg times) against the same steps
fed from a device-resident image, graph replay against eager launches and
depth-limited against full tile lists.  The step is deterministic (no float
atomics anywhere on it: sb_blend_bwd_det, the loss's fixed-order block
reduction), so all of these must agree BITWISE."""

import numpy as np
import pytest
import torch

import paper_2404_06926_b200 as sb
from paper_2404_06926_b200.synthetic import view_map

from parity import assert_logs_identical, assert_maps_identical

pytestmark = pytest.mark.gpu


def _mapper(arrays, img, W, H, f):
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs())
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    entry = mp.store.add(sb.CameraFrame(pose=sb.CameraPose.identity(), intrinsics=intr,
                                        image=img), cfg.lr_exposure)
    return mp, entry


@pytest.mark.parametrize("graphs", [False, True])
def test_optimize_keyframe_host_image_matches_device_image(graphs):
    rng = np.random.default_rng(3)
    W, H, f = 96, 64, 80.0
    arrays = [a.astype(np.float32) if a.dtype != bool else a for a in view_map(rng, 500, W, H, f)]
    img0 = rng.uniform(0, 1, (H, W, 3))
    imgs = [rng.uniform(0, 1, (H, W, 3)).astype(np.float32) for _ in range(4)]

    a, ea = _mapper(arrays, img0, W, H, f)
    b, eb = _mapper(arrays, img0, W, H, f)
    a.use_graphs = b.use_graphs = graphs
    # first step sizes the pair buffers (synchronous binning) in both
    ha = [a.optimize_keyframe(ea)]
    hb = [b.optimize_keyframe(eb)]
    for im in imgs:
        pinned = torch.from_numpy(im).pin_memory()
        ha.append(a.optimize_keyframe(ea, pinned))
        eb.gt.copy_(torch.from_numpy(im).cuda())
        q = np.clip(np.round(np.clip(im.astype(np.float64), 0, 1) * 255.0), 0, 255)
        eb.gt8.copy_(torch.from_numpy(q.astype(np.uint8)).cuda())
        hb.append(b.optimize_keyframe(eb))
    la, lb = a.collect(ha), b.collect(hb)
    assert len(a.training_log) == 5
    assert [x["iteration"] for x in la] == [y["iteration"] for y in lb]
    assert_logs_identical(la, lb)
    assert_maps_identical(a, b)
    assert torch.equal(ea.gt, eb.gt)


def _scene(seed=5, n=800):
    rng = np.random.default_rng(seed)
    W, H, f = 96, 64, 80.0
    arrays = [a.astype(np.float32) if a.dtype != bool else a for a in view_map(rng, n, W, H, f)]
    img = rng.uniform(0, 1, (H, W, 3))
    return arrays, img, W, H, f


@pytest.mark.parametrize("graphs", [False, True])
def test_tile_caps_match_full_lists(graphs):
    """Lists truncated behind the previous saturation depth (engine.use_caps)
    give the same iterations as full lists."""
    arrays, img, W, H, f = _scene()
    a, ea = _mapper(arrays, img, W, H, f)
    b, eb = _mapper(arrays, img, W, H, f)
    a.use_graphs = b.use_graphs = graphs
    b.engine.use_caps = False
    la = a.collect([a.optimize_keyframe(ea) for _ in range(6)])
    lb = b.collect([b.optimize_keyframe(eb) for _ in range(6)])
    assert_logs_identical(la, lb)
    assert_maps_identical(a, b)
    # the limits did apply somewhere: saturated tiles carry a finite depth limit
    lim = next(iter(a.engine.caps.values()))
    assert int(torch.isfinite(lim).sum()) > 0


def test_tile_caps_too_small_rerun():
    """A depth limit in front of a tile's saturation depth is detected by the
    forward blend (status overflow); that iteration and those queued behind
    it are re-run with full lists -- bitwise the full-list trajectory."""
    arrays, img, W, H, f = _scene(seed=9)
    a, ea = _mapper(arrays, img, W, H, f)
    b, eb = _mapper(arrays, img, W, H, f)
    b.engine.use_caps = False
    la = a.collect([a.optimize_keyframe(ea) for _ in range(2)])
    lb = b.collect([b.optimize_keyframe(eb) for _ in range(2)])
    for lim in a.engine.caps.values():
        lim.fill_(1e-3)                    # in front of every Gaussian
    # the invalid iteration halts the engine: the two queued behind it are
    # device no-ops too (sb_bin / sb_blend_fwd halt flag), all three re-run
    hs = [a.optimize_keyframe(ea) for _ in range(3)]
    flags = [int(h[3][6:8].view(torch.int64)[1].item()) for h in hs]
    assert flags == [1, 1, 1], flags
    la += a.collect(hs)
    assert a.reruns == 3
    lb += b.collect([b.optimize_keyframe(eb) for _ in range(3)])
    assert_logs_identical(la, lb)
    assert_maps_identical(a, b)


def test_render_image_matches_render_view():
    """Mapper.render_image (sync-free device binning, the view's depth
    limits reused across renders, heavy-first schedule) produces exactly
    render_view's targets, including after map updates, and the limits do
    apply (fewer pairs binned once they exist)."""
    rng = np.random.default_rng(12)
    W, H, f = 160, 96, 120.0
    arrays = [a.astype(np.float32) if a.dtype != bool else a
              for a in view_map(rng, 20000, W, H, f, opacity=(0.8, 0.95))]
    img = rng.uniform(0, 1, (H, W, 3))
    mp, entry = _mapper(arrays, img, W, H, f)
    pose, intr = entry.frame.pose, entry.frame.intrinsics
    kept = []
    for it in range(4):
        st = torch.zeros(2, dtype=torch.int64, device="cuda")
        out = mp.engine.render(mp.map, pose, intr, key="t", status=st)
        torch.cuda.synchronize()
        kept.append(int(st[0].item()))
        assert int(st[1].item()) == 0
        ref = mp.render_view(pose, intr)[2]
        got = mp.render_image(pose, intr, key="t")
        for k in ("color", "depth", "transmittance", "n_contrib"):
            np.testing.assert_array_equal(got[k].cpu().numpy(),
                                          getattr(ref, k).cpu().numpy(), err_msg=k)
        if it == 1:
            mp._optimize_step(entry)    # the map changes between renders
    assert min(kept[1:]) < kept[0], kept


def test_render_image_empty_view_and_size_change():
    """render_image with nothing in view (camera turned away: no pairs) and
    after the image size changes (the render path re-sizes itself)."""
    rng = np.random.default_rng(5)
    W, H, f = 96, 64, 80.0
    arrays = [a.astype(np.float32) if a.dtype != bool else a for a in view_map(rng, 3000, W, H, f)]
    mp, entry = _mapper(arrays, rng.uniform(0, 1, (H, W, 3)), W, H, f)
    away = sb.CameraPose(np.diag([-1.0, 1.0, -1.0]), np.zeros(3))    # looking along -z
    intr = entry.frame.intrinsics
    out = mp.render_image(away, intr, key="away")
    ref = mp.render_view(away, intr)[2]
    assert float(out["transmittance"].min().item()) == 1.0
    np.testing.assert_array_equal(out["color"].cpu().numpy(), ref.color.cpu().numpy())
    intr2 = sb.CameraIntrinsics(f, f, 40.0, 30.0, 80, 60)
    for _ in range(2):
        got = mp.render_image(entry.frame.pose, intr2, key="small")
        ref2 = mp.render_view(entry.frame.pose, intr2)[2]
        np.testing.assert_array_equal(got["color"].cpu().numpy(), ref2.color.cpu().numpy())
        np.testing.assert_array_equal(got["n_contrib"].cpu().numpy(),
                                      ref2.n_contrib.cpu().numpy())


def test_hostmem_pinned_huge_pages_upload():
    """hostmem.pinned_from: a pinned CPU tensor that uploads bit-exactly (the
    staging buffer the e2e bench feeds optimize_keyframe from)."""
    from paper_2404_06926_b200 import hostmem
    img = np.random.default_rng(2).uniform(0, 1, (64, 96, 3)).astype(np.float32)
    t = hostmem.pinned_from(img)
    assert t.is_pinned() and t.shape == img.shape
    d = t.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d.cpu().numpy(), img)
