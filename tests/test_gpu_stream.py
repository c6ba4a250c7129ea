"""The incremental mapping loop and map growth against a run of the REFERENCE
(VERDICT r1 #7): tests/golden/stream/stream16.npz was recorded from
splatmap.Mapper.process_frame by tests/golden/make_stream.py.

The same 16 frames go through this package's Mapper.process_frame
(mapper.py:332-374).  Checked:

* bootstrap (first-frame points + the seeded sky shell, mapper.py:124-161,
  214-233) and every keyframe's expansion (mapper.py:245-281): map.count after
  every frame and the appended rows as seeded (before the frame's first
  optimisation round) BIT-EXACT (float64 seed arithmetic cast to float32,
  _seed_arrays 106-118); the expansion mask's rendered opacity against the
  reference's to the float noise of two optimised float32 maps, every pixel
  whose mask bit differs explained by that noise (the reference's opacity
  closer to the 0.99 threshold than the two renders are to each other);
* optimize_map's seeded sample-and-shuffle order (mapper.py:285-297) and the
  training log's iteration numbers: exact; its losses to the float noise of
  two float32 trajectories (the reference's own f32/f64 drift);
* render_view / render_image with include_sky=False (mapper.py:202-204)
  against the oracle's render of the non-sky rows.
"""

import os

import numpy as np
import pytest

from parity import GOLDEN, oracle

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def stream():
    import paper_2404_06926_b200 as sb
    z = dict(np.load(os.path.join(GOLDEN, "stream", "stream16.npz")))
    cfg_kw = {str(k): v for k, v in zip(z["cfg_keys"], z["cfg_vals"])}
    cfg_kw = {k: (int(v) if k in ("sky_count", "keyframe_interval", "replay_keyframes",
                                  "iterations_per_keyframe") else float(v))
              for k, v in cfg_kw.items()}
    cfg = sb.MapperConfig(**cfg_kw)
    mp = sb.Mapper(cfg, seed=0)
    W, H, F = int(z["W"]), int(z["H"]), float(z["F"])
    intr = sb.CameraIntrinsics(F, F, W / 2, H / 2, W, H)
    out = {"z": z, "counts": [], "logs_len": [], "opacity": [], "added": {}, "mp": mp,
           "intr": intr}
    snap = {}
    plain = mp.optimize_map

    def optimize_map():          # the rows as seeded: before the first round
        if not snap:
            snap.update({k: _np(v).copy() for k, v in mp.map.arrays().items()})
        return plain()
    mp.optimize_map = optimize_map
    off = 0
    for i in range(len(z["counts"])):
        n = int(z["n_points"][i])
        pts = [sb.ColoredPoint(z["points"][off + k], z["rgbs"][off + k]) for k in range(n)]
        off += n
        pose = sb.CameraPose(z["R"][i], z["t"][i])
        img = z["images_u8"][i].astype(np.float64) / 255.0
        if i in set(z["kf_index"].tolist()):
            out["opacity"].append(_np(mp.render_view(pose, intr)[2].opacity).copy())
        before = mp.map.count
        snap.clear()
        mp.process_frame(sb.CameraFrame(pose=pose, intrinsics=intr, image=img, points=pts,
                                        frame_index=i))
        after = mp.map.count
        if after > before:
            out["added"][i] = {k: v[before:after].copy() for k, v in snap.items()}
        out["counts"].append(after)
        out["logs_len"].append(len(mp.training_log))
    out["log"] = list(mp.training_log)
    out["final_sky"] = _np(mp.map.is_sky).copy()
    return out


def test_counts_after_every_frame(stream):
    z = stream["z"]
    assert stream["counts"] == z["counts"].tolist()
    assert stream["logs_len"] == z["logs_len"].tolist()


def test_expansion_mask_opacity(stream):
    z = stream["z"]
    thr = 0.99
    for got, want in zip(stream["opacity"], z["kf_opacity"]):
        g, w = got.astype(np.float64), want.astype(np.float64)
        np.testing.assert_allclose(g, w, atol=2e-3)
        flip = (g < thr) != (w < thr)
        assert np.all(np.abs(w[flip] - thr) <= np.abs(g[flip] - w[flip])), int(flip.sum())


def test_appended_rows_bitexact(stream):
    z = stream["z"]
    frames = z["add_frame"]
    for i, rows in stream["added"].items():
        sel = frames == i
        for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
            np.testing.assert_array_equal(rows[k], z["add_" + k][sel], err_msg=f"frame {i} {k}")
    assert sorted(stream["added"]) == sorted(set(frames.tolist()))
    np.testing.assert_array_equal(stream["final_sky"], z["final_is_sky"])


def test_optimize_map_order_and_log(stream):
    z = stream["z"]
    log = stream["log"]
    assert [r["iteration"] for r in log] == z["log_iteration"].tolist()
    assert [r["keyframe"] for r in log] == z["log_keyframe"].tolist()
    got = np.array([r["loss"] for r in log])
    np.testing.assert_allclose(got, z["log_loss"], rtol=2e-3)
    np.testing.assert_allclose([r["l1"] for r in log], z["log_l1"], rtol=2e-3)
    np.testing.assert_allclose([r["psnr"] for r in log], z["log_psnr"], atol=0.05)


def test_render_without_sky(stream):
    """mapper.py:202-204: include_sky=False renders only the non-sky rows."""
    mp, intr = stream["mp"], stream["intr"]
    z = stream["z"]
    o = oracle()
    import paper_2404_06926_b200 as sb
    pose = sb.CameraPose(z["R"][-1], z["t"][-1])
    gm = {k: _np(v).copy() for k, v in mp.map.arrays().items()}
    gm["is_sky"] = _np(mp.map.is_sky).copy()
    assert gm["is_sky"].any() and not gm["is_sky"].all()
    cam = o.Camera(W=z["R"][-1], t=z["t"][-1], fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy,
                   width=intr.width, height=intr.height)
    _, _, ref = o.render_view(gm, cam, include_sky=False)
    _, _, ref_sky = o.render_view(gm, cam, include_sky=True)
    _, _, t = mp.render_view(pose, intr, include_sky=False)
    np.testing.assert_allclose(_np(t.color), ref["color"], atol=1e-6)
    np.testing.assert_array_equal(_np(t.n_contrib), ref["n_contrib"])
    img = mp.render_image(pose, intr, key="nosky", include_sky=False)
    np.testing.assert_array_equal(_np(img["color"]), _np(t.color))
    # the sky does contribute when included
    assert np.abs(ref_sky["color"] - ref["color"]).max() > 1e-3
