"""Record a small incremental-mapping stream from the REFERENCE (splatmap).

Run in the build container only (the reference lives at /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_stream.py

A seeded 16-frame stream (64x48 images, a teacher map's centres as the frame
points, 300-Gaussian sky) is fed to ``splatmap.Mapper.process_frame``
(mapper.py:332-374) with keyframes every 5 frames, 3 replayed keyframes per
round and 2 rounds per keyframe.  Recorded in ``tests/golden/stream/stream16.npz``:

* the inputs: poses, intrinsics, images and points of every frame, the config;
* after every frame: map.count and len(training_log);
* for every keyframe: the rendered opacity the expansion mask is taken from
  (mapper.py:252-257) and the rows ``expand`` appended (mapper.py:259-281,
  _seed_arrays 106-118), as seeded -- read before the frame's first
  optimize_map;
* the bootstrap rows (first-frame points + init_sky, mapper.py:124-161, 214-233),
  likewise before optimisation;
* the whole training log (iteration, keyframe, l1, dssim, loss, psnr) -- the
  keyframe column is optimize_map's seeded sample-and-shuffle order
  (mapper.py:285-297);
* the final map.

tests/test_gpu_stream.py replays the same frames through this package.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from splatmap import mapper as ref_mapper  # noqa: E402
from splatmap import scene as ref_scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

W, H, F = 64, 48, 56.0
N_FRAMES = 16
CFG = dict(sky_count=300, sky_radius=100.0, keyframe_interval=5, replay_keyframes=3,
           iterations_per_keyframe=2, mask_threshold=0.99)


def teacher(rng, n=3000):
    z = rng.uniform(4.0, 12.0, n)
    u = rng.uniform(-8, W + 8, n)
    v = rng.uniform(-6, H + 6, n)
    pos = np.stack([(u - W / 2) * z / F, (v - H / 2) * z / F, z], axis=1)
    rgb = rng.uniform(0.05, 0.95, (n, 3))
    return pos, rgb


def frames():
    rng = np.random.default_rng(2024)
    pos, rgb = teacher(rng)
    out = []
    for i in range(N_FRAMES):
        yaw = 0.012 * i
        R = np.array([[np.cos(yaw), 0.0, np.sin(yaw)], [0.0, 1.0, 0.0],
                      [-np.sin(yaw), 0.0, np.cos(yaw)]])
        t = np.array([0.02 * i, 0.0, 0.0])
        img = rng.integers(0, 256, (H, W, 3)) / 255.0     # exact in the uint8 fixture
        sel = rng.choice(pos.shape[0], 120, replace=False)
        out.append((R, t, img, pos[sel], rgb[sel]))
    return out


class RecordingMapper(ref_mapper.Mapper):
    """The reference Mapper, snapshotting the map when a frame's first
    optimisation round starts (the rows as seeded)."""

    snap = None

    def optimize_map(self):
        if self.snap is None:
            self.snap = {k: np.asarray(getattr(self.map, k)).copy()
                         for k in ("positions", "log_scales", "rotations", "opacity_logits",
                                   "sh_coeffs")}
        return super().optimize_map()


def main():
    cfg = ref_mapper.MapperConfig(**CFG)
    mp = RecordingMapper(cfg, seed=0, dtype=np.float32)
    intr = ref_scene.CameraIntrinsics(fx=F, fy=F, cx=W / 2, cy=H / 2, width=W, height=H)
    rec = {"W": W, "H": H, "F": F, "cfg_keys": np.array(list(CFG)),
           "cfg_vals": np.array([float(v) for v in CFG.values()])}
    counts, logs_len = [], []
    kf_opacity, kf_index = [], []
    add_rows = {k: [] for k in ("positions", "log_scales", "rotations", "opacity_logits",
                                "sh_coeffs")}
    add_frame = []
    Rs, ts, imgs, pts, rgbs, npts = [], [], [], [], [], []
    for i, (R, t, img, p, c) in enumerate(frames()):
        pose = ref_scene.CameraPose(R, t)
        frame = ref_scene.CameraFrame(
            pose=pose, intrinsics=intr, image=img,
            points=[ref_scene.ColoredPoint(p[k], c[k]) for k in range(p.shape[0])],
            frame_index=i)
        is_kf = i % cfg.keyframe_interval == 0
        if is_kf and i > 0:
            _, _, tg = mp.render_view(pose, intr)
            kf_opacity.append(np.asarray(tg.opacity, np.float32))
            kf_index.append(i)
        before = mp.map.count
        mp.snap = None
        mp.process_frame(frame)
        after = mp.map.count
        if after > before:
            for k in add_rows:
                add_rows[k].append(mp.snap[k][before:after].copy())
            add_frame += [i] * (after - before)
        counts.append(after)
        logs_len.append(len(mp.training_log))
        Rs.append(R)
        ts.append(t)
        imgs.append(img)
        pts.append(p)
        rgbs.append(c)
        npts.append(p.shape[0])
    rec.update(R=np.array(Rs), t=np.array(ts),
               images_u8=np.round(np.array(imgs) * 255.0).astype(np.uint8),
               points=np.concatenate(pts),
               rgbs=np.concatenate(rgbs), n_points=np.array(npts), counts=np.array(counts),
               logs_len=np.array(logs_len), kf_opacity=np.array(kf_opacity),
               kf_index=np.array(kf_index), add_frame=np.array(add_frame),
               scene_extent=np.float64(mp.scene_extent))
    for k, v in add_rows.items():
        rec["add_" + k] = np.concatenate(v)
    log = mp.training_log
    rec["log_iteration"] = np.array([r["iteration"] for r in log])
    rec["log_keyframe"] = np.array([r["keyframe"] for r in log])
    for k in ("l1", "dssim", "loss", "psnr"):
        rec["log_" + k] = np.array([float(r[k]) for r in log])
    for k in add_rows:
        rec["final_" + k] = np.asarray(getattr(mp.map, k)).copy()
    rec["final_is_sky"] = np.asarray(mp.map.is_sky).copy()
    path = os.path.join(OUT, "stream", "stream16.npz")
    np.savez_compressed(path, **rec)
    print(path, "frames", N_FRAMES, "final count", counts[-1], "log rows", len(log),
          "added", len(add_frame))


if __name__ == "__main__":
    main()
