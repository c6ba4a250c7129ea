"""Record a small checkpoint written by the reference Mapper
(splatmap/mapper.py:378-419) as a fixture for the checkpoint-compatibility
test (tests/test_gpu_checkpoint.py).

Run in the build container only (the reference lives at /root/reference):

    python tests/golden/make_checkpoint.py

Writes tests/golden/ckpt_ref/{map.bin, map_summary.txt, state.npz,
mapper.json}: a 60-Gaussian map (with a sky row), an Adam state after three
steps over a subset, two keyframes with non-trivial exposures and exposure
Adam states, a point buffer and an advanced RNG.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from splatmap import adam as radam  # noqa: E402
from splatmap.mapper import Mapper, MapperConfig  # noqa: E402
from splatmap.scene import CameraFrame, CameraIntrinsics, CameraPose  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ckpt_ref")


def main():
    rng = np.random.default_rng(17)
    cfg = MapperConfig()
    m = Mapper(cfg, seed=5)
    n = 60
    pos = rng.normal(0, 1, (n, 3)) + np.array([0, 0, 5.0])
    ls = np.log(rng.uniform(0.05, 0.3, (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.normal(0, 1, n)
    sh = rng.normal(0, 0.3, (n, 16, 3))
    sky = np.zeros(n, bool)
    sky[-3:] = True
    m.map.append_arrays(pos.astype(np.float32), ls.astype(np.float32), q.astype(np.float32),
                        op.astype(np.float32), sh.astype(np.float32), sky)
    m.scene_extent = 2.5
    m.adam = radam.AdamState(m.map.count, m._lrs())
    params = m._params()
    for _ in range(3):
        grads = {k: rng.normal(0, 1e-2, v.shape).astype(np.float32) for k, v in params.items()}
        radam.adam_step(params, grads, m.adam, active=rng.uniform(size=n) < 0.7)
    for k in range(2):
        intr = CameraIntrinsics(fx=30.0, fy=30.0, cx=16.0, cy=12.0, width=32, height=24)
        a = 0.1 * k
        R = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
        frame = CameraFrame(pose=CameraPose(R, np.array([0.1 * k, 0.0, 0.0])), intrinsics=intr,
                            image=rng.uniform(0, 1, (24, 32, 3)), points=[],
                            frame_index=3 + 4 * k, is_keyframe=True)
        e = m.store.add(frame, cfg.lr_exposure)
        e.exposure.matrix[:] = e.exposure.matrix + rng.normal(0, 0.02, (3, 4))
        for _ in range(2 + k):
            e.exposure_opt.step(e.exposure.matrix, rng.normal(0, 0.1, (3, 4)))
    m.point_buffer = [rng.normal(0, 1, (7, 6))]
    m.frames_received = 11
    m.last_frame_index = 9
    m.global_iteration = 42
    m.rng.random(13)
    m.save_checkpoint(OUT)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
