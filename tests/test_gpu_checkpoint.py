"""Checkpoint compatibility (mapper.py:378-464): a
checkpoint written by the reference Mapper (tests/golden/ckpt_ref, recorded by
tests/golden/make_checkpoint.py) loads into the B200 Mapper, and saving it
again reproduces the reference's files: map.bin and map_summary.txt byte for
byte, state.npz array for array, mapper.json field for field."""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ckpt_ref")


def test_reference_checkpoint_round_trip(tmp_path):
    import paper_2404_06926_b200 as sb
    cfg = sb.MapperConfig()
    m = sb.Mapper.load_checkpoint(REF, cfg)
    meta = json.loads(open(os.path.join(REF, "mapper.json")).read())
    assert m.global_iteration == meta["global_iteration"] == 42
    assert m.frames_received == 11 and m.last_frame_index == 9
    assert m.map.count == 60 and m.map.sky_count == 3
    assert len(m.store) == 2
    with np.load(os.path.join(REF, "state.npz")) as ref:
        np.testing.assert_array_equal(m.adam.steps.cpu().numpy(), ref["adam_steps"])
        np.testing.assert_array_equal(m.adam.m["sh"].cpu().numpy(), ref["adam_m_sh"])
        for i, e in enumerate(m.store.entries):
            np.testing.assert_array_equal(e.exposure.matrix, ref["kf_exposures"][i])
            st = e.exposure.state.cpu().numpy()
            np.testing.assert_array_equal(st[:12].reshape(3, 4), ref["kf_exp_m"][i])
            np.testing.assert_array_equal(st[12:24].reshape(3, 4), ref["kf_exp_v"][i])
            assert int(st[24]) == int(ref["kf_exp_t"][i])

    out = tmp_path / "ckpt"
    m.save_checkpoint(out)
    for name in ("map.bin", "map_summary.txt"):
        assert open(os.path.join(REF, name), "rb").read() == open(out / name, "rb").read(), name
    with np.load(os.path.join(REF, "state.npz")) as ref, np.load(out / "state.npz") as got:
        assert sorted(ref.files) == sorted(got.files)
        for k in ref.files:
            assert ref[k].dtype == got[k].dtype, k
            np.testing.assert_array_equal(ref[k], got[k], err_msg=k)
    assert json.loads(open(out / "mapper.json").read()) == meta

    # the resumed mapper keeps the reference's RNG stream
    m2 = sb.Mapper.load_checkpoint(out, cfg)
    assert np.array_equal(m.rng.random(5), m2.rng.random(5))
    torch.cuda.synchronize()


def test_resume_equals_uninterrupted(tmp_path):
    """Training resumed from a checkpoint continues bit for bit like the run
    that never stopped: the map, both Adam moments, the step counters and
    the exposure after 6 + 6 iterations of one keyframe.  The loaded Adam
    state rebuilds its touched-row mask from the moments (AdamState.from_dict
    -> moments_written), so the resumed run's touched-row skip elides exactly
    the identity updates the uninterrupted run elides."""
    import paper_2404_06926_b200 as sb
    from paper_2404_06926_b200 import synthetic
    scene = synthetic.config(1)
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False, capacity=scene.n)

    def fresh():
        mp = sb.Mapper(cfg)
        mp.map.append_arrays(*scene.arrays)
        mp.scene_extent = 1.0
        mp.adam = sb.AdamState(mp.map.count, mp._lrs())
        pose = sb.CameraPose(scene.W, scene.t)
        intr = sb.CameraIntrinsics(scene.fx, scene.fy, scene.cx, scene.cy, scene.width,
                                   scene.height)
        entry = mp.store.add(sb.CameraFrame(pose=pose, intrinsics=intr, image=scene.image),
                             cfg.lr_exposure, torch.float32)
        entry.exposure.matrix = scene.E
        return mp, entry

    a, ea = fresh()
    a.collect([a.optimize_keyframe(ea) for _ in range(6)])
    a.save_checkpoint(tmp_path / "ckpt")
    b = sb.Mapper.load_checkpoint(tmp_path / "ckpt", cfg)
    eb = b.store.entries[0]
    a.collect([a.optimize_keyframe(ea) for _ in range(6)])
    b.collect([b.optimize_keyframe(eb) for _ in range(6)])
    torch.cuda.synchronize()
    for k, v in a.map.arrays().items():
        assert torch.equal(v, b.map.arrays()[k]), k
    for g in a.adam._m:
        n = a.adam.count
        assert a.adam._m[g][:n].cpu().numpy().tobytes() == b.adam._m[g][:n].cpu().numpy().tobytes(), g
        assert a.adam._v[g][:n].cpu().numpy().tobytes() == b.adam._v[g][:n].cpu().numpy().tobytes(), g
    assert torch.equal(a.adam.steps, b.adam.steps)
    np.testing.assert_array_equal(ea.exposure.matrix, eb.exposure.matrix)
