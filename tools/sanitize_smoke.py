"""A small run of every sm_100a kernel family for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck --error-exitcode 99 python tools/sanitize_smoke.py

the public stage API (project, bin, render, loss, deterministic backward,
chain, sparse Adam) in float32 and float64, the mapping engine's step
(eager, then graph replay with depth limits), the keyframe-batch step with
first-touch accumulation and the packed exchange at world 1, map growth and
the render path.  Small scenes: the tools slow kernels down 10-100x."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_06926_b200 as sb  # noqa: E402
from paper_2404_06926_b200.synthetic import view_map  # noqa: E402


def stage_api(dt):
    rng = np.random.default_rng(3)
    W, H, f = 48, 32, 40.0
    arrays = [a.astype(dt) if a.dtype != bool else a for a in view_map(rng, 300, W, H, f)]
    gm = sb.GaussianMap(dtype=dt)
    gm.append_arrays(*arrays)
    pose, intr = sb.CameraPose.identity(), sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    scr = sb.project_gaussians(*[gm.arrays()[k] for k in ("positions", "log_scales", "rotations",
                                                          "opacity_logits", "sh_coeffs")],
                               pose, intr)
    grid = sb.bin_and_sort(scr, intr)
    t = sb.render(grid, scr, intr)
    img = rng.uniform(0, 1, (H, W, 3))
    _, d_r, _, _ = sb.photometric_loss(t.color, img, sb.ExposureAffine.identity(), 0.2)
    buf = sb.backward_per_gaussian(t, d_r, scr, grid, gm, pose, intr)
    st = sb.AdamState(gm.count, {"position": 1e-3, "log_scale": 1e-3, "rotation": 1e-3,
                                 "opacity_logit": 1e-2, "sh0": 1e-3, "sh_rest": 1e-4}, dtype=dt)
    a = gm.arrays()
    sb.adam_step({"position": a["positions"], "log_scale": a["log_scales"],
                  "rotation": a["rotations"], "opacity_logit": a["opacity_logits"],
                  "sh": a["sh_coeffs"]},
                 {"position": buf.d_position, "log_scale": buf.d_log_scale,
                  "rotation": buf.d_rotation, "opacity_logit": buf.d_opacity_logit,
                  "sh": buf.d_sh}, st, active=np.arange(0, gm.count, 2))


def engine_and_batch():
    rng = np.random.default_rng(5)
    W, H, f = 64, 48, 56.0
    arrays = [a.astype(np.float32) if a.dtype != bool else a for a in view_map(rng, 800, W, H, f)]
    cfg = sb.MapperConfig(scene_extent=1.0, sky_enabled=False)
    mp = sb.Mapper(cfg)
    mp.map.append_arrays(*arrays)
    mp.scene_extent = 1.0
    mp.adam = sb.AdamState(mp.map.count, mp._lrs())
    intr = sb.CameraIntrinsics(f, f, W / 2, H / 2, W, H)
    e = mp.store.add(sb.CameraFrame(pose=sb.CameraPose.identity(), intrinsics=intr,
                                    image=rng.uniform(0, 1, (H, W, 3))), cfg.lr_exposure)
    mp.collect([mp.optimize_keyframe(e) for _ in range(4)])     # eager, then graphs + limits
    mp.render_image(e.frame.pose, intr, key="v")
    mp.render_image(e.frame.pose, intr, key="v")
    import torch.distributed as dist
    from paper_2404_06926_b200.batch import DeviceBatchCompute, PackedBatchStep
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        step = PackedBatchStep(DeviceBatchCompute(mp), always_reduce=True, lazy=True)
        for _ in range(4):
            step.step([e])
        step.flush()
    finally:
        dist.destroy_process_group()
    # growth: append rows, step again (re-sizing)
    mp.map.append_arrays(*[a[:50] for a in arrays])
    mp.adam.resize(mp.map.count)
    mp.collect([mp.optimize_keyframe(e) for _ in range(2)])


if __name__ == "__main__":
    torch.cuda.set_device(0)
    stage_api(np.float32)
    stage_api(np.float64)
    engine_and_batch()
    torch.cuda.synchronize()
    print("sanitize smoke ok")
