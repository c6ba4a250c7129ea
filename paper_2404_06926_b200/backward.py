"""Backward rasteriser and chain rule on the device (a6, a7).

backward_per_gaussian: backward.py:516-527 -> csrc/blend_bwd.cu (pixel stage)
+ csrc/preprocess.cu (chain to parameters).  The reference's two pixel-stage
variants (per-pixel and per-(tile, Gaussian)) compute the same function; on
the GPU one kernel serves both names: each CTA replays its tile front to back
with one thread per pixel and reduces the per-Gaussian adjoints with warp
shuffles (the per-Gaussian privatisation of backward.py realised in
registers and shared memory); the per-(tile, Gaussian) sums are then merged
per row in ascending tile order (backward.py:92-98) through the binning's
pair slot map (sb_blend_bwd_det): deterministic, no float atomics.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .forward import _SCRATCH, TERMINATION_THRESHOLD, RenderTargets, TileGrid
from .projection import SplatScreen
from .scene import CameraIntrinsics, CameraPose, GaussianMap, as_device


@dataclass
class GradientBuffer:
    """Per-parameter gradients aligned with the GaussianMap (backward.py:30-50)."""

    d_position: torch.Tensor
    d_log_scale: torch.Tensor
    d_rotation: torch.Tensor
    d_opacity_logit: torch.Tensor
    d_sh: torch.Tensor
    d_exposure: object = field(default=None)

    @classmethod
    def zeros(cls, n: int, dtype=torch.float32, device=None) -> "GradientBuffer":
        if not isinstance(dtype, torch.dtype):
            dtype = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        dev = device if device is not None else torch.device("cuda")
        z = lambda *s: torch.zeros(s, dtype=dtype, device=dev)  # noqa: E731
        return cls(z(n, 3), z(n, 3), z(n, 4), z(n), z(n, 16, 3), np.zeros((3, 4)))


def pixel_stage(targets: RenderTargets, d_color_image, screen: SplatScreen, grid: TileGrid,
                intr: CameraIntrinsics, early_termination=True,
                term_threshold=TERMINATION_THRESHOLD):
    """Screen-space adjoints per screen row: (d_mean2d M x 2, d_conic M x 3
    (aa, ab, cc), d_opacity M, d_color M x 3)."""
    dt = screen.dtype
    m = len(screen)
    dev = screen.mean2d.device
    out = [torch.zeros((max(m, 1),) + s, dtype=dt, device=dev) for s in ((2,), (3,), (), (3,))]
    if grid.n_pairs and m:
        rec = grid.records if grid.records is not None else screen.records()[0]
        dC = as_device(d_color_image, dt)
        cf = targets.color.contiguous()
        same = (bool(early_termination) == targets.early_termination
                and float(term_threshold) == targets.term_threshold)
        last = targets.last if (same and targets.last is not None) else None
        if grid.bin_workspace is None:
            raise ValueError("TileGrid carries no binning workspace (make it with bin_and_sort)")
        code = N.dtype_code(dt)
        wsb = N.load().sb_blend_bwd_workspace_bytes(code, grid.bin_capacity, intr.width,
                                                     intr.height)
        ws = _SCRATCH.get("bwd", wsb, dev)
        N.call("sb_blend_bwd_det", code, N.ptr(rec), N.ptr(grid.pair_gaussian32),
               N.ptr(grid.offsets32), intr.width, intr.height, 16, int(bool(early_termination)),
               float(term_threshold), N.ptr(dC), N.ptr(cf), N.ptr(last), *[N.ptr(t) for t in out],
               None, grid.bin_rows, grid.bin_capacity, 0, N.ptr(grid.bin_workspace), N.ptr(ws),
               ws.numel(), N.stream_ptr())
    return [t[:m] for t in out]


def _chain(adj, screen: SplatScreen, gmap, pose, intr) -> GradientBuffer:
    arrays = _map_arrays(gmap)
    dt = arrays["positions"].dtype
    n = arrays["positions"].shape[0]
    buf = GradientBuffer.zeros(n, dtype=dt, device=arrays["positions"].device)
    m = len(screen)
    if m == 0:
        return buf
    # hold contiguous copies for the duration of the launch
    f = {k: getattr(screen, k).contiguous() for k in ("inv_cov2d", "t_cam", "t_clamped",
                                                      "view_dir", "basis", "color_raw", "opacity")}
    f["clamped_x"] = screen.clamped_x.to(torch.uint8).contiguous()
    f["clamped_y"] = screen.clamped_y.to(torch.uint8).contiguous()
    sc = N.SbChainScreen(**{k: v.data_ptr() for k, v in f.items()})
    cam = N.camera(pose, intr)
    src = screen.source_index.contiguous()
    N.call("sb_preprocess_bwd", N.dtype_code(dt), m, N.ptr(src),
           N.ptr(arrays["positions"]), N.ptr(arrays["log_scales"]), N.ptr(arrays["rotations"]),
           N.ptr(arrays["sh_coeffs"]), N.C.byref(sc), *[N.ptr(a) for a in adj],
           N.C.byref(cam), N.ptr(buf.d_position), N.ptr(buf.d_log_scale), N.ptr(buf.d_rotation),
           N.ptr(buf.d_opacity_logit), N.ptr(buf.d_sh), N.stream_ptr())
    return buf


def _map_arrays(gmap) -> dict:
    if isinstance(gmap, GaussianMap):
        return gmap.arrays()
    dt = None
    out = {}
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        v = getattr(gmap, k)
        t = v if isinstance(v, torch.Tensor) else as_device(v)
        if dt is None:
            dt = t.dtype
        out[k] = t.to(dt).contiguous()
    return out


def backward_per_gaussian(targets: RenderTargets, d_color_image, screen: SplatScreen,
                          grid: TileGrid, gmap, pose: CameraPose, intr: CameraIntrinsics,
                          early_termination: bool = True,
                          term_threshold: float = TERMINATION_THRESHOLD) -> GradientBuffer:
    """backward.py:516-527 on the device."""
    if targets.n_contrib is None:
        raise ValueError("render targets carry no backward state")
    adj = pixel_stage(targets, d_color_image, screen, grid, intr, early_termination,
                      term_threshold)
    return _chain(adj, screen, gmap, pose, intr)


def backward_per_pixel(targets: RenderTargets, d_color_image, screen: SplatScreen,
                       grid: TileGrid, gmap, pose: CameraPose, intr: CameraIntrinsics,
                       early_termination: bool = True,
                       term_threshold: float = TERMINATION_THRESHOLD) -> GradientBuffer:
    """backward.py:503-513: same function; the GPU kernel is shared (module doc)."""
    if targets.n_contrib is None:
        raise ValueError("render targets carry no backward state")
    return backward_per_gaussian(targets, d_color_image, screen, grid, gmap, pose, intr,
                                 early_termination, term_threshold)
