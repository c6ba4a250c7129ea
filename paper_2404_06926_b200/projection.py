"""Per-Gaussian projection on the device (a2; projection.py:307-392).

``project_gaussians`` keeps the reference signature and returns a compacted
``SplatScreen`` whose rows are the kept Gaussians in map order
(``source_index``), exactly like the reference; every field is a CUDA tensor.
The sm_100a kernel (csrc/preprocess.cu) computes all rows map-indexed in one
pass; compaction is a device gather.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .scene import CameraIntrinsics, CameraPose, as_device

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
DILATION_FLOOR = 0.3        # projection.py:21
ALPHA_CLAMP = 0.99          # projection.py:22
ALPHA_CUTOFF = 1.0 / 255.0  # projection.py:23
FRUSTUM_GUARD = 1.3         # projection.py:27


def rgb_to_sh0(rgb):
    return (np.asarray(rgb) - 0.5) / SH_C0


def sh0_to_rgb(coeff):
    return np.asarray(coeff) * SH_C0 + 0.5


def logit(p: float) -> float:
    return float(np.log(p) - np.log1p(-p))


@dataclass
class ProjectedGaussian:
    """Scalar screen-space Gaussian (projection.py:228-239), host float64."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    inv_cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    source_index: int = 0


class SplatScreen:
    """Per-view projected Gaussians (projection.py:251-290), device SoA."""

    FIELDS = ("mean2d", "cov2d", "inv_cov2d", "depth", "color", "opacity", "source_index",
              "t_cam", "t_clamped", "clamped_x", "clamped_y", "view_dir", "basis", "color_raw",
              "radius_cut", "q_cut")

    def __init__(self, mean2d, cov2d, inv_cov2d, depth, color, opacity, source_index, t_cam,
                 t_clamped, clamped_x, clamped_y, view_dir, basis, color_raw, radius_cut, q_cut):
        dt = mean2d.dtype if isinstance(mean2d, torch.Tensor) else None
        if dt is None:
            dt = torch.float64 if np.asarray(mean2d).dtype == np.float64 else torch.float32

        def f(x, shape_tail):
            t = as_device(x, dt)
            return t.reshape((-1,) + shape_tail)

        self.mean2d = f(mean2d, (2,))
        m = self.mean2d.shape[0]
        self.cov2d = f(cov2d, (2, 2))
        self.inv_cov2d = f(inv_cov2d, (2, 2))
        self.depth = f(depth, ())
        self.color = f(color, (3,))
        self.opacity = f(opacity, ())
        self.source_index = as_device(source_index, torch.int64).reshape(m)
        self.t_cam = f(t_cam, (3,))
        self.t_clamped = f(t_clamped, (3,))
        self.clamped_x = as_device(clamped_x, torch.bool).reshape(m)
        self.clamped_y = as_device(clamped_y, torch.bool).reshape(m)
        self.view_dir = f(view_dir, (3,))
        self.basis = f(basis, (16,))
        self.color_raw = f(color_raw, (3,))
        self.radius_cut = f(radius_cut, ())
        self.q_cut = f(q_cut, ())

    @property
    def dtype(self):
        return self.mean2d.dtype

    def __len__(self) -> int:
        return self.mean2d.shape[0]

    def get(self, i: int) -> ProjectedGaussian:
        return ProjectedGaussian(
            mean2d=self.mean2d[i].double().cpu().numpy(), cov2d=self.cov2d[i].double().cpu().numpy(),
            inv_cov2d=self.inv_cov2d[i].double().cpu().numpy(), depth=float(self.depth[i]),
            color=self.color[i].double().cpu().numpy(), opacity=float(self.opacity[i]),
            source_index=int(self.source_index[i]))

    def records(self):
        """Pack the binning/blend record (12 reals/row) + depth sort keys."""
        m = len(self)
        dev = self.mean2d.device
        rec = torch.empty((max(m, 1), N.RECORD_REALS), dtype=self.dtype, device=dev)
        valid = torch.empty(max(m, 1), dtype=torch.uint8, device=dev)
        kdt = torch.int64 if self.dtype == torch.float64 else torch.int32
        keys = torch.empty(max(m, 1), dtype=kdt, device=dev)
        vals = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        if m:
            # keep every contiguous copy alive across the call (a temporary
            # freed while building the argument list could be reused by the next)
            fields = [t.contiguous() for t in (self.mean2d, self.inv_cov2d, self.opacity,
                                               self.q_cut, self.radius_cut, self.color,
                                               self.depth)]
            N.call("sb_pack_records", N.dtype_code(self.dtype), m, *[N.ptr(t) for t in fields],
                   N.ptr(rec), N.ptr(valid), N.ptr(keys), N.ptr(vals), N.stream_ptr())
        return rec, valid, keys, vals


def project_gaussians(positions, log_scales, rotations, opacity_logits, sh_coeffs,
                      pose: CameraPose, intr: CameraIntrinsics, near: float = 0.01,
                      dilation: float = DILATION_FLOOR, select=None) -> SplatScreen:
    """projection.py:307-392 on the device."""
    pos = positions if isinstance(positions, torch.Tensor) else as_device(positions)
    dt = pos.dtype
    n = pos.shape[0]
    args = [as_device(a, dt) for a in (pos, log_scales, rotations, opacity_logits, sh_coeffs)]
    dev = args[0].device
    sel = None
    if select is not None:
        s = select if isinstance(select, torch.Tensor) else torch.from_numpy(np.asarray(select))
        s = s.to(dev)
        if s.dtype == torch.bool:
            sel = s.to(torch.uint8).contiguous()
        else:
            sel = torch.zeros(n, dtype=torch.uint8, device=dev)
            sel[s.long()] = 1
    E = lambda *shape: torch.empty((max(n, 1),) + shape, dtype=dt, device=dev)  # noqa: E731
    out = {"cov2d": E(2, 2), "inv_cov2d": E(2, 2), "t_cam": E(3), "t_clamped": E(3),
           "view_dir": E(3), "basis": E(16), "color_raw": E(3), "mean2d": E(2), "depth": E(),
           "color": E(3), "opacity": E(), "radius_cut": E(), "q_cut": E()}
    out["clamped_x"] = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    out["clamped_y"] = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    ex = N.SbScreenExtras(**{k: v.data_ptr() for k, v in out.items()})
    rec = E(N.RECORD_REALS)
    valid = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    kdt = torch.int64 if dt == torch.float64 else torch.int32
    keys = torch.empty(max(n, 1), dtype=kdt, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cam = N.camera(pose, intr)
    if n:
        N.call("sb_preprocess_fwd", N.dtype_code(dt), n, *[N.ptr(a) for a in args], N.ptr(sel),
               N.C.byref(cam), float(near), float(dilation), 0.1, N.ptr(rec), N.ptr(valid),
               N.ptr(keys), N.ptr(vals), None, N.C.byref(ex), None, N.stream_ptr())
    idx = torch.nonzero(valid[:n]).squeeze(1)
    f = {k: v[:n].index_select(0, idx) for k, v in out.items()}
    return SplatScreen(mean2d=f["mean2d"], cov2d=f["cov2d"], inv_cov2d=f["inv_cov2d"],
                       depth=f["depth"], color=f["color"], opacity=f["opacity"],
                       source_index=idx, t_cam=f["t_cam"], t_clamped=f["t_clamped"],
                       clamped_x=f["clamped_x"].bool(), clamped_y=f["clamped_y"].bool(),
                       view_dir=f["view_dir"], basis=f["basis"], color_raw=f["color_raw"],
                       radius_cut=f["radius_cut"], q_cut=f["q_cut"])


def sigmoid(x):
    """projection.py:293-300 (host helper)."""
    x = np.asarray(x)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out
