"""The mapping iteration as one device pipeline (a1-a10, mapper.py:299-328).

``MappingEngine.step`` runs Mapper._optimize_step's sequence on one stream
with persistent, capacity-sized buffers and no host round trip except the
pair count the radix sort needs:

  K1+K2  sb_preprocess_fwd   frustum mask + projection, map-indexed records
  K3-K5  sb_bin              depth sort, cull+count, scan, emit, tile sort, ranges
  K6     sb_blend_fwd        blend + exposure epilogue (Y = M C + b)
  K7     sb_loss_fused       L1 + D-SSIM, dY -> d_rendered, dE (f64)
  K8     sb_blend_bwd        termination-aware replay, shuffle-reduced atomics
  K9+K10 sb_chain_adam_rows  chain rule fused into the frustum-sparse Adam
  K11    sb_exposure_adam    ScalarAdam in f64 on the device
  log    sb_psnr8_sse        psnr_8bit of clip(exposure(C)) for the training log

The log row (loss, l1, dssim, ssim, psnr-sse) stays on the device; callers
read it back in batches.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .adam import AdamState, lr_vector
from .forward import _SCRATCH, run_bin
from .loss import run_loss
from .scene import GaussianMap

LOG_FIELDS = ("loss", "l1", "dssim", "ssim", "psnr")


class DeviceExposure:
    """Per-keyframe exposure affine E = [M | b] (float64 master copy) and its
    ScalarAdam state, both on the device (loss.py:17-28, adam.py:125-140)."""

    def __init__(self, matrix=None, dtype=torch.float32, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        m = np.concatenate([np.eye(3), np.zeros((3, 1))], 1) if matrix is None else matrix
        self.mat = torch.as_tensor(np.asarray(m, np.float64).reshape(12)).to(dev)
        self.real = self.mat.to(dtype)
        self.state = torch.zeros(25, dtype=torch.float64, device=dev)

    @property
    def matrix(self) -> np.ndarray:
        return self.mat.cpu().numpy().reshape(3, 4)

    @matrix.setter
    def matrix(self, value):
        self.mat.copy_(torch.as_tensor(np.asarray(value, np.float64).reshape(12)))
        self.real.copy_(self.mat.to(self.real.dtype))


class MappingEngine:
    def __init__(self, dtype=torch.float32):
        self.dtype = dtype
        self.bufs: dict = {}
        self.binout: dict = {}
        self.fwd: dict = {}
        self.loss: dict = {}
        self.last_pairs = 0
        self.identity = None

    def _buf(self, name, shape, dtype):
        dev = torch.device("cuda", torch.cuda.current_device())
        t = self.bufs.get(name)
        need = int(np.prod(shape))
        if t is None or t.numel() < need or t.dtype != dtype:
            rows = shape[0]
            grow = (max(int(rows * 1.25), rows),) + tuple(shape[1:])
            t = torch.empty(grow, dtype=dtype, device=dev)
            self.bufs[name] = t
        return t.reshape(-1)[:need].reshape(shape)

    def step(self, gmap: GaussianMap, adam: AdamState, pose, intr, gt, gt8, exposure,
             lam=0.2, near=0.01, margin=0.1, dilation=0.3, early=True, thresh=1e-4,
             lr_exposure=1e-2, update_exposure=True, log_out=None):
        """One mapping iteration; returns the device log row (float64[5])."""
        dt = self.dtype
        code = N.dtype_code(dt)
        n = gmap.count
        W, H = intr.width, intr.height
        dev = gmap.positions.device
        st = N.stream_ptr()
        arrays = gmap.arrays()
        cam = N.camera(pose, intr)
        rec = self._buf("records", (max(n, 1), N.RECORD_REALS), dt)
        valid = self._buf("valid", (max(n, 1),), torch.uint8)
        keys = self._buf("keys", (max(n, 1),), torch.int64 if dt == torch.float64 else torch.int32)
        vals = self._buf("vals", (max(n, 1),), torch.int32)
        frustum = self._buf("frustum", (max(n, 1),), torch.uint8)
        if exposure is None:
            if self.identity is None or self.identity.real.dtype != dt:
                self.identity = DeviceExposure(dtype=dt, device=dev)
            exposure = self.identity
        # K1 + K2
        N.call("sb_preprocess_fwd", code, n, *[N.ptr(arrays[k]) for k in (
            "positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")], None,
            N.C.byref(cam), float(near), float(dilation), float(margin), N.ptr(rec),
            N.ptr(valid), N.ptr(keys), N.ptr(vals), N.ptr(frustum), None, st)
        # K3-K5
        cap = max(int(self.last_pairs * 1.25), 4 * n, 1024)
        pg, pt, off, P = run_bin(dt, n, rec, valid, keys, vals, W, H, True, cap,
                                 out=self.binout)
        self.last_pairs = P
        # K6 + exposure epilogue
        from .forward import run_blend_fwd
        o = run_blend_fwd(dt, rec, pg, off, W, H, early, thresh, exposure.real, out=self.fwd)
        # K7
        lo = run_loss(o["color"], gt, exposure.real, lam, y=o["y"], out=self.loss)
        # K8
        dm = self._buf("d_mean2d", (max(n, 1), 2), dt)
        dc = self._buf("d_conic", (max(n, 1), 3), dt)
        do = self._buf("d_opacity", (max(n, 1),), dt)
        dcol = self._buf("d_color", (max(n, 1), 3), dt)
        for t in (dm, dc, do, dcol):
            N.call("sb_memset_async", N.ptr(t), 0, t.numel() * t.element_size(), st)
        N.call("sb_blend_bwd", code, N.ptr(rec), N.ptr(pg), N.ptr(off), W, H, 16, int(early),
               float(thresh), N.ptr(lo["d_rendered"]), N.ptr(o["color"]), N.ptr(o["last"]),
               N.ptr(dm), N.ptr(dc), N.ptr(do), N.ptr(dcol), st)
        # K9 + K10
        G = adam.groups({"position": arrays["positions"], "log_scale": arrays["log_scales"],
                         "rotation": arrays["rotations"], "opacity_logit": arrays["opacity_logits"],
                         "sh": arrays["sh_coeffs"]}, None)
        lrs = lr_vector(adam.lrs)
        N.call("sb_chain_adam_rows", code, n, N.ptr(valid), N.ptr(frustum), N.C.byref(cam),
               float(dilation), N.ptr(dm), N.ptr(dc), N.ptr(do), N.ptr(dcol), N.C.byref(G),
               N.ptr(adam._steps), lrs.ctypes.data_as(N.vp), st)
        # K11
        if update_exposure and exposure is not self.identity:
            N.call("sb_exposure_adam", code, N.ptr(exposure.mat), N.ptr(exposure.real),
                   N.ptr(lo["d_E"]), N.ptr(exposure.state), float(lr_exposure), st)
        # training-log PSNR (mapper.py:319-327), with the updated exposure
        log = log_out if log_out is not None else torch.empty(6, dtype=torch.float64, device=dev)
        sse = log[5:6].view(torch.int64)
        N.call("sb_memset_async", N.ptr(sse), 0, 8, st)
        if gt8 is not None:
            N.call("sb_psnr8_sse", code, W * H, N.ptr(o["color"]), N.ptr(exposure.real),
                   N.ptr(gt8), N.ptr(sse), st)
        log[:4].copy_(lo["parts"])
        self.last = {"targets": o, "loss": lo, "n_pairs": P, "frustum": frustum[:n],
                     "valid": valid[:n]}
        return log


def log_dict(row: np.ndarray, npx: int) -> dict:
    """Host view of a device log row (metrics.py:16-27 PSNR convention)."""
    sse = int(np.asarray(row[5:6]).view(np.int64)[0])
    mse = sse / (3.0 * npx)
    psnr = 99.0 if mse == 0.0 else min(10.0 * math.log10(255.0 ** 2 / mse), 99.0)
    return {"l1": float(row[1]), "dssim": float(row[2]), "loss": float(row[0]), "psnr": psnr}


def quantize_8bit(img) -> np.ndarray:
    """metrics.py:12-13."""
    a = np.asarray(img)
    return np.clip(np.round(np.clip(a, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)
