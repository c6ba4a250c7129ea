"""Image metrics and the per-view evaluation path on the device (SURVEY §8f
row 3): metrics.py:12-34 (psnr_8bit on 8-bit quantised images, SSIM on
floats) and the body of cli.py:_render_views (render, exposure-compensate,
clip, score)."""

from __future__ import annotations

import math

import torch

from . import _native as N
from .loss import ExposureAffine, apply_exposure, exposure_real, ssim
from .scene import as_device

PSNR_CAP = 99.0


def quantize_8bit(img) -> torch.Tensor:
    """metrics.py:12-13 on the device (sb_quantize8): clip, *255, round half
    to even, uint8, in double like numpy."""
    a = img if isinstance(img, torch.Tensor) else as_device(img)
    if a.dtype not in (torch.float32, torch.float64):
        a = a.to(torch.float64)
    a = a.contiguous()
    q = torch.empty(a.shape, dtype=torch.uint8, device=a.device)
    N.call("sb_quantize8", N.dtype_code(a.dtype), a.numel(), N.ptr(a), N.ptr(q), N.stream_ptr())
    return q


def psnr_8bit(a, b) -> float:
    """metrics.py:16-27: PSNR of two [0, 1] images after 8-bit quantisation,
    capped at 99 dB (identical images).  The squared error is the integer
    reduction of sb_psnr8_sse."""
    x = a if isinstance(a, torch.Tensor) else as_device(a)
    x = x.contiguous()
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    q = quantize_8bit(b).contiguous()
    npx = x.numel() // 3
    sse = torch.zeros(1, dtype=torch.int64, device=x.device)
    e = exposure_real(ExposureAffine.identity(), x.dtype, x.device)
    N.call("sb_psnr8_sse", N.dtype_code(x.dtype), npx, N.ptr(x), N.ptr(e), N.ptr(q), N.ptr(sse),
           N.stream_ptr())
    mse = int(sse.item()) / (3.0 * npx)
    if mse == 0.0:
        return PSNR_CAP
    return min(10.0 * math.log10(255.0 ** 2 / mse), PSNR_CAP)


def ssim_metric(a, b) -> float:
    """metrics.py:30-34: mean SSIM of two (H, W, 3) images, in float64."""
    x = (a if isinstance(a, torch.Tensor) else as_device(a)).to(torch.float64)
    return ssim(x, as_device(b, torch.float64))


def evaluate_view(mapper, pose, intr, gt, exposure=None) -> dict:
    """cli.py:_render_views for one view: render the map, apply the view's
    exposure (identity for novel views), clip to [0, 1], score against the
    ground truth.  Returns psnr, ssim and the compensated image (device)."""
    _, _, targets = mapper.render_view(pose, intr)
    E = ExposureAffine.identity() if exposure is None else exposure
    img = torch.clamp(apply_exposure(E, targets.color), 0.0, 1.0)
    return {"psnr": psnr_8bit(img, gt), "ssim": ssim_metric(img, gt), "image": img,
            "targets": targets}


__all__ = ["PSNR_CAP", "evaluate_view", "psnr_8bit", "quantize_8bit", "ssim_metric"]
