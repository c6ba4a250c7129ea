"""Training objective on the device (a5; loss.py:143-177): fused L1 + D-SSIM
on exposure-compensated renders with exact gradients (csrc/loss.cu)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .forward import _SCRATCH
from .scene import as_device

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


@dataclass
class ExposureAffine:
    """3x4 colour transform [M | b] in float64 on the host (loss.py:17-28)."""

    matrix: np.ndarray

    def __post_init__(self):
        self.matrix = np.asarray(self.matrix, dtype=np.float64).reshape(3, 4)

    @staticmethod
    def identity() -> "ExposureAffine":
        return ExposureAffine(np.concatenate([np.eye(3), np.zeros((3, 1))], axis=1))


def exposure_real(E, dtype, device) -> torch.Tensor:
    """E cast to the working dtype (loss.py:155-158: E.matrix.astype(dt))."""
    m = E.matrix if isinstance(E, ExposureAffine) else np.asarray(E, np.float64)
    return torch.as_tensor(np.asarray(m, np.float64).reshape(12)).to(device=device, dtype=dtype)


def apply_exposure(E, color_image):
    """loss.py:31-36: out = C M^T + b, no clamp."""
    img = color_image if isinstance(color_image, torch.Tensor) else as_device(color_image)
    img = img.contiguous()
    out = torch.empty_like(img)
    e = exposure_real(E, img.dtype, img.device)
    npx = img.numel() // 3
    N.call("sb_apply_exposure", N.dtype_code(img.dtype), npx, N.ptr(img), N.ptr(e), N.ptr(out),
           N.stream_ptr())
    return out


def run_loss(rendered, gt, e_real, lam, y=None, out=None):
    """Launch the fused loss; returns device tensors (d_rendered, d_E f64[12],
    parts f64[4] = loss, l1, dssim, ssim) without synchronising."""
    H, W, _ = rendered.shape
    dev = rendered.device
    o = out if out is not None else {}
    if o.get("d_rendered") is None or o["d_rendered"].shape != rendered.shape \
            or o["d_rendered"].dtype != rendered.dtype:
        o["d_rendered"] = torch.empty_like(rendered)
        o["d_E"] = torch.empty(12, dtype=torch.float64, device=dev)
    if o.get("parts") is None:
        o["parts"] = torch.empty(4, dtype=torch.float64, device=dev)
    wsb = N.load().sb_loss_workspace_bytes(W, H)
    ws = _SCRATCH.get("loss", wsb, dev)
    N.call("sb_loss_fused", N.dtype_code(rendered.dtype), W, H, N.ptr(rendered), N.ptr(y),
           N.ptr(gt), N.ptr(e_real), float(lam), N.ptr(o["d_rendered"]), N.ptr(o["d_E"]),
           N.ptr(o["parts"]), N.ptr(ws), ws.numel(), N.stream_ptr())
    return o


def photometric_loss(rendered, ground_truth, E, lam: float = 0.2):
    """loss.py:143-177.  Returns (loss, d_rendered, d_E, parts) like the
    reference: loss and parts as Python floats (one device sync), d_rendered a
    device tensor, d_E a host (3, 4) array in the working dtype."""
    r = rendered if isinstance(rendered, torch.Tensor) else as_device(rendered)
    if tuple(r.shape) != tuple(ground_truth.shape):
        raise ValueError(
            f"shape mismatch: rendered {tuple(r.shape)} vs gt {tuple(ground_truth.shape)}")
    r = r.contiguous()
    gt = as_device(ground_truth, r.dtype)
    e = exposure_real(E, r.dtype, r.device)
    o = run_loss(r, gt, e, lam)
    parts = o["parts"].cpu().numpy()
    d_E = o["d_E"].cpu().numpy().reshape(3, 4)
    npdt = np.float32 if r.dtype == torch.float32 else np.float64
    return (float(parts[0]), o["d_rendered"], d_E.astype(npdt),
            {"l1": float(parts[1]), "dssim": float(parts[2]), "ssim": float(parts[3])})


def ssim(x, y) -> float:
    """Metric-only mean SSIM (loss.py:137-140), through the fused kernel with
    lam = 1 and identity exposure: loss = (1 - ssim) / 2."""
    a = x if isinstance(x, torch.Tensor) else as_device(x)
    a = a.contiguous()
    if a.dtype not in (torch.float32, torch.float64):
        a = a.to(torch.float64)
    b = as_device(y, a.dtype)
    e = exposure_real(ExposureAffine.identity(), a.dtype, a.device)
    o = run_loss(a, b, e, 1.0)
    return float(o["parts"][3].item())
