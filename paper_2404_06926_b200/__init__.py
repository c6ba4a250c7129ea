"""paper_2404_06926_b200: B200-native (sm_100a) drop-in for the online 3D
Gaussian map-optimisation hot path of Gaussian-LIC (arXiv 2404.06926).

The public names mirror the reference package ``splatmap``
(splatmap/__init__.py:6-32) for the hot path: projection, binning, blend,
loss, backward, sparse Adam and the Mapper step.  Everything computes in
libsplatb200.so (hand-written CUDA for sm_100a, csrc/); there is no CPU
fallback -- calls raise RuntimeError without a CUDA device or the library.
"""

__version__ = "0.1.0"

from .adam import AdamState, ScalarAdam, adam_step  # noqa: F401
from .backward import GradientBuffer, backward_per_gaussian, backward_per_pixel  # noqa: F401
from .engine import DeviceExposure, MappingEngine  # noqa: F401
from .forward import RenderTargets, TileGrid, bin_and_sort, render  # noqa: F401
from .loss import ExposureAffine, apply_exposure, photometric_loss, ssim  # noqa: F401
from .mapper import Mapper, MapperConfig, init_sky  # noqa: F401
from .metrics import evaluate_view, psnr_8bit, quantize_8bit, ssim_metric  # noqa: F401
from .projection import SplatScreen, project_gaussians  # noqa: F401
from .scene import (CameraFrame, CameraIntrinsics, CameraPose, CapacityError,  # noqa: F401
                    ColoredPoint, Gaussian, GaussianMap, frustum_contains, frustum_mask)

__all__ = [
    "AdamState", "CameraFrame", "CameraIntrinsics", "CameraPose", "CapacityError",
    "ColoredPoint", "DeviceExposure", "ExposureAffine", "Gaussian", "GaussianMap",
    "GradientBuffer", "Mapper", "MapperConfig", "MappingEngine", "RenderTargets", "ScalarAdam",
    "SplatScreen", "TileGrid", "adam_step", "apply_exposure", "backward_per_gaussian",
    "backward_per_pixel", "bin_and_sort", "frustum_contains", "frustum_mask", "init_sky",
    "photometric_loss", "project_gaussians", "psnr_8bit", "quantize_8bit", "render", "ssim",
    "ssim_metric", "evaluate_view", "__version__",
]
