"""ctypes binding of libsplatb200.so (include/splatb200.h).

This is the ONLY compute backend of the package: there is no CPU fallback.
Importing works anywhere (so the CPU test suite can check the library's
exports), but every call requires a CUDA device and raises RuntimeError
loudly when the extension or the device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsplatb200.so")

SB_OK, SB_ERR_INVALID, SB_ERR_CUDA, SB_ERR_CAPACITY = 0, -1, -2, -3
SB_F32, SB_F64 = 0, 1
RECORD_REALS = 12
TILE = 16

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double
sz = C.c_size_t


class SbCamera(C.Structure):
    _fields_ = [("W", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class SbScreenExtras(C.Structure):
    _fields_ = [(n, vp) for n in ("cov2d", "inv_cov2d", "t_cam", "t_clamped", "clamped_x",
                                  "clamped_y", "view_dir", "basis", "color_raw", "mean2d", "depth",
                                  "color", "opacity", "radius_cut", "q_cut")]


class SbChainScreen(C.Structure):
    _fields_ = [(n, vp) for n in ("inv_cov2d", "t_cam", "t_clamped", "view_dir", "basis",
                                  "color_raw", "opacity", "clamped_x", "clamped_y")]


class SbAdamGroups(C.Structure):
    _fields_ = [("param", vp * 5), ("grad", vp * 5), ("m", vp * 5), ("v", vp * 5)]


# name -> (restype, argtypes)
_SIGS = {
    "sb_version": (i32, []),
    "sb_last_error": (C.c_char_p, []),
    "sb_frustum_mask": (i32, [i32, i64, vp, vp, f64, f64, vp, vp]),
    "sb_preprocess_fwd": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, f64, f64, f64, vp, vp, vp,
                                vp, vp, vp, vp, vp]),
    "sb_pack_records": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sb_bin_workspace_bytes": (sz, [i64, i64, i32, i32]),
    "sb_bin": (i32, [i32, i64, vp, vp, vp, vp, i32, i32, i32, i32, i64, vp, vp, vp, vp, vp, sz,
                     vp, vp, i64, vp, vp]),
    "sb_blend_fwd": (i32, [i32, vp, vp, vp, i32, i32, i32, i32, f64, vp, vp, vp, vp, vp, vp, vp,
                           vp, vp, vp, vp, vp, vp, i32, vp]),
    "sb_loss_workspace_bytes": (sz, [i32, i32]),
    "sb_loss_fused": (i32, [i32, i32, i32, vp, vp, vp, vp, f64, vp, vp, vp, vp, sz, vp]),
    "sb_blend_bwd": (i32, [i32, vp, vp, vp, i32, i32, i32, i32, f64, vp, vp, vp, vp, vp, vp, vp,
                           vp, vp]),
    "sb_blend_bwd_workspace_bytes": (sz, [i32, i64, i32, i32]),
    "sb_blend_bwd_det": (i32, [i32, vp, vp, vp, i32, i32, i32, i32, f64, vp, vp, vp, vp, vp, vp,
                               vp, vp, i64, i64, i64, vp, vp, sz, vp]),
    "sb_blend_bwd_partials": (i32, [i32, vp, vp, vp, i32, i32, i32, i32, f64, vp, vp, vp, vp, i64,
                                    i64, vp, vp, sz, vp]),
    "sb_gather_adjoints": (i32, [i32, i64, i64, i32, i32, i64, vp, vp, sz, vp, vp, vp, vp, vp,
                                 vp]),
    "sb_preprocess_bwd": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                vp, vp, vp]),
    "sb_preprocess_bwd_rows": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, f64, vp, vp, vp, vp,
                                     vp, vp, vp, vp, vp, i32, vp]),
    "sb_sparse_adam": (i32, [i32, i64, vp, vp, vp, vp, vp]),
    "sb_chain_adam_workspace_bytes": (sz, [i32, i64]),
    "sb_chain_adam_rows": (i32, [i32, i64, vp, vp, vp, f64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                 vp, sz, i32, vp, vp]),
    "sb_exposure_adam": (i32, [i32, vp, vp, vp, vp, f64, vp, vp]),
    "sb_apply_exposure": (i32, [i32, i64, vp, vp, vp, vp]),
    "sb_psnr8_sse": (i32, [i32, i64, vp, vp, vp, vp, vp]),
    "sb_quantize8": (i32, [i32, i64, vp, vp, vp]),
    "sb_memset_async": (i32, [vp, i32, sz, vp]),
    "sb_pack_rows": (i32, [i32, i64, vp, vp, i64, vp, vp, vp]),
    "sb_unpack_rows": (i32, [i32, i64, vp, vp, i64, vp, vp]),
    "sb_expand_select": (i32, [i64, vp, vp, f64, i32, vp, f64, vp, vp]),
    "sb_depth_limits_gate": (i32, [vp, i64, vp, vp, i32, vp]),
    "sb_sparse_adam_workspace_bytes": (sz, [i32, i64]),
    "sb_sparse_adam_flat": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp]),
    "sb_chain_accumulate_workspace_bytes": (sz, [i32, i64]),
    "sb_chain_accumulate": (i32, [i32, i64, vp, vp, vp, vp, vp, vp, vp, f64, vp, vp, vp, vp, vp,
                                  vp, vp, vp, vp, vp, i32, vp, vp, sz, vp]),
}

EXPORTS = tuple(_SIGS)
ABI_VERSION = 11100   # sb_version() of the library these signatures describe

_LIB = None


def load(require_cuda: bool = True):
    """Load the extension; with require_cuda also insist on a CUDA device."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2404_06926_b200.build` "
                "(this package has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sb_version() != ABI_VERSION:
            # a stale build with other signatures would be called with the
            # wrong arguments: refuse it
            raise RuntimeError(f"{LIB_PATH} has ABI {lib.sb_version()}, this package needs "
                               f"{ABI_VERSION}: rebuild with `python -m paper_2404_06926_b200.build`")
        _LIB = lib
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2404_06926_b200 needs a CUDA device (sm_100a); none found")
    return _LIB


class CapacityExceeded(Exception):
    def __init__(self, needed):
        super().__init__(f"capacity exceeded, need {needed}")
        self.needed = needed


def check(rc: int, what: str) -> None:
    if rc == SB_OK:
        return
    msg = (_LIB.sb_last_error() or b"").decode(errors="replace")
    if rc == SB_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == SB_ERR_CAPACITY:
        raise CapacityExceeded(msg)
    raise RuntimeError(f"{what}: {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return vp(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return vp(s.cuda_stream)


def dtype_code(dt) -> int:
    import torch
    if dt in (torch.float32, np.float32):
        return SB_F32
    if dt in (torch.float64, np.float64):
        return SB_F64
    raise ValueError(f"unsupported dtype {dt}: float32 (production) or float64 (verification)")


def camera(pose, intr) -> SbCamera:
    s = SbCamera()
    s.W[:] = [float(v) for v in np.asarray(pose.rotation_wc, np.float64).reshape(9)]
    s.t[:] = [float(v) for v in np.asarray(pose.translation_wc, np.float64).reshape(3)]
    s.fx, s.fy = float(intr.fx), float(intr.fy)
    s.cx, s.cy = float(intr.cx), float(intr.cy)
    s.width, s.height = int(intr.width), int(intr.height)
    return s
