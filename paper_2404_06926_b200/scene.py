"""Scene data model on the device: cameras, the Gaussian map store, frustum
culling.  Mirrors ``splatmap.scene`` (scene.py:1-298) with the map's
structure-of-arrays living in HBM as torch tensors.

Layout: positions N x 3, log_scales N x 3, rotations N x 4
(w, x, y, z), opacity_logits N, sh_coeffs N x 16 x 3 (coefficient-major,
channel innermost), is_sky N -- 236 B of float32 per Gaussian, each group one
contiguous allocation so kernels stream it with 16-byte loads.  Buffers are
reserved geometrically up to ``capacity`` (hard cap, CapacityError) so
appends during map growth do not reallocate every keyframe.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N

DEFAULT_CAPACITY = 4_000_000   # scene.py:12
DEFAULT_NEAR = 0.01
DEFAULT_FRUSTUM_MARGIN = 0.1
MAP_MAGIC = b"GMAP"
MAP_VERSION = 1


class CapacityError(RuntimeError):
    """Raised when appending would exceed the map's hard capacity (scene.py:20-21)."""


class PointSource(Enum):
    LIDAR = 0
    SFM = 1


def _device():
    N.load()
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, dtype=None) -> torch.Tensor:
    """numpy/tensor -> contiguous CUDA tensor (no copy if already there)."""
    dev = _device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=dtype if dtype is not None else x.dtype)
    else:
        arr = np.ascontiguousarray(np.asarray(x))
        if not arr.flags.writeable:     # e.g. arrays read from an .npz archive
            arr = arr.copy()
        t = torch.from_numpy(arr).to(device=dev)
        if dtype is not None:
            t = t.to(dtype)
    return t.contiguous()


def torch_dtype(dt) -> torch.dtype:
    if isinstance(dt, torch.dtype):
        return dt
    dt = np.dtype(dt)
    if dt == np.float32:
        return torch.float32
    if dt == np.float64:
        return torch.float64
    raise ValueError(f"unsupported dtype {dt}")


@dataclass
class Gaussian:
    """Single host-side Gaussian (scene.py:29-49)."""

    position: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    opacity_logit: float
    sh_coeffs: np.ndarray
    is_sky: bool = False

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.log_scale = np.asarray(self.log_scale, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.sh_coeffs = np.asarray(self.sh_coeffs, dtype=np.float64).reshape(16, 3)


@dataclass
class CameraIntrinsics:
    """scene.py:51-64."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 < self.cx < self.width and 0 < self.cy < self.height):
            raise ValueError("principal point must lie inside the image")


@dataclass
class CameraPose:
    """World-to-camera transform x_cam = rotation_wc @ x_world + translation_wc
    (scene.py:66-84), kept in float64 on the host."""

    rotation_wc: np.ndarray
    translation_wc: np.ndarray

    def __post_init__(self):
        self.rotation_wc = np.asarray(self.rotation_wc, dtype=np.float64).reshape(3, 3)
        self.translation_wc = np.asarray(self.translation_wc, dtype=np.float64).reshape(3)

    def camera_center(self) -> np.ndarray:
        return -self.rotation_wc.T @ self.translation_wc

    @staticmethod
    def identity() -> "CameraPose":
        return CameraPose(np.eye(3), np.zeros(3))


@dataclass
class ColoredPoint:
    position_w: np.ndarray
    rgb: np.ndarray
    source: PointSource = PointSource.LIDAR

    def __post_init__(self):
        self.position_w = np.asarray(self.position_w, dtype=np.float64).reshape(3)
        self.rgb = np.asarray(self.rgb, dtype=np.float64).reshape(3)


@dataclass
class CameraFrame:
    """scene.py:98-110.  ``image`` may be numpy or a tensor (H, W, 3)."""

    pose: CameraPose
    intrinsics: CameraIntrinsics
    image: object
    points: list = field(default_factory=list)
    frame_index: int = 0
    is_keyframe: bool = False

    def __post_init__(self):
        h, w = tuple(self.image.shape[:2])
        if (h, w) != (self.intrinsics.height, self.intrinsics.width):
            raise ValueError("image dimensions do not match intrinsics")


_GROUPS = (("positions", (3,)), ("log_scales", (3,)), ("rotations", (4,)),
           ("opacity_logits", ()), ("sh_coeffs", (16, 3)))


class GaussianMap:
    """Device structure-of-arrays store (scene.py:113-260).

    Single writer: appends must not overlap a render or step in flight on
    another stream.  ``positions`` etc. are views of the first ``count`` rows.
    """

    def __init__(self, capacity: int = DEFAULT_CAPACITY, dtype=torch.float32,
                 reserve: int = 0):
        self.capacity = int(capacity)
        self.dtype = torch_dtype(dtype)
        self._n = 0
        self._reserved = 0
        self._buf: dict = {}
        self._sky = None
        self._grow(max(int(reserve), 0))

    # --- storage -----------------------------------------------------------
    def _grow(self, rows: int) -> None:
        if rows <= self._reserved and self._buf:
            return
        dev = _device()
        new = {}
        for name, shape in _GROUPS:
            t = torch.zeros((rows,) + shape, dtype=self.dtype, device=dev)
            if name in self._buf and self._n:
                t[: self._n] = self._buf[name][: self._n]
            new[name] = t
        sky = torch.zeros(rows, dtype=torch.bool, device=dev)
        if self._sky is not None and self._n:
            sky[: self._n] = self._sky[: self._n]
        self._buf, self._sky, self._reserved = new, sky, rows

    def reserve(self, rows: int) -> None:
        self._grow(min(max(rows, self._reserved), self.capacity))

    @property
    def count(self) -> int:
        return self._n

    def __len__(self) -> int:
        return self._n

    @property
    def positions(self):
        return self._buf["positions"][: self._n]

    @property
    def log_scales(self):
        return self._buf["log_scales"][: self._n]

    @property
    def rotations(self):
        return self._buf["rotations"][: self._n]

    @property
    def opacity_logits(self):
        return self._buf["opacity_logits"][: self._n]

    @property
    def sh_coeffs(self):
        return self._buf["sh_coeffs"][: self._n]

    @property
    def is_sky(self):
        return self._sky[: self._n]

    @property
    def sky_count(self) -> int:
        return int(self.is_sky.sum().item())

    def arrays(self) -> dict:
        return {name: self._buf[name][: self._n] for name, _ in _GROUPS}

    # --- appends (scene.py:134-187) --------------------------------------------
    def append_arrays(self, positions, log_scales, rotations, opacity_logits, sh_coeffs,
                      is_sky) -> int:
        n = int(len(positions))
        if n == 0:
            return self._n
        if self._n + n > self.capacity:
            raise CapacityError(
                f"appending {n} Gaussians would exceed capacity {self.capacity} "
                f"(current count {self._n})")
        need = self._n + n
        if need > self._reserved:
            self._grow(min(self.capacity, max(need, 2 * self._reserved, 1024)))
        lo, hi = self._n, need
        for (name, shape), arr in zip(_GROUPS, (positions, log_scales, rotations, opacity_logits,
                                                sh_coeffs)):
            self._buf[name][lo:hi] = as_device(arr, self.dtype).reshape((n,) + shape)
        self._sky[lo:hi] = as_device(is_sky, torch.bool).reshape(n)
        self._n = hi
        return self._n

    def append(self, gaussians: list) -> int:
        n = len(gaussians)
        if n == 0:
            return self._n
        return self.append_arrays(
            np.array([g.position for g in gaussians]).reshape(n, 3),
            np.array([g.log_scale for g in gaussians]).reshape(n, 3),
            np.array([g.rotation for g in gaussians]).reshape(n, 4),
            np.array([g.opacity_logit for g in gaussians]).reshape(n),
            np.array([g.sh_coeffs for g in gaussians]).reshape(n, 16, 3),
            np.array([g.is_sky for g in gaussians], dtype=bool).reshape(n))

    def get(self, index: int) -> Gaussian:
        return Gaussian(
            position=self.positions[index].double().cpu().numpy(),
            log_scale=self.log_scales[index].double().cpu().numpy(),
            rotation=self.rotations[index].double().cpu().numpy(),
            opacity_logit=float(self.opacity_logits[index].item()),
            sh_coeffs=self.sh_coeffs[index].double().cpu().numpy(),
            is_sky=bool(self.is_sky[index].item()))

    def bounding_box(self):
        if self._n == 0:
            return np.zeros(3), np.zeros(3)
        p = self.positions
        return p.min(dim=0).values.cpu().numpy(), p.max(dim=0).values.cpu().numpy()

    # --- GMAP v1 serialisation, byte-compatible with scene.py:208-251 ---------
    def save(self, path) -> None:
        n = self._n
        with open(path, "wb") as f:
            f.write(MAP_MAGIC)
            f.write(struct.pack("<IQQ", MAP_VERSION, n, self.sky_count))
            for t in (self.positions, self.log_scales, self.rotations, self.opacity_logits,
                      self.sh_coeffs, self.is_sky.to(torch.float32)):
                f.write(np.ascontiguousarray(t.detach().cpu().numpy(), dtype="<f4").tobytes())

    @classmethod
    def load(cls, path, capacity: int = DEFAULT_CAPACITY, dtype=torch.float32) -> "GaussianMap":
        with open(path, "rb") as f:
            magic = f.read(4)
            if magic != MAP_MAGIC:
                raise ValueError(f"not a Gaussian map file (magic {magic!r})")
            version, n, _sky = struct.unpack("<IQQ", f.read(20))
            if version != MAP_VERSION:
                raise ValueError(f"unsupported map version {version}")
            capacity = max(capacity, n)

            def read(shape):
                count = int(np.prod(shape))
                buf = f.read(count * 4)
                if len(buf) != count * 4:
                    raise ValueError("truncated map file")
                return np.frombuffer(buf, dtype="<f4").reshape(shape)

            arrs = [read((n, 3)), read((n, 3)), read((n, 4)), read((n,)), read((n, 16, 3))]
            sky = read((n,)) > 0.5
        m = cls(capacity=capacity, dtype=dtype, reserve=n)
        m.append_arrays(*arrs, sky)
        return m

    def summary(self) -> str:
        lo, hi = self.bounding_box()
        return (f"count = {self.count}\nsky_count = {self.sky_count}\n"
                f"bbox_min = {lo[0]:.6g} {lo[1]:.6g} {lo[2]:.6g}\n"
                f"bbox_max = {hi[0]:.6g} {hi[1]:.6g} {hi[2]:.6g}\n")


def frustum_contains(pose: CameraPose, intr: CameraIntrinsics, point_w,
                     near: float = DEFAULT_NEAR, margin: float = DEFAULT_FRUSTUM_MARGIN) -> bool:
    """Scalar twin (scene.py:263-280), evaluated in float64 on the host."""
    p = np.asarray(point_w, dtype=np.float64).reshape(3)
    pc = pose.rotation_wc @ p + pose.translation_wc
    if pc[2] <= near:
        return False
    u = intr.fx * pc[0] / pc[2] + intr.cx
    v = intr.fy * pc[1] / pc[2] + intr.cy
    mx, my = margin * intr.width, margin * intr.height
    return (-mx <= u <= intr.width - 1 + mx) and (-my <= v <= intr.height - 1 + my)


def frustum_mask(pose: CameraPose, intr: CameraIntrinsics, points_w,
                 near: float = DEFAULT_NEAR, margin: float = DEFAULT_FRUSTUM_MARGIN):
    """a1 (scene.py:283-298) on the device: bool[N] tensor."""
    pts = points_w if isinstance(points_w, torch.Tensor) else as_device(points_w)
    if pts.dtype not in (torch.float32, torch.float64):
        pts = pts.to(torch.float32)
    pts = pts.contiguous()
    n = pts.shape[0]
    out = torch.empty(n, dtype=torch.uint8, device=pts.device)
    cam = N.camera(pose, intr)
    N.call("sb_frustum_mask", N.dtype_code(pts.dtype), n, N.ptr(pts), N.C.byref(cam),
           float(near), float(margin), N.ptr(out), N.stream_ptr())
    return out.bool()
