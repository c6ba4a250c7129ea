"""Adam with the frustum-restricted sparse mode on the device (a8, a9;
adam.py:1-140).  Per-Gaussian int64 step counters; inactive rows untouched."""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .scene import as_device

BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-15
GROUPS = ("position", "log_scale", "rotation", "opacity_logit", "sh")
SHAPES = {"position": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (),
          "sh": (16, 3)}


def lr_vector(lrs: dict) -> np.ndarray:
    """{position, log_scale, rotation, opacity_logit, sh0, sh_rest} (adam.py:67-73)."""
    return np.array([lrs["position"], lrs["log_scale"], lrs["rotation"], lrs["opacity_logit"],
                     lrs["sh0"], lrs["sh_rest"]], dtype=np.float64)


class AdamState:
    """Moments parallel to the GaussianMap plus per-Gaussian counters (adam.py:20-64)."""

    def __init__(self, count: int, lrs: dict, dtype=torch.float32, reserve: int = 0):
        if not isinstance(dtype, torch.dtype):
            dtype = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        self.lrs = dict(lrs)
        self.dtype = dtype
        self.shapes = SHAPES
        self._n = 0
        self._reserved = 0
        self._m: dict = {}
        self._v: dict = {}
        self._steps = None
        self._touched = None       # uint8 per row: moments possibly non-zero
        self._touched_ok = True    # False: recompute from the moments first
        self._alloc(max(count, reserve))
        self._n = int(count)

    def _alloc(self, rows: int) -> None:
        dev = torch.device("cuda", torch.cuda.current_device())
        N.load()
        for d in (self._m, self._v):
            for g in GROUPS:
                t = torch.zeros((rows,) + SHAPES[g], dtype=self.dtype, device=dev)
                if g in d and self._n:
                    t[: self._n] = d[g][: self._n]
                d[g] = t
        s = torch.zeros(rows, dtype=torch.int64, device=dev)
        tch = torch.zeros(rows, dtype=torch.uint8, device=dev)
        if self._steps is not None and self._n:
            s[: self._n] = self._steps[: self._n]
            tch[: self._n] = self._touched[: self._n]
        self._steps = s
        self._touched = tch
        self._reserved = rows

    @property
    def count(self) -> int:
        return self._n

    @property
    def m(self) -> dict:
        self._touched_ok = False   # the caller may write through these views
        return {g: t[: self._n] for g, t in self._m.items()}

    @property
    def v(self) -> dict:
        self._touched_ok = False
        return {g: t[: self._n] for g, t in self._v.items()}

    def moments_written(self) -> None:
        """The moments were written outside the Adam kernels (a gather, a
        load): the touched-row mask is recomputed before the next step."""
        self._touched_ok = False

    def touched(self) -> torch.Tensor:
        """uint8[reserved]: 1 where a row's moments may be non-zero (the
        touched-row skip of sb_chain_adam_rows / sb_sparse_adam_flat; rows
        with 0 have m = v = +0 exactly).  Kept by the Adam kernels; rebuilt
        from the moments' bits after any outside write."""
        if not self._touched_ok:
            n = self._n
            if n:
                t = torch.zeros(n, dtype=torch.bool, device=self._touched.device)
                it = torch.int32 if self.dtype == torch.float32 else torch.int64
                for d in (self._m, self._v):
                    for g in GROUPS:
                        t |= (d[g][:n].reshape(n, -1).view(it) != 0).any(dim=1)
                self._touched[:n] = t.to(torch.uint8)
            self._touched[n:].zero_()
            self._touched_ok = True
        return self._touched

    @property
    def steps(self):
        return self._steps[: self._n]

    def resize(self, new_count: int) -> None:
        """Grow for appended Gaussians: zero moments, zero steps (adam.py:37-48)."""
        extra = new_count - self._n
        if extra < 0:
            raise ValueError("Adam state cannot shrink")
        if extra == 0:
            return
        if new_count > self._reserved:
            self._alloc(max(new_count, 2 * self._reserved))
        for d in (self._m, self._v):
            for g in GROUPS:
                d[g][self._n:new_count].zero_()
        self._steps[self._n:new_count].zero_()
        self._touched[self._n:new_count].zero_()
        self._n = new_count

    def to_dict(self) -> dict:
        out = {"steps": self.steps.cpu().numpy()}
        for g in GROUPS:
            out[f"m_{g}"] = self._m[g][: self._n].cpu().numpy()
            out[f"v_{g}"] = self._v[g][: self._n].cpu().numpy()
        return out

    @classmethod
    def from_dict(cls, data: dict, lrs: dict, dtype=torch.float32) -> "AdamState":
        st = cls(int(np.asarray(data["steps"]).shape[0]), lrs, dtype=dtype)
        st._steps[: st._n] = as_device(np.asarray(data["steps"], np.int64))
        for g in GROUPS:
            st._m[g][: st._n] = as_device(data[f"m_{g}"], dtype)
            st._v[g][: st._n] = as_device(data[f"v_{g}"], dtype)
        st.moments_written()
        return st

    def groups(self, params: dict, grads: dict | None) -> N.SbAdamGroups:
        G = N.SbAdamGroups()
        for i, g in enumerate(GROUPS):
            p = params[g]
            if not (p.is_contiguous() and p.dtype == self.dtype):
                raise ValueError(f"param {g} must be a contiguous {self.dtype} tensor")
            G.param[i] = p.data_ptr()
            G.grad[i] = grads[g].data_ptr() if grads is not None else None
            G.m[i] = self._m[g].data_ptr()
            G.v[i] = self._v[g].data_ptr()
        return G

    def groups_rows(self, params: dict, grads: dict, lo: int, hi: int) -> N.SbAdamGroups:
        """Group pointers for the row block [lo, hi): parameters and moments
        offset to row lo, gradients given for the block itself."""
        G = N.SbAdamGroups()
        for i, g in enumerate(GROUPS):
            p = params[g]
            if not (p.is_contiguous() and p.dtype == self.dtype):
                raise ValueError(f"param {g} must be a contiguous {self.dtype} tensor")
            G.param[i] = _row_ptr(p, lo)
            G.grad[i] = grads[g].data_ptr()
            G.m[i] = _row_ptr(self._m[g], lo)
            G.v[i] = _row_ptr(self._v[g], lo)
        return G

    def reserve(self, rows: int) -> None:
        """Storage for at least ``rows`` rows (moments and counters)."""
        if rows > self._reserved:
            self._alloc(rows)


def _row_ptr(t: torch.Tensor, lo: int) -> int:
    return t.data_ptr() + lo * t[0].numel() * t.element_size()


def active_mask(active, n: int, device):
    if active is None:
        return None
    a = active if isinstance(active, torch.Tensor) else torch.from_numpy(np.asarray(active))
    a = a.to(device)
    if a.dtype == torch.bool:
        return a.to(torch.uint8).contiguous()
    mask = torch.zeros(n, dtype=torch.uint8, device=device)
    if a.numel():
        mask[a.long()] = 1
    return mask


def adam_step(params: dict, grads: dict, state: AdamState, active=None) -> None:
    """One Adam step over ``params`` in place (adam.py:76-122)."""
    n = state.count
    dev = params["position"].device
    g = {k: (v if isinstance(v, torch.Tensor) else as_device(v)).to(state.dtype).contiguous()
         for k, v in grads.items()}
    mask = active_mask(active, n, dev)
    if mask is not None and not bool(mask.any()):
        return
    G = state.groups(params, g)
    lrs = lr_vector(state.lrs)
    code = N.dtype_code(state.dtype)
    if mask is None:
        N.call("sb_sparse_adam", code, n, N.C.byref(G), N.ptr(state._steps), None,
               lrs.ctypes.data_as(N.vp), N.stream_ptr())
        state.moments_written()    # this kernel keeps no touched-row mask
        return
    from .forward import _SCRATCH
    ws = _SCRATCH.get("sparse_adam", N.load().sb_sparse_adam_workspace_bytes(code, n), dev)
    N.call("sb_sparse_adam_flat", code, n, N.C.byref(G), N.ptr(state._steps), N.ptr(mask), None,
           N.ptr(state.touched()), lrs.ctypes.data_as(N.vp), N.ptr(ws), ws.numel(), None,
           N.stream_ptr())


class ScalarAdam:
    """Plain Adam for the exposure block, float64 (adam.py:125-140).  Host
    object for the drop-in API; the mapping engine keeps its state on the
    device (sb_exposure_adam)."""

    def __init__(self, shape, lr: float, dtype=np.float64):
        self.lr = lr
        self.m = np.zeros(shape, dtype=dtype)
        self.v = np.zeros(shape, dtype=dtype)
        self.t = 0

    def step(self, param: np.ndarray, grad) -> None:
        grad = grad.cpu().numpy() if isinstance(grad, torch.Tensor) else np.asarray(grad)
        self.t += 1
        self.m = BETA1 * self.m + (1 - BETA1) * grad
        self.v = BETA2 * self.v + (1 - BETA2) * grad * grad
        m_hat = self.m / (1 - BETA1 ** self.t)
        v_hat = self.v / (1 - BETA2 ** self.t)
        param -= self.lr * m_hat / (np.sqrt(v_hat) + EPS)
