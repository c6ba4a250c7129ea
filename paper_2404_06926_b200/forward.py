"""Tile binning and forward blend on the device (a3, a4).

bin_and_sort: forward.py:184-255 (csrc/binning.cu)
render:       forward.py:345-368 (csrc/blend.cu)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _native as N
from .projection import SplatScreen
from .scene import CameraIntrinsics

DEFAULT_TILE_SIZE = 16
TERMINATION_THRESHOLD = 1e-4


class Scratch:
    """Grow-only named device byte buffers (the library never allocates)."""

    def __init__(self):
        self._bufs: dict = {}

    def get(self, name: str, nbytes: int, device) -> torch.Tensor:
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes or b.device != device:
            b = torch.empty(max(int(nbytes * 1.25), 256), dtype=torch.uint8, device=device)
            self._bufs[name] = b
        return b


_SCRATCH = Scratch()


@dataclass
class TileGrid:
    """Depth-sorted (tile, row) pairs in CSR layout (forward.py:39-60)."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    pair_gaussian32: torch.Tensor
    pair_tile32: torch.Tensor
    offsets32: torch.Tensor
    records: torch.Tensor = field(default=None, repr=False)
    # the sb_bin workspace that made these pairs (its pair slot map feeds the
    # deterministic backward, sb_blend_bwd_det) and that call's sizes
    bin_workspace: torch.Tensor = field(default=None, repr=False)
    bin_rows: int = 0
    bin_capacity: int = 0

    @property
    def pair_gaussian(self):
        return self.pair_gaussian32.long()

    @property
    def pair_tile(self):
        return self.pair_tile32.long()

    @property
    def offsets(self):
        return self.offsets32.long()

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    @property
    def n_pairs(self) -> int:
        return int(self.pair_gaussian32.shape[0])

    def tile_list(self, tx: int, ty: int):
        t = ty * self.tiles_x + tx
        lo, hi = int(self.offsets32[t]), int(self.offsets32[t + 1])
        return self.pair_gaussian32[lo:hi].long()


@dataclass
class RenderTargets:
    """Rendered images + backward state (forward.py:63-71).  ``last`` is the
    per-pixel replay length recorded by the forward blend."""

    color: torch.Tensor
    depth: torch.Tensor
    opacity: torch.Tensor
    transmittance: torch.Tensor
    n_contrib: torch.Tensor
    last: torch.Tensor = field(default=None, repr=False)
    early_termination: bool = True
    term_threshold: float = TERMINATION_THRESHOLD


def run_bin(dt, m, records, valid, keys, vals, width, height, cull=True, pair_capacity=None,
            scratch: Scratch = _SCRATCH, out=None):
    """sb_bin with one capacity retry.  ``out`` (optional dict) keeps the pair
    buffers across calls and receives the call's workspace and sizes
    (``bin_ws``, ``bin_m``, ``bin_cap``, ``bin_sort_cap``: what
    sb_blend_bwd_det needs).  Returns (pair_gaussian32, pair_tile32,
    offsets32, P)."""
    dev = records.device
    n_tiles = ((width + 15) // 16) * ((height + 15) // 16)
    store = out if out is not None else {}
    if store.get("offsets") is None or store["offsets"].numel() != n_tiles + 1:
        store["offsets"] = torch.empty(n_tiles + 1, dtype=torch.int32, device=dev)
    offsets = store["offsets"]
    cap = max(int(pair_capacity or 0), 1024)
    lib = N.load()
    for attempt in range(2):
        if store.get("pairs_cap", 0) < cap:
            store["pair_gaussian"] = torch.empty(cap, dtype=torch.int32, device=dev)
            store["pair_tile"] = torch.empty(cap, dtype=torch.int32, device=dev)
            store["pairs_cap"] = cap
        cap = store["pairs_cap"]
        pg, pt = store["pair_gaussian"], store["pair_tile"]
        ws = scratch.get("bin", lib.sb_bin_workspace_bytes(m, cap, width, height), dev)
        npairs = N.C.c_int64(0)
        rc = lib.sb_bin(N.dtype_code(dt), m, N.ptr(records), N.ptr(valid), N.ptr(keys),
                        N.ptr(vals), width, height, 16, int(bool(cull)), cap, N.ptr(pg),
                        N.ptr(pt), N.ptr(offsets), N.C.byref(npairs), N.ptr(ws), ws.numel(),
                        None, None, 0, None, N.stream_ptr())
        if rc == N.SB_ERR_CAPACITY and attempt == 0:
            cap = int(npairs.value * 1.25) + 1024
            continue
        N.check(rc, "sb_bin")
        P = int(npairs.value)
        store.update(bin_ws=ws, bin_m=m, bin_cap=cap, bin_sort_cap=0)
        return pg[:P], pt[:P], offsets, P
    raise RuntimeError("sb_bin: capacity retry failed")


def bin_and_sort(screen: SplatScreen, intr: CameraIntrinsics,
                 tile_size: int = DEFAULT_TILE_SIZE, cull: bool = True) -> TileGrid:
    """forward.py:184-255 on the device."""
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValueError(f"tile_size {tile_size} unsupported (sm_100a kernels use 16)")
    rec, valid, keys, vals = screen.records()
    m = len(screen)
    tiles_x = (intr.width + tile_size - 1) // tile_size
    tiles_y = (intr.height + tile_size - 1) // tile_size
    # a private workspace: the grid keeps the slot map its backward reads
    store = {}
    pg, pt, off, _ = run_bin(screen.dtype, m, rec, valid, keys, vals, intr.width, intr.height,
                             cull, scratch=Scratch(), out=store)
    return TileGrid(tile_size, tiles_x, tiles_y, pg, pt, off, records=rec,
                    bin_workspace=store["bin_ws"], bin_rows=m, bin_capacity=store["bin_cap"])


def run_blend_fwd(dt, records, pg, off, width, height, early=True,
                  thresh=TERMINATION_THRESHOLD, exposure=None, out=None, depth_limit=None,
                  status=None, coarse_limit=None, sched=None, halt=None, fast_exp=False):
    dev = records.device
    o = out if out is not None else {}

    def buf(name, shape, tdt):
        t = o.get(name)
        if t is None or tuple(t.shape) != shape or t.dtype != tdt:
            t = torch.empty(shape, dtype=tdt, device=dev)
            o[name] = t
        return t

    H, W = height, width
    c = buf("color", (H, W, 3), dt)
    d = buf("depth", (H, W), dt)
    t = buf("transmittance", (H, W), dt)
    op = buf("opacity", (H, W), dt)
    nc = buf("n_contrib", (H, W), torch.int32)
    last = buf("last", (H, W), torch.int32)
    y = buf("y", (H, W, 3), dt) if exposure is not None else None
    # heavy-first tile schedule: [forward order | replay lengths | backward
    # order], the last two for a following sb_blend_bwd
    n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
    if sched is None:
        if o.get("sched") is None or o["sched"].numel() != 3 * n_tiles:
            o["sched"] = torch.zeros(3 * n_tiles, dtype=torch.int32, device=dev)
        sched = o["sched"]
    o["sched_used"] = sched
    N.call("sb_blend_fwd", N.dtype_code(dt), N.ptr(records), N.ptr(pg), N.ptr(off), W, H, 16,
           int(bool(early)), float(thresh), N.ptr(exposure), N.ptr(c), N.ptr(d), N.ptr(t),
           N.ptr(op), N.ptr(nc), N.ptr(last), N.ptr(y), N.ptr(depth_limit), N.ptr(status),
           N.ptr(coarse_limit), N.ptr(sched), N.ptr(halt), int(bool(fast_exp)), N.stream_ptr())
    return o


def render(grid: TileGrid, screen: SplatScreen, intr: CameraIntrinsics,
           early_termination: bool = True,
           term_threshold: float = TERMINATION_THRESHOLD) -> RenderTargets:
    """forward.py:345-368 on the device."""
    rec = grid.records if grid.records is not None else screen.records()[0]
    o = run_blend_fwd(screen.dtype, rec, grid.pair_gaussian32, grid.offsets32, intr.width,
                      intr.height, early_termination, term_threshold)
    return RenderTargets(color=o["color"], depth=o["depth"], opacity=o["opacity"],
                         transmittance=o["transmittance"], n_contrib=o["n_contrib"],
                         last=o["last"], early_termination=bool(early_termination),
                         term_threshold=float(term_threshold))
