"""Pinned host staging buffers backed by transparent huge pages.

The keyframe image a mapping loop uploads every iteration (11 MB at
1280x720) goes host->device by DMA.  Pinned memory from ``pin_memory()`` /
cudaHostAlloc is made of 4 KB pages; on the B200 boxes here (a VM behind an
IOMMU) its DMA runs at 16-18 GB/s, while the same copy from a 2 MB-page
mapping registered with cudaHostRegister runs at 54 GB/s
(``tools/h2d_probe.py``).  ``pinned_empty`` returns such a buffer as a CPU
tensor (``is_pinned()`` is True), falling back to ``pin_memory()`` when the
kernel refuses huge pages or the registration fails.
"""

from __future__ import annotations

import ctypes
import mmap

import numpy as np
import torch

_HUGE = 2 << 20
_MADV_HUGEPAGE = 14
_libc = None
_registered: list = []   # (ptr, mmap): kept for the process lifetime or release()


def _madvise(ptr: int, size: int) -> None:
    global _libc
    if _libc is None:
        _libc = ctypes.CDLL("libc.so.6", use_errno=True)
    _libc.madvise(ctypes.c_void_p(ptr), ctypes.c_size_t(size), _MADV_HUGEPAGE)


def huge_page_bytes(ptr: int) -> int | None:
    """AnonHugePages of the mapping containing ``ptr`` (/proc/self/smaps), or
    None when unavailable: how much of a staging buffer got 2 MB pages."""
    try:
        with open("/proc/self/smaps") as f:
            inside = False
            for line in f:
                head = line.split()
                if "-" in head[0] and len(head) > 4 and ":" in head[3]:
                    lo, hi = (int(x, 16) for x in head[0].split("-"))
                    inside = lo <= ptr < hi
                elif inside and line.startswith("AnonHugePages:"):
                    return int(head[1]) * 1024
    except Exception:
        return None
    return None


def pinned_empty(shape, dtype=torch.float32) -> torch.Tensor:
    """A pinned CPU tensor on huge pages (contents zero)."""
    shape = tuple(int(s) for s in shape)
    npdt = torch.empty((), dtype=dtype).numpy().dtype
    count = int(np.prod(shape)) if shape else 1
    nbytes = count * npdt.itemsize
    try:
        size = (nbytes + _HUGE - 1) // _HUGE * _HUGE
        m = mmap.mmap(-1, size + _HUGE, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        base = ctypes.addressof(ctypes.c_char.from_buffer(m))
        off = (-base) % _HUGE
        ptr = base + off
        _madvise(ptr, size)
        ctypes.memset(ptr, 0, size)                     # fault the pages in
        rc = torch.cuda.cudart().cudaHostRegister(ptr, size, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister: {rc}")
        _registered.append((ptr, m))
        arr = np.frombuffer(m, dtype=npdt, count=count, offset=off)   # keeps m alive
        return torch.from_numpy(arr).view(shape)
    except Exception:
        return torch.empty(shape, dtype=dtype).pin_memory()


def pinned_from(array) -> torch.Tensor:
    """``pinned_empty`` filled with ``array`` (numpy or CPU tensor)."""
    src = torch.as_tensor(array)
    t = pinned_empty(src.shape, src.dtype)
    t.copy_(src)
    return t
