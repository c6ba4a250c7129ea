"""Host->device bandwidth of an 11 MB pinned buffer: torch pin_memory vs a
transparent-huge-page mapping registered with cudaHostRegister."""
import ctypes
import mmap
import os
import sys
import time

import torch

print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
      if os.path.exists("/sys/kernel/mm/transparent_hugepage/enabled") else "n/a")
nbytes = 1280 * 720 * 3 * 4
dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")


def bw(host, reps=50):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


a = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
print("pin_memory GB/s", round(bw(a), 1), round(bw(a), 1))

libc = ctypes.CDLL("libc.so.6", use_errno=True)
size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
m = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
base = ctypes.addressof(ctypes.c_char.from_buffer(m))
aligned = (base + (2 << 20) - 1) // (2 << 20) * (2 << 20)
MADV_HUGEPAGE = 14
print("madvise", libc.madvise(ctypes.c_void_p(aligned), ctypes.c_size_t(size), MADV_HUGEPAGE))
ctypes.memset(aligned, 0, size)
rc = torch.cuda.cudart().cudaHostRegister(aligned, size, 0)
print("cudaHostRegister", rc)
buf = (ctypes.c_float * (nbytes // 4)).from_address(aligned)
import numpy as np  # noqa: E402
h = torch.from_numpy(np.frombuffer(buf, dtype=np.float32))
print("is_pinned", h.is_pinned())
print("THP-registered GB/s", round(bw(h), 1), round(bw(h), 1))
with open("/proc/self/smaps") as f:
    txt = f.read()
print("AnonHugePages lines >0:", sum(1 for l in txt.splitlines() if l.startswith("AnonHugePages:") and not l.split()[1] == "0"))
