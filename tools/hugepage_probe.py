"""Pinned host buffers for the H2D feed: cudaHostAlloc pages vs a THP-backed (2 MB pages)
region registered with cudaHostRegister, written by the CPU first (diagnostic)."""
import ctypes
import mmap
import sys

import torch

sys.path.insert(0, ".")
import paper_2311_12716_b200 as amz  # noqa: E402
from paper_2311_12716_b200 import _lib  # noqa: E402

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      [ln for ln in open("/proc/meminfo") if "Huge" in ln][:3])
nb = 5259264
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = ctypes.CDLL("libcudart.so.12") if False else None
SZ = 16 << 20
raw = libc.mmap(None, SZ + (2 << 20), mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
base = (raw + (2 << 20) - 1) & ~((2 << 20) - 1)
print("madvise", libc.madvise(base, SZ, 14))  # MADV_HUGEPAGE
ctypes.memset(base, 1, SZ)
smaps = open("/proc/self/smaps").read()
print("AnonHugePages total kB", sum(int(ln.split()[1]) for ln in smaps.splitlines() if ln.startswith("AnonHugePages")))
r = torch.cuda.cudart().cudaHostRegister(base, SZ, 0)
print("cudaHostRegister", r)
dbig = torch.empty(nb, dtype=torch.uint8, device="cuda")
hw = amz.pinned_empty((nb,), torch.uint8)
hw.copy_(torch.randint(0, 3, (nb,), dtype=torch.uint8))
st = torch.cuda.current_stream()


def timeit(fn, k=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1000, 1)


import numpy as np  # noqa: E402

ht = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * nb).from_address(base)))
print("registered tensor is_pinned", ht.is_pinned())
for name, t in (("cudaHostAlloc cpu-written", hw), ("THP registered cpu-written", ht)):
    ptr = t.data_ptr()
    ce = timeit(lambda: dbig.copy_(t, non_blocking=True))
    kern = timeit(lambda: _lib.call("amz_copy_h2d", dbig.data_ptr(), ptr, nb, 32, st.cuda_stream))
    print(f"{name:28s} CE us {ce}  kernel us {kern}")
