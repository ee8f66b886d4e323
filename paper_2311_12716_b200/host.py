"""Pinned host staging buffers for the host->device trajectory feed.

``pinned_empty`` allocates through the library (``amz_host_alloc``: 2 MB transparent
huge pages registered with cudaHostRegister, else cudaHostAlloc) and wraps the block as
a CPU torch tensor; the block is freed when the last tensor viewing it goes away.
Copies of CPU-written data from it to the device run at the PCIe rate (measured 49-53
GB/s on the B200 hosts, where the same data in 4 KB cudaHostAlloc pages read at 11-25
GB/s: tools/hugepage_probe.py), so an input feed (actions, values from a host-side
actor) should stage through it.
"""

from __future__ import annotations

import ctypes
import math

from . import _lib


def _torch():
    import torch

    return torch


class _HostBlock:
    __slots__ = ("ptr",)

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _lib.call("amz_host_alloc", nbytes, ctypes.byref(p))
        self.ptr = p.value

    def __del__(self):
        if self.ptr:
            try:
                _lib.lib().amz_host_free(ctypes.c_void_p(self.ptr))
            except Exception:  # interpreter shutdown
                pass
            self.ptr = None


def pinned_empty(shape, dtype):
    """Uninitialised pinned CPU tensor of ``shape``/``dtype`` from amz_host_alloc."""
    torch = _torch()
    torch.cuda.init()  # torch reports (and copies) host memory as pinned only once CUDA is up
    shape = tuple(int(x) for x in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    n = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
    blk = _HostBlock(max(n, 1))
    raw = (ctypes.c_uint8 * max(n, 1)).from_address(blk.ptr)
    raw._amz_block = blk  # the tensor's storage holds raw, raw holds the block
    return torch.frombuffer(raw, dtype=torch.uint8)[:n].view(dtype).reshape(shape)
