"""Node-shared host tier: one copy of a host table for all of a node's GPU processes.

Legion keeps the uncached feature rows (and the full topology) in host memory that
every GPU reads over PCIe (PAPER.md, unified cache; the reference's CPU tier,
simulator.py:161-202). With one process per GPU a per-process pinned copy would hold
the table K times — 8 x 57 GB at papers100M shape, more than the box has. Here the
node's first rank creates the table in POSIX shared memory (/dev/shm), every rank maps
it and registers the mapping with CUDA (cudaHostRegister, mapped + portable, via
gc_host_register), so each GPU reads the same physical pages zero-copy through UVA.
The file is unlinked as soon as every rank has mapped it: the pages live until the
last process unmaps them, and nothing is left behind if a rank dies.
"""

from __future__ import annotations

import ctypes
import mmap
import os

import numpy as np
import torch

from . import _lib

_SHM_DIR = "/dev/shm"


class SharedHostTensor:
    """A host tensor backed by a named /dev/shm file, pinned and GPU-mapped in this process.

    create=True makes (and sizes) the file; create=False attaches to it. Call
    unlink() on the creator once every process has attached."""

    def __init__(self, name: str, shape: tuple, dtype: torch.dtype, create: bool, register: bool = True):
        if "/" in name:
            raise ValueError("shared host tensor names are plain file names")
        self.path = os.path.join(_SHM_DIR, name)
        self.shape = tuple(int(s) for s in shape)
        itemsize = torch.empty((), dtype=dtype).element_size()
        numel = int(np.prod(self.shape)) if self.shape else 1
        self.nbytes = numel * itemsize
        size = max(self.nbytes, mmap.PAGESIZE)
        flags = os.O_RDWR | (os.O_CREAT | os.O_TRUNC if create else 0)
        fd = os.open(self.path, flags, 0o600)
        try:
            if create:
                os.ftruncate(fd, size)
            elif os.fstat(fd).st_size < size:
                raise ValueError(f"{self.path} is smaller than the requested {size} bytes")
            self._mm = mmap.mmap(fd, size, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self.tensor = torch.frombuffer(self._mm, dtype=dtype, count=numel).view(self.shape)
        self.creator = create
        self._registered = False
        if register and self.nbytes:
            alias = ctypes.c_void_p()
            _lib.check(_lib.lib().gc_host_register(self.tensor.data_ptr(), self.nbytes, ctypes.byref(alias)),
                       "host_register")
            self._registered = True
            if alias.value != self.tensor.data_ptr():
                raise RuntimeError("mapped host memory is not at its host address (UVA required)")

    def unlink(self) -> None:
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass

    def close(self) -> None:
        if self._registered:
            _lib.check(_lib.lib().gc_host_unregister(self.tensor.data_ptr()), "host_unregister")
            self._registered = False
        self.tensor = None
        if self._mm is not None:
            try:
                self._mm.close()
            except BufferError:  # views still alive: the mapping goes with the process
                pass
            self._mm = None
        if self.creator:
            self.unlink()


def shared_host_table(name: str, shape: tuple, dtype: torch.dtype, local_rank: int, fill=None, barrier=None
                      ) -> SharedHostTensor:
    """Collective over one node's ranks: local rank 0 creates and fills (fill(tensor)),
    everyone attaches and registers, then the file is unlinked. barrier() must
    synchronise the node's ranks (dist.barrier for torch.distributed)."""
    barrier = barrier or (lambda: None)
    if local_rank == 0:
        t = SharedHostTensor(name, shape, dtype, create=True)
        if fill is not None:
            fill(t.tensor)
        barrier()
        barrier()  # every rank has attached
        t.unlink()
        barrier()
        return t
    barrier()  # the creator has filled it
    t = SharedHostTensor(name, shape, dtype, create=False)
    barrier()
    barrier()  # the name is gone: nothing outlives the processes
    return t
